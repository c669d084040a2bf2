"""Summarise ncu captures (run on the dev box, ncu -i needs no GPU) into profiles/<tag>/.

    python scripts/ncu_summary.py gpurun_out/r1h profiles/r1

Writes summary.md (human) and summary.json (machine: per capture the duration,
DRAM bytes read/written, throughputs, launch config) and copies the launch list
with per-kernel shares of the step.
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "launch__shared_mem_per_block_dynamic", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
       "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
       "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
       "dram__bytes.sum.peak_sustained", "dram__cycles_elapsed.avg.per_second"]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for name in RAW:
            if name in hdr:
                i = hdr.index(name)
                d[name] = (r[i], units[i])
        res.append(d)
    return res


def to_bytes(v):
    val, unit = v
    f = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return f * scale


def to_ns(v):
    val, unit = v
    f = float(val.replace(",", ""))
    return f * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)


def launches(csv_path):
    if not os.path.exists(csv_path):
        return None
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    hdr = rows[0]
    agg = defaultdict(list)
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "")
            agg[name].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot} for k, v in agg.items()}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    summary = {"source": src, "captures": {}}
    md = [f"# ncu summary ({os.path.basename(src)})", "",
          "Captures: `ncu --set full --clock-control none` (one launch each, cold L2, serialised).", ""]
    for f in sorted(os.listdir(src)):
        if not f.endswith(".ncu-rep"):
            continue
        for d in raw_metrics(os.path.join(src, f)):
            dur = to_ns(d["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in d else None
            rd = to_bytes(d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
            wr = to_bytes(d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
            entry = {"kernel": d["kernel"][:120], "duration_ns": dur, "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "dram_GBps": (rd + wr) / dur if dur and rd is not None else None}
            if "dram__bytes.sum.peak_sustained" in d and "dram__cycles_elapsed.avg.per_second" in d:
                # ncu's DRAM peak: bytes per DRAM cycle x DRAM clock
                v, u = d["dram__bytes.sum.peak_sustained"]
                bpc = float(v.replace(",", "")) * {"byte/cycle": 1, "Kbyte/cycle": 1e3, "Mbyte/cycle": 1e6}.get(u, 1)
                v, u = d["dram__cycles_elapsed.avg.per_second"]
                hz = float(v.replace(",", "")) * {"hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}.get(u, 1)
                entry["dram_peak_gbs"] = round(bpc * hz / 1e9, 1)
            for k in RAW[3:]:
                if k in d:
                    entry[k] = d[k][0]
            summary["captures"][f] = entry
            md += [f"## {f}", "", f"- kernel: `{entry['kernel']}`",
                   f"- duration: {dur / 1e3:.2f} us" if dur else "- duration: ?",
                   f"- DRAM read {rd / 1e6:.2f} MB, write {wr / 1e6:.3f} MB -> {entry['dram_GBps']:.0f} GB/s"
                   if rd is not None and dur else "- DRAM: ?"]
            for k in RAW[3:]:
                if k in d:
                    md.append(f"- {k}: {d[k][0]} {d[k][1]}")
            md.append("")
    ls = launches(os.path.join(src, "launches.csv"))
    if ls:
        summary["launch_list"] = ls
        md += ["## Launch list (short bench run, `--metrics gpu__time_duration.sum`)", "",
               "| kernel | launches | mean us | share of kernel time |", "|---|---|---|---|"]
        for k, v in sorted(ls.items(), key=lambda kv: -kv[1]["share"]):
            md.append(f"| `{k}` | {v['launches']} | {v['mean_ns'] / 1e3:.2f} | {100 * v['share']:.1f} % |")
        shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches.csv"))
    for extra in ("bench.json", "kbench.jsonl", "gpu.txt"):
        if os.path.exists(os.path.join(src, extra)):
            shutil.copy(os.path.join(src, extra), os.path.join(dst, extra))
    json.dump(summary, open(os.path.join(dst, "summary.json"), "w"), indent=1)
    open(os.path.join(dst, "summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()

"""Per-SASS-instruction executed counts and stall samples from an ncu report (source page),
printed as the hottest instructions and totals per address window.
    python scripts/ncu_source.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1] if rows[0][0] == "Kernel Name" else rows[0]
    body = rows[2:] if rows[0][0] == "Kernel Name" else rows[1:]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex, ism = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    recs = []
    for i, r in enumerate(body):
        try:
            recs.append((i, r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ism] or 0)))
        except (ValueError, IndexError):
            pass
    tot_ex = sum(r[3] for r in recs)
    tot_sm = sum(r[4] for r in recs)
    print(f"instructions {tot_ex}  samples {tot_sm}")
    print("-- hottest by executed")
    for r in sorted(recs, key=lambda r: -r[3])[:top]:
        print(f"{r[0]:5d} {r[3]:10d} {r[4]:7d}  {r[2][:70]}")
    print("-- hottest by stall samples")
    for r in sorted(recs, key=lambda r: -r[4])[:top]:
        print(f"{r[0]:5d} {r[3]:10d} {r[4]:7d}  {r[2][:70]}")


if __name__ == "__main__":
    main()

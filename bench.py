#!/usr/bin/env python
"""Benchmark: the MCAP-routed decode-linear stack of Llama-3.2-1B (BASELINE.json
configs[1]) on B200, through the C ABI (libmcapq.so).

A "step" = one pass of the whole hot path over one batch-1 decode token: 16
layers x {q, k, v, o, gate, up, down} routed by the MCAP profile (layer 15 ->
W4A16, the other 15 -> W4A8 with their 4 activation quantisations each), the
step replayed as one CUDA graph.  Synthetic seeded bf16
weights/activations (synth_inputs), random-init, no checkpoints.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, or self-launched when --gpus N is given without a launcher): every
rank runs its own replica of the stack (independent decode streams; "scaling":
"weak": the 1B step does not shard), and the line's `sharded`
object carries the column-sharded Llama-3.1-8B lm_head (M = 1, 64) and MLP gate /
down with their NCCL all-gather: T(1), T(P), comm us and E(P) = T(1) / (P T(P)).
One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import itertools
import json
import math
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth_inputs as si  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
GOLDEN_PROFILE = os.path.join(ROOT, "tests", "golden", "llama32_1b_profile.json")
SLOTS = ["q", "k", "v", "o", "gate", "up", "down"]
WORKLOAD = ("llama-3.2-1b 16-layer decode linear stack (q,k,v,o,gate,up,down), MCAP mask from tab:per_layer_scores "
            "(L15 W4A16, 15 layers W4A8), batch 1, chained (x_o=y_q, x_gate/up=y_o, x_down=y_up, "
            "x_qkv(l+1)=y_down(l)), one CUDA graph")
INPUT_ID = {"q": 0, "k": 0, "v": 0, "o": 1, "gate": 2, "up": 2, "down": 3}
MODEL = "llama-3.2-1b"
CONFIG_ID = 2


def traffic_from_profiles(kernel_prefix):
    """DRAM bytes (read + write) per launch of `kernel_prefix` from the newest committed
    ncu --set full summary (profiles/<round>/summary.json), or None."""
    pdir = os.path.join(ROOT, "profiles")
    if not os.path.isdir(pdir):
        return None, None
    for sub in sorted(os.listdir(pdir), reverse=True):
        p = os.path.join(pdir, sub, "summary.json")
        if not os.path.exists(p):
            continue
        for cap, e in json.load(open(p)).get("captures", {}).items():
            if kernel_prefix in e.get("kernel", "") and e.get("dram_read_bytes") is not None:
                return int(e["dram_read_bytes"] + (e.get("dram_write_bytes") or 0)), f"profiles/{sub}/summary.json:{cap}"
    return None, None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_dram_peak():
    """ncu's DRAM peak (dram__bytes.sum.peak_sustained x dram__cycles_elapsed.avg.per_second)
    from the newest committed summary, GB/s, or None (SURVEY 8(d) D.2 denominator (i))."""
    pdir = os.path.join(ROOT, "profiles")
    if not os.path.isdir(pdir):
        return None, None
    for sub in sorted(os.listdir(pdir), reverse=True):
        p = os.path.join(pdir, sub, "summary.json")
        if os.path.exists(p):
            for cap, e in json.load(open(p)).get("captures", {}).items():
                if e.get("dram_peak_gbs"):
                    return float(e["dram_peak_gbs"]), f"profiles/{sub}/summary.json:{cap}"
    return None, None


def read_ceiling(mq, dev, stream, gib=1, reps=10):
    """Pure-read HBM ceiling in this run (D.2 (iii)): mcapq_debug_read_bw streaming a
    `gib` GiB buffer (> 8 x L2), median of `reps` CUDA-event-timed reads, GB/s."""
    buf = torch.empty(gib << 30, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    times = []
    with torch.cuda.stream(stream):
        mq.debug_read_bw(buf, sink, stream=stream)
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mq.debug_read_bw(buf, sink, stream=stream)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    del buf
    return buf_bytes_gbs(gib << 30, statistics.median(times))


def buf_bytes_gbs(nbytes, ms):
    return round(nbytes / (ms * 1e-3) / 1e9, 1)


def bf16_peak_tflops():
    """Dense bf16 tensor peak: MEASURED_PEAKS.json bf16_tflops (cuBLAS burst), else 2250."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if "bf16_tflops" in d:
            return float(d["bf16_tflops"])
    return 2250.0


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- workload
# The decode chain through the linears: each group's input is the output that feeds
# it in the model, with the non-linear ops between them (attention, residual+RMSNorm,
# SiLU*mul) elided: x_o = y_q, x_gate/up = y_o, x_down = y_up, x_q/k/v(l+1) = y_down(l).
# Only layer 0's q/k/v input is a step input.
CHAIN_SRC = {1: "q", 2: "o", 3: "up"}      # input_id -> slot of the same layer producing it


def build_stack(mq, dev, routes, m=1, chain=True):
    """Pack the 16-layer Llama-3.2-1B linear stack, chained (CHAIN_SRC); returns
    (stack, weights, xs, ys).  The outputs live in one device arena in (layer, slot)
    order, so mcapq_stack_step_host moves each direction with one copy."""
    L = si.MODELS[MODEL]["layers"]
    st = mq.Stack(routes, max_m=m)
    shapes = {slot: si.linear_shape(MODEL, slot) for slot in SLOTS}
    yarena = torch.empty(L * m * sum(n for n, _ in shapes.values()), dtype=torch.bfloat16, device=dev)
    ys, off = {}, 0
    for l in range(L):
        for slot in SLOTS:
            n = shapes[slot][0]
            ys[(l, slot)] = yarena[off:off + m * n].view(m, n)
            off += m * n
    xs = {}
    for l in range(L):
        for iid in sorted(set(INPUT_ID.values())):
            if not chain:      # diagnostic: every input a step input (no dependencies)
                slot = next(sl for sl in SLOTS if INPUT_ID[sl] == iid)
                xs[(l, iid)] = si.activation(m, shapes[slot][1], si.seed_for(CONFIG_ID, l, slot, True),
                                             si.activation_kind(slot)).to(dev)
            elif iid == 0:
                xs[(l, 0)] = (si.activation(m, shapes["q"][1], si.seed_for(CONFIG_ID, 0, "q", True)).to(dev)
                              if l == 0 else ys[(l - 1, "down")])
            else:
                xs[(l, iid)] = ys[(l, CHAIN_SRC[iid])]
    weights = {}
    for l in range(L):
        for s_id, slot in enumerate(SLOTS):
            n, k = shapes[slot]
            w = si.weight(n, k, si.seed_for(CONFIG_ID, l, slot)).to(dev)
            pw = mq.pack_w4(w)
            del w
            st.set(l, s_id, INPUT_ID[slot], pw, xs[(l, INPUT_ID[slot])], ys[(l, slot)])
            weights[(l, slot)] = pw
    return st, weights, xs, ys


def stack_with_routes(mq, routes, weights, xs, ys, m=1):
    st = mq.Stack(routes, max_m=m)
    L = len(routes)
    for l in range(L):
        for s_id, slot in enumerate(SLOTS):
            st.set(l, s_id, INPUT_ID[slot], weights[(l, slot)], xs[(l, INPUT_ID[slot])], ys[(l, slot)])
    return st


def time_graph(st, stream, steps, warmup, dist=None):
    for _ in range(warmup):
        st.replay(stream=stream)
    stream.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        st.replay(stream=stream)
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    return e0.elapsed_time(e1) / steps


def step_percentiles(st, stream, steps):
    """Per-step times (ms) of `steps` back-to-back graph replays, one CUDA event between
    consecutive replays on the launching stream: p10 / p50 / p90 (D.4)."""
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(stream)
    for i in range(steps):
        st.replay(stream=stream)
        evs[i + 1].record(stream)
    evs[-1].synchronize()
    t = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(steps))
    q = lambda f: t[min(len(t) - 1, int(f * len(t)))]
    return {"p10_ms": round(q(0.10), 5), "p50_ms": round(q(0.50), 5), "p90_ms": round(q(0.90), 5), "steps": steps}


def time_dominant_kernel(mq, weights, xs, stream, reps_per_layer=4):
    """The stack's dominant kernel: the grouped W4A8 gate+up launch (2 x 8192x2048,
    stream_linear<DP4A> with the quantiser fused), exactly as the stack launches it
    (mcapq_linear_group), rotating over the 16 layers' weights (16 x 18.9 MB > L2)
    so every launch streams from HBM.  CUDA events on the launching stream."""
    L = si.MODELS[MODEL]["layers"]
    dev = xs[(0, 0)].device
    n = weights[(0, "gate")].n
    outs = [torch.empty(1, n, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    seq = [l for _ in range(reps_per_layer) for l in range(L)]
    with torch.cuda.stream(stream):
        def call(l):
            mq.linear_group(0, [weights[(l, "gate")], weights[(l, "up")]], xs[(l, INPUT_ID["gate"])], outs=outs,
                            stream=stream)
        for l in seq[:4]:
            call(l)
        stream.synchronize()
        # capture the launches in a graph: the timed region holds kernels only, no host work
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for l in seq:
                call(l)
        g.replay()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(4):
            g.replay()
        e1.record(stream)
        e1.synchronize()
    per_launch_ms = e0.elapsed_time(e1) / (4 * len(seq))
    w = weights[(0, "gate")]
    alg_bytes = 2 * (w.n * w.k // 2 + w.n * (w.k // 32) * 2) + 2 * w.k + 2 * 2 * w.n
    return per_launch_ms, alg_bytes, len(seq)


def _graph_us(fns, stream, reps, dist=None):
    """Per-call us of `reps` calls captured in one CUDA graph, call r = fns[r % len(fns)]
    (rotating weight copies, so repeated calls stream from HBM, not L2); CUDA events on
    the launching stream after one warm replay; max over ranks when dist is given."""
    dev = torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.stream(stream):
        for f in fns:
            f()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for r in range(reps):
                fns[r % len(fns)]()
        g.replay()
        stream.synchronize()
        if dist is not None:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1000 / reps], device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del g
    return float(t.item())


def _copies(pw, l2):
    """Distinct HBM copies of a packed weight, together >= 4 x L2 (at most 16)."""
    c = max(1, min(16, -(-4 * l2 // pw.nbytes)))
    return [pw] + [type(pw)(pw.nib.clone(), pw.scale.clone()) for _ in range(c - 1)]


# the sharded layers of north_star (configs 4 and 5): (slot, M, graph reps)
SHARDED = (("lm_head", 1, 20), ("lm_head", 64, 4), ("gate", 1, 64), ("down", 1, 64))


def time_sharded(mq, dev, stream, dist, world, rank, force_comm=False, slots=None):
    """Rows a8 / NEXT-2 at P = world: the Llama-3.1-8B lm_head
    (M = 1, 64) and MLP gate / down column-sharded over the job's ranks.  Per layer and
    route: T(1) = the unsharded linear on one GPU (no collective), T(P) = the sharded
    linear + NCCL all-gather into the replicated y (mcapq_linear_colshard), t_local = the
    rank's shard alone, comm = T(P) - t_local, E(P) = T(1) / (P T(P)); at M = 1 also the
    fused epilogue (NVLink stores into NCCL symmetric-window replicas + one LSA barrier:
    fused_TP_us, fused_comm_us, fused_E); for the lm_head also greedy decode (local argmax +
    P x M key gather, mcapq_linear_colshard_argmax).
    Every time is a CUDA graph of repeated calls over rotating weight copies (>= 4 x L2
    together), CUDA events, max over ranks."""
    comm = mq.Comm() if world > 1 or force_comm else None   # force_comm: the P = 1 path check
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    rows = []
    for slot, m, reps in (slots or SHARDED):
        n, k = si.linear_shape("llama-3.1-8b", slot)
        per = n // world
        w = si.weight(n, k, si.seed_for(5 if slot == "lm_head" else 4, 0, slot))
        pw_full = mq.pack_w4(w.to(dev))
        del w
        pw = pw_full.shard(world, rank) if world > 1 else pw_full
        x = si.activation(m, k, si.seed_for(5 if slot == "lm_head" else 4, 0, slot, True)).to(dev)
        wbytes = n * k // 2 + n * (k // 32) * 2
        full_c, shard_c = _copies(pw_full, l2), (_copies(pw, l2) if comm is not None else None)
        for route, name in ((0, "w4a8"), (1, "w4a16")):
            y = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
            yl = torch.empty(m, per, dtype=torch.bfloat16, device=dev)
            ws = torch.empty(max(256, mq.workspace_bytes(route, m, n, k)), dtype=torch.uint8, device=dev)
            t1 = _graph_us([lambda c=c: mq.linear(route, c, x, out=y, ws=ws, stream=stream) for c in full_c],
                           stream, reps, dist)
            row = {"model": "llama-3.1-8b", "slot": slot, "N": n, "K": k, "M": m, "route": name, "P": world,
                   "rows_per_rank": per, "T1_us": round(t1, 3), "T1_gbs": round(wbytes / t1 / 1e3, 1),
                   "weight_copies": [len(full_c), len(shard_c) if shard_c else 0]}
            if comm is not None:
                tl = _graph_us([lambda c=c: mq.linear(route, c, x, out=yl, ws=ws, stream=stream) for c in shard_c],
                               stream, reps, dist)
                wsc = torch.empty(max(256, comm.workspace_bytes(route, m, n, k)), dtype=torch.uint8, device=dev)
                tp = _graph_us([lambda c=c: mq.linear_colshard(comm, route, c, n, x, out=y, ws=wsc, stream=stream)
                                for c in shard_c], stream, reps, dist)
                row.update({"t_local_us": round(tl, 3), "TP_us": round(tp, 3), "comm_us": round(tp - tl, 3),
                            "E": round(t1 / (world * tp), 3), "gbs_total": round(wbytes / tp / 1e3, 1)})
                if m == 1:
                    # a8 fused epilogue: NVLink stores into every rank's window replica + one LSA
                    # barrier instead of the all-gather (mcapq_linear_colshard fused_epilogue=1)
                    try:
                        yw = comm.window(n)
                        tf = _graph_us([lambda c=c: mq.linear_colshard(comm, route, c, n, x, out=yw, ws=wsc,
                                                                       stream=stream, fused=True) for c in shard_c],
                                       stream, reps, dist)
                        comm.free_window(yw)
                        row.update({"fused_TP_us": round(tf, 3), "fused_comm_us": round(tf - tl, 3),
                                    "fused_E": round(t1 / (world * tf), 3)})
                    except Exception as e:   # the headline line must still print
                        row["fused_error"] = f"{type(e).__name__}: {e}"[:160]
                if slot == "down" and k % (32 * world) == 0:
                    # NEXT-2 Megatron pairing: down row-parallel (K-sharded, the partner of a
                    # column-sharded up) -- this rank's K-slice partial + NCCL sum all-reduce
                    # (mcapq_linear_rowshard), and at M = 1 the fused NVLink slot stores + LSA
                    # barriers + rank-order sum
                    try:
                        kp = k // world
                        ks_c = _copies(pw_full.kshard(world, rank), l2)
                        xs = x[:, rank * kp:(rank + 1) * kp].contiguous()
                        wsr = torch.empty(max(256, comm.rowshard_workspace_bytes(route, m, n, kp)), dtype=torch.uint8,
                                          device=dev)
                        tr = _graph_us([lambda c=c: mq.linear_rowshard(comm, route, c, xs, out=y, ws=wsr,
                                                                       stream=stream) for c in ks_c], stream, reps, dist)
                        row.update({"rowpar_TP_us": round(tr, 3), "rowpar_E": round(t1 / (world * tr), 3)})
                        if m == 1 and kp % 256 == 0 and kp >= 2048:
                            win = comm.window(n, torch.float32, rows=world)
                            trf = _graph_us([lambda c=c: mq.linear_rowshard(comm, route, c, xs, out=y, ws=win,
                                                                            stream=stream, fused=True) for c in ks_c],
                                            stream, reps, dist)
                            comm.free_window(win)
                            row.update({"rowpar_fused_TP_us": round(trf, 3), "rowpar_fused_E": round(t1 / (world * trf), 3)})
                        del ks_c
                    except Exception as e:   # the headline line must still print
                        row["rowpar_error"] = f"{type(e).__name__}: {e}"[:160]
                if slot == "lm_head":
                    wsa = torch.empty(max(256, mq.argmax_workspace_bytes(route, m, per, k, world)),
                                      dtype=torch.uint8, device=dev)
                    ws1 = torch.empty(max(256, mq.argmax_workspace_bytes(route, m, n, k)), dtype=torch.uint8,
                                      device=dev)
                    ta = _graph_us([lambda c=c: mq.linear_colshard_argmax(comm, route, c, n, x, ws=wsa, stream=stream)
                                    for c in shard_c], stream, reps, dist)
                    t1a = _graph_us([lambda c=c: mq.linear_argmax(route, c, x, ws=ws1, stream=stream) for c in full_c],
                                    stream, reps, dist)
                    row.update({"greedy_T1_us": round(t1a, 3), "greedy_TP_us": round(ta, 3),
                                "greedy_E": round(t1a / (world * ta), 3)})
            rows.append(row)
        del pw_full, pw, full_c, shard_c
    del comm
    return {"timing": "CUDA graph of repeated calls over rotating weight copies (>= 4 x L2), CUDA events, max "
                      "over ranks; T(1) unsharded on one GPU, "
                      "T(P) sharded + NCCL all-gather (E = T(1) / (P T(P))); down also row-parallel "
                      "(rowpar_*: K-sharded + all-reduce, NEXT-2)", "rows": rows}


def time_mlp8b_stack(mq, dev, stream, layers=8, steps=20):
    """cfg4 shapes in the decode setting: an 8-layer Llama-3.1-8B MLP stack (gate/up
    14336x4096, down 4096x14336) chained like decode (x_gate/up(l) = y_down(l-1),
    x_down(l) = y_up(l)), one persistent stack_step launch per step, all W4A8 and all
    W4A16.  One packed layer cloned per layer (distinct HBM copies: 793 MB per step > L2)."""
    shapes = {s_: si.linear_shape("llama-3.1-8b", s_) for s_ in ("gate", "up", "down")}
    base = {s_: mq.pack_w4(si.weight(n, k, si.seed_for(4, 0, s_)).to(dev)) for s_, (n, k) in shapes.items()}
    weights = {(l, s_): mq.PackedW4(base[s_].nib.clone(), base[s_].scale.clone())
               for l in range(layers) for s_ in shapes}
    ys = {(l, s_): torch.empty(1, shapes[s_][0], dtype=torch.bfloat16, device=dev) for l in range(layers)
          for s_ in shapes}
    x0 = si.activation(1, shapes["gate"][1], si.seed_for(4, 0, "gate", True)).to(dev)
    wbytes = sum(w.nbytes for w in weights.values())
    out = {"layers": layers, "weight_bytes_per_step": wbytes, "shapes": "gate/up 14336x4096, down 4096x14336"}
    for route, name in ((0, "w4a8"), (1, "w4a16")):
        st = mq.Stack([route] * layers, max_m=1)
        for l in range(layers):
            xg = x0 if l == 0 else ys[(l - 1, "down")]
            st.set(l, 0, 0, weights[(l, "gate")], xg, ys[(l, "gate")])
            st.set(l, 1, 0, weights[(l, "up")], xg, ys[(l, "up")])
            st.set(l, 2, 1, weights[(l, "down")], ys[(l, "up")], ys[(l, "down")])
        with torch.cuda.stream(stream):
            st.capture(1, stream=stream)
        ms = time_graph(st, stream, steps, 3)
        out[f"{name}_us_per_layer"] = round(ms * 1000 / layers, 3)
        out[f"{name}_gbs"] = round(wbytes / (ms * 1e-3) / 1e9, 1)
        out[f"{name}_frac"] = round(wbytes / (ms * 1e-3) / 1e9 / peaks()[0], 4)
        out[f"{name}_kernels_per_step"] = st.launches(1)
        del st
    del weights, base
    torch.cuda.empty_cache()
    return out


def time_single_linears(mq, dev, stream):
    """Single-linear rows of the metric at the other configs (cfg1 q_proj, cfg4 8B MLP,
    cfg5 lm_head), both routes, M = 1, rotating weight copies so each launch reads HBM."""
    out = []
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for cfg, model, slot, m in ((1, "llama-3.2-1b", "q", 1), (4, "llama-3.1-8b", "gate", 1),
                                (4, "llama-3.1-8b", "gate+up", 1),
                                (4, "llama-3.1-8b", "down", 1), (5, "llama-3.1-8b", "lm_head", 1),
                                (3, "llama-3.2-3b", "up", 1), (3, "llama-3.2-3b", "up", 16),
                                (3, "llama-3.2-3b", "up", 64), (3, "llama-3.2-3b", "q", 64),
                                (5, "llama-3.1-8b", "lm_head", 64)):
        # "a+b": the linears sharing one input in ONE grouped launch (mcapq_linear_group: the
        # fused gate/up of P:977), as the framework launches the 8B MLP up-projections
        members = slot.split("+")
        dims = [si.linear_shape(model, s_) for s_ in members]
        n, k = dims[0]
        wbytes = sum(n_ * k_ // 2 + n_ * (k_ // 32) * 2 for n_, k_ in dims)
        copies = max(2, min(32, math.ceil(4 * l2 / wbytes)))
        ws = []
        pw0s = []
        for s_, (n_, k_) in zip(members, dims):
            base = si.weight(n_, k_, si.seed_for(cfg, 0, s_)).to(dev)
            pw0s.append(mq.pack_w4(base))
            del base
        for c in range(copies):
            ws.append([mq.PackedW4(p_.nib.clone(), p_.scale.clone()) for p_ in pw0s])
        x = si.activation(m, k, si.seed_for(cfg, 0, members[0], True), si.activation_kind(members[0])).to(dev)
        ys_ = [torch.empty(m, n_, dtype=torch.bfloat16, device=dev) for n_, _ in dims]
        y = ys_[0]
        grouped = len(members) > 1
        row = {"config": cfg, "model": model, "slot": slot, "N": sum(n_ for n_, _ in dims) if grouped else n, "K": k,
               "M": m, "weight_bytes": wbytes}
        if grouped:
            row["launch"] = "one grouped launch (mcapq_linear_group)"
        with torch.cuda.stream(stream):
            wsp = torch.empty(mq.workspace_bytes(0, m, max(n_ for n_, _ in dims), k), dtype=torch.uint8, device=dev)
            combos = list(itertools.product(((0, "w4a8"), (1, "w4a16")), (True, False)))
            if m == 1 and not grouped:
                # the paper's two-kernel W4A8 design on this GPU (app:kernels): a separate
                # quantisation kernel (mcapq_quant_a8) + a warp-per-row dp4a GEMV on the pre-quantised
                # activations (mcapq_w4a8), PDL-chained -- the baseline the fused TMA path replaces
                combos.append(((3, "w4a8_twokernel"), True))
                qbuf = (torch.empty((m, k), dtype=torch.int8, device=dev),
                        torch.empty((m, k // 32), dtype=torch.float32, device=dev),
                        torch.empty((m, k // 32), dtype=torch.int32, device=dev))
            if m > 1 and not grouped:   # a6 with bf16-dequantised weights on tcgen05 (mcapq_w4a16_bf16deq)
                combos.append(((2, "w4a16_bf16deq"), True))
            for (route, name), pdl in combos:
                # pdl: back-to-back linears as a decode engine launches them (mcapq_set_pdl: the
                # next weight stream starts under the previous kernel's tail); also without
                prev = mq.set_pdl(pdl)
                name_ = name if pdl else name + "_nopdl"

                def call(pws):
                    if grouped:
                        mq.linear_group(route, pws, x, outs=ys_, ws=wsp, stream=stream)
                        return
                    pw = pws[0]
                    if route == 0:
                        mq.linear(0, pw, x, out=y, ws=wsp, stream=stream)
                    elif route == 1:
                        mq.w4a16(pw, x, out=y, stream=stream)
                    elif route == 2:
                        mq.w4a16_bf16deq(pw, x, out=y, stream=stream)
                    else:
                        mq.quant_a8(x, stream=stream, out=qbuf)
                        mq.w4a8(pw, *qbuf, out=y, stream=stream)
                for pw in ws:        # every copy once: TMA descriptors are encoded outside the capture
                    call(pw)
                reps = max(copies, 20)
                stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for i in range(reps):
                        call(ws[i % copies])
                g.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(3):
                    g.replay()
                e1.record(stream)
                e1.synchronize()
                us = e0.elapsed_time(e1) * 1000 / (3 * reps)
                mq.set_pdl(prev)
                row[f"{name_}_us"] = round(us, 3)
                row[f"{name_}_gbs"] = round(wbytes / us / 1e3, 1)
                if pdl:
                    row[f"{name_}_frac"] = round(wbytes / us / 1e3 / peaks()[0], 4)
                if m > 1 and pdl:   # batched rows are judged on the tensor pipe too: int8 / bf16 MMA ops per second
                    row[f"{name_}_tops"] = round(2 * m * n * k / (us * 1e-6) / 1e12, 1)
                    if route == 2:   # useful bf16 FLOP/s against the measured dense bf16 peak
                        row[f"{name_}_tensor_frac"] = round(2 * m * n * k / (us * 1e-6) / 1e12 / bf16_peak_tflops(), 4)
        row["w4a8_over_w4a16"] = round(row["w4a16_us"] / row["w4a8_us"], 3)
        if m > 1:   # which batched W4A8 kernel ran (launch_gemm's dispatch, DESIGN 6.4 / 6.4b)
            mode = os.environ.get("MCAPQ_GEMM_A8_TC05", "1")
            tc = m >= 9 and (mode == "2" or (mode == "1" and m > 32 and (n + 127) // 128 >= mq.device_sms()))
            row["w4a8_kernel"] = ("tc05_w4a8 (tcgen05 kind::i8, TMEM read-back per block)" if tc
                                  else ("stream_linear<IMMA>" if m <= 8 else "gemm_w4<A8> (mma.sync IMMA)"))
            mode16 = os.environ.get("MCAPQ_GEMM_A16_TC05", "1")
            tc16 = m >= 9 and (mode16 == "2" or (mode16 == "1" and (n + 127) // 128 >= mq.device_sms()))
            row["w4a16_kernel"] = ("tc05_w4a16x (tcgen05 kind::f16, exact per-block read-back)" if tc16
                                   else ("stream_linear<HMMA>" if m <= 8 else "gemm_w4<A16> (mma.sync HMMA)"))
        out.append(row)
        del ws, pw0s
        torch.cuda.empty_cache()
    return out


def time_prefill(mq, dev, stream):
    """NEXT-4 rows: the 8B gate (14336 x 4096) and down at prefill sizes -- dequantise once
    (mcapq_dequant_w4_bf16) + the tcgen05 bf16 GEMM (mcapq_bf16w_gemm), CUDA-graph timed;
    useful bf16 FLOP/s against MEASURED_PEAKS.json bf16_tflops."""
    out = []
    for slot, m in (("gate", 1024), ("gate", 4096), ("down", 1024)):
        n, k = si.linear_shape("llama-3.1-8b", slot)
        pw = mq.pack_w4(si.weight(n, k, si.seed_for(4, 0, slot)).to(dev))
        x = si.activation(m, k, si.seed_for(4, 0, slot, True), si.activation_kind(slot)).to(dev)
        y = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
        wdq = mq.dequant_w4_bf16(pw)
        res = {}
        with torch.cuda.stream(stream):
            for name, fn in (("dequant", lambda: mq.dequant_w4_bf16(pw, out=wdq, stream=stream)),
                             ("gemm", lambda: mq.bf16w_gemm(wdq, x, out=y, stream=stream))):
                fn()
                stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(10):
                        fn()
                g.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(3):
                    g.replay()
                e1.record(stream)
                e1.synchronize()
                res[name] = e0.elapsed_time(e1) * 1000 / 30
        fl = 2.0 * m * n * k
        out.append({"model": "llama-3.1-8b", "slot": slot, "N": n, "K": k, "M": m,
                    "dequant_us": round(res["dequant"], 2), "gemm_us": round(res["gemm"], 2),
                    "gemm_tflops": round(fl / res["gemm"] / 1e6, 1),
                    "gemm_tensor_frac": round(fl / res["gemm"] / 1e6 / bf16_peak_tflops(), 4),
                    "prefill_tflops": round(fl / (res["gemm"] + res["dequant"]) / 1e6, 1)})
        del pw, x, y, wdq
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- CPU oracle
def oracle_prepare(layers=(0, 15)):
    """Pack (outside any timing) the sample layers of the stack for the oracle:
    layer 0 (a W4A8 layer, like 15 of the 16) and layer 15 (the W4A16 layer)."""
    import oracle
    oracle.build()
    _, _, routes = oracle.routes_from_profile(open(GOLDEN_PROFILE).read())
    prep = []
    for l in layers:
        packed, xin = {}, {}
        for slot in SLOTS:
            n, k = si.linear_shape(MODEL, slot)
            w = si.weight(n, k, si.seed_for(CONFIG_ID, l, slot)).float().numpy()
            packed[slot] = oracle.pack_w4(w)
            key = INPUT_ID[slot]
            if key not in xin:
                xin[key] = si.activation(1, k, si.seed_for(CONFIG_ID, l, slot, True),
                                         si.activation_kind(slot)).float().numpy()
        prep.append((l, routes[l], packed, xin))
    return routes, prep


def oracle_step(routes, prep):
    """One bounded sample: the oracle (as it stands) runs every sample layer in full
    (quantise once per distinct input + 7 linears); the stack's GB/s is extrapolated
    from the per-route layer times with the mask's route counts (15 W4A8 + 1 W4A16)."""
    import oracle
    t_route, b_layer = {}, {}
    for (l, route, packed, xin) in prep:
        t0 = time.perf_counter()
        qcache, nbytes = {}, 0
        for slot in SLOTS:
            nib, sc = packed[slot]
            x = xin[INPUT_ID[slot]]
            if route == oracle.W4A8:
                if INPUT_ID[slot] not in qcache:
                    qcache[INPUT_ID[slot]] = oracle.quant_a8(x)
                oracle.w4a8(nib, sc, *qcache[INPUT_ID[slot]])
            else:
                oracle.w4a16(nib, sc, x)
            nbytes += nib.nbytes + sc.nbytes
        t_route[route] = time.perf_counter() - t0
        b_layer[route] = nbytes
    total_t = sum(t_route[r] for r in routes)
    total_b = sum(b_layer[r] for r in routes)
    return total_b / total_t / 1e9, sum(t_route.values())


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_baseline(steps=5, warmup=1):
    """The oracle on all the process's cores: `warmup` untimed samples, then the median
    of `steps` timed ones (the same procedure as --impl reference)."""
    routes, prep = oracle_prepare()
    for _ in range(warmup):
        oracle_step(routes, prep)
    vals, secs = [], 0.0
    for _ in range(steps):
        v, t = oracle_step(routes, prep)
        vals.append(v)
        secs += t
    return statistics.median(vals), len(os.sched_getaffinity(0)), secs


def oracle_baseline_1core(steps=3, warmup=1):
    """The same sample on ONE core: a child process pinned to one CPU with one OpenMP
    thread (the oracle's row loop is OpenMP), so the thread count is what it says."""
    import subprocess
    cpu = sorted(os.sched_getaffinity(0))[0]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    code = ("import os, sys, json; os.sched_setaffinity(0, {%d}); sys.path.insert(0, %r); import bench; "
            "v, c, t = bench.oracle_baseline(%d, %d); print(json.dumps([v, c, t]))" % (cpu, ROOT, steps, warmup))
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        v, c, t = json.loads(out.stdout.strip().splitlines()[-1])
        return v, c, t
    except Exception as e:   # the headline line must still print
        return None, 1, f"{type(e).__name__}: {e}"[:120]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    routes, prep = oracle_prepare()
    for _ in range(args.warmup):
        oracle_step(routes, prep)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        v, t = oracle_step(routes, prep)
        vals.append(v)
        secs += t
    v = statistics.median(vals)
    cores = len(os.sched_getaffinity(0))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "s8xu4->s32,f32 (W4A8) | f32 (W4A16)", "data": "synthetic",
        "config": {"workload": WORKLOAD, "m": 1, "layers": 16, "routes": "".join(str(r) for r in routes)},
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": "per step: layer 0 (W4A8) and layer 15 (W4A16) of the stack run in full by the "
                                   f"C oracle, extrapolated to the 15+1 mask; {secs:.1f} s of CPU work in total"},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip per-config single-linear rows")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start the N ranks ourselves
        # (one process per GPU, NCCL over 127.0.0.1), rank 0 prints the line
        import socket
        import subprocess
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; timing {world} rank(s)", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist = tdist
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)

    import paper_2604_21026_b200 as mq
    mq.load()

    prof = mq.profile_parse(open(GOLDEN_PROFILE).read())
    routes = prof.routes()
    st, weights, xs, ys = build_stack(mq, dev, routes)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        st.capture(1, stream=stream)
    wbytes = st.weight_bytes
    act_bytes = sum(v.numel() * 2 for v in xs.values()) + sum(v.numel() * 2 for v in ys.values())
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size

    with ClockSampler(local) as clk:
        ms = time_graph(st, stream, args.steps, args.warmup, dist)
    pct = step_percentiles(st, stream, args.steps)
    # max over ranks
    t = torch.tensor([ms], device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * wbytes / (ms_max * 1e-3) / 1e9
    L = len(routes)

    # route endpoints (tab:threshold all-W4A8 / all-W4A16), same weights
    st8 = stack_with_routes(mq, [0] * L, weights, xs, ys)
    st16 = stack_with_routes(mq, [1] * L, weights, xs, ys)
    with torch.cuda.stream(stream):
        st8.capture(1, stream=stream)
        st16.capture(1, stream=stream)
    ms8 = time_graph(st8, stream, args.steps, args.warmup)
    ms16 = time_graph(st16, stream, args.steps, args.warmup)

    # e2e: pinned host inputs -> H2D -> graph -> D2H, through mcapq_stack_step_host
    bi, bo = st.host_bytes(1)
    xh = torch.empty(bi, dtype=torch.uint8).pin_memory()
    yh = torch.empty(bo, dtype=torch.uint8).pin_memory()
    x0 = xs[(0, 0)].cpu().view(torch.uint8).flatten()     # the step's one input (layer 0's q/k/v input)
    assert bi == x0.numel(), (bi, x0.numel())
    xh[:bi] = x0
    for _ in range(args.warmup):
        st.step_host(xh, yh, 1, stream=stream)
    stream.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        st.step_host(xh, yh, 1, stream=stream)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    te = torch.tensor([e2e_ms], device=dev)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * wbytes / (float(te.item()) * 1e-3) / 1e9

    # roofline of the dominant kernel: the step graph holds ONE kernel (stack_step, the
    # whole routed step), so its per-launch time is the timed region's per-step time
    # (CUDA events on the launching stream).  Algorithmic bytes per launch = the step's
    # packed weights + every activation read once + every output written once.
    peak, peak_src = peaks()
    dram_peak, dram_peak_src = ncu_dram_peak()
    read_ceil = read_ceiling(mq, dev, stream)
    kernels_per_step = st.launches(1)
    step_alg_bytes = wbytes + act_bytes
    achieved = step_alg_bytes / (ms_max * 1e-3) / 1e9
    traffic, traffic_src = traffic_from_profiles("stack_step")
    # the per-linear kernel (what a non-persistent decode launches per linear): grouped gate+up
    k_ms, k_bytes, k_reps = time_dominant_kernel(mq, weights, xs, stream)
    k_traffic, k_traffic_src = traffic_from_profiles("stream_linear<0>")

    extras = [] if args.no_extras or rank != 0 else time_single_linears(mq, dev, stream)
    mlp8b = None if args.no_extras or rank != 0 else time_mlp8b_stack(mq, dev, stream)
    prefill = None if args.no_extras or rank != 0 else time_prefill(mq, dev, stream)
    sharded = None
    if world > 1 and not args.no_extras:
        try:
            sharded = time_sharded(mq, dev, stream, dist, world, rank)
        except Exception as e:   # the headline line must still print
            sharded = {"error": f"{type(e).__name__}: {e}"[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gbs, cores, secs = oracle_baseline()
        g1, _, s1 = oracle_baseline_1core()
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": "layer 0 (W4A8) + layer 15 (W4A16) of the same stack, each run in full by the C oracle "
                         f"(1 warm-up + median of 5, {secs:.1f} s timed), extrapolated to the 15+1 mask",
               "value_1core": None if g1 is None else round(g1, 4),
               "sample_1core": f"the same sample pinned to one CPU, OMP_NUM_THREADS=1 (1 warm-up + median of 3"
                               + (f", {s1:.1f} s timed)" if g1 is not None else f"; failed: {s1})")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "s8xu4->s32,f32 (W4A8) | bf16->f32 (W4A16)",
            "data": "synthetic (seeded bf16 weights/activations, random init)",
            "config": {"workload": WORKLOAD,
                       "m": 1, "layers": L, "routes": "".join(str(r) for r in routes),
                       "weight_bytes_per_step": wbytes, "activation_bytes_per_step": act_bytes,
                       "l2_policy": f"no flush: {wbytes / 1e6:.0f} MB of weights per step > {l2 / 1e6:.0f} MB L2",
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
            "step_ms_percentiles": pct,
            "us_per_layer": round(ms_max * 1000 / L, 3),
            "us_per_linear": round(ms_max * 1000 / (L * len(SLOTS)), 3),
            "routes_endpoints": {"all_w4a8_gbs": round(wbytes / (ms8 * 1e-3) / 1e9, 1),
                                 "all_w4a16_gbs": round(wbytes / (ms16 * 1e-3) / 1e9, 1),
                                 "all_w4a8_us_per_layer": round(ms8 * 1000 / L, 3),
                                 "all_w4a16_us_per_layer": round(ms16 * 1000 / L, 3),
                                 "w4a8_over_w4a16": round(ms16 / ms8, 3)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "stack_step (persistent routed decode step: all 112 linears, one launch)"
                         if kernels_per_step == 1 else "stack (per-linear launches)",
                         "alg_bytes_per_launch": step_alg_bytes, "us_per_launch": round(ms_max * 1000, 3),
                         "launches_timed": args.steps, "peak_source": peak_src,
                         "other_denominators": {
                             "ncu_dram_peak_gbs": dram_peak, "frac_ncu_dram_peak":
                                 round(achieved / dram_peak, 4) if dram_peak else None,
                             "ncu_dram_peak_source": dram_peak_src,
                             "read_ceiling_gbs": read_ceil, "frac_read_ceiling": round(achieved / read_ceil, 4),
                             "read_ceiling_source": "mcapq_debug_read_bw, 1 GiB streaming LDG.128, this run"}},
            "per_linear_kernel": {"kernel": "stream_linear<DP4A> grouped gate+up (2 x 8192x2048, M=1, fused "
                                            "quantiser), launched alone, rotating 16 layers' weights",
                                  "achieved": round(k_bytes / (k_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
                                  "frac": round(k_bytes / (k_ms * 1e-3) / 1e9 / peak, 4),
                                  "alg_bytes_per_launch": k_bytes, "us_per_launch": round(k_ms * 1000, 3),
                                  "launches_timed": k_reps, "traffic": k_traffic, "traffic_source": k_traffic_src},
            "e2e": {"value": round(e2e_value, 1), "unit": "GB/s", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
                    "ms_per_step": round(float(te.item()), 5), "api": "mcapq_stack_step_host"},
            "gpu_launches": kernels_per_step * args.steps,
            "kernels_per_step": kernels_per_step,
            "clocks": clk.report(),
            "single_linears": extras,
            "mlp_8b_stack": mlp8b,
            "prefill_8b": prefill,
            "sharded": sharded,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

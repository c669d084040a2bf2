"""Per-linear timeline of the persistent step kernel (MCAPQ_STREAM_TRACE=1), one graph
replay of the 1B stack.  Per op, medians over the CTAs that own tiles (us):
go (barrier wait), stage (x load + quantise), wfirst (first weight stage after
staging), compute (first stage -> last tile's compute), epi (last epilogue), and the
op's span.  Diagnostic only.

    MCAPQ_STREAM_TRACE=1 python scripts/trace_step.py [--routes 0|1|golden] [--independent]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_21026_b200 as mq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--routes", default="golden")
    ap.add_argument("--independent", action="store_true")
    ap.add_argument("--ops", type=int, default=64)
    ap.add_argument("--mlp8b", action="store_true", help="the 8-layer Llama-3.1-8B MLP stack instead")
    ap.add_argument("--no-epilogue", action="store_true", help="a build without the epilogue records (A/B)")
    args = ap.parse_args()
    assert os.environ.get("MCAPQ_STREAM_TRACE") == "1"
    dev = torch.device("cuda:0")
    mq.load()
    routes = (mq.profile_parse(open(bench.GOLDEN_PROFILE).read()).routes() if args.routes == "golden"
              else [int(args.routes)] * 16)
    if args.mlp8b:
        import synth_inputs as si
        L = 8
        route = 0 if args.routes in ("golden", "0") else 1
        shapes = {s_: si.linear_shape("llama-3.1-8b", s_) for s_ in ("gate", "up", "down")}
        base = {s_: mq.pack_w4(si.weight(n, k, 7 + i).to(dev)) for i, (s_, (n, k)) in enumerate(shapes.items())}
        keep = []
        st = mq.Stack([route] * L, max_m=1)
        prev = si.activation(1, 4096, 9).to(dev)
        for l in range(L):
            w = {s_: mq.PackedW4(base[s_].nib.clone(), base[s_].scale.clone()) for s_ in shapes}
            y = {s_: torch.empty(1, shapes[s_][0], dtype=torch.bfloat16, device=dev) for s_ in shapes}
            st.set(l, 0, 0, w["gate"], prev, y["gate"])
            st.set(l, 1, 0, w["up"], prev, y["up"])
            st.set(l, 2, 1, w["down"], y["up"], y["down"])
            keep.append((w, y, prev))
            prev = y["down"]
    else:
        st, _, _, _ = bench.build_stack(mq, dev, routes, chain=not args.independent)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        st.run(1, stream=stream)
        stream.synchronize()
        st.capture(1, stream=stream)
        for _ in range(3):
            st.replay(stream=stream)
        stream.synchronize()
    buf = np.zeros((1 << 16, 8), np.uint64)
    n = mq.load().mcapq_debug_stream_trace(ctypes.c_void_p(buf.ctypes.data), buf.shape[0])
    rec = buf[:n].astype(np.int64)
    half = n if args.no_epilogue else n // 2
    ep = rec[half:n]          # epilogue records: [op][cta] {last tile start, stores issued}
    rec = rec[:half]
    nops_ = half // max(1, int(rec[:, 1].max() >> 48) + 1) if half else 0
    t0 = rec[rec[:, 2] > 0, 2].min()
    print(f"{'op':>3} {'ctas':>4} {'start':>8} {'go':>6} {'stage':>6} {'wfirst':>6} {'compute':>7} {'epi':>6} "
          f"{'end_med':>8} {'end_max':>8} {'stages':>6} {'stalled':>7} {'load':>6} {'ep_med':>8} {'ep_max':>8}")
    tot = np.zeros(5)
    for op in range(min(args.ops, int(rec[:, 0].max()) + 1)):
        r = rec[(rec[:, 0] == op) & (rec[:, 6] > 0)]
        if len(r) == 0:
            continue
        d = np.median(np.stack([r[:, 3] - r[:, 2], r[:, 4] - r[:, 3], r[:, 6] - r[:, 4], r[:, 7] - r[:, 6],
                                r[:, 5] - r[:, 7]], 1), 0) / 1000
        load = np.median((r[:, 1] >> 32) & 0xFFFF) / 1000   # go -> input loaded and checked
        tot += d
        grid = int(rec[:, 1].max() >> 48) + 1
        e = ep[op * grid:(op + 1) * grid]
        e = e[e[:, 1] > 0]
        ep_s = f"{(np.median(e[:, 1]) - t0) / 1000:8.2f} {(e[:, 1].max() - t0) / 1000:8.2f}" if len(e) else ""
        print(f"{op:3d} {len(r):4d} {(np.median(r[:, 2]) - t0) / 1000:8.2f} {d[0]:6.2f} {d[1]:6.2f} {d[2]:6.2f} "
              f"{d[3]:7.2f} {d[4]:6.2f} {(np.median(r[:, 5]) - t0) / 1000:8.2f} {(r[:, 5].max() - t0) / 1000:8.2f} "
              f"{np.mean(r[:, 1] & 0xFFFF):6.2f} {np.mean((r[:, 1] >> 16) & 0xFFFF):7.2f} {load:6.2f} {ep_s}")
    print("sum of medians (go, stage, wfirst, compute, epi):", np.round(tot, 2))
    print("total span us:", (rec[:, 5].max() - t0) / 1000)


if __name__ == "__main__":
    main()

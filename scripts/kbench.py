"""Kernel microbenchmark: per-launch time of the routed decode linears, launches
captured in a CUDA graph (no host overhead), rotating over enough weight copies
to defeat the 126 MB L2.  One JSON line per (case, route).

    python scripts/kbench.py [--cases a,b] [--reps N] [--tag T]

Environment knobs of the stream kernel (MCAPQ_STREAM_*) are read once at load.
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_21026_b200 as mq  # noqa: E402
import synth_inputs as si  # noqa: E402

CASES = {
    # name: (list of (n, k) sharing one input, m)
    "gateup_1b": ([(8192, 2048), (8192, 2048)], 1),
    "qkv_1b": ([(2048, 2048), (512, 2048), (512, 2048)], 1),
    "o_1b": ([(2048, 2048)], 1),
    "down_1b": ([(2048, 8192)], 1),
    "gate_8b": ([(14336, 4096)], 1),
    "gateup_8b": ([(14336, 4096), (14336, 4096)], 1),
    "down_8b": ([(4096, 14336)], 1),
    "lmhead_8b": ([(128256, 4096)], 1),
    "up_3b_m16": ([(8192, 3072)], 16),
    "q_3b_m64": ([(3072, 3072)], 64),
    "lmhead_8b_m64": ([(128256, 4096)], 64),
    "lmhead_8b_m16": ([(128256, 4096)], 16),
    "lmhead_8b_m32": ([(128256, 4096)], 32),
    "up_3b_m64": ([(8192, 3072)], 64),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="gateup_1b,qkv_1b,down_1b,gate_8b,down_8b,lmhead_8b")
    ap.add_argument("--routes", default="0,1")
    ap.add_argument("--reps", type=int, default=0)
    ap.add_argument("--tag", default="")
    ap.add_argument("--pdl", type=int, default=1, help="launch with programmatic dependent launch (mcapq_set_pdl)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    mq.load()
    mq.set_pdl(bool(args.pdl))
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    stream = torch.cuda.Stream()
    env = {k: v for k, v in os.environ.items() if k.startswith("MCAPQ_")}
    for name in args.cases.split(","):
        shapes, m = CASES[name]
        wbytes = sum(n * k // 2 + n * (k // 32) * 2 for n, k in shapes)
        copies = max(2, min(64, math.ceil(3 * l2 / wbytes)))
        base = [mq.pack_w4(si.weight(n, k, 7 + i).to(dev)) for i, (n, k) in enumerate(shapes)]
        sets = [[mq.PackedW4(b.nib.clone(), b.scale.clone()) for b in base] for _ in range(copies)]
        k = shapes[0][1]
        x = si.activation(m, k, 9).to(dev)
        outs = [torch.empty(m, n, dtype=torch.bfloat16, device=dev) for n, _ in shapes]
        for route in [int(r) for r in args.routes.split(",")]:
            reps = args.reps or max(copies, 32)
            ws = torch.empty(max(256, mq.workspace_bytes(min(route, 1), m, max(n for n, _ in shapes), k)), dtype=torch.uint8,
                             device=dev)

            def call(i):
                if route == 2:   # a6 with bf16-dequantised weights (tcgen05 kernel)
                    for w_, y_ in zip(sets[i % copies], outs):
                        mq.w4a16_bf16deq(w_, x, out=y_, stream=stream)
                else:
                    mq.linear_group(route, sets[i % copies], x, outs=outs, ws=ws, stream=stream)

            with torch.cuda.stream(stream):
                for i in range(copies):     # descriptors of every copy encoded outside the capture
                    call(i)
                stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for i in range(reps):
                        call(i)
                g.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                best = 1e30
                for _ in range(5):
                    e0.record(stream)
                    g.replay()
                    e1.record(stream)
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1) * 1000 / reps)
            print(json.dumps({"tag": args.tag, "case": name, "route": ["w4a8", "w4a16", "w4a16_bf16deq"][route], "m": m,
                              "us": round(best, 3), "GBps": round(wbytes / best / 1e3, 1), "weight_bytes": wbytes,
                              "copies": copies, "reps": reps, "env": env}), flush=True)
        del sets, base
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

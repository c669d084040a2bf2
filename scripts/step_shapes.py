"""Diagnostic: stream rate of the persistent step kernel on uniform synthetic
programs (MCAPQ_STEP_FLAGS applies).  One JSON line per program."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_21026_b200 as mq  # noqa: E402
import synth_inputs as si  # noqa: E402

PROGRAMS = {
    "gateup16": (16, [(8192, 2048), (8192, 2048)]),     # 16 ops of 2 x 8192x2048 (one group each)
    "down16": (16, [(2048, 8192)]),
    "q16": (16, [(2048, 2048)]),
    "big4": (4, [(32768, 4096)]),
    "big1": (1, [(131072, 4096)]),
}


def main():
    dev = torch.device("cuda:0")
    mq.load()
    for name, (L, shapes) in PROGRAMS.items():
        st = mq.Stack([0] * L, max_m=1)
        keep = []
        for l in range(L):
            k = shapes[0][1]
            x = si.activation(1, k, 5 + l).to(dev)
            for sl, (n, kk) in enumerate(shapes):
                w = mq.PackedW4(torch.randint(0, 255, (n, kk // 2), dtype=torch.uint8, device=dev),
                                torch.full((n, kk // 32), 0x2000, dtype=torch.int16, device=dev))
                y = torch.empty(1, n, dtype=torch.bfloat16, device=dev)
                st.set(l, sl, 0, w, x, y)
                keep.append((w, x, y))
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            st.capture(1, stream=stream)
        ms = bench.time_graph(st, stream, 50, 5)
        print(json.dumps({"program": name, "env": {k: v for k, v in os.environ.items() if k.startswith("MCAPQ_")},
                          "ms": round(ms, 4), "GBps": round(st.weight_bytes / ms / 1e6, 1),
                          "launches": st.launches(1)}), flush=True)
        del st, keep
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

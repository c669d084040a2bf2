"""Time one graph replay of the persistent 1B decode-step kernel (diagnostic).
Environment knobs (MCAPQ_STEP_FLAGS: 1 no compute, 2 no barrier, 4 no staging;
MCAPQ_STEP_SMEM_KB) are read once at library load.  Prints one JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_21026_b200 as mq  # noqa: E402


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--routes", default="golden")
    ap.add_argument("--independent", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    mq.load()
    if args.routes == "golden":
        routes = mq.profile_parse(open(bench.GOLDEN_PROFILE).read()).routes()
    else:
        routes = [int(args.routes)] * 16
    st, weights, xs, ys = bench.build_stack(mq, dev, routes, chain=not args.independent)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        st.capture(1, stream=stream)
    ms = bench.time_graph(st, stream, 100, 10)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MCAPQ_")},
                      "routes": args.routes, "chain": not args.independent,
                      "ms_per_step": round(ms, 4), "GBps": round(st.weight_bytes / ms / 1e6, 1),
                      "launches": st.launches(1)}), flush=True)


if __name__ == "__main__":
    main()

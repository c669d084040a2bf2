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


def build_mlp8b(mq, dev, route, L=8):
    import synth_inputs as si
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
    return st, keep


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--routes", default="golden")
    ap.add_argument("--independent", action="store_true")
    ap.add_argument("--mlp8b", action="store_true", help="the 8-layer Llama-3.1-8B MLP stack instead")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    mq.load()
    if args.routes == "golden":
        routes = mq.profile_parse(open(bench.GOLDEN_PROFILE).read()).routes()
    else:
        routes = [int(args.routes)] * 16
    if args.mlp8b:
        st, keep = build_mlp8b(mq, dev, 0 if args.routes in ("golden", "0") else 1)
    else:
        st, weights, xs, ys = bench.build_stack(mq, dev, routes, chain=not args.independent)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        st.capture(1, stream=stream)
    ms = bench.time_graph(st, stream, 100, 10)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MCAPQ_")},
                      "routes": args.routes, "chain": not args.independent, "mlp8b": args.mlp8b,
                      "us_per_layer": round(ms * 1000 / (8 if args.mlp8b else 16), 3),
                      "ms_per_step": round(ms, 4), "GBps": round(st.weight_bytes / ms / 1e6, 1),
                      "launches": st.launches(1)}), flush=True)


if __name__ == "__main__":
    main()

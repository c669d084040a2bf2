"""A small persistent-step program for compute-sanitizer (racecheck / synccheck / memcheck):
2 layers (W4A8, W4A16) of a reduced decode chain, x_o = y_q, x_gate/up = y_o, x_down = y_up
with K = 4096 for down (so the W4A8 layer's down reads producer-quantised records across
the cluster pair), run once eagerly and replayed twice from a graph; outputs checked
against the per-linear path.
    compute-sanitizer --tool racecheck python scripts/sanitize_step.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_21026_b200 as mq  # noqa: E402
import synth_inputs as si  # noqa: E402

DIMS = {"q": (2048, 2048), "k": (256, 2048), "v": (256, 2048), "o": (2048, 2048), "gate": (4096, 2048),
        "up": (4096, 2048), "down": (2048, 4096)}
INP = {"q": 0, "k": 0, "v": 0, "o": 1, "gate": 2, "up": 2, "down": 3}
SRC = {"o": "q", "gate": "o", "up": "o", "down": "up"}


def main():
    dev = torch.device("cuda:0")
    mq.load()
    routes = [0, 1]
    st = mq.Stack(routes, max_m=1)
    ops, ys = [], {}
    prev = si.activation(1, 2048, 3000).to(dev)
    for l, r in enumerate(routes):
        for sid, (slot, (n, k)) in enumerate(DIMS.items()):
            x = prev if slot in ("q", "k", "v") else ys[(l, SRC[slot])]
            if x.shape[-1] != k:   # shapes chosen to chain exactly
                raise SystemExit(f"shape chain broken at {slot}")
            pw = mq.pack_w4(si.weight(n, k, 3001 + 16 * l + sid).to(dev))
            y = torch.empty(1, n, dtype=torch.bfloat16, device=dev)
            st.set(l, sid, INP[slot], pw, x, y)
            ys[(l, slot)] = y
            ops.append((r, pw, x, y))
        prev = ys[(l, "down")]
    st.run(1)
    torch.cuda.synchronize()
    first = [y.clone() for (_, _, _, y) in ops]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.capture(1, stream=s)
        for _ in range(2):
            st.replay(stream=s)
    s.synchronize()
    bad = 0
    for a, (r, pw, x, y) in zip(first, ops):
        ref = mq.linear(r, pw, x.clone(), out_dtype=torch.bfloat16)
        bad += int(not torch.equal(ref, y)) + int(not torch.equal(a, y))
    torch.cuda.synchronize()
    print("launches", st.launches(1), "mismatches", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

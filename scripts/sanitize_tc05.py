"""The tcgen05 batched W4A8 kernel (tc05_w4a8) and the row-parallel reduction under
compute-sanitizer (memcheck / synccheck / racecheck): MCAPQ_GEMM_A8_TC05=2 forces the
tcgen05 path at any N; passes of 16, 33 and 64 tokens (MP = 16 / 64, the two-set and
one-set epilogues, ragged N); outputs checked against the oracle within reading T.
    MCAPQ_GEMM_A8_TC05=2 compute-sanitizer --tool memcheck python scripts/sanitize_tc05.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2604_21026_b200 as mq  # noqa: E402
import synth_inputs as si  # noqa: E402


def main():
    assert os.environ.get("MCAPQ_GEMM_A8_TC05") == "2", "run with MCAPQ_GEMM_A8_TC05=2"
    dev = torch.device("cuda:0")
    mq.load()
    n, k = 200, 1024
    w = si.weight(n, k, 4100)
    pw = mq.pack_w4(w.to(dev))
    nib, sc = oracle.pack_w4(w.float().numpy())
    worst = 0.0
    for m in (16, 33, 64):
        x = si.activation(m, k, 4101 + m)
        y = mq.linear(mq.W4A8, pw, x.to(dev), out_dtype=torch.float32)
        torch.cuda.synchronize()
        _, ref = oracle.w4a8_from_x(nib, sc, x.float().numpy())
        rms = np.sqrt(np.mean(ref ** 2))
        err = np.abs(y.cpu().numpy().astype(np.float64) - ref) / np.maximum(np.abs(ref), rms)
        worst = max(worst, float(err.max()))
    parts = torch.randn(3, 5, 40, device=dev)
    r = mq.rowshard_reduce(parts, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(r, parts[0] + parts[1] + parts[2])
    assert worst <= 1e-3, worst
    print(f"ok: tc05_w4a8 M = 16/33/64 max rel err {worst:.2e}; rowshard_reduce exact")


if __name__ == "__main__":
    main()

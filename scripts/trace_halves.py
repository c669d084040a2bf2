"""Per-op end times split by CTA halves (gate/up: CTAs of the gate tiles vs the up tiles),
from one traced replay of the 1B golden step.  MCAPQ_STREAM_TRACE=1 python scripts/trace_halves.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2604_21026_b200 as mq  # noqa: E402

dev = torch.device("cuda:0")
mq.load()
routes = mq.profile_parse(open(bench.GOLDEN_PROFILE).read()).routes()
st, _, _, _ = bench.build_stack(mq, dev, routes, chain=True)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    st.run(1, stream=s)
    s.synchronize()
    st.capture(1, stream=s)
    for _ in range(3):
        st.replay(stream=s)
    s.synchronize()
buf = np.zeros((1 << 16, 8), np.uint64)
n = mq.load().mcapq_debug_stream_trace(ctypes.c_void_p(buf.ctypes.data), buf.shape[0])
rec = buf[:n].astype(np.int64)
half = n // 2
ep = rec[half:n]
rec = rec[:half]
t0 = rec[rec[:, 2] > 0, 2].min()
grid = int(rec[:, 1].max() >> 48) + 1
for op in (2, 3, 6, 7, 10, 11):
    r = rec[(rec[:, 0] == op) & (rec[:, 6] > 0)]
    cta = (r[:, 1] >> 48)
    e = ep[op * grid:(op + 1) * grid]
    lo, hi = cta < grid // 2, cta >= grid // 2
    f = lambda m, col: (np.median(r[m, col]) - t0) / 1000
    eg = ep[op * grid:(op + 1) * grid]
    el = eg[:grid // 2]; eh = eg[grid // 2:]
    el = el[el[:, 1] > 0]; eh = eh[eh[:, 1] > 0]
    print(f"op {op}: compute-end med lo {f(lo, 7):.2f} hi {f(hi, 7):.2f} | end med lo {f(lo, 5):.2f} hi {f(hi, 5):.2f} "
          f"| ep lo med {(np.median(el[:, 1]) - t0) / 1000 if len(el) else 0:.2f} max {(el[:, 1].max() - t0) / 1000 if len(el) else 0:.2f} "
          f"hi med {(np.median(eh[:, 1]) - t0) / 1000 if len(eh) else 0:.2f} max {(eh[:, 1].max() - t0) / 1000 if len(eh) else 0:.2f}")

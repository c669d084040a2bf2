"""Timeline of one graph replay of the 1B decode-linear stack (MCAPQ_STREAM_TRACE=1):
per launch, the first CTA start, the median 'after griddepcontrol.wait',
'activations ready' and CTA end, relative to the replay start.  Diagnostic only.

    MCAPQ_STREAM_TRACE=1 python scripts/trace_stack.py [--routes 0|1|golden] [--launches 16]
"""
import argparse
import ctypes
import os
import statistics
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
    ap.add_argument("--launches", type=int, default=24)
    args = ap.parse_args()
    assert os.environ.get("MCAPQ_STREAM_TRACE") == "1"
    dev = torch.device("cuda:0")
    mq.load()
    if args.routes == "golden":
        routes = mq.profile_parse(open(bench.GOLDEN_PROFILE).read()).routes()
    else:
        routes = [int(args.routes)] * 16
    st, weights, xs, ys = bench.build_stack(mq, dev, routes)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        st.run(1, stream=stream)          # allocates the trace buffer outside the capture
        stream.synchronize()
        st.capture(1, stream=stream)
        for _ in range(3):
            st.replay(stream=stream)
        stream.synchronize()
    buf = np.zeros((1 << 16, 8), np.uint64)
    n = mq.load().mcapq_debug_stream_trace(ctypes.c_void_p(buf.ctypes.data), buf.shape[0])
    rec = buf[:n]
    launches = sorted(set(int(v) for v in rec[:, 0]))
    t0 = None
    print(f"{'launch':>6} {'ctas':>5} {'start_min':>9} {'start_med':>9} {'wait_med':>9} {'x_med':>9} {'ready_med':>9} "
          f"{'stage1':>9} {'end_med':>9} {'end_max':>9}  (us, relative to the first launch's first CTA start)")
    rows = []
    for lid in launches:
        r = rec[rec[:, 0] == lid]
        r = r[r[:, 2] > 0]
        if len(r) == 0:
            continue
        rows.append((lid, r))
    t0 = min(int(r[:, 2].min()) for _, r in rows)
    for lid, r in rows[: args.launches]:
        f = lambda col: (r[:, col].astype(np.int64) - t0) / 1000.0  # noqa: E731
        fx = np.median(f(6)) if (r[:, 6] > 0).all() else float("nan")
        print(f"{lid:6d} {len(r):5d} {f(2).min():9.2f} {np.median(f(2)):9.2f} {np.median(f(3)):9.2f} {fx:9.2f} "
              f"{np.median(f(4)):9.2f} {np.median(f(7)):9.2f} {np.median(f(5)):9.2f} {f(5).max():9.2f}")
    ends = [((r[:, 5].astype(np.int64) - t0).max()) / 1000 for _, r in rows]
    print("total span us:", max(ends))


if __name__ == "__main__":
    main()

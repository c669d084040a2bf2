"""NEXT-4 microbenchmark: dequantise-once + tcgen05 bf16 GEMM (mcapq_w4a16_bf16deq_prefill) and the
GEMM alone on a resident W^ (mcapq_bf16w_gemm), CUDA-graph timed; one JSON line per case.
    python scripts/prefill_bench.py [--cases gate_8b:512,lmhead_8b:256]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_21026_b200 as mq  # noqa: E402
import synth_inputs as si  # noqa: E402

SHAPES = {"gate_8b": (14336, 4096), "down_8b": (4096, 14336), "lmhead_8b": (128256, 4096), "up_3b": (8192, 3072)}


def timed(fn, stream, reps=10):
    with torch.cuda.stream(stream):
        fn()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                fn()
        g.replay()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(3):
            e0.record(stream)
            g.replay()
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1000 / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="gate_8b:256,gate_8b:1024,gate_8b:4096,lmhead_8b:256,down_8b:1024")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    mq.load()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 2250.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 2250.0
    stream = torch.cuda.Stream()
    for case in args.cases.split(","):
        name, m = case.split(":")
        m = int(m)
        n, k = SHAPES[name]
        pw = mq.pack_w4(si.weight(n, k, 11).to(dev))
        x = si.activation(m, k, 12).to(dev)
        y = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
        ws = torch.empty(mq.load().mcapq_prefill_workspace_bytes(n, k), dtype=torch.uint8, device=dev)
        wdq = mq.dequant_w4_bf16(pw)
        t_pre = timed(lambda: mq.w4a16_bf16deq_prefill(pw, x, out=y, ws=ws, stream=stream), stream)
        t_gemm = timed(lambda: mq.bf16w_gemm(wdq, x, out=y, stream=stream), stream)
        t_dq = timed(lambda: mq.dequant_w4_bf16(pw, out=wdq, stream=stream), stream)
        fl = 2.0 * m * n * k
        print(json.dumps({"case": name, "M": m, "N": n, "K": k, "prefill_us": round(t_pre, 2),
                          "gemm_us": round(t_gemm, 2), "dequant_us": round(t_dq, 2),
                          "prefill_tflops": round(fl / t_pre / 1e6, 1), "gemm_tflops": round(fl / t_gemm / 1e6, 1),
                          "gemm_tensor_frac": round(fl / t_gemm / 1e6 / peak, 4),
                          "dequant_gbs": round(n * k * (0.5625 + 2.0) / t_dq / 1e3, 1)}), flush=True)
        del pw, x, y, ws, wdq
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

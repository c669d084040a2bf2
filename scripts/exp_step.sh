#!/bin/bash
# step-kernel A/B: probe (1B chain, golden mask), trace, 8B MLP stack bench rows, step parity tests
O=${1:-gpurun_out/step}; mkdir -p $O
ROUTES=golden TRACE=0 bash scripts/step_matrix.sh $O "MCAPQ_STEP_FLAGS=0"
MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes 0 > $O/trace.txt 2>&1
MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes 0 --mlp8b > $O/trace8b.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "step or stack or quant" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt

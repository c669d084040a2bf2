#!/bin/bash
# step-kernel iteration: parity tests of the step paths, probe matrix, one trace
# usage: bash scripts/step_ab.sh OUTDIR "ENV1;ENV2;..."
O=${1:-gpurun_out/step}; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -x -q -k "step or stack" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
ROUTES=golden TRACE=0 bash scripts/step_matrix.sh $O "${2:-MCAPQ_STEP_FLAGS=0}"
env ${TRACE_ENV:-MCAPQ_STEP_FLAGS=0} MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace.txt 2>&1

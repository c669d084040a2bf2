O=gpurun_out/diag1; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
ROUTES=golden TRACE=0 bash scripts/step_matrix.sh $O "MCAPQ_STEP_FLAGS=0;MCAPQ_STEP_FLAGS=8;MCAPQ_STEP_FLAGS=520;MCAPQ_STEP_FLAGS=9;MCAPQ_STEP_FLAGS=256;MCAPQ_STEP_FLAGS=1;MCAPQ_STEP_EP_LOG2=3;MCAPQ_STEP_FLAGS=0"
MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace0.txt 2>&1
MCAPQ_STEP_EP_LOG2=3 MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace_ep3.txt 2>&1
MCAPQ_STEP_FLAGS=8 MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace_f8.txt 2>&1
MCAPQ_STEP_FLAGS=1 MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace_f1.txt 2>&1

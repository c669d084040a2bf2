O=gpurun_out/exp2; mkdir -p $O
for c in 1 2; do for kb in 112 226; do for nc in 0 1; do
  MCAPQ_STREAM_CTAS_PER_SM=$c MCAPQ_STREAM_SMEM_KB=$kb MCAPQ_STREAM_NOCOMPUTE=$nc timeout 120 python scripts/kbench.py --cases lmhead_8b,gate_8b --routes 0 --tag "c$c-kb$kb-nc$nc" >> $O/kb.jsonl 2>>$O/err.txt
done; done; done
ROUTES=0 TRACE=0 bash scripts/step_matrix.sh $O "MCAPQ_STEP_FLAGS=13 MCAPQ_STEP_SMEM_KB=120;MCAPQ_STEP_FLAGS=13 MCAPQ_STEP_SMEM_KB=160;MCAPQ_STEP_FLAGS=13 MCAPQ_STEP_SMEM_KB=226;MCAPQ_STEP_FLAGS=0 MCAPQ_STEP_SMEM_KB=226;MCAPQ_STEP_FLAGS=0 MCAPQ_STEP_SMEM_KB=160"

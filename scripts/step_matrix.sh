#!/bin/bash
# Step-kernel diagnostic matrix (one JSON line per probe) + per-op traces.
#   bash scripts/step_matrix.sh OUTDIR "ENV1;ENV2;..."   (each ENV a space-separated VAR=VAL list)
OUT=${1:-gpurun_out/sm}
CASES=${2:-"MCAPQ_STEP_FLAGS=0"}
ROUTES=${ROUTES:-"0 1"}
mkdir -p $OUT
IFS=';' read -ra CS <<< "$CASES"
for r in $ROUTES; do
  for c in "${CS[@]}"; do
    env $c timeout 120 python scripts/step_probe.py --routes $r $PROBE_ARGS >> $OUT/probe.jsonl 2>>$OUT/err.txt
  done
done
if [ "${TRACE:-1}" = "1" ]; then
  for r in $ROUTES; do
    env ${TRACE_ENV:-MCAPQ_STEP_FLAGS=0} MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes $r > $OUT/trace_r$r.txt 2>&1
  done
fi

#!/bin/bash
# A/B of library builds on the step kernel: bash scripts/ab.sh OUTDIR "lib1 lib2 ..." "ENV1;ENV2"
# (each lib a path; "cur" = the in-tree build).  Runs the step parity tests on the in-tree
# build first, then one step_probe line per (lib, env, routes).
O=${1:-gpurun_out/ab}; mkdir -p $O
LIBS=${2:-"cur"}
CASES=${3:-"MCAPQ_STEP_FLAGS=0"}
ROUTES=${ROUTES:-"golden"}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTK:-step or stack}" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
fi
IFS=';' read -ra CS <<< "$CASES"
for rep in $(seq 1 ${REPS:-2}); do
for lib in $LIBS; do
  for r in $ROUTES; do
    for c in "${CS[@]}"; do
      if [ "$lib" = "cur" ]; then L=""; else L="MCAPQ_LIB=$lib"; fi
      echo -n "{\"lib\": \"$lib\", \"rep\": $rep, \"probe\": " >> $O/ab.jsonl
      env $L $c timeout 120 python scripts/step_probe.py --routes $r $PROBE_ARGS >> $O/ab.jsonl 2>>$O/err.txt || echo "null" >> $O/ab.jsonl
      sed -i '$ s/$/}/' $O/ab.jsonl
    done
  done
done
done

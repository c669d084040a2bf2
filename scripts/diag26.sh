O=gpurun_out/diag26; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for rep in 1 2; do for c in "MCAPQ_STEP_REC_SPIN=64" "MCAPQ_STEP_REC_SPIN=0" "MCAPQ_STEP_REC_SPIN=256" "MCAPQ_STEP_REC_SPIN=1024" "MCAPQ_STEP_REC_R=0.45" "MCAPQ_STEP_REC_R=0.75"; do
  echo -n "$c " >> $O/probe.txt; env $c timeout 60 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
  echo -n "$c " >> $O/probe.txt; env $c timeout 60 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.txt 2>>$O/err.txt
done; done

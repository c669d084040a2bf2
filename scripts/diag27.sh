O=gpurun_out/diag27; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for rep in 1 2; do for c in "MCAPQ_STEP_REC_MINK=4096" "MCAPQ_STEP_REC_MINK=2048" "MCAPQ_STEP_REC_MINK=2048 MCAPQ_STEP_REC_R=0.3" "MCAPQ_STEP_REC_MINK=2048 MCAPQ_STEP_REC_R=1.5"; do
  echo -n "$c|" >> $O/probe.txt; env $c timeout 60 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
done; done
MCAPQ_STEP_REC_MINK=2048 timeout 300 python -m pytest tests -m gpu -x -q -k "step or stack or record" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt

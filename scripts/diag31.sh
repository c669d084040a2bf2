O=gpurun_out/diag31; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for rep in 1 2; do for c in "MCAPQ_STEP_EP_LOG2=1" "MCAPQ_STEP_EP_LOG2=2" "MCAPQ_STEP_SMEM_KB=180" "MCAPQ_STEP_SMEM_KB=220" "MCAPQ_STEP_HOLD=0" "MCAPQ_STEP_SPIN_NS=32" "MCAPQ_STEP_POLLS=2"; do
  echo -n "$c|" >> $O/probe.txt; env $c timeout 60 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
  echo -n "$c|" >> $O/probe.txt; env $c timeout 60 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.txt 2>>$O/err.txt
done; done

O=gpurun_out/diag12; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "step or stack or record" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for e in "MCAPQ_STEP_ILV=1" "MCAPQ_STEP_ILV=0"; do
  env $e timeout 120 python scripts/step_probe.py --routes golden >> $O/probe.jsonl 2>>$O/err.txt
  env $e timeout 120 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.jsonl 2>>$O/err.txt
done; done
MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace_ilv.txt 2>&1

O=gpurun_out/diag6; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for rep in 1 2; do for e in "MCAPQ_STEP_FLAGS=0" "MCAPQ_STEP_FLAGS=2048"; do
  env $e timeout 120 python scripts/step_probe.py --routes golden >> $O/probe.jsonl 2>>$O/err.txt
  env $e timeout 120 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.jsonl 2>>$O/err.txt
done; done
MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace0.txt 2>&1
timeout 300 python scripts/kbench.py --cases lmhead_8b,gate_8b,down_8b --routes 1 > $O/kb.txt 2>&1
timeout 600 python scripts/sharded_p1.py > $O/sharded_p1.json 2> $O/sharded_p1.err
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt

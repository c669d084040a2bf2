O=gpurun_out/diag2; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for e in "MCAPQ_STEP_FLAGS=0" "MCAPQ_STEP_FLAGS=128" "MCAPQ_STEP_HOLD=0" "MCAPQ_STEP_FLAGS=4"; do
  env $e timeout 120 python scripts/step_probe.py --routes golden >> $O/probe.jsonl 2>>$O/err.txt
  env $e MCAPQ_STREAM_TRACE=1 timeout 120 python scripts/trace_step.py --routes golden > $O/trace_$(echo $e | tr '=' '_').txt 2>&1
done
# W4A16 M=1 stream kernel A/B: base vs lean vs lean-1CTA
for lib in base lean v1cta; do
  for c in "" "MCAPQ_STREAM_CTAS_PER_SM=1"; do
    echo "== $lib $c" >> $O/kb.txt
    env MCAPQ_LIB=_ab/$lib/libmcapq.so $c timeout 300 python scripts/kbench.py --cases lmhead_8b,gate_8b,down_8b,gateup_1b,down_1b --routes 1 >> $O/kb.txt 2>&1
  done
done
timeout 600 python -m pytest tests -m gpu -x -q -k "w4a16 or a16 or hmma or W4A16 or route" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt

O=gpurun_out/diag3; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for c in "" "MCAPQ_STREAM_SMEM_KB=160" "MCAPQ_STREAM_SMEM_KB=200"; do
  echo "== cur $c" >> $O/kb.txt
  env $c timeout 300 python scripts/kbench.py --cases lmhead_8b,gate_8b,down_8b,gateup_1b,down_1b,qkv_1b,o_1b --routes 1 >> $O/kb.txt 2>&1
done
echo "== cur a8" >> $O/kb.txt
timeout 300 python scripts/kbench.py --cases lmhead_8b,gate_8b,down_8b --routes 0 >> $O/kb.txt 2>&1
for lib in base cur; do
  for r in golden 1; do
    if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
    env $L timeout 120 python scripts/step_probe.py --routes $r >> $O/probe_$lib.jsonl 2>>$O/err.txt
  done
  env $L timeout 120 python scripts/step_probe.py --mlp8b --routes 1 >> $O/probe_$lib.jsonl 2>>$O/err.txt
done

O=gpurun_out/diag29; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "bf16deq or tc05 or prefill or bf16w" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for lib in head7 cur; do
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  echo "== $lib" >> $O/kb.txt; env $L timeout 200 python scripts/kbench.py --cases up_3b_m16,lmhead_8b_m16,lmhead_8b_m64 --routes 2 >> $O/kb.txt 2>&1
  echo "== $lib pf" >> $O/kb.txt; env $L timeout 200 python scripts/prefill_bench.py --cases gate_8b:4096,lmhead_8b:256 >> $O/kb.txt 2>&1
done; done

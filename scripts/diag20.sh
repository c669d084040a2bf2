O=gpurun_out/diag20; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "bf16deq or tc05 or prefill or bf16w" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for lib in head5 cur; do
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  echo "== $lib" >> $O/pf.txt; env $L timeout 200 python scripts/prefill_bench.py >> $O/pf.txt 2>&1
done; done

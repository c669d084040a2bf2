O=gpurun_out/diag21; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
MCAPQ_GEMM_A8_TC05=2 timeout 300 python -m pytest tests -m gpu -x -q -k "batched or adversarial" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for lib in head6 cur; do
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  for d in 0 3; do
  echo "== $lib dbg$d" >> $O/kb.txt; env $L MCAPQ_GEMM_A8_TC05=2 MCAPQ_TC05_DBG=$d timeout 200 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 0 >> $O/kb.txt 2>&1
  done
done; done

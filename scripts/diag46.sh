# tc05_w4a16x: E ring of 8 slices (cur) vs 4 (_ab/head)
O=gpurun_out/diag46; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for ts in 0 1; do
MCAPQ_GEMM_A16_TC05=2 MCAPQ_TC05_TS=$ts timeout 600 python -m pytest tests -m gpu -x -q -k "w4a16 or gemm or batched or tc05 or linear or wide or full_size" > $O/pytest_ts$ts.txt 2>&1; echo "rc $?" >> $O/pytest_ts$ts.txt
done
for rep in 1 2; do for lib in head cur; do
  echo "lib $lib" >> $O/kb.txt
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  env $L timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m32,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done; done

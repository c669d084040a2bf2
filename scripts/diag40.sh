# tc05_w4a16x with A in TMEM: one tcgen05.wait::st per slice (cur) vs per atom pair (_ab/pre),
# then what is left without conversion (1), read-back (4), E ring (64)
O=gpurun_out/diag40; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
MCAPQ_GEMM_A16_TC05=2 MCAPQ_TC05_TS=1 timeout 600 python -m pytest tests -m gpu -x -q -k "w4a16 or gemm or batched or tc05 or linear or wide or full_size" > $O/pytest_ts.txt 2>&1; echo "rc $?" >> $O/pytest_ts.txt
timeout 600 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -x -q -k "wide_batched or full_size_sampled" > $O/pytest_new.txt 2>&1; echo "rc $?" >> $O/pytest_new.txt
for rep in 1 2; do for lib in pre cur; do for ts in 0 1; do
  echo "lib $lib ts $ts" >> $O/kb.txt
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  env $L MCAPQ_TC05_TS=$ts timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done; done; done
for d in 1 4 5 16 69; do
  echo "dbg $d" >> $O/kb.txt
  MCAPQ_TC05_TS=1 MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done

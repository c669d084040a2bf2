# tc05_w4a16x: dequantise warps load the slice's four blocks up front and release the stage early
O=gpurun_out/diag39; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
MCAPQ_GEMM_A16_TC05=2 timeout 900 python -m pytest tests -m gpu -x -q -k "w4a16 or gemm or batched or tc05 or linear" > $O/pytest_forced.txt 2>&1; echo "rc $?" >> $O/pytest_forced.txt
MCAPQ_GEMM_A16_TC05=2 MCAPQ_TC05_TS=1 timeout 900 python -m pytest tests -m gpu -x -q -k "w4a16 or gemm or batched or tc05 or linear" > $O/pytest_forced_ts.txt 2>&1; echo "rc $?" >> $O/pytest_forced_ts.txt
for ts in 0 1; do
  echo "ts $ts" >> $O/kb.txt
  MCAPQ_TC05_TS=$ts timeout 200 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done

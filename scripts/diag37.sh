# tc05_w4a16x with the A operand in tensor memory (MCAPQ_TC05_TS=1, default) vs shared memory
O=gpurun_out/diag37; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
MCAPQ_GEMM_A16_TC05=2 timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_forced.txt 2>&1; echo "rc $?" >> $O/pytest_forced.txt
for ts in 0 1; do
  echo "ts $ts" >> $O/kb.txt
  MCAPQ_TC05_TS=$ts timeout 200 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,q_3b_m64,lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
  MCAPQ_GEMM_A16_TC05=2 MCAPQ_TC05_TS=$ts timeout 200 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,q_3b_m64 --routes 1 >> $O/kb.txt 2>&1
done

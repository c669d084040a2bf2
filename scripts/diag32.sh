O=gpurun_out/diag32; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
MCAPQ_GEMM_A16_TC05=2 timeout 300 python -m pytest tests -m gpu -x -q -k "batched or adversarial or full_size or wide_range" > $O/pytest2.txt 2>&1; echo "rc $?" >> $O/pytest2.txt
tail -30 $O/pytest2.txt
for c in "MCAPQ_GEMM_A16_TC05=0" "MCAPQ_GEMM_A16_TC05=2"; do
  echo "== $c" >> $O/kb.txt; env $c timeout 200 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,q_3b_m64,lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done

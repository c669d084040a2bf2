O=gpurun_out/diag7; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "batched or adversarial or prequantised or full_size or lm_head or group" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
tail -30 $O/pytest.txt
for c in "" "MCAPQ_GEMM_A8_TC05=0"; do
  echo "== $c" >> $O/kb.txt
  env $c timeout 300 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,q_3b_m64,lmhead_8b_m16,lmhead_8b_m64 --routes 0 >> $O/kb.txt 2>&1
done

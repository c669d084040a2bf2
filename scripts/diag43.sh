# tc05_w4a8 with two MMA issuer warps: GPU suite, forced tcgen05 W4A8 subset, A/B vs _ab/pre
O=gpurun_out/diag43; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
MCAPQ_GEMM_A8_TC05=2 timeout 600 python -m pytest tests -m gpu -x -q -k "w4a8 or gemm or batched or tc05 or linear or wide or full_size or adversarial" > $O/pytest_a8.txt 2>&1; echo "rc $?" >> $O/pytest_a8.txt
for rep in 1 2; do for lib in pre cur; do
  echo "lib $lib" >> $O/kb.txt
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  env $L timeout 120 python scripts/kbench.py --cases lmhead_8b_m64 --routes 0 >> $O/kb.txt 2>&1
  env $L MCAPQ_GEMM_A8_TC05=2 timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,up_3b_m64 --routes 0 >> $O/kb.txt 2>&1
done; done

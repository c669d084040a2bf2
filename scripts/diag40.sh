# tc05_w4a16x with A in TMEM (TS = 1): what is left without conversion (1), read-back (4), E ring (64)
O=gpurun_out/diag40; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -x -q -k "wide_batched or full_size_sampled" > $O/pytest_new.txt 2>&1; echo "rc $?" >> $O/pytest_new.txt
for d in 0 1 4 5 16 69; do
  echo "dbg $d" >> $O/kb.txt
  MCAPQ_TC05_TS=1 MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done

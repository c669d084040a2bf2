# full GPU suite (default dispatch + the wide ragged test), A-in-TMEM forced subset, and the TS
# elimination with the MMAs removed (8)
O=gpurun_out/diag41; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
MCAPQ_GEMM_A16_TC05=2 MCAPQ_TC05_TS=1 timeout 600 python -m pytest tests -m gpu -x -q -k "w4a16 or gemm or batched or tc05 or linear or wide or full_size" > $O/pytest_ts.txt 2>&1; echo "rc $?" >> $O/pytest_ts.txt
for d in 0 8 13 77; do
  echo "dbg $d" >> $O/kb.txt
  MCAPQ_TC05_TS=1 MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done

# tc05_w4a16x: A-atom ring depth (MCAPQ_TC05_NA) x stage cap, full and without compute (dbg 13)
O=gpurun_out/diag36; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for d in 0 13; do for na in 4 6 8 12; do for sc in 3 8; do
  echo "dbg $d na $na stages $sc" >> $O/kb.txt
  MCAPQ_TC05_NA=$na MCAPQ_TC05_STAGES=$sc MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done; done; done

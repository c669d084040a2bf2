# tc05_w4a16x: the TMA stream alone (MCAPQ_TC05_DBG=16) vs full, and the stage-count cap
O=gpurun_out/diag35; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for d in 0 16 13; do for sc in 4 8; do
  echo "dbg $d stages $sc" >> $O/kb.txt
  MCAPQ_TC05_STAGES=$sc MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64,lmhead_8b --routes 1 >> $O/kb.txt 2>&1
done; done

# tc05_w4a16x handshake costs (TS = 0): dbg 13 (no convert / MMA / TMEM) + 32 (no proxy fence)
# + 64 (no E ring) + 128 (no atom-ring protection); also 16 (TMA stream only)
O=gpurun_out/diag38; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for d in 16 13 45 77 141 237 0 32 128; do
  echo "dbg $d" >> $O/kb.txt
  MCAPQ_TC05_TS=0 MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done

O=gpurun_out/diag10; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for c in "MCAPQ_TC05_DBG=0" "MCAPQ_TC05_DBG=1" "MCAPQ_TC05_DBG=2" "MCAPQ_TC05_DBG=3"; do
  echo "== $c" >> $O/kb.txt
  env $c timeout 300 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 0 >> $O/kb.txt 2>&1
done

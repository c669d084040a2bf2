# tc05_w4a16x bottleneck by elimination (MCAPQ_TC05_DBG: 1 no code conversion, 2 no epilogue
# math, 4 no TMEM read-back, 8 no MMAs) + one ncu capture per token pass width
O=gpurun_out/diag34; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for d in 0 1 2 4 8 5 12 13; do
  echo "dbg $d" >> $O/kb.txt
  MCAPQ_TC05_DBG=$d timeout 120 python scripts/kbench.py --cases lmhead_8b_m16,lmhead_8b_m64 --routes 1 >> $O/kb.txt 2>&1
done
for c in m16 m64; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a16x -s 2 -c 1 \
  -o $O/prof_x_$c python scripts/kbench.py --cases lmhead_8b_$c --routes 1 --reps 2 > $O/ncu_$c.log 2>&1
python scripts/ncu_stalls.py $O/prof_x_$c.ncu-rep > $O/stalls_$c.txt 2>&1
python scripts/ncu_source.py $O/prof_x_$c.ncu-rep 60 > $O/source_$c.txt 2>&1
done
rm -f $O/*.ncu-rep

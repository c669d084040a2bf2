O=gpurun_out/diag28; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a16 -s 2 -c 1 \
   -o $O/prof python scripts/kbench.py --cases lmhead_8b_m64 --routes 2 --reps 2 > $O/ncu.log 2>&1
python scripts/ncu_source.py $O/prof.ncu-rep 50 > $O/source.txt 2>&1
python scripts/ncu_stalls.py $O/prof.ncu-rep > $O/stalls.txt 2>&1
rm -f $O/*.ncu-rep

O=gpurun_out/diag8; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a8 -s 2 -c 1 \
   -o $O/prof_a8tc python scripts/kbench.py --cases lmhead_8b_m16 --routes 0 --reps 2 > $O/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a8 -s 2 -c 1 \
   -o $O/prof_a8tc64 python scripts/kbench.py --cases lmhead_8b_m64 --routes 0 --reps 2 > $O/ncu64.log 2>&1
python scripts/ncu_summary.py $O $O/sum > $O/sum.log 2>&1
for r in prof_a8tc prof_a8tc64; do
python scripts/ncu_source.py $O/$r.ncu-rep 60 > $O/sum/${r}_source.txt 2>&1
python scripts/ncu_stalls.py $O/$r.ncu-rep > $O/sum/${r}_stalls.txt 2>&1
done
rm -f $O/*.ncu-rep

O=gpurun_out/diag9; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "batched or adversarial" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,lmhead_8b_m16,lmhead_8b_m64 --routes 0 > $O/kb.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tc05_w4a8 -s 2 -c 1 \
   -o $O/prof python scripts/kbench.py --cases lmhead_8b_m16 --routes 0 --reps 2 > $O/ncu.log 2>&1
ncu -i $O/prof.ncu-rep --page raw --csv > $O/raw.csv 2>&1
python scripts/ncu_source.py $O/prof.ncu-rep 60 > $O/source.txt 2>&1
rm -f $O/*.ncu-rep

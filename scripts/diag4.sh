O=gpurun_out/diag4; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "rowshard" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_linear -s 2 -c 1 \
   -o $O/prof_w4a16 python scripts/kbench.py --cases lmhead_8b --routes 1 --reps 2 > $O/ncu_w4a16.log 2>&1
python scripts/ncu_summary.py $O $O/sum > $O/sum.log 2>&1
python scripts/ncu_source.py $O/prof_w4a16.ncu-rep 40 > $O/sum/prof_w4a16_source.txt 2>&1
python scripts/ncu_stalls.py $O/prof_w4a16.ncu-rep > $O/sum/prof_w4a16_stalls.txt 2>&1
rm -f $O/*.ncu-rep

O=gpurun_out/diag16; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "w4a16 or a16 or hmma or W4A16 or step or stack or wide_range or edges or batched" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for lib in head3 cur; do
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  echo -n "$lib " >> $O/probe.txt; env $L timeout 60 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
  echo -n "$lib " >> $O/probe.txt; env $L timeout 60 python scripts/step_probe.py --routes 1 >> $O/probe.txt 2>>$O/err.txt
  echo -n "$lib " >> $O/probe.txt; env $L timeout 60 python scripts/step_probe.py --mlp8b --routes 1 >> $O/probe.txt 2>>$O/err.txt
  echo "== $lib" >> $O/kb.txt; env $L timeout 200 python scripts/kbench.py --cases lmhead_8b,gate_8b,down_8b --routes 1 >> $O/kb.txt 2>&1
done; done

O=gpurun_out/diag13; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "step or stack or record" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for lib in head cur; do
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  echo -n "$lib " >> $O/probe.txt; env $L timeout 120 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
  echo -n "$lib " >> $O/probe.txt; env $L timeout 120 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.txt 2>>$O/err.txt
done; done

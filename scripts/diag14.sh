O=gpurun_out/diag14; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "step or stack or record" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
tail -25 $O/pytest.txt
for rep in 1 2; do for lib in head2 cur; do
  if [ $lib = cur ]; then L=""; else L="MCAPQ_LIB=_ab/$lib/libmcapq.so"; fi
  echo -n "$lib " >> $O/probe.txt; env $L timeout 60 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
  echo -n "$lib " >> $O/probe.txt; env $L timeout 60 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.txt 2>>$O/err.txt
  echo -n "$lib " >> $O/probe.txt; env $L timeout 60 python scripts/step_probe.py --routes 1 >> $O/probe.txt 2>>$O/err.txt
done; done
MCAPQ_STREAM_TRACE=1 timeout 60 python scripts/trace_step.py --routes golden > $O/trace.txt 2>&1

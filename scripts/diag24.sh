O=gpurun_out/diag24; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "step or stack or record" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for rep in 1 2; do for c in "L=head6" "MCAPQ_STEP_REC_R=0.8" "MCAPQ_STEP_REC_R=0.6" "MCAPQ_STEP_REC_R=1.0"; do
  if [ "$c" = "L=head6" ]; then E="MCAPQ_LIB=_ab/head6/libmcapq.so"; else E="$c"; fi
  echo -n "$c " >> $O/probe.txt; env $E timeout 60 python scripts/step_probe.py --routes golden >> $O/probe.txt 2>>$O/err.txt
  echo -n "$c " >> $O/probe.txt; env $E timeout 60 python scripts/step_probe.py --mlp8b --routes 0 >> $O/probe.txt 2>>$O/err.txt
done; done

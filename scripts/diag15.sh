O=gpurun_out/diag15; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
export MCAPQ_GEMM_A8_TC05=2
timeout 300 python scripts/sanitize_tc05.py > $O/plain.txt 2>&1
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_tc05.py > $O/$t.txt 2>&1; echo "exit $?" >> $O/$t.txt
done

O=gpurun_out/diag17; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
for c in "MCAPQ_STREAM_CTAS_PER_SM=0" "MCAPQ_STREAM_CTAS_PER_SM=2" "MCAPQ_STREAM_CTAS_PER_SM=2 MCAPQ_STREAM_SMEM_KB=96" "MCAPQ_STREAM_CTAS_PER_SM=1 MCAPQ_STREAM_SMEM_KB=160" "MCAPQ_STREAM_CTAS_PER_SM=1 MCAPQ_STREAM_SMEM_KB=200" "MCAPQ_STREAM_CTAS_PER_SM=1 MCAPQ_STREAM_SMEM_KB=80"; do
  echo "== $c" >> $O/kb.txt
  env $c timeout 200 python scripts/kbench.py --cases gate_8b,down_8b,gateup_8b,down_1b,gateup_1b --routes 0 >> $O/kb.txt 2>&1
done

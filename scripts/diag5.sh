O=gpurun_out/diag5; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/gpu.txt 2>&1
(cd scripts/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu && timeout 120 ./tmem_ld) > $O/tmem_ld.jsonl 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err

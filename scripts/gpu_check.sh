#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list + one full capture.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
python __graft_entry__.py > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gemv|tc_linear|quant_a8|stream_linear' -c 300 --csv \
     --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_linear -s 42 -c 1 \
     -o $OUT/prof_w4a8 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_linear -s 62 -c 1 \
     -o $OUT/prof_w4a16 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_full16.log 2>&1
fi
echo done > $OUT/DONE

#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list + full captures.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
python __graft_entry__.py > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ "${ONLY_NCU:-0}" = "1" ]; then :; fi
timeout 400 python scripts/kbench.py --cases o_1b,qkv_1b,gateup_1b,down_1b,gate_8b,down_8b,lmhead_8b,up_3b_m16,q_3b_m64,lmhead_8b_m16,lmhead_8b_m64 > $OUT/kbench.jsonl 2>&1
timeout 300 python scripts/kbench.py --cases up_3b_m16,up_3b_m64,q_3b_m64,lmhead_8b_m16,lmhead_8b_m64 --routes 2 >> $OUT/kbench.jsonl 2>&1
if [ "${NCU:-1}" = "1" ]; then
  # every launch of a short bench run with its device time (cold-cache, serialised: compare shares)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'stack_step|stream_linear|gemv|tc_linear|quant_a8|gemm_w4|tc05' \
     -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_launch.log 2>&1
  # the headline step kernel (whole 16-layer step in one launch)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stack_step -s 3 -c 1 \
     -o $OUT/prof_step python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_step.log 2>&1
  # the 8B MLP stack step (records path: clusters of 2, producer-side quantisation), both routes
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stack_step -s 3 -c 1 \
     -o $OUT/prof_step_mlp8b python scripts/step_probe.py --mlp8b --routes 0 > $OUT/ncu_step_mlp8b.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stack_step -s 3 -c 1 \
     -o $OUT/prof_step_mlp8b_a16 python scripts/step_probe.py --mlp8b --routes 1 > $OUT/ncu_step_mlp8b_a16.log 2>&1
  # the dominant per-linear kernel: W4A8 grouped gate+up (bench's roofline kernel)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_linear -s 8 -c 1 \
     -o $OUT/prof_w4a8 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_w4a8.log 2>&1
  # W4A16 (HMMA1 engine) on the 8B lm_head
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_linear -s 2 -c 1 \
     -o $OUT/prof_w4a16 python scripts/kbench.py --cases lmhead_8b --routes 1 --reps 2 > $OUT/ncu_w4a16.log 2>&1
  # batched decode (a5/a6): 8B lm_head at M = 64, both routes
  # W4A8 batched: tcgen05 kind::i8 at M = 64 (tc05_w4a8), mma.sync IMMA at M = 16 (gemm_w4)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a8 -s 2 -c 1 \
     -o $OUT/prof_tc05_a8 python scripts/kbench.py --cases lmhead_8b_m64 --routes 0 --reps 2 > $OUT/ncu_tc05_a8.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_w4 -s 2 -c 1 \
     -o $OUT/prof_gemm_a8 python scripts/kbench.py --cases lmhead_8b_m16 --routes 0 --reps 2 > $OUT/ncu_gemm_a8.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_w4 -s 2 -c 1 \
     -o $OUT/prof_gemm_a16 python scripts/kbench.py --cases lmhead_8b_m64 --routes 1 --reps 2 > $OUT/ncu_gemm_a16.log 2>&1
  # exact batched W4A16 on tcgen05 (tc05_w4a16x: A from TMEM at M = 16, from smem at M = 64)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a16x -s 2 -c 1 \
     -o $OUT/prof_tc05x_m16 python scripts/kbench.py --cases lmhead_8b_m16 --routes 1 --reps 2 > $OUT/ncu_tc05x_m16.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc05_w4a16x -s 2 -c 1 \
     -o $OUT/prof_tc05x_m64 python scripts/kbench.py --cases lmhead_8b_m64 --routes 1 --reps 2 > $OUT/ncu_tc05x_m64.log 2>&1
  # batched W4A16 with bf16-dequantised weights on tcgen05 (8B lm_head, M = 64)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc05 -s 2 -c 1 \
     -o $OUT/prof_tc05 python scripts/kbench.py --cases lmhead_8b_m64 --routes 2 --reps 2 > $OUT/ncu_tc05.log 2>&1
fi
# summarise on the box (ncu -i needs no GPU) and keep only what fits the 64 MiB return:
# the summaries, the source-level hot spots of the step kernels, and the 1B step report
python scripts/ncu_summary.py $OUT $OUT/sum > $OUT/sum.log 2>&1
for r in prof_step prof_step_mlp8b prof_step_mlp8b_a16 prof_w4a16 prof_tc05_a8 prof_tc05x_m16 prof_tc05x_m64; do
  [ -f $OUT/$r.ncu-rep ] && python scripts/ncu_source.py $OUT/$r.ncu-rep 40 > $OUT/sum/${r}_source.txt 2>&1
  [ -f $OUT/$r.ncu-rep ] && python scripts/ncu_stalls.py $OUT/$r.ncu-rep > $OUT/sum/${r}_stalls.txt 2>&1
done
for f in $OUT/*.ncu-rep; do [ "$(basename $f)" = "prof_step.ncu-rep" ] || rm -f $f; done
echo done > $OUT/DONE

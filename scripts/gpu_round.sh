#!/bin/bash
# One GPU call: build, gpu tests, smoke, bench (N=1), launch list of the bench.
set -x
OUT=gpurun_out/${1:-run}
mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/gputest.log

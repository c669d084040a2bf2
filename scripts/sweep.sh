#!/bin/bash
# Stream-kernel tuning sweep (one gpurun call).  Usage: bash scripts/sweep.sh TAG
TAG=${1:-sweep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
python - > $OUT/read_ceiling.json 2>&1 <<'EOF'
import torch, json
x = torch.empty(2 * 1024**3 // 4, dtype=torch.int32, device="cuda")
x.fill_(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); s = x.sum(); e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"read_ceiling_GBps": round(x.numel() * 4 / best / 1e6, 1), "bytes": x.numel() * 4, "ms": best}))
EOF
CASES=${CASES:-gateup_1b,qkv_1b,down_1b,gate_8b,lmhead_8b}
while read -r envs; do
  env $envs timeout 300 python scripts/kbench.py --cases $CASES --tag "$envs" >> $OUT/kbench.jsonl 2>> $OUT/kbench.err
done <<EOF
MCAPQ_X=0
MCAPQ_STREAM_PDL=1
MCAPQ_STREAM_NOCOMPUTE=1
MCAPQ_STREAM_SMEM_KB=200
MCAPQ_STREAM_SMEM_KB=200 MCAPQ_STREAM_NOCOMPUTE=1
MCAPQ_STREAM_SMEM_KB=200 MCAPQ_STREAM_PDL=1
MCAPQ_STREAM_STAGES=2
MCAPQ_STREAM_STAGES=3
EOF
echo done > $OUT/DONE

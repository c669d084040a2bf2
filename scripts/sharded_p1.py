"""The bench's sharded rows (bench.time_sharded) through the real NCCL paths at P = 1 on
this pod's one GPU (a code-path check of what SCALE runs at P = 2/4/8; E(1) is ~1 by
construction).  python scripts/sharded_p1.py"""
import json
import os
import socket
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2604_21026_b200 as mq  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
dev = torch.device("cuda:0")
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0, device_id=dev)
mq.load()
stream = torch.cuda.Stream()
res = bench.time_sharded(mq, dev, stream, dist, 1, 0, force_comm=True,
                         slots=(("lm_head", 1, 8), ("gate", 1, 32), ("down", 1, 32), ("down", 16, 16)))
print(json.dumps(res))
dist.destroy_process_group()

"""World-size-2 `gloo` tests (CPU) of the multi-GPU host logic (rows a8 and NEXT-2):
the NCCL unique-id bootstrap over a torch process group, the rank-major row
partition (reading A22) and the all-gather reassembly.  Each rank computes its
shard with the oracle; the gathered result must equal the unsharded one
bit-for-bit, for M = 1 (in-place gather order) and M > 1 (rank-major + permute).  The
row-parallel (K-sharded) partition: each rank's K-slice partial, summed by an
all-reduce, equals the oracle's sharded sum and the unsharded linear."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2604_21026_b200 as mq
        import synth_inputs as si
        # 1. the NCCL id bootstrap: every rank sees rank 0's 128 bytes
        uid = mq.Comm.bootstrap_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(i == ids[0] for i in ids)
        # 2. shard + gather reassembly on the oracle
        n, k = 64, 256
        w = si.weight(n, k, 5).float().numpy()
        nib, sc = oracle.pack_w4(w)
        pw = mq.PackedW4(torch.from_numpy(nib), torch.from_numpy(sc.view(np.int16)))
        mine = pw.shard(world, rank)
        a, b = oracle.colshard_rows(n, world, rank)
        assert mine.n == b - a and torch.equal(mine.nib, pw.nib[a:b])
        for m in (1, 3):
            x = si.activation(m, k, 6 + m).float().numpy()
            for route in (oracle.W4A8, oracle.W4A16):
                if route == oracle.W4A8:
                    y_local, _ = oracle.w4a8_from_x(mine.nib.numpy(), mine.scale.numpy().view(np.uint16), x)
                else:
                    y_local, _ = oracle.w4a16(mine.nib.numpy(), mine.scale.numpy().view(np.uint16), x)
                # rank-major all-gather of the [m, N/P] slices, then the permute to [m, N]
                flat = torch.from_numpy(np.ascontiguousarray(y_local)).flatten()
                parts = [torch.empty_like(flat) for _ in range(world)]
                dist.all_gather(parts, flat)
                gathered = torch.stack(parts).view(world, m, n // world)
                y = gathered.permute(1, 0, 2).reshape(m, n).numpy()
                full = oracle.colshard_linear(route, nib, sc, x, 1)
                assert np.array_equal(y, full)
        # 3. NEXT-2 row-parallel: this rank's K-slice (PackedW4.kshard) partial, then the sum
        # all-reduce; equal to the oracle's rank-order sharded sum and, within fp32
        # rounding, to the unsharded linear
        k2 = 512
        w2 = si.weight(n, k2, 9).float().numpy()
        nib2, sc2 = oracle.pack_w4(w2)
        pw2 = mq.PackedW4(torch.from_numpy(nib2), torch.from_numpy(sc2.view(np.int16)))
        ks = pw2.kshard(world, rank)
        a, b = oracle.rowshard_cols(k2, world, rank)
        assert ks.k == b - a and torch.equal(ks.nib, pw2.nib[:, a // 2:b // 2])
        for m in (1, 3):
            x = si.activation(m, k2, 10 + m).float().numpy()
            for route in (oracle.W4A8, oracle.W4A16):
                fn = oracle.w4a8_from_x if route == oracle.W4A8 else oracle.w4a16
                p32, p64 = fn(ks.nib.numpy(), ks.scale.numpy().view(np.uint16), x[:, a:b])
                t = torch.from_numpy(np.ascontiguousarray(p64))
                dist.all_reduce(t)
                _, u64 = fn(nib2, sc2, x)
                _, r64 = oracle.rowshard_linear(route, nib2, sc2, x, world)
                scale = np.maximum(np.abs(u64), np.sqrt(np.mean(u64 ** 2)))
                assert np.max(np.abs(t.numpy() - r64) / scale) < 1e-12
                assert np.max(np.abs(t.numpy() - u64) / scale) < 1e-12
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_shard_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res

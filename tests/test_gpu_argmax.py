"""NEXT-2 on the GPU: greedy decode on the lm_head, fused into the linear's
epilogue at M = 1, and its column-sharded form (local argmax + key gather) emulated P
ways on one GPU.  The argmax is a decision taken on fp32 logits, so (reading T, DESIGN
§2) both sides take it in the same precision: the GPU index must equal the oracle's
argmax_first of the GPU's own fp32 logits (bit-exact), its value must be that logit, and
the index must be a valid maximiser of the oracle's fp64 logits within tolerance T."""
import numpy as np
import pytest
import torch

import synth_inputs as si
from test_gpu_parity import DEV, _f32, _pack_both, mq  # noqa: F401

pytestmark = pytest.mark.gpu


def _y64(orc, route, nib, sc, x):
    return (orc.w4a8_from_x(nib, sc, _f32(x)) if route == 0 else orc.w4a16(nib, sc, _f32(x)))[1]


def _check(mq, orc, route, pw, nib, sc, x, idx, val):
    y32 = mq.linear(route, pw, x.to(DEV), out_dtype=torch.float32).cpu().numpy()
    idx, val = idx.cpu().numpy(), val.cpu().numpy()
    assert np.array_equal(idx, orc.argmax_first(y32))                     # same decision, same precision
    assert np.array_equal(val.view(np.uint32), y32[np.arange(len(idx)), idx].view(np.uint32))
    y64 = np.asarray(_y64(orc, route, nib, sc, x)).reshape(y32.shape)
    for i in range(y64.shape[0]):                                          # a valid maximiser within T
        tol = 1e-3 * max(abs(y64[i].max()), np.sqrt(np.mean(y64[i] ** 2)))
        assert y64[i, idx[i]] >= y64[i].max() - 2 * tol


@pytest.mark.parametrize("route", [0, 1])
@pytest.mark.parametrize("n,k,m", [(4096, 2048, 1), (3000, 4096, 1), (4096, 2048, 4), (2048, 2048, 64),
                                   (1000, 800, 1), (600, 800, 3)])
def test_linear_argmax_vs_oracle(mq, orc, route, n, k, m):
    w = si.weight(n, k, 3000 + n + k)
    x = si.activation(m, k, 3001 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    idx, val = mq.linear_argmax(route, pw, x.to(DEV))
    _check(mq, orc, route, pw, nib, sc, x, idx, val)


@pytest.mark.parametrize("route", [0, 1])
@pytest.mark.parametrize("m", [1, 16])
def test_argmax_ties_take_the_first_index(mq, orc, route, m):
    """Rows 100 and 3000 are the same packed row scaled up: their logits are bit-identical
    (the per-row order depends on K only, A22) and maximal; the first index wins, also
    when the two rows sit in different shards."""
    n, k = 4096, 2048
    w = si.weight(n, k, 3100)
    w[100] = w[100].float().mul(6.0).to(torch.bfloat16)
    w[3000] = w[100]
    pw = mq.pack_w4(w.to(DEV))
    x = si.activation(m, k, 3101)
    y32 = mq.linear(route, pw, x.to(DEV), out_dtype=torch.float32)
    assert torch.equal(y32[:, 100], y32[:, 3000])
    idx, _ = mq.linear_argmax(route, pw, x.to(DEV))
    want = torch.tensor(orc.argmax_first(y32.cpu().numpy()))
    assert torch.equal(idx.cpu(), want)
    for P in (2, 4, 8):
        per = n // P
        keys = torch.stack([mq.argmax_keys(route, pw.shard(P, r), x.to(DEV), row_offset=r * per) for r in range(P)])
        assert torch.equal(mq.argmax_combine(keys)[0].cpu(), want)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 64])
@pytest.mark.parametrize("route", [0, 1])
def test_colshard_argmax_emulated(mq, orc, P, m, route):
    """Rank r's local keys (global indices r N/P + n) in slot r, combined: the index and
    value mcapq_linear_colshard_argmax computes after its key all-gather -- equal to the
    unsharded greedy decode and to the oracle's sharded argmax of the same fp32 logits."""
    n, k = 4096, 2048
    w = si.weight(n, k, 3200 + P)
    x = si.activation(m, k, 3201 + m).to(DEV)
    pw = mq.pack_w4(w.to(DEV))
    per = n // P
    keys = torch.empty(P, m, dtype=torch.int64, device=DEV)
    for r in range(P):
        mq.argmax_keys(route, pw.shard(P, r), x, row_offset=r * per, out=keys[r])
    idx, val = mq.argmax_combine(keys)
    ref_idx, ref_val = mq.linear_argmax(route, pw, x)
    assert torch.equal(idx, ref_idx) and torch.equal(val, ref_val)
    y32 = mq.linear(route, pw, x, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(idx.cpu().numpy(), orc.colshard_argmax(y32, P))


@pytest.mark.parametrize("route", [0, 1])
def test_full_size_lm_head_argmax(mq, orc, route):
    """cfg5 8B lm_head (128256 x 4096), M = 1, the fused epilogue argmax."""
    n, k = si.linear_shape("llama-3.1-8b", "lm_head")
    w = si.weight(n, k, si.seed_for(5, 0, "lm_head"))
    x = si.activation(1, k, si.seed_for(5, 0, "lm_head", True))
    pw, nib, sc = _pack_both(mq, orc, w)
    idx, val = mq.linear_argmax(route, pw, x.to(DEV))
    _check(mq, orc, route, pw, nib, sc, x, idx, val)


def test_argmax_graph_capture(mq):
    n, k = 4096, 2048
    pw = mq.pack_w4(si.weight(n, k, 3300).to(DEV))
    x = si.activation(1, k, 3301).to(DEV)
    ws = torch.empty(mq.argmax_workspace_bytes(0, 1, n, k), dtype=torch.uint8, device=DEV)
    ref = mq.linear_argmax(0, pw, x, ws=ws)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            out = mq.linear_argmax(0, pw, x, ws=ws, stream=s)
        for _ in range(3):
            g.replay()
    s.synchronize()
    assert torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1])

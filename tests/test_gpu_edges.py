"""GPU parity on the inputs most likely to break the production engines (SURVEY §8(c)
"Adversarial inputs"), and the column-shard data path (row a8) emulated P ways on one
GPU.  Every check is against the CPU oracle on identical seeded inputs: integer stages
bit-exact, outputs within reading T:
    |y - y*| <= rtol * max(|y*_n|, rms(y*)),  y* = oracle fp64, rtol 1e-3 (fp32 out).

Engines reached (K % 256 == 0, K >= 2048 unless noted):
    M = 1 W4A8  -> stream_linear<DP4A> (fused quantiser a8_quad_store)
    M = 1 W4A16 -> stream_linear<HMMA1>
    M = 4       -> stream_linear<IMMA> / <HMMA>
    M = 16, 64  -> gemm_w4<A8> / <A16>  (quant_a8 kernel + TMA-fed mma.sync)
    bf16deq     -> tc05_w4a16 (tcgen05, reading A13')
    stack       -> stack_step (row-lane DP4A, octet/quad quantisers, HMMA1)
"""
import numpy as np
import pytest
import torch

import synth_inputs as si
from test_gpu_parity import DEV, _assert_close, _f32, _pack_both, mq  # noqa: F401

pytestmark = pytest.mark.gpu


def _oracle_y64(orc, route, nib, sc, x):
    if route == 0:
        return orc.w4a8_from_x(nib, sc, _f32(x))[1]
    return orc.w4a16(nib, sc, _f32(x))[1]


# ---------------------------------------------------------------- adversarial inputs, every engine
ENGINES = [(1, 0), (1, 1), (4, 0), (4, 1), (16, 0), (16, 1), (64, 0), (64, 1)]


@pytest.mark.parametrize("k", [2048, 4096])
@pytest.mark.parametrize("m,route", ENGINES)
def test_adversarial_through_engines(mq, orc, m, route, k):
    n = 176                                   # 11 row tiles of 16: ragged against every CTA tile
    w = si.adversarial_weight(n, k, 2000 + k + m)
    x = si.adversarial_activation(m, k, 2001 + k + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    for out_dtype, rtol in ((torch.float32, 1e-3), (torch.bfloat16, 2e-3)):
        y = mq.linear(route, pw, x.to(DEV), out_dtype=out_dtype)
        _assert_close(y, _oracle_y64(orc, route, nib, sc, x), rtol)


@pytest.mark.parametrize("m", [1, 4, 16, 64])
def test_wide_range_activations_w4a16(mq, orc, m):
    """W4A16 engines that accumulate (128 + c) x and add -136 sum x (HMMA1 / HMMA): groups
    spanning ~14 binades with x100 outliers, where that correction cancels the most."""
    n, k = 176, 4096
    w = si.weight(n, k, 2101)
    x = si.wide_range_activation(m, k, 2102 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    y = mq.linear(1, pw, x.to(DEV), out_dtype=torch.float32)
    _assert_close(y, _oracle_y64(orc, 1, nib, sc, x), 1e-3)


@pytest.mark.parametrize("m", [1, 16, 64])
def test_adversarial_bf16deq(mq, orc, m):
    n, k = 176, 2048
    w = si.adversarial_weight(n, k, 2201 + m)
    x = si.adversarial_activation(m, k, 2202 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    y = mq.w4a16_bf16deq(pw, x.to(DEV), out_dtype=torch.float32)
    _, y64 = orc.w4a16_bf16deq(nib, sc, _f32(x))
    _assert_close(y, y64, 1e-3)


@pytest.mark.parametrize("k", [2048, 4096, 14336])
def test_stream_quantiser_and_group_dots_bit_exact(mq, orc, k):
    """The stream kernel's fused quantiser (a8_quad_store, its IEEE-division fallback near
    half-integers, amax = 0 groups) and its block_D: q, sx, sq and every D bit-exact."""
    n = 48
    w = si.adversarial_weight(n, k, 2300 + k)
    x = si.adversarial_activation(1, k, 2301 + k)
    pw, nib, sc = _pack_both(mq, orc, w)
    q, sx, sq, D = mq.stream_w4a8_dump(pw, x.to(DEV))
    oq, os_, osq = orc.quant_a8(_f32(x))
    torch.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), oq.reshape(-1))
    assert np.array_equal(sx.cpu().numpy().view(np.uint32), os_.reshape(-1).view(np.uint32))
    assert np.array_equal(sq.cpu().numpy(), osq.reshape(-1))
    oD = orc.w4a8_group_dots(nib, oq, osq)
    assert np.array_equal(D.cpu().numpy(), oD.reshape(n, k // 32))


# ---------------------------------------------------------------- the persistent step on adversarial data
ADV_STEP = {"q": (256, 2048), "k": (64, 2048), "v": (64, 2048), "o": (256, 2048), "gate": (512, 2048),
            "up": (512, 2048), "down": (256, 4096)}
ADV_INPUT = {"q": 0, "k": 0, "v": 0, "o": 1, "gate": 2, "up": 2, "down": 3}


def test_step_kernel_adversarial(mq, orc):
    """stack_step with adversarial weights and adversarial step inputs (every input a step
    input: K = 2048 takes the octet quantiser, K = 4096 the quad quantiser), routes W4A8 and
    W4A16; each linear against the oracle."""
    routes = (0, 1)
    st = mq.Stack(list(routes), max_m=1)
    ops, xs = [], {}
    for l in range(len(routes)):
        for sid, (slot, (n, k)) in enumerate(ADV_STEP.items()):
            key = (l, ADV_INPUT[slot])
            if key not in xs:
                xs[key] = si.adversarial_activation(1, k, 2400 + 16 * l + sid)
                xs[key] = (xs[key], xs[key].to(DEV))
            w = si.adversarial_weight(n, k, 2450 + 16 * l + sid)
            pw = mq.pack_w4(w.to(DEV))
            y = torch.empty(1, n, dtype=torch.float32, device=DEV)
            st.set(l, sid, ADV_INPUT[slot], pw, xs[key][1], y)
            ops.append((l, w, xs[key][0], y))
    st.run(1)
    torch.cuda.synchronize()
    assert st.launches(1) == 1
    for (l, w, x, y) in ops:
        nib, sc = orc.pack_w4(_f32(w))
        _assert_close(y, _oracle_y64(orc, routes[l], nib, sc, x), 1e-3)


# ---------------------------------------------------------------- a8: P-way column shards on one GPU
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 64])
@pytest.mark.parametrize("route", [0, 1])
def test_colshard_emulated_vs_oracle(mq, orc, P, m, route):
    """Rank r's linear on rows [r N/P, (r+1) N/P) into slot r of the rank-major buffer
    (what mcapq_linear_colshard computes before the all-gather fills the other slots),
    then mcapq_colshard_assemble: equal to the oracle's sharded linear (reading A22) and
    bit-identical to the unsharded GPU call."""
    n, k = 2048, 2048
    w = si.weight(n, k, 2500 + P)
    x = si.activation(m, k, 2501 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    xd = x.to(DEV)
    per = n // P
    y64 = _oracle_y64(orc, route, nib, sc, x)
    for dt, rtol in ((torch.float32, 1e-3), (torch.bfloat16, 2e-3)):
        rank_major = torch.empty(P, m, per, dtype=dt, device=DEV)
        for r in range(P):
            mq.linear(route, pw.shard(P, r), xd, out=rank_major[r])
        y = mq.colshard_assemble(rank_major, P)
        full = mq.linear(route, pw, xd, out_dtype=dt)
        torch.cuda.synchronize()
        assert torch.equal(y, full)
        if dt == torch.float32:
            _assert_close(y, y64, rtol)
    y32c = orc.colshard_linear(route, nib, sc, _f32(x), P)
    y32 = (orc.w4a8_from_x(nib, sc, _f32(x)) if route == 0 else orc.w4a16(nib, sc, _f32(x)))[0]
    assert np.array_equal(y32c, y32)          # the oracle's own shard invariant


def test_colshard_assemble_f32_ragged_m(mq):
    P, m, per = 4, 5, 24
    src = torch.randn(P, m, per, device=DEV)
    y = mq.colshard_assemble(src, P)
    assert torch.equal(y, src.permute(1, 0, 2).reshape(m, P * per))


# ---------------------------------------------------------------- producer-side quantisation records
@pytest.mark.parametrize("route_down", [0])
def test_step_records_edge_groups(mq, orc, route_down):
    """The producer-quantised records (step kernel, a W4A8 consumer with K >= 4096): the
    up linear's output is made to contain all-zero 32-row groups (amax = 0: s = +0,
    codes 0), groups with one x100 outlier row, and groups whose two 16-row halves come
    from the two CTAs of a cluster; down (K = 8192) reads the records.  Each linear
    against the oracle on the input it actually read, and down bit-identical to the
    per-linear path (which quantises the same bf16 words itself)."""
    n_up, k = 8192, 2048
    w_up = si.weight(n_up, k, 2600)
    g = torch.arange(n_up) // 32
    w_up[(g % 7) == 3] = 0.0                         # whole groups of zero rows -> y = 0
    w_up[(torch.arange(n_up) % 224) == 17] *= 100.0   # one x100 outlier row in some groups
    w_down = si.weight(2048, n_up, 2601)
    x = si.activation(1, k, 2602).to(DEV)
    y_up = torch.empty(1, n_up, dtype=torch.bfloat16, device=DEV)
    y_down = torch.empty(1, 2048, dtype=torch.bfloat16, device=DEV)
    pw_up, pw_down = mq.pack_w4(w_up.to(DEV)), mq.pack_w4(w_down.to(DEV))
    st = mq.Stack([route_down], max_m=1)
    st.set(0, 0, 0, pw_up, x, y_up)
    st.set(0, 1, 1, pw_down, y_up, y_down)
    st.run(1)
    torch.cuda.synchronize()
    assert st.launches(1) == 1
    assert (y_up.view(-1)[(g % 7 == 3).to(DEV)] == 0).all()
    nib, sc = orc.pack_w4(_f32(w_down))
    _assert_close(y_down, _oracle_y64(orc, route_down, nib, sc, y_up), 2e-3)
    ref = mq.linear(route_down, pw_down, y_up.clone(), out_dtype=torch.bfloat16)
    assert torch.equal(ref, y_down)
    # replays: records carry the new epoch's tag every launch
    first = y_down.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.capture(1, stream=s)
        for _ in range(3):
            y_down.zero_()
            st.replay(stream=s)
            s.synchronize()
            assert torch.equal(first, y_down)


# ---------------------------------------------------------------- a8 fused epilogue (NVLink stores)
@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("route", [0, 1])
def test_fused_colshard_peer_stores_emulated(mq, orc, P, route):
    """The fused column-shard epilogue on one GPU: P emulated replicas of y_full in one
    buffer; 'rank' r runs its N/P rows with mcapq_debug_linear_peers, storing every row
    into all P replicas (the per-peer stores the fused path issues over NVLink).  Every
    replica must equal the unsharded linear bit-for-bit and the oracle's sharded linear."""
    n, k = 2048, 2048
    w = si.weight(n, k, 2700 + P)
    x = si.activation(1, k, 2710 + P).to(DEV)
    pw = mq.pack_w4(w.to(DEV))
    per = n // P
    reps = torch.full((P, n), float("nan"), dtype=torch.bfloat16, device=DEV)
    es = 2
    for r in range(P):
        shard = pw.shard(P, r)
        y_local = reps[r, r * per:(r + 1) * per]
        deltas = [(p - r) * n * es for p in range(P)]     # replica p's row block r, from replica r's
        mq.debug_linear_peers(route, shard, x, y_local, deltas)
    torch.cuda.synchronize()
    ref = mq.linear(route, pw, x, out_dtype=torch.bfloat16)
    for p in range(P):
        assert torch.equal(reps[p:p + 1], ref), f"replica {p}"
    nib, sc = orc.pack_w4(_f32(w))
    y64 = (orc.w4a8_from_x(nib, sc, _f32(x)) if route == 0 else orc.w4a16(nib, sc, _f32(x)))[1]
    y32c = orc.colshard_linear(route, nib, sc, _f32(x), P)
    assert np.array_equal(y32c, (orc.w4a8_from_x(nib, sc, _f32(x)) if route == 0 else orc.w4a16(nib, sc, _f32(x)))[0])
    _assert_close(reps[0:1], y64, 2e-3)


# ---------------------------------------------------------------- NEXT-2: P-way row shards on one GPU
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 4, 64])
@pytest.mark.parametrize("route", [0, 1])
def test_rowshard_emulated_vs_oracle(mq, orc, P, m, route):
    """Row-parallel (K-sharded) linear emulated P ways: rank r's routed linear on its
    K-slice (PackedW4.kshard, x[:, r K/P ..]) into slot r of [P, M, N] fp32 partials (what
    each rank computes before the all-reduce / the fused path's slot stores), then
    mcapq_rowshard_reduce (the rank-order sum every rank runs): equal to the oracle's
    sharded linear within the north-star tolerance, each partial equal to the unsharded
    oracle's partial over the same groups, and the reduce an exact fp32 rank-order sum."""
    n, k = 2048, 16384 if P == 8 else 8192
    w = si.weight(n, k, 2800 + P)
    x = si.activation(m, k, 2801 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    xd = x.to(DEV)
    kp = k // P
    parts = torch.empty(P, m, n, dtype=torch.float32, device=DEV)
    for r in range(P):
        mq.linear(route, pw.kshard(P, r), xd[:, r * kp:(r + 1) * kp].contiguous(), out=parts[r])
    y = mq.rowshard_reduce(parts, out_dtype=torch.float32)
    yb = mq.rowshard_reduce(parts, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    _, y64 = orc.rowshard_linear(route, nib, sc, _f32(x), P)
    _assert_close(y, y64, 1e-3)
    _assert_close(yb, y64, 2e-3)
    ref = parts[0].clone()
    for r in range(1, P):
        ref += parts[r]
    assert torch.equal(y, ref)
    for r in (0, P - 1):
        a = r * kp
        p64 = _oracle_y64(orc, route, nib[:, a // 2:(a + kp) // 2], sc[:, a // 32:(a + kp) // 32], x[:, a:a + kp])
        _assert_close(parts[r], p64, 1e-3)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("route", [0, 1])
def test_fused_rowshard_peer_stores_emulated(mq, orc, P, route):
    """The fused row-shard all-reduce on one GPU: P emulated windows of [P][N] fp32 slots
    in one buffer; 'rank' r's GEMV (mcapq_debug_linear_peers) stores its K-slice partial
    into slot r of EVERY window (the per-peer NVLink stores), then each window's rank-order
    sum (mcapq_rowshard_reduce): every rank's y identical, equal to the oracle's sharded
    linear."""
    n, k = 2048, 2048 * P
    w = si.weight(n, k, 2900 + P)
    x = si.activation(1, k, 2910 + P)
    pw, nib, sc = _pack_both(mq, orc, w)
    xd = x.to(DEV)
    kp = k // P
    wins = torch.full((P, P, n), float("nan"), dtype=torch.float32, device=DEV)   # [window p][slot r][n]
    for r in range(P):
        y_local = wins[r, r]
        deltas = [(p - r) * P * n * 4 for p in range(P)]     # window p's slot r, from window r's slot r
        mq.debug_linear_peers(route, pw.kshard(P, r), xd[:, r * kp:(r + 1) * kp].contiguous(), y_local.view(1, n),
                              deltas)
    ys = [mq.rowshard_reduce(wins[p].view(P, 1, n), out_dtype=torch.bfloat16) for p in range(P)]
    torch.cuda.synchronize()
    for p in range(1, P):
        assert torch.equal(ys[p], ys[0]), f"rank {p}"
    _, y64 = orc.rowshard_linear(route, nib, sc, _f32(x), P)
    _assert_close(ys[0], y64, 2e-3)


def test_rowshard_reduce_ragged(mq):
    P, m, n = 3, 5, 37
    src = torch.randn(P, m, n, device=DEV)
    y = mq.rowshard_reduce(src, out_dtype=torch.float32)
    assert torch.equal(y, src[0] + src[1] + src[2])


def test_rowshard_rejects_partial_groups(mq):
    pw = mq.pack_w4(si.weight(64, 96, 2950).to(DEV))
    with pytest.raises(mq.McapqError):
        pw.kshard(2, 0)


# ---------------------------------------------------------------- wide batched linears (tcgen05 dispatch)
@pytest.mark.parametrize("m", [9, 70])
def test_wide_batched_default_dispatch_ragged(mq, orc, m):
    """At least one 128-row tile per SM sends batched decode to the tcgen05 kernels by default
    (kernels_stream.cu launch_gemm): W4A16 -> tc05_w4a16x (A operand in TMEM for passes of
    <= 32 tokens, in shared memory at 64), W4A8 -> tc05_w4a8 for passes of > 32 tokens.  N is
    148 tiles + a ragged 72 rows, M = 9 is one ragged 16-token pass, M = 70 a full 64-token
    pass plus a 6-token one (tok0 = 64).  Whole output against the oracle (reading T)."""
    n, k = 148 * 128 + 72, 512             # ragged against the 128-row tile, ldy % 8 == 0
    w = si.weight(n, k, 4100 + m)
    x = si.activation(m, k, 4101 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    xd = x.to(DEV)
    for route in (0, 1):
        y = mq.linear(route, pw, xd, out_dtype=torch.float32)
        _assert_close(y, _oracle_y64(orc, route, nib, sc, x), 1e-3)

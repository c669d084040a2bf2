"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on identical
seeded inputs (synth_inputs).  Integer stages bit-exact; outputs within the
north-star tolerance (reading T):
    |y - y*| <= rtol * max(|y*_n|, rms(y*)),  y* = oracle fp64 reference,
    rtol = 1e-3 (fp32 output), 2e-3 (bf16 output).
"""
import json
import os

import numpy as np
import pytest
import torch

import synth_inputs as si

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def mq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_21026_b200 as mq
    mq.load()
    return mq


DEV = "cuda:0"


def _f32(t):
    return t.float().cpu().numpy()


def _pack_both(mq, orc, w_bf16):
    pw = mq.pack_w4(w_bf16.to(DEV))
    nib, sc = orc.pack_w4(_f32(w_bf16))
    return pw, nib, sc


def _half_ulp_bf16(v):
    # half a bf16 ulp of |v| (8 significant bits): 2^(floor(log2|v|) - 8)
    a = np.maximum(np.abs(v), np.finfo(np.float32).tiny)
    return np.exp2(np.floor(np.log2(a)) - 8)


def _assert_close(y_gpu, y64, rtol):
    """Reading T.  fp32 output: |y - y*| <= 1e-3 max(|y*|, rms).  bf16 output (rtol
    2e-3): the fp32 bound plus half a bf16 ulp elementwise (bf16's own unit
    roundoff 2^-8 exceeds 2e-3, so 2e-3 is enforced normwise)."""
    y = y_gpu.float().cpu().numpy().astype(np.float64)
    ref = np.asarray(y64, np.float64).reshape(y.shape)
    rms = np.sqrt(np.mean(ref ** 2)) if ref.size else 0.0
    if y_gpu.dtype == torch.bfloat16:
        tol = 1e-3 * np.maximum(np.abs(ref), rms) + _half_ulp_bf16(ref)
        if ref.size >= 512:       # a statistic of RNE rounding (~1.7e-3): noisy on short vectors
            nrm = np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300)
            assert nrm <= rtol, f"normwise rel err {nrm:.3e} > {rtol}"
    else:
        tol = rtol * np.maximum(np.abs(ref), rms)
    bad = np.abs(y - ref) > tol
    assert not bad.any(), (f"{bad.sum()} of {bad.size} outside tolerance; worst rel "
                           f"{(np.abs(y - ref) / np.maximum(np.abs(ref), rms + 1e-300)).max():.3e}")


# ---------------------------------------------------------------- a1 pack
@pytest.mark.parametrize("n,k,kind", [(64, 256, "synth"), (37, 4096, "synth"), (1, 32, "synth"),
                                      (48, 512, "adv"), (200, 2048, "adv")])
def test_pack_bit_exact(mq, orc, n, k, kind):
    w = si.weight(n, k, 11 + n) if kind == "synth" else si.adversarial_weight(n, k, 12 + n)
    pw, nib, sc = _pack_both(mq, orc, w)
    torch.cuda.synchronize()
    assert np.array_equal(pw.nib.cpu().numpy(), nib)
    assert np.array_equal(pw.scale.cpu().numpy().view(np.uint16), sc)


def test_pack_f32_input_and_ldw(mq, orc):
    w = (torch.randn(33, 96 + 32, generator=torch.Generator().manual_seed(3)) * 0.05)
    w[5, 40] = 0.0
    wd = w.to(DEV)
    sub = wd[:, :96]                    # ldw = 128 > k = 96
    pw = mq.pack_w4(sub)
    nib, sc = orc.pack_w4(w[:, :96].numpy())
    assert np.array_equal(pw.nib.cpu().numpy(), nib)
    assert np.array_equal(pw.scale.cpu().numpy().view(np.uint16), sc)


def test_pack_dev_err_flags(mq, orc):
    w = torch.zeros(2, 64, dtype=torch.float32)
    w[0, 3] = float("inf")
    w[1, 40] = 6e5                      # |m|/8 > 65504 -> fp16 overflow (A4)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    pw = mq.pack_w4(w.to(DEV), dev_err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0x3
    st, nib, sc = orc.pack_w4_status(w.numpy())
    assert st == 3
    assert np.array_equal(pw.nib.cpu().numpy(), nib)
    assert np.array_equal(pw.scale.cpu().numpy().view(np.uint16), sc)


# ---------------------------------------------------------------- a2 quant
@pytest.mark.parametrize("m,k,kind", [(1, 2048, "synth"), (3, 4096, "swiglu"), (16, 1024, "adv"), (64, 3072, "synth")])
def test_quant_a8_bit_exact(mq, orc, m, k, kind):
    if kind == "adv":
        x = si.adversarial_activation(m, k, 21)
    else:
        x = si.activation(m, k, 22 + m, "swiglu" if kind == "swiglu" else "rmsnorm")
    q, s, sq = mq.quant_a8(x.to(DEV))
    oq, os_, osq = orc.quant_a8(_f32(x))
    torch.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), oq)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), os_.view(np.uint32))
    assert np.array_equal(sq.cpu().numpy(), osq)


# ---------------------------------------------------------------- integer stage
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n,k,m", [(40, 512, 1), (33, 1024, 5), (16, 2048, 16)])
def test_group_dots_bit_exact(mq, orc, mode, n, k, m):
    w = si.adversarial_weight(n, k, 31 + n)
    x = si.activation(m, k, 32 + m)
    pw, nib, sc = _pack_both(mq, orc, w)
    q, s, sq = mq.quant_a8(x.to(DEV))
    D = mq.w4a8_group_dots(pw, q, sq, mode=mode)
    oq, os_, osq = orc.quant_a8(_f32(x))
    oD = orc.w4a8_group_dots(nib, oq, osq)
    assert np.array_equal(D.cpu().numpy(), oD)


# ---------------------------------------------------------------- a3-a6 outputs
# K % 256 == 0 takes the persistent TMA stream path; K = 800 the generic kernels
SHAPES = [(200, 2048), (3072, 1024), (48, 14336), (512, 3072), (72, 800)]


@pytest.mark.parametrize("m", [1, 3, 8, 11])
@pytest.mark.parametrize("route", [0, 1])
def test_grouped_launch_bit_identical_to_separate(mq, route, m):
    # fused QKV / gate-up launch: same bits as one launch per linear
    k = 2048
    ws = [mq.pack_w4(si.weight(n, k, 300 + n).to(DEV)) for n in (2048, 512, 512)]
    x = si.activation(m, k, 301 + m).to(DEV)
    outs = mq.linear_group(route, ws, x)
    for w, y in zip(ws, outs):
        assert torch.equal(y, mq.linear(route, w, x))


@pytest.mark.parametrize("n,k", SHAPES)
@pytest.mark.parametrize("m", [1, 2, 5, 8, 16, 64])
@pytest.mark.parametrize("route", [0, 1])
def test_linear_vs_oracle(mq, orc, route, m, n, k):
    if m == 64 and n * k > 3072 * 1024:
        pytest.skip("oracle time")
    w = si.weight(n, k, 41 + n + k)
    x = si.activation(m, k, 42 + m + k, "swiglu" if k >= 8192 else "rmsnorm")
    pw, nib, sc = _pack_both(mq, orc, w)
    xd = x.to(DEV)
    for out_dtype, rtol in ((torch.float32, 1e-3), (torch.bfloat16, 2e-3)):
        y = mq.linear(route, pw, xd, out_dtype=out_dtype)
        if route == 0:
            _, y64 = orc.w4a8_from_x(nib, sc, _f32(x))
        else:
            _, y64 = orc.w4a16(nib, sc, _f32(x))
        _assert_close(y, y64, rtol)


@pytest.mark.parametrize("m", [1, 8, 16])
def test_w4a8_prequantised_matches_fused(mq, orc, m):
    n, k = 96, 2048
    pw, nib, sc = _pack_both(mq, orc, si.weight(n, k, 51))
    xd = si.activation(m, k, 52).to(DEV)
    q, s, sq = mq.quant_a8(xd)
    y1 = mq.w4a8(pw, q, s, sq)          # separate quantiser + generic kernel
    y2 = mq.w4a8_x(pw, xd)              # TMA stream kernel, quantiser fused
    torch.cuda.synchronize()
    if m == 1 or m >= 9:
        # m = 1: both dp4a paths sum a lane's blocks l, l+32, ... in the same order;
        # m >= 9: both run the batched kernel on the same quantised activations
        assert torch.equal(y1, y2)
    _, y64 = orc.w4a8(nib, sc, *orc.quant_a8(_f32(xd.cpu())))
    _assert_close(y1, y64, 1e-3)
    _assert_close(y2, y64, 1e-3)


# ---------------------------------------------------------------- a5/a6 batched kernel (m >= 9)
GEMM_SHAPES = [(200, 256), (1000, 2048), (4000, 512), (96, 4096)]


@pytest.mark.parametrize("n,k", GEMM_SHAPES)
@pytest.mark.parametrize("m", [9, 16, 17, 33, 64, 100])
@pytest.mark.parametrize("route", [0, 1])
def test_batched_vs_oracle(mq, orc, route, m, n, k):
    """One weight pass per 64 tokens; ragged token passes (9, 17, 33, 100 = 64 + 36), ragged
    row tiles (200, 1000, 4000 rows over 32/64/128-row tiles), K from one 256-slice up."""
    w = si.weight(n, k, 1401 + n + k)
    x = si.activation(m, k, 1402 + m + k)
    pw, nib, sc = _pack_both(mq, orc, w)
    y = mq.linear(route, pw, x.to(DEV), out_dtype=torch.float32)
    if route == 0:
        _, y64 = orc.w4a8_from_x(nib, sc, _f32(x))
    else:
        _, y64 = orc.w4a16(nib, sc, _f32(x))
    _assert_close(y, y64, 1e-3)


@pytest.mark.parametrize("route", [0, 1])
def test_batched_ldx_ldy_and_rows_beyond_n(mq, orc, route):
    """Strided activations/outputs; the last row tile is mostly out of bounds (TMA zero
    fill must never leak into stored rows)."""
    n, k, m = 40, 1024, 20
    w = si.weight(n, k, 1501)
    xs = si.activation(m, k + 64, 1502)
    pw, nib, sc = _pack_both(mq, orc, w)
    xd = xs.to(DEV)[:, :k]
    yd = torch.full((m, n + 24), 7.0, dtype=torch.float32, device=DEV)
    mq.linear(route, pw, xd, out=yd[:, :n])
    if route == 0:
        _, y64 = orc.w4a8_from_x(nib, sc, _f32(xs[:, :k].contiguous()))
    else:
        _, y64 = orc.w4a16(nib, sc, _f32(xs[:, :k].contiguous()))
    _assert_close(yd[:, :n], y64, 1e-3)
    assert torch.all(yd[:, n:] == 7.0)


# ---------------------------------------------------------------- a6, bf16-dequant semantics (tcgen05)
@pytest.mark.parametrize("n,k", GEMM_SHAPES)
@pytest.mark.parametrize("m", [1, 9, 16, 33, 64, 100])
def test_bf16deq_vs_oracle(mq, orc, m, n, k):
    """tcgen05 kernel vs oracle_w4a16_bf16deq (W^ = bf16_rne(d (c - 8)), fp32 accumulation):
    ragged row tiles over 128-row CTAs, token passes of 16/32/64 (+ a second pass at 100),
    K from one 256-slice up; reading T."""
    w = si.weight(n, k, 1451 + n + k)
    x = si.activation(m, k, 1452 + m + k)
    pw, nib, sc = _pack_both(mq, orc, w)
    y = mq.w4a16_bf16deq(pw, x.to(DEV), out_dtype=torch.float32)
    _, y64 = orc.w4a16_bf16deq(nib, sc, _f32(x))
    _assert_close(y, y64, 1e-3)


def test_bf16deq_rounds_the_weights(mq, orc):
    """The kernel really applies the bf16 rounding of d (c - 8): its distance to the
    bf16-dequant oracle is far below the distance between the two semantics."""
    n, k, m = 1024, 2048, 32
    w = si.weight(n, k, 1461)
    x = si.activation(m, k, 1462)
    pw, nib, sc = _pack_both(mq, orc, w)
    y = mq.w4a16_bf16deq(pw, x.to(DEV)).cpu().numpy().astype(np.float64)
    _, yb = orc.w4a16_bf16deq(nib, sc, _f32(x))
    _, ye = orc.w4a16(nib, sc, _f32(x))
    gap = np.linalg.norm(yb - ye)
    assert gap > 0
    assert np.linalg.norm(y - yb) < 0.05 * gap


def test_bf16deq_strides_bf16_out_rows_beyond_n(mq, orc):
    """Strided x / y, bf16 output, last row tile mostly out of bounds (never stored)."""
    n, k, m = 40, 1024, 20
    w = si.weight(n, k, 1471)
    xs = si.activation(m, k + 64, 1472)
    pw, nib, sc = _pack_both(mq, orc, w)
    yd = torch.full((m, n + 24), 7.0, dtype=torch.bfloat16, device=DEV)
    mq.w4a16_bf16deq(pw, xs.to(DEV)[:, :k], out=yd[:, :n])
    _, y64 = orc.w4a16_bf16deq(nib, sc, _f32(xs[:, :k].contiguous()))
    _assert_close(yd[:, :n], y64, 2e-3)
    assert torch.all(yd[:, n:] == 7.0)


def test_bf16deq_full_size_lm_head_sampled_rows(mq, orc):
    """Config 5 at its full size (8B lm_head 128256 x 4096, M = 64), in the launch
    configuration bench.py times; sampled rows (incl. the last) against the oracle."""
    n, k, m = 128256, 4096, 64
    w = si.weight(n, k, 1481)
    x = si.activation(m, k, 1482)
    pw = mq.pack_w4(w.to(DEV))
    y = mq.w4a16_bf16deq(pw, x.to(DEV), out_dtype=torch.float32)
    rows = np.unique(np.concatenate([np.linspace(0, n - 1, 48).astype(np.int64), [127, 128, n - 128, n - 1]]))
    nib, sc = orc.pack_w4(_f32(w[rows]))
    _, y64 = orc.w4a16_bf16deq(nib, sc, _f32(x))
    _assert_close(y[:, rows], y64, 1e-3)


def test_bf16deq_rejects_k_not_multiple_of_256(mq):
    pw = mq.pack_w4(si.weight(64, 288, 1491).to(DEV))
    with pytest.raises(mq.McapqError):
        mq.w4a16_bf16deq(pw, si.activation(16, 288, 1492).to(DEV))


# ---------------------------------------------------------------- NEXT-4 prefill (dequantise once + tcgen05 GEMM)
@pytest.mark.parametrize("n,k", [(200, 256), (37, 4096), (1000, 2048)])
def test_dequant_w4_bf16_bit_exact(mq, orc, n, k):
    """W^ = bf16_rne(f32(d) (c - 8)) bit-for-bit: the oracle's exact dequantisation
    (oracle_dequant_w4) rounded by the oracle's RNE fp32 -> bf16."""
    w = si.weight(n, k, 1521 + n)
    pw, nib, sc = _pack_both(mq, orc, w)
    got = mq.dequant_w4_bf16(pw).cpu().view(torch.int16).numpy().view(np.uint16)
    ref = orc.f32_to_bf16_bits(orc.dequant_w4(nib, sc))
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n,k", [(200, 256), (1000, 2048), (4000, 512)])
@pytest.mark.parametrize("m", [64, 100, 256, 300])
def test_prefill_vs_oracle(mq, orc, m, n, k):
    """Dequantise once + tcgen05 GEMM vs oracle_w4a16_bf16deq: token passes of 64/128/256
    (300 = 256 + 44), ragged 128-row tiles; reading T."""
    w = si.weight(n, k, 1531 + n + k)
    x = si.activation(m, k, 1532 + m + k)
    pw, nib, sc = _pack_both(mq, orc, w)
    y = mq.w4a16_bf16deq_prefill(pw, x.to(DEV), out_dtype=torch.float32)
    _, y64 = orc.w4a16_bf16deq(nib, sc, _f32(x))
    _assert_close(y, y64, 1e-3)


def test_bf16w_gemm_strides_bf16_out_rows_beyond_n(mq, orc):
    n, k, m = 40, 1024, 70
    w = si.weight(n, k, 1541)
    xs = si.activation(m, k + 64, 1542)
    pw, nib, sc = _pack_both(mq, orc, w)
    wdq = mq.dequant_w4_bf16(pw)
    yd = torch.full((m, n + 24), 7.0, dtype=torch.bfloat16, device=DEV)
    mq.bf16w_gemm(wdq, xs.to(DEV)[:, :k], out=yd[:, :n])
    _, y64 = orc.w4a16_bf16deq(nib, sc, _f32(xs[:, :k].contiguous()))
    _assert_close(yd[:, :n], y64, 2e-3)
    assert torch.all(yd[:, n:] == 7.0)


def test_prefill_and_bf16deq_graph_capture_and_pdl(mq):
    """Both tcgen05 paths are stream-ordered and capturable: a CUDA graph of
    prefill + batched bf16-dequant calls (with programmatic dependent launch on) replays
    to the same bits as eager launches."""
    n, k, m = 1000, 2048, 96
    pw = mq.pack_w4(si.weight(n, k, 1561).to(DEV))
    x = si.activation(m, k, 1562).to(DEV)
    ref_p = mq.w4a16_bf16deq_prefill(pw, x)
    ref_b = mq.w4a16_bf16deq(pw, x)
    yp = torch.empty_like(ref_p)
    yb = torch.empty_like(ref_b)
    ws = torch.empty(mq.load().mcapq_prefill_workspace_bytes(n, k), dtype=torch.uint8, device=DEV)
    prev = mq.set_pdl(True)
    try:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            mq.w4a16_bf16deq_prefill(pw, x, out=yp, ws=ws, stream=s)
            mq.w4a16_bf16deq(pw, x, out=yb, stream=s)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                mq.w4a16_bf16deq_prefill(pw, x, out=yp, ws=ws, stream=s)
                mq.w4a16_bf16deq(pw, x, out=yb, stream=s)
            yp.zero_()
            yb.zero_()
            g.replay()
            s.synchronize()
    finally:
        mq.set_pdl(prev)
    assert torch.equal(yp, ref_p) and torch.equal(yb, ref_b)


def test_bf16w_gemm_rejects_k_not_multiple_of_64(mq):
    pw = mq.pack_w4(si.weight(64, 288, 1551).to(DEV))
    with pytest.raises(mq.McapqError):
        mq.w4a16_bf16deq_prefill(pw, si.activation(64, 288, 1552).to(DEV))


def test_zero_activation_and_impulse_rows(mq, orc):
    # S:315 / S:324-325 special cases through the GPU path
    k = 256
    w = torch.zeros(16, k)
    picks = [(r, (r * 13) % k, float(r - 8) or 1.0) for r in range(16)]
    for r, col, v in picks:
        w[r, col] = v
    pw = mq.pack_w4(w.to(torch.bfloat16).to(DEV))
    z = torch.zeros(1, k, dtype=torch.bfloat16, device=DEV)
    assert torch.count_nonzero(mq.w4a8_x(pw, z)) == 0
    assert torch.count_nonzero(mq.w4a16(pw, z)) == 0
    x = si.activation(1, k, 61)
    y = mq.w4a16(pw, x.to(DEV)).cpu()
    for r, col, v in picks:
        assert y[0, r].item() == np.float32(v) * np.float32(x[0, col].float().item())


def test_column_shards_bit_identical(mq):
    # A22: per-row arithmetic depends on K only -> any row slice reproduces the full result bit-for-bit
    n, k = 1024, 4096
    pw = mq.pack_w4(si.weight(n, k, 71).to(DEV))
    for m in (1, 16):
        x = si.activation(m, k, 72 + m).to(DEV)
        for route in (0, 1):
            full = mq.linear(route, pw, x)
            for P in (2, 4, 8):
                parts = [mq.linear(route, pw.shard(P, r), x) for r in range(P)]
                assert torch.equal(torch.cat(parts, dim=1), full)


def test_deterministic(mq):
    n, k = 2048, 2048
    pw = mq.pack_w4(si.weight(n, k, 81).to(DEV))
    x = si.activation(4, k, 82).to(DEV)
    for route in (0, 1):
        a = mq.linear(route, pw, x)
        b = mq.linear(route, pw, x)
        assert torch.equal(a, b)


def test_linear_host_e2e(mq, orc):
    n, k, m = 512, 2048, 1
    w = si.weight(n, k, 91)
    x = si.activation(m, k, 92)
    pw = mq.pack_w4(w.to(DEV))
    xh = x.pin_memory()
    for route in (0, 1):
        yh = torch.empty(m, n, dtype=torch.float32).pin_memory()
        ws = torch.empty(mq.host_workspace_bytes(route, m, n, k), dtype=torch.uint8, device=DEV)
        mq.linear_host(route, pw, xh, yh, ws)
        torch.cuda.synchronize()
        yd = mq.linear(route, pw, x.to(DEV))
        assert torch.equal(yh, yd.cpu())


# ---------------------------------------------------------------- full-size configs, sampled rows
FULL = [("llama-3.1-8b", "gate", 1), ("llama-3.1-8b", "down", 1), ("llama-3.1-8b", "lm_head", 1),
        ("llama-3.1-8b", "lm_head", 16), ("llama-3.1-8b", "lm_head", 24), ("llama-3.1-8b", "lm_head", 64),
        ("llama-3.2-3b", "up", 16), ("llama-3.2-3b", "q", 64)]


@pytest.mark.parametrize("model,slot,m", FULL)
def test_full_size_sampled_rows(mq, orc, model, slot, m):
    n, k = si.linear_shape(model, slot)
    w = si.weight(n, k, si.seed_for(5, 0, slot))
    x = si.activation(m, k, si.seed_for(5, 0, slot, True), si.activation_kind(slot))
    pw = mq.pack_w4(w.to(DEV))
    rows = np.sort(np.random.default_rng(n + k).choice(n, size=48, replace=False))
    rows[-1] = n - 1
    nib, sc = orc.pack_w4(_f32(w[rows]))
    assert np.array_equal(pw.nib[rows].cpu().numpy(), nib)
    assert np.array_equal(pw.scale[rows].cpu().numpy().view(np.uint16), sc)
    xd = x.to(DEV)
    for route in (0, 1):
        y = mq.linear(route, pw, xd, out_dtype=torch.bfloat16)
        if route == 0:
            _, y64 = orc.w4a8_from_x(nib, sc, _f32(x))
        else:
            _, y64 = orc.w4a16(nib, sc, _f32(x))
        _assert_close(y[:, rows], y64, 2e-3)


# ---------------------------------------------------------------- a7 + a9 stack
STACK_DIMS = {
    # K < 2048: generic kernels, separate quantiser launches (4 + 7 per W4A8 layer, 7 per W4A16 layer)
    "generic": ({"q": (256, 512), "k": (64, 512), "v": (64, 512), "o": (512, 256), "gate": (1024, 512),
                 "up": (1024, 512), "down": (512, 1024)}, 2 * (4 + 7) + 2 * 7),
    # K >= 2048: TMA stream kernels, grouped qkv / o / gate-up / down launches, quantiser fused
    "stream": ({"q": (256, 2048), "k": (64, 2048), "v": (64, 2048), "o": (512, 2048), "gate": (384, 2048),
                "up": (384, 2048), "down": (256, 2048)}, 4 * 4),
}


@pytest.mark.parametrize("kind", ["generic", "stream"])
def test_stack_matches_oracle_and_graph_replay(mq, orc, kind):
    prof = mq.profile_parse(open(os.path.join(GOLD, "llama32_1b_profile.json")).read())
    routes = prof.routes()
    assert routes == [0] * 15 + [1]
    L = 4
    routes = [0, 1, 0, 1]
    dims, launches = STACK_DIMS[kind]
    inputs = {"q": 0, "k": 0, "v": 0, "o": 1, "gate": 2, "up": 2, "down": 3}
    st = mq.Stack(routes, max_m=2)
    ref = []
    xs = {}
    for l in range(L):
        for slot_id, (slot, (n, k)) in enumerate(dims.items()):
            w = si.weight(n, k, si.seed_for(2, l, slot))
            key = (l, inputs[slot])
            if key not in xs:
                xa = si.activation(2, k, si.seed_for(2, l, slot, True), si.activation_kind(slot))
                xs[key] = (xa, xa.to(DEV))     # slots sharing an input share the device tensor
            x, xd = xs[key]
            pw = mq.pack_w4(w.to(DEV))
            y = torch.empty(2, n, dtype=torch.bfloat16, device=DEV)
            st.set(l, slot_id, inputs[slot], pw, xd, y)
            ref.append((l, y, w, x))
    assert st.launches(2) == launches
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.run(2, stream=s)
    s.synchronize()
    first = [y.clone() for (_, y, _, _) in ref]
    for (l, y, w, x) in ref:
        nib, sc = orc.pack_w4(_f32(w))
        if routes[l] == 0:
            _, y64 = orc.w4a8_from_x(nib, sc, _f32(x))
        else:
            _, y64 = orc.w4a16(nib, sc, _f32(x))
        _assert_close(y, y64, 2e-3)
    for (_, y, _, _) in ref:
        y.zero_()
    torch.cuda.synchronize()
    st.capture(2, stream=s)
    st.replay(stream=s)
    s.synchronize()
    for a, (_, y, _, _) in zip(first, ref):
        assert torch.equal(a, y)
    assert st.weight_bytes == sum(pw_n * k // 2 + pw_n * k // 32 * 2 for pw_n, k in dims.values()) * L


# ---------------------------------------------------------------- a9: the persistent step kernel (M = 1)
# Llama-3.2-1B widths at 4 layers (K up to 8192: multi-round staging), routes [0, 1, 0, 1].
STEP_DIMS = {"q": (2048, 2048), "k": (512, 2048), "v": (512, 2048), "o": (2048, 2048), "gate": (8192, 2048),
             "up": (8192, 2048), "down": (2048, 8192)}
STEP_INPUT = {"q": 0, "k": 0, "v": 0, "o": 1, "gate": 2, "up": 2, "down": 3}


def _step_stack(mq, mode, L=4, routes=(0, 1, 0, 1)):
    """mode: 'independent' (every input a step input), 'dataflow' (the decode chain:
    x_o = y_q, x_gate/up = y_o, x_down = y_up, x_q(l+1) = y_down(l) -- exact aliases,
    passed by tagged dataflow), 'barrier' (x_q(l+1) is a view half-overlapping
    y_down(l): a partial alias -> grid-barrier dependency)."""
    st = mq.Stack(list(routes), max_m=1)
    ops, ys, xs = [], {}, {}
    for l in range(L):
        for slot_id, (slot, (n, k)) in enumerate(STEP_DIMS.items()):
            key = (l, STEP_INPUT[slot])
            if key not in xs:
                if mode == "dataflow" and not (l == 0 and slot == "q"):
                    src = {"q": (l - 1, "down"), "o": (l, "q"), "gate": (l, "o"), "down": (l, "up")}[slot]
                    xs[key] = ys[src]
                elif mode == "barrier" and l > 0 and slot == "q":
                    xs[key] = ys[("buf", l - 1)][1024:1024 + k].view(1, k)
                else:
                    xs[key] = si.activation(1, k, si.seed_for(2, l, slot, True), si.activation_kind(slot)).to(DEV)
            w = si.weight(n, k, si.seed_for(2, l, slot))
            pw = mq.pack_w4(w.to(DEV))
            if mode == "barrier" and slot == "down":
                buf = si.activation(1, 2 * n, si.seed_for(3, l, slot, True)).to(DEV).view(-1)
                ys[("buf", l)] = buf
                y = buf[:n].view(1, n)
            else:
                y = torch.empty(1, n, dtype=torch.bfloat16, device=DEV)
            ys[(l, slot)] = y
            st.set(l, slot_id, STEP_INPUT[slot], pw, xs[key], y)
            ops.append((l, slot, w, xs[key], y))
    return st, ops


def test_bench_step_full_size_sampled(mq, orc):
    """Row a9 at BASELINE's full size, in the launch configuration bench.py times: the
    16-layer Llama-3.2-1B chained stack under the golden MCAP mask (tab:per_layer_scores,
    layer 15 W4A16), one stack_step launch captured in a graph.  Sampled rows of every
    linear of layers 0, 7, 14 (W4A8) and 15 (W4A16) against the oracle on the linear's
    actual input (the same per-linear check as the small step tests)."""
    import bench
    routes = mq.profile_parse(open(bench.GOLDEN_PROFILE).read()).routes()
    assert list(routes) == [0] * 15 + [1]
    st, _, xs, ys = bench.build_stack(mq, torch.device(DEV), routes)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.capture(1, stream=s)
        st.replay(stream=s)
    s.synchronize()
    assert st.launches(1) == 1
    rng = np.random.default_rng(260421026)
    for l in (0, 7, 14, 15):
        for slot in bench.SLOTS:
            n, k = si.linear_shape(bench.MODEL, slot)
            rows = np.sort(rng.choice(n, size=16, replace=False))
            rows[-1] = n - 1
            w = si.weight(n, k, si.seed_for(bench.CONFIG_ID, l, slot))
            nib, sc = orc.pack_w4(_f32(w[rows]))
            x = _f32(xs[(l, bench.INPUT_ID[slot])])
            if routes[l] == 0:
                _, y64 = orc.w4a8_from_x(nib, sc, x)
            else:
                _, y64 = orc.w4a16(nib, sc, x)
            _assert_close(ys[(l, slot)][:, rows], y64, 2e-3)


@pytest.mark.parametrize("mode", ["independent", "dataflow", "barrier"])
def test_step_kernel_m1_vs_oracle(mq, orc, mode):
    routes = (0, 1, 0, 1)
    st, ops = _step_stack(mq, mode, routes=routes)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.run(1, stream=s)
    s.synchronize()
    assert st.launches(1) == 1        # one persistent kernel per step
    # every linear against the oracle on the input it actually read (for chained
    # linears: the GPU's own output of the producing linear, final after the step)
    first = []
    for (l, slot, w, x, y) in ops:
        nib, sc = orc.pack_w4(_f32(w))
        xin = _f32(x)
        if routes[l] == 0:
            _, y64 = orc.w4a8_from_x(nib, sc, xin)
        else:
            _, y64 = orc.w4a16(nib, sc, xin)
        _assert_close(y, y64, 2e-3)
        first.append(y.clone())
    # replays (the epoch advances every launch; counters reset by the kernel) are bit-identical
    with torch.cuda.stream(s):
        st.capture(1, stream=s)
        for _ in range(3):
            for (_, _, _, _, y) in ops:    # every output is recomputed (chained inputs included)
                y.zero_()
            st.replay(stream=s)
            s.synchronize()
            for a, (_, _, _, _, y) in zip(first, ops):
                assert torch.equal(a, y)


def test_step_kernel_equals_per_linear_path(mq):
    """The persistent step kernel (M = 1, chained) and single mcapq_linear calls on
    the same inputs give bit-identical outputs (same engines, same K-only order)."""
    routes = (0, 1, 0, 1)
    st, ops = _step_stack(mq, "dataflow", routes=routes)
    st.run(1)
    torch.cuda.synchronize()
    for (l, slot, w, x, y) in ops:
        pw = mq.pack_w4(w.to(DEV))
        ref = mq.linear(routes[l], pw, x.clone(), out_dtype=torch.bfloat16)
        assert torch.equal(ref, y), (l, slot)


@pytest.mark.parametrize("m", [1, 4, 16, 64])
def test_pdl_chain_matches_plain(mq, m):
    """mcapq_set_pdl(1): a chain of dependent linears (each input the previous output)
    launched with programmatic dependent launch gives the same bits as plain launches
    (activations/outputs wait for the predecessor; only weights stream early)."""
    k = 2048
    ws = [mq.pack_w4(si.weight(k, k, 1600 + i).to(DEV)) for i in range(4)]
    x0 = si.activation(m, k, 1610 + m).to(DEV)
    torch.cuda.synchronize()

    def chain():
        y = x0
        outs = []
        for i, w in enumerate(ws):
            y = mq.linear(i % 2, w, y, out_dtype=torch.bfloat16)
            outs.append(y)
        return outs

    ref = chain()
    prev = mq.set_pdl(True)
    try:
        got = chain()
    finally:
        mq.set_pdl(prev)
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_colshard_nccl_world1(mq):
    """a8 through NCCL on this box's one GPU: mcapq_comm_init + mcapq_linear_colshard
    (local rows, ncclAllGather, the rank-major permute for M > 1) equals mcapq_linear."""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                            device_id=torch.device(DEV))
    try:
        comm = mq.Comm()
        n, k = 4096, 2048
        pw = mq.pack_w4(si.weight(n, k, 1701).to(DEV))
        for m in (1, 16):
            x = si.activation(m, k, 1702 + m).to(DEV)
            for route in (0, 1):
                y = mq.linear_colshard(comm, route, pw.shard(1, 0), n, x)
                torch.cuda.synchronize()
                assert torch.equal(y, mq.linear(route, pw, x, out_dtype=torch.bfloat16))
        del comm
    finally:
        dist.destroy_process_group()


def test_colshard_fused_nccl_world1(mq):
    """a8 fused epilogue through a real NCCL symmetric window on this box's one GPU:
    mcapq_comm_window_alloc (ncclMemAlloc + symmetric registration + an ncclDevComm with an
    LSA barrier), the GEMV epilogue storing into every LSA peer's replica, the LSA barrier
    kernel: y_full equals the plain linear bit-for-bit, for both routes; replays from a
    captured graph give the same bits."""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                            device_id=torch.device(DEV))
    try:
        comm = mq.Comm()
        n, k = 4096, 2048
        pw = mq.pack_w4(si.weight(n, k, 1721).to(DEV))
        x = si.activation(1, k, 1722).to(DEV)
        y = comm.window(n)
        for route in (0, 1):
            y.zero_()
            mq.linear_colshard(comm, route, pw.shard(1, 0), n, x, out=y, fused=True)
            torch.cuda.synchronize()
            ref = mq.linear(route, pw, x, out_dtype=torch.bfloat16)
            assert torch.equal(y, ref)
            st = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(st):
                ws = torch.empty(max(256, comm.workspace_bytes(route, 1, n, k)), dtype=torch.uint8, device=DEV)
                with torch.cuda.graph(g, stream=st):
                    mq.linear_colshard(comm, route, pw.shard(1, 0), n, x, out=y, ws=ws, stream=st, fused=True)
            y.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y, ref)
        comm.free_window(y)
        del comm
    finally:
        dist.destroy_process_group()


def test_rowshard_nccl_world1(mq, orc):
    """NEXT-2 through NCCL on this box's one GPU: mcapq_linear_rowshard (local K-slice
    partial, ncclAllReduce in place, conversion) for M = 1 / 16 and both routes, and the
    fused path through a real symmetric window (LSA barrier, epilogue stores into the
    window slots, LSA barrier, rank-order sum), eager and graph-replayed: at P = 1 both
    equal the plain linear (the sum of one partial is the partial)."""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                            device_id=torch.device(DEV))
    try:
        comm = mq.Comm()
        n, k = 2048, 4096
        pw = mq.pack_w4(si.weight(n, k, 1731).to(DEV))
        for m in (1, 16):
            x = si.activation(m, k, 1732 + m).to(DEV)
            for route in (0, 1):
                for dt in (torch.float32, torch.bfloat16):
                    y = mq.linear_rowshard(comm, route, pw.kshard(1, 0), x, out_dtype=dt)
                    torch.cuda.synchronize()
                    assert torch.equal(y, mq.linear(route, pw, x, out_dtype=dt))
        win = comm.window(n, torch.float32, rows=1)
        x = si.activation(1, k, 1740).to(DEV)
        for route in (0, 1):
            ref = mq.linear(route, pw, x, out_dtype=torch.bfloat16)
            y = mq.linear_rowshard(comm, route, pw.kshard(1, 0), x, ws=win, fused=True)
            torch.cuda.synchronize()
            assert torch.equal(y, ref)
            st = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            y2 = torch.empty_like(ref)
            with torch.cuda.stream(st):
                with torch.cuda.graph(g, stream=st):
                    mq.linear_rowshard(comm, route, pw.kshard(1, 0), x, out=y2, ws=win, stream=st, fused=True)
            y2.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y2, ref)
        comm.free_window(win)
        del comm
    finally:
        dist.destroy_process_group()


def test_step_kernel_k14336_chain(mq, orc):
    """The 8B MLP chain through the persistent step (K = 14336 input: 4 staging rounds per
    thread; both routes), each linear against the oracle on the input it actually read."""
    L, routes = 2, (0, 1)
    gate_n, hid = 14336, 2048
    st = mq.Stack(list(routes), max_m=1)
    ops = []
    prev = si.activation(1, hid, 1801).to(DEV)
    for l in range(L):
        shapes = (("gate", (gate_n, hid)), ("up", (gate_n, hid)), ("down", (hid, gate_n)))
        ws = {s_: si.weight(n, k, 1810 + 3 * l + i) for i, (s_, (n, k)) in enumerate(shapes)}
        y = {s_: torch.empty(1, w.shape[0], dtype=torch.bfloat16, device=DEV) for s_, w in ws.items()}
        pw = {s_: mq.pack_w4(w.to(DEV)) for s_, w in ws.items()}
        st.set(l, 0, 0, pw["gate"], prev, y["gate"])
        st.set(l, 1, 0, pw["up"], prev, y["up"])
        st.set(l, 2, 1, pw["down"], y["up"], y["down"])
        ops += [(l, ws["gate"], prev, y["gate"]), (l, ws["up"], prev, y["up"]), (l, ws["down"], y["up"], y["down"])]
        prev = y["down"]
    st.run(1)
    torch.cuda.synchronize()
    assert st.launches(1) == 1
    for (l, w, x, y) in ops:
        nib, sc = orc.pack_w4(_f32(w))
        if routes[l] == 0:
            _, y64 = orc.w4a8_from_x(nib, sc, _f32(x))
        else:
            _, y64 = orc.w4a16(nib, sc, _f32(x))
        _assert_close(y, y64, 2e-3)


def test_stack_step_host_chained(mq):
    """mcapq_stack_step_host on a chained stack: only the step input crosses H2D (one copy),
    every output comes back (one copy when the outputs share an arena), and the host copy of
    the outputs equals the device outputs of a plain run."""
    routes = (0, 1, 0, 1)
    st, ops = _step_stack(mq, "dataflow", routes=routes)
    bi, bo = st.host_bytes(1)
    k0 = STEP_DIMS["q"][1]
    assert bi == 2 * k0                          # layer 0's q/k/v input only
    assert bo == 2 * sum(n for n, _ in STEP_DIMS.values()) * len(routes)
    x0 = ops[0][3]
    xh = x0.cpu().view(torch.uint8).flatten().clone().pin_memory()
    yh = torch.empty(bo, dtype=torch.uint8).pin_memory()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.capture(1, stream=s)
        st.step_host(xh, yh, 1, stream=s)
    s.synchronize()
    off = 0
    for (_, _, _, _, y) in ops:
        nb = y.numel() * 2
        assert torch.equal(yh[off:off + nb].view(torch.bfloat16).view(y.shape), y.cpu())
        off += nb

"""Pins for the oracle's linears: W4A8 (rows a3/a5),
W4A16 exact (row a4) and W4A16 bf16-dequant (row a6; P:982,
reading A13).  Brute force in exact rationals on tiny shapes, closed forms and
special cases; the nibble unpacking used here is the test's own."""
from fractions import Fraction

import numpy as np
import pytest
import torch


def _codes(nib):
    # the test's own unpack of the split layout: byte t of a block holds
    # element t (low nibble) and element t+16 (high nibble)
    n, kh = nib.shape
    out = np.zeros((n, kh * 2), np.int64)
    for r in range(n):
        for g in range(kh // 16):
            for t in range(16):
                b = int(nib[r, 16 * g + t])
                out[r, 32 * g + t] = b & 15
                out[r, 32 * g + t + 16] = b >> 4
    return out


def _d(scale):
    return scale.view(np.float16).astype(np.float64)


def _bf16(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _rand(shape, seed, scale=1.0):
    return _bf16(np.random.default_rng(seed).standard_normal(shape) * scale)


def test_deferred_correction_identity(orc):
    # sumi - 8 sum_x == sum (c - 8) q, exactly, for random codes and activations
    rng = np.random.default_rng(21)
    w = _rand((24, 256), 1, 0.02)
    x = _rand((3, 256), 2)
    nib, sc = orc.pack_w4(w)
    q, s, sq = orc.quant_a8(x)
    D = orc.w4a8_group_dots(nib, q, sq)
    c = _codes(nib)
    centered = ((c[None, :, :] - 8) * q[:, None, :].astype(np.int64)).reshape(3, 24, 8, 32).sum(-1)
    assert np.array_equal(D.astype(np.int64), centered)
    # and the unsigned form with the explicit sum_x from the raw codes (sumi uses w_uns in [0, 15])
    sumi = (c[None] * q[:, None, :].astype(np.int64)).reshape(3, 24, 8, 32).sum(-1)
    sumx = q.astype(np.int64).reshape(3, 8, 32).sum(-1)
    assert np.array_equal(D.astype(np.int64), sumi - 8 * sumx[:, None, :])
    assert np.abs(D).max() <= 32 * 8 * 127


def test_w4a8_zero_activation_is_zero(orc):
    # all activation codes 0 -> output exactly 0
    nib, sc = orc.pack_w4(_rand((8, 64), 3))
    y32, y64 = orc.w4a8_from_x(nib, sc, np.zeros((1, 64), np.float32))
    assert np.all(y32 == 0) and np.all(y64 == 0)


def test_w4a8_brute_force(orc):
    # y = sum_g d_g s_g D_g computed in exact rationals; y64 within fp64 summation error,
    # y32 within the fp32 bound of its (G-term) sum
    for seed, (n, k, m) in enumerate([(5, 64, 1), (7, 32, 3), (4, 96, 2)]):
        w = _rand((n, k), 10 + seed, 0.05)
        x = _rand((m, k), 20 + seed, 2.0)
        nib, sc = orc.pack_w4(w)
        q, s, sq = orc.quant_a8(x)
        y32, y64 = orc.w4a8(nib, sc, q, s, sq)
        c = _codes(nib)
        d = _d(sc)
        for i in range(m):
            for r in range(n):
                exact = Fraction(0)
                absum = Fraction(0)
                for g in range(k // 32):
                    Dg = sum((int(c[r, 32 * g + j]) - 8) * int(q[i, 32 * g + j]) for j in range(32))
                    t = Fraction(float(d[r, g])) * Fraction(float(s[i, g])) * Dg
                    exact += t
                    absum += abs(t)
                G = k // 32
                assert abs(Fraction(float(y64[i, r])) - exact) <= absum * G * Fraction(2) ** -52
                assert abs(Fraction(float(y32[i, r])) - exact) <= absum * (G + 2) * Fraction(2) ** -23


def test_w4a8_vs_fp64_dequantised_product(orc):
    # vs full precision (dequantised weights . dequantised activations), rel err <= 1e-6
    for seed in range(20):
        w = _rand((16, 64), 100 + seed)
        x = _rand((1, 64), 200 + seed)
        nib, sc = orc.pack_w4(w)
        q, s, sq = orc.quant_a8(x)
        y32, y64 = orc.w4a8(nib, sc, q, s, sq)
        wd = orc.dequant_w4(nib, sc).astype(np.float64)
        xd = q.astype(np.float64) * np.repeat(s.astype(np.float64), 32, axis=1)
        ref = wd @ xd[0]
        tol = 1e-6 * np.abs(wd) @ np.abs(xd[0])
        assert np.all(np.abs(y64[0] - ref) <= tol)
        assert np.all(np.abs(y32[0] - ref) <= 1e-5 * np.abs(wd) @ np.abs(xd[0]))


def test_w4a16_zero_and_impulse_rows(orc):
    # S:324 x = 0 -> 0;  S:325 impulse rows (one code != 8 per row) -> y = d (c - 8) x_k exactly
    k = 128
    w = np.zeros((6, k), np.float32)
    picks = [(0, -8.0), (5, 7.0), (40, -3.0), (77, 0.5), (100, 1.0), (127, -0.25)]
    for r, (col, v) in enumerate(picks):
        w[r, col] = v
    nib, sc = orc.pack_w4(w)
    y32, _ = orc.w4a16(nib, sc, np.zeros((1, k), np.float32))
    assert np.all(y32 == 0)
    x = _rand((1, k), 7, 3.0)
    y32, y64 = orc.w4a16(nib, sc, x)
    for r, (col, v) in enumerate(picks):
        # the only non-zero weight is the block max -> code 0 -> d (0 - 8) = v exactly
        assert y32[0, r] == np.float32(v) * x[0, col]
        assert y64[0, r] == float(v) * float(x[0, col])


def test_w4a16_terms_exact_in_fp32(orc):
    # reading A10: f32(d) (c - 8) x is exact in fp32 (11 x 4 x 8 significand bits <= 24)
    nib, sc = orc.pack_w4(_rand((64, 256), 31, 0.03))
    x = _rand((1, 256), 32, 5.0)
    d = np.repeat(_d(sc), 32, axis=1)
    c = _codes(nib)
    t32 = (d.astype(np.float32) * (c - 8).astype(np.float32)) * x[0].astype(np.float32)
    t64 = d * (c - 8) * x[0].astype(np.float64)
    assert np.array_equal(t32.astype(np.float64), t64)


def test_w4a16_brute_force(orc):
    for seed, (n, k, m) in enumerate([(5, 64, 1), (3, 32, 4), (6, 96, 2)]):
        w = _rand((n, k), 40 + seed, 0.05)
        x = _rand((m, k), 50 + seed, 2.0)
        nib, sc = orc.pack_w4(w)
        y32, y64 = orc.w4a16(nib, sc, x)
        c = _codes(nib)
        d = _d(sc)
        for i in range(m):
            for r in range(n):
                terms = [Fraction(float(d[r, j // 32])) * (int(c[r, j]) - 8) * Fraction(float(x[i, j])) for j in range(k)]
                exact = sum(terms, Fraction(0))
                absum = sum((abs(t) for t in terms), Fraction(0))
                assert abs(Fraction(float(y64[i, r])) - exact) <= absum * k * Fraction(2) ** -53
                assert abs(Fraction(float(y32[i, r])) - exact) <= absum * k * Fraction(2) ** -24


def test_w4a16_bf16deq_matches_bf16_rounded_weights(orc):
    # A13: W^ = bf16_rne(d (c - 8)); y = X W^T with fp32 accumulation.  The test rounds
    # with torch's converter (independent), then multiplies in fp64.
    nib, sc = orc.pack_w4(_rand((32, 512), 61, 0.02))
    x = _rand((4, 512), 62)
    y32, y64 = orc.w4a16_bf16deq(nib, sc, x)
    wd = (np.repeat(_d(sc), 32, axis=1) * (_codes(nib) - 8)).astype(np.float32)
    wb = _bf16(wd).astype(np.float64)
    ref = x.astype(np.float64) @ wb.T
    bound = np.abs(x.astype(np.float64)) @ np.abs(wb.T)
    assert np.all(np.abs(y64 - ref) <= bound * 512 * 2.0 ** -53)
    assert np.all(np.abs(y32 - ref) <= bound * 512 * 2.0 ** -24)
    # and it genuinely differs from exact dequant (the reason A13 exists)
    ye, _ = orc.w4a16(nib, sc, x)
    assert not np.array_equal(ye, y32)


def test_routes_do_not_change_row_results(orc):
    # A22 (sharding): every row is an independent K-length dot product
    w = _rand((32, 128), 71, 0.02)
    x = _rand((2, 128), 72)
    nib, sc = orc.pack_w4(w)
    for P in (2, 4, 8):
        for route in (orc.W4A8, orc.W4A16):
            full = orc.colshard_linear(route, nib, sc, x, 1)
            sh = orc.colshard_linear(route, nib, sc, x, P)
            assert np.array_equal(full, sh)
    with pytest.raises(orc.OracleError):
        orc.colshard_rows(30, 4, 0)

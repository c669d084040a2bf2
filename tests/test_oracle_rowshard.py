"""Pins for the oracle's row-parallel (K-sharded) linear (NEXT-2: "row-parallel
o/down with reduce-scatter or all-reduce"): the sharded sum against the unsharded
linear (the K-sum splits over whole groups: an identity up to fp64 rounding), the
locality of the per-token quantiser and of the per-group int32 dots (P:2346-2353,
P:937-942: a group never straddles two ranks, so the shard's codes and dots are slices
of the unsharded ones, bit for bit), and an exact-rational brute force of one tiny
sharded W4A16 product (tests/fractions_ref.py, independent of oracle/)."""
from fractions import Fraction

import numpy as np
import pytest

import synth_inputs as si
from fractions_ref import to_f16


def _inputs(n, k, m, seed):
    w = si.weight(n, k, seed).float().numpy()
    x = si.activation(m, k, seed + 1).float().numpy()
    return w, x


@pytest.mark.parametrize("route", [0, 1])
@pytest.mark.parametrize("P", [2, 4])
def test_sharded_sum_equals_unsharded(orc, route, P):
    n, k, m = 48, 1024, 3
    w, x = _inputs(n, k, m, 11 + P)
    nib, sc = orc.pack_w4(w)
    y32, y64 = orc.rowshard_linear(route, nib, sc, x, P)
    if route == 0:
        u32, u64 = orc.w4a8_from_x(nib, sc, x)
    else:
        u32, u64 = orc.w4a16(nib, sc, x)
    scale = np.maximum(np.abs(u64), np.sqrt(np.mean(u64 ** 2)))
    assert np.max(np.abs(y64 - u64) / scale) < 1e-12
    # the fp32 rank-order sum of fp32 partials: within fp32 rounding of the fp64 result
    assert np.max(np.abs(y32.astype(np.float64) - u64) / scale) < 1e-5


def test_quantiser_and_group_dots_are_rank_local(orc):
    n, k, m, P = 40, 2048, 2, 4
    w, x = _inputs(n, k, m, 21)
    nib, sc = orc.pack_w4(w)
    q, s, sq = orc.quant_a8(x)
    D = orc.w4a8_group_dots(nib, q, sq)
    for r in range(P):
        a, b = orc.rowshard_cols(k, P, r)
        qr, sr, sqr = orc.quant_a8(x[:, a:b])
        assert np.array_equal(qr, q[:, a:b])
        assert np.array_equal(sr.view(np.uint32), s[:, a // 32:b // 32].view(np.uint32))
        assert np.array_equal(sqr, sq[:, a // 32:b // 32])
        Dr = orc.w4a8_group_dots(nib[:, a // 2:b // 2], qr, sqr)
        assert np.array_equal(Dr, D[:, :, a // 32:b // 32])


def test_bad_slices_rejected(orc):
    with pytest.raises(orc.OracleError):
        orc.rowshard_cols(96, 2, 0)        # 48 columns per rank: not whole 32-groups
    with pytest.raises(orc.OracleError):
        orc.rowshard_cols(100, 3, 0)


def test_brute_force_tiny_w4a16(orc):
    """y = sum over ranks of sum over k of d(c - 8) x, exactly, for a 2 x 128 weight at P = 2:
    the oracle's fp64 rank sum must equal the exact rational to fp64 precision."""
    n, k, P = 2, 128, 2
    w, x = _inputs(n, k, 1, 31)
    nib, sc = orc.pack_w4(w)
    c = orc.codes(nib).astype(np.int64)
    d = orc.f16_bits_to_f32(sc).astype(np.float64)
    # the scale is an fp16 value: check the oracle's decoding against the exact rounding of d
    for v in d.ravel()[:4]:
        assert Fraction(float(v)) == to_f16(Fraction(float(v)))
    _, y64 = orc.rowshard_linear(1, nib, sc, x, P)
    for i in range(n):
        exact = Fraction(0)
        for kk in range(k):
            exact += Fraction(float(d[i, kk // 32])) * (int(c[i, kk]) - 8) * Fraction(float(x[0, kk]))
        assert abs(float(exact) - y64[0, i]) <= 1e-12 * max(1.0, abs(float(exact)))

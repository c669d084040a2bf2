"""Pins for the oracle's Q4_0 weight pack (row a1).

Readings pinned here: A2 (d = m / -8), A3 (first index on ties), A4 (codes from
the stored fp16 scale; zero / overflow edges), A5 (half away from zero; the
saturation-aware error bound), A21 (+0 scale for zero blocks).
"""
from fractions import Fraction

import numpy as np
import pytest

from fractions_ref import round_half_away, to_f16


def _block(vals):
    b = np.zeros((1, 32), np.float32)
    b[0, : len(vals)] = vals
    return b


def test_q4_0_is_18_bytes_per_32_and_4_5_bpw(orc):
    # P:932 "18 bytes per 32 elements"; "4.5 bpw"
    w = np.random.default_rng(0).standard_normal((3, 64)).astype(np.float32)
    nib, sc = orc.pack_w4(w)
    aos = orc.export_q4_0_aos(nib, sc)
    assert len(aos) == 3 * 2 * 18
    assert len(aos) * 8 / w.size == 4.5
    assert nib.nbytes + sc.nbytes == len(aos)


def test_zero_block(orc):
    # S:289 "all zeros -> d=0, all codes 8, dequantizes to zeros"; A21: d stored as +0
    for z in (0.0, -0.0):
        nib, sc = orc.pack_w4(np.full((1, 32), z, np.float32))
        assert sc[0, 0] == 0x0000
        assert np.all(nib == 0x88)
        assert np.all(orc.dequant_w4(nib, sc) == 0)


def test_extreme_value_worked_example(orc):
    # block = [-8, 0 x 31] -> m = -8, d = 1, code_0 = 0, dequant = -8 exactly
    nib, sc = orc.pack_w4(_block([-8.0]))
    assert sc[0, 0] == 0x3C00                 # fp16 1.0
    assert nib[0, 0] == 0x80                   # c_0 = 0 (low), c_16 = 8 (high)  -- P:933 split layout
    assert np.all(nib[0, 1:] == 0x88)
    dq = orc.dequant_w4(nib, sc)
    assert dq[0, 0] == -8.0 and np.all(dq[0, 1:] == 0)


def test_split_nibble_layout(orc):
    # P:933 / S:270: byte t = c_t | c_{t+16} << 4.  Build codes c_j = j % 16 with d = 1:
    # x_j = c_j - 8, but the max-magnitude element must be -8 (c=0) first.
    c = np.array([(j * 7) % 16 for j in range(32)])
    c[0] = 0
    x = (c - 8).astype(np.float32)[None, :]
    nib, sc = orc.pack_w4(x)
    assert sc[0, 0] == 0x3C00
    expect = np.array([c[t] | (c[t + 16] << 4) for t in range(16)], np.uint8)
    assert np.array_equal(nib[0], expect)
    assert np.array_equal(orc.codes(nib)[0], c)


def test_tie_break_first_index(orc):
    # A3: +a at index i and -a at j: the first decides the sign of d
    for i, j in [(0, 5), (5, 0), (31, 30), (3, 17)]:
        x = np.zeros((1, 32), np.float32)
        x[0, i], x[0, j] = 3.0, -3.0
        nib, sc = orc.pack_w4(x)
        d = np.array([sc[0, 0]], np.uint16).view(np.float16)[0]
        first = x[0, min(i, j)]
        assert d == np.float16(first / -8.0)
        c = orc.codes(nib)[0]
        assert c[min(i, j)] == 0                  # the extreme maps to code 0 (A2)
        assert c[max(i, j)] == 15                 # the opposite sign saturates at +7 (A5)


def test_rounding_boundaries(orc):
    # A5: codes for x = (k +- 0.5) d and +-1 ulp around them, d = 1/8 (m = -1)
    d = 0.125
    for k in range(-8, 8):
        for center in (k - 0.5, k + 0.5):
            for ulps in (-1, 0, 1):
                v = np.float32(center * d)
                if ulps:
                    v = np.nextafter(v, np.float32(np.inf * ulps), dtype=np.float32)
                if abs(v) >= 1.0:
                    continue
                x = _block([-1.0, v])
                nib, sc = orc.pack_w4(x)
                assert sc[0, 0] == 0x3000              # fp16 0.125
                q = float(v) / d
                if ulps == 0:                         # exact half-way: away from zero
                    r = np.sign(q) * np.floor(abs(q) + 0.5)
                else:
                    r = np.round(q)                   # not a tie: nearest
                expect = int(min(max(r, -8), 7)) + 8
                assert orc.codes(nib)[0, 1] == expect, (k, center, ulps, v)


def test_brute_force_exact_rationals(orc):
    # Recompute d and every code with exact rationals (fractions_ref), from bf16 inputs.
    rng = np.random.default_rng(3)
    import torch
    w = torch.from_numpy(rng.standard_normal((16, 64)).astype(np.float32) * 0.02).to(torch.bfloat16).float().numpy()
    w[3, :32] *= 1e-5                            # fp16-subnormal d
    nib, sc = orc.pack_w4(w)
    c = orc.codes(nib)
    for r in range(16):
        for g in range(2):
            blk = w[r, 32 * g: 32 * g + 32]
            idx = int(np.argmax(np.abs(blk)))      # numpy argmax: first index on ties
            m = Fraction(float(blk[idx]))
            d = to_f16(m / -8)
            got_d = float(np.array([sc[r, g]], np.uint16).view(np.float16)[0])
            assert float(d) == got_d
            for j in range(32):
                if d == 0:
                    e = 8
                else:
                    e = min(max(round_half_away(Fraction(float(blk[j])) / d), -8), 7) + 8
                assert c[r, 32 * g + j] == e


@pytest.mark.parametrize("dist", ["normal", "uniform", "cauchy"])
def test_round_trip_saturation_aware_bound(orc, dist):
    # A5 invariant: |x - d(c-8)| <= |d|/2 for non-saturated codes, <= |d|(1 + 2^-8) at code 15
    rng = np.random.default_rng({"normal": 1, "uniform": 2, "cauchy": 3}[dist])
    n = 10000
    if dist == "normal":
        w = rng.standard_normal((n, 32))
    elif dist == "uniform":
        w = rng.uniform(-1, 1, (n, 32))
    else:
        w = np.clip(rng.standard_cauchy((n, 32)), -1e3, 1e3)
    w = w.astype(np.float32)
    nib, sc = orc.pack_w4(w)
    dq = orc.dequant_w4(nib, sc).astype(np.float64)
    d = np.abs(sc.view(np.float16).astype(np.float64))        # [n, 1]
    err = np.abs(dq - w.astype(np.float64))
    c = orc.codes(nib)
    sat = c == 15
    # non-saturated: half a step, plus the fp16 rounding of d moving the grid (x/d ≤ 8(1+2^-11))
    dd = np.broadcast_to(d, err.shape)
    assert np.all(err[~sat] <= dd[~sat] * 0.5 * (1 + 2.0 ** -20))
    assert np.all(err[sat] <= dd[sat] * (1 + 2.0 ** -8))
    assert sat.any(1).mean() > 0.05                # the naive |d|/2 bound really fails here


def test_idempotence(orc):
    # pack(dequant(pack(W))) == pack(W), byte-identical (S:297 fixpoint)
    rng = np.random.default_rng(5)
    w = rng.standard_normal((2000, 64)).astype(np.float32)
    nib, sc = orc.pack_w4(w)
    nib2, sc2 = orc.pack_w4(orc.dequant_w4(nib, sc))
    assert np.array_equal(nib, nib2) and np.array_equal(sc, sc2)


def test_fp16_overflow_and_nonfinite_are_errors(orc):
    # A4: |m|/8 rounds to fp16 inf -> ERANGE; non-finite input -> error
    st, _, _ = orc.pack_w4_status(_block([6e5]))
    assert st == 3
    st, _, _ = orc.pack_w4_status(_block([5.2e5]))     # 5.2e5/8 = 65000 < 65520: fine
    assert st == 0
    st, _, _ = orc.pack_w4_status(_block([np.nan]))
    assert st == 3
    with pytest.raises(orc.OracleError):
        orc.pack_w4(_block([np.inf]))


def test_k_must_be_multiple_of_32(orc):
    with pytest.raises(orc.OracleError):
        orc.pack_w4(np.zeros((2, 48), np.float32))


def test_golden_extreme_block_bytes(orc):
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "q4_0_extreme_block.txt")
    lines = {l.split(":")[0]: l.split(":")[1].split() for l in open(path) if not l.startswith("#") and ":" in l}
    x = np.array([[float(v) for v in lines["input"]]], np.float32)
    nib, sc = orc.pack_w4(x)
    assert orc.export_q4_0_aos(nib, sc) == bytes(int(b, 16) for b in lines["aos18"])

"""Pins for the oracle's per-group int8 activation quantiser (row a2;
P:929-931; readings A6, A7, A8, A21)."""
from fractions import Fraction

import numpy as np
import pytest
import torch

from fractions_ref import round_half_away, to_f32


def test_unit_scale_worked_example(orc):
    # group with amax = 127 -> s = 1, codes = rounded inputs
    x = np.zeros((1, 32), np.float32)
    x[0, :5] = [127.0, -3.5, 2.5, 0.49, -126.6]
    q, s, sq = orc.quant_a8(x)
    assert s[0, 0] == 1.0
    assert list(q[0, :5]) == [127, -4, 3, 0, -127]
    assert sq[0, 0] == 127 - 4 + 3 + 0 - 127


def test_zero_group(orc):
    # S:307 / A21: all zeros -> s = +0, all codes 0
    q, s, sq = orc.quant_a8(np.zeros((2, 64), np.float32))
    assert np.all(q == 0) and np.all(sq == 0)
    assert np.all(s.view(np.uint32) == 0)


def test_brute_force_exact_rationals(orc):
    # s = fp32(amax / 127) (IEEE quotient), q = round_half_away(fp32(x / s))
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.standard_normal((3, 128)).astype(np.float32) * 3).to(torch.bfloat16).float().numpy()
    x[1, 40] = 0.0
    q, s, sq = orc.quant_a8(x)
    for i in range(3):
        for g in range(4):
            grp = x[i, 32 * g: 32 * g + 32]
            amax = max(abs(Fraction(float(v))) for v in grp)
            sx = to_f32(amax / 127)
            assert float(sx) == float(s[i, g])
            tot = 0
            for j in range(32):
                e = min(max(round_half_away(to_f32(Fraction(float(grp[j])) / sx)), -127), 127)
                assert q[i, 32 * g + j] == e
                tot += e
            assert sq[i, g] == tot                         # sum_x


def test_error_bound_and_clamp_never_needed(orc):
    # A7: |s q - x| <= s (1/2 + 127 * 2^-24); the +-127 clamp only absorbs the quotient's rounding
    rng = np.random.default_rng(12)
    x = (rng.standard_normal((500, 1024)) * np.exp(rng.uniform(-5, 5, (500, 1)))).astype(np.float32)
    q, s, sq = orc.quant_a8(x)
    sg = np.repeat(s, 32, axis=1).astype(np.float64)
    err = np.abs(sg * q - x.astype(np.float64))
    assert np.all(err <= sg * (0.5 + 127 * 2.0 ** -24))
    assert np.abs(q).max() == 127
    assert np.array_equal(sq, q.reshape(500, 32, 32).astype(np.int64).sum(-1))


def test_per_token_rows_independent(orc):
    # A6: quantisation is per token row and per 32-group: rows never interact
    rng = np.random.default_rng(13)
    x = rng.standard_normal((4, 96)).astype(np.float32)
    q, s, sq = orc.quant_a8(x)
    for i in range(4):
        qi, si, sqi = orc.quant_a8(x[i:i + 1])
        assert np.array_equal(qi[0], q[i]) and np.array_equal(si[0], s[i]) and np.array_equal(sqi[0], sq[i])


def test_nonfinite_is_error(orc):
    x = np.zeros((1, 32), np.float32)
    x[0, 3] = np.inf
    with pytest.raises(orc.OracleError):
        orc.quant_a8(x)

"""Host-side pins of the arithmetic identities the fused W4A8 quantiser relies on
(no GPU, no product code: the identities are checked in exact rational arithmetic).

The activation scale is s = fl(amax / 127) in IEEE round-to-nearest (PAPER.md P:2351,
app:kernels; reading A7).  The kernels compute it without a division, as one
correction step from r = fl(1/127):  q0 = fl(a r);  e = fl(a - 127 q0) (one FMA);
s = fl(q0 + e r) (one FMA).  amax is the magnitude of a bf16 activation, so every
possible input is enumerable: this test checks all 32640 finite non-negative bf16
magnitudes (subnormals included) against the correctly rounded quotient.
"""
import math
import struct
from fractions import Fraction as F

import pytest


def _rnd32(q: F) -> F:
    """Round a rational to the nearest fp32 value (ties to even), subnormals included."""
    if q == 0:
        return F(0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while F(2) ** e > a:
        e -= 1
    while F(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)
    ulp = F(2) ** (e - 23)
    m = a / ulp
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > F(1, 2) or (rem == F(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * fl * ulp


def _bf16(bits: int) -> F:
    return F(struct.unpack("<f", struct.pack("<I", bits << 16))[0])


def test_rnd32_matches_hardware_rounding():
    # the helper itself against numpy's fp32 rounding on values with a plain decimal form
    import numpy as np
    for x in (1 / 3, 2 / 7, 1e-40, 3.4e38, 0.1, 127.5, 2.0 ** -149 * 1.5):
        assert _rnd32(F(x)) == F(float(np.float32(x)))


def test_div127_one_correction_step_is_exact_for_every_bf16_magnitude():
    r = _rnd32(F(1, 127))
    assert float(r) == float.fromhex("0x1.020408p-7")      # the constant in div127_rn
    bad = []
    for b in range(0, 0x7F80):                               # all finite bf16 magnitudes
        a = _bf16(b)
        q0 = _rnd32(a * r)
        e = _rnd32(a - 127 * q0)                             # fma(-q0, 127, a)
        s = _rnd32(e * r + q0)                               # fma(e, r, q0)
        if s != _rnd32(a / 127):
            bad.append(hex(b))
    assert not bad, bad[:8]


@pytest.mark.parametrize("amax_bits", [0x0001, 0x0080, 0x3F80, 0x42FE, 0x7F7F])
def test_scale_never_underflows_to_zero(amax_bits):
    # live <=> amax != 0: the smallest bf16 subnormal / 127 is still a nonzero fp32
    assert _rnd32(_bf16(amax_bits) / 127) != 0


# ---------------------------------------------------------------------------
# tcgen05 bf16-dequant path (mcapq_w4a16_bf16deq, reading A13'): the kernel forms
# W^ = bf16_rne(f32(d) (c - 8)) in bf16x2 arithmetic as rn(hi (c - 8) + lo (c - 8)) with
# hi = bf16_rne(d), lo = d - hi.  That is one rounding of the exact product iff lo and
# lo (c - 8) are exact in bf16 (8 significant bits) -- checked here for every finite fp16 d
# and every code, in exact binary arithmetic (float64 holds all these values exactly).
def _sig_bits(v):
    """Significant bits of each (exactly float64-representable) value; 0 for zero."""
    import numpy as np
    v = np.abs(np.asarray(v, np.float64))
    m, _ = np.frexp(v)                       # v = m 2^e, m in [0.5, 1)
    bits = np.zeros(v.shape, np.int64)
    nz = v != 0
    mant = (m[nz] * 2.0 ** 53).astype(np.uint64)
    tz = np.zeros(mant.shape, np.int64)
    x = mant.copy()
    for _ in range(53):
        z = (x & np.uint64(1)) == 0
        tz += z & (x != 0)
        x = np.where(z, x >> np.uint64(1), x)
    bits[nz] = 53 - tz
    return bits


def _bf16_rne(v):
    import numpy as np
    import torch
    return torch.from_numpy(np.asarray(v, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def test_bf16deq_split_scale_is_one_rounding():
    import numpy as np
    h = np.arange(0, 0x10000, dtype=np.uint32).astype(np.uint16)
    d = h.view(np.float16).astype(np.float64)
    d = d[np.isfinite(d)]
    hi = _bf16_rne(d)
    lo = d - hi                                        # exact in float64
    assert (_sig_bits(lo) <= 8).all()                  # lo is a bf16 value
    assert (np.abs(hi) < 3.0e38).all()
    for c in range(16):
        e = lo * (c - 8)
        assert (_sig_bits(e) <= 8).all(), c            # lo (c - 8) is exact in bf16
        exact = d * (c - 8)                            # = hi (c - 8) + e, exactly
        assert np.array_equal(hi * (c - 8) + e, exact)

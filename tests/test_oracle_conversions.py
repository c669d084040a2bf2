"""Pins for the oracle's IEEE conversions (conversions).

fp32->fp16 RNE is checked EXHAUSTIVELY (all 2^32 inputs) against the x86 F16C
hardware converter; fp16->fp32 over all 65536 halves.  fp32->bf16 RNE is checked
against torch's converter over every exponent with random and tie mantissas, and
against exact-rational rounding.
"""
import os
import shutil
import subprocess
from fractions import Fraction

import numpy as np
import pytest
import torch

from fractions_ref import to_bf16, to_f16

HERE = os.path.dirname(os.path.abspath(__file__))


def _has_f16c():
    try:
        with open("/proc/cpuinfo") as f:
            return " f16c" in f.read()
    except OSError:
        return False


@pytest.mark.skipif(not _has_f16c() or shutil.which("gcc") is None, reason="needs x86 F16C + gcc")
def test_f16_exhaustive_vs_f16c(orc, tmp_path):
    exe = tmp_path / "f16c"
    libdir = os.path.dirname(str(orc.build()))
    subprocess.run(["gcc", "-O2", "-mf16c", "-fopenmp", os.path.join(HERE, "pins", "f16c_exhaustive.c"),
                    str(orc.build()), f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.split() == ["0", "0"]


def test_f16_specials_vs_exact_rounding(orc):
    vals = [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26,
            2.0 ** -14, 2.0 ** -14 - 2.0 ** -25, 1.0 / 3, 0.1, 1e-7, 12345.678]
    x = np.array(vals, np.float32)
    got = orc.f32_to_f16_bits(x).view(np.float16).astype(np.float64)
    for v32, g in zip(x, got):
        ref = to_f16(Fraction(float(v32)))
        assert float(ref) == g or (np.isinf(g) and np.isinf(float(ref)))


def test_bf16_vs_torch_all_exponents(orc):
    rng = np.random.default_rng(7)
    exps = np.arange(0, 256, dtype=np.uint32)
    mant = rng.integers(0, 1 << 23, size=(256, 64), dtype=np.uint32)
    mant[:, 0] = 0x8000          # exact tie, even keep
    mant[:, 1] = 0x18000         # exact tie, odd keep
    mant[:, 2] = 0x7FFF
    mant[:, 3] = 0x7FFFFF        # carries into the exponent
    u = (exps[:, None] << 23) | mant
    u = np.concatenate([u, u | 0x80000000]).ravel()
    f = u.view(np.float32)
    finite = np.isfinite(f)
    got = orc.f32_to_bf16_bits(f)
    ref = torch.from_numpy(f.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got[finite], ref[finite])
    # non-finite: inf stays inf, nan stays nan
    g_nan = got[np.isnan(f)]
    assert np.all((g_nan & 0x7F80) == 0x7F80) and np.all(g_nan & 0x7F)


def test_bf16_vs_exact_rounding(orc):
    rng = np.random.default_rng(11)
    f = (rng.standard_normal(2000) * np.exp(rng.uniform(-30, 30, 2000))).astype(np.float32)
    got = orc.bf16_bits_to_f32(orc.f32_to_bf16_bits(f))
    for a, g in zip(f, got):
        assert float(to_bf16(Fraction(float(a)))) == float(g)


def test_f16_to_f32_subnormals(orc):
    h = np.arange(0, 1024, dtype=np.uint16)
    got = orc.f16_bits_to_f32(h)
    assert np.array_equal(got.astype(np.float64), np.arange(1024) * 2.0 ** -24)

"""Exact-rational brute-force helpers for the oracle pins.

Independent of oracle/: nothing here imports it.  IEEE rounding is written out
on Fractions (round-to-nearest-even to a given significand width), so a pin
built from these helpers checks the oracle against the mathematics, not
against itself.
"""
from fractions import Fraction
import math
import struct


def f32_bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def bits_f32(u: int) -> float:
    return struct.unpack("<f", struct.pack("<I", u & 0xFFFFFFFF))[0]


def round_to_binary(v: Fraction, mant_bits: int, emin: int, emax: int):
    """Round an exact rational to the nearest binary float with `mant_bits`
    significand bits (incl. hidden), min normal exponent emin, max exponent emax,
    ties to even.  Returns a Fraction, or +-inf as float."""
    if v == 0:
        return Fraction(0)
    sign = -1 if v < 0 else 1
    a = abs(v)
    e = math.floor(math.log2(a.numerator) - math.log2(a.denominator))
    # fix e so that 2^e <= a < 2^(e+1)
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, emin)                       # subnormal range: fixed quantum
    q = Fraction(2) ** (e - (mant_bits - 1))
    n = a / q
    fl = n.numerator // n.denominator
    rem = n - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    r = fl * q
    if r >= Fraction(2) ** (emax + 1):
        return sign * math.inf
    return sign * r


def to_f32(v: Fraction):
    return round_to_binary(v, 24, -126, 127)


def to_f16(v: Fraction):
    return round_to_binary(v, 11, -14, 15)


def to_bf16(v: Fraction):
    return round_to_binary(v, 8, -126, 127)


def round_half_away(v: Fraction) -> int:
    a = abs(v)
    fl = a.numerator // a.denominator
    r = fl + 1 if a - fl >= Fraction(1, 2) else fl
    return -r if v < 0 else r

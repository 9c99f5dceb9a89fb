"""Exact rational reference arithmetic used to PIN the oracle (not the oracle
itself): IEEE binary32 round-to-nearest-even of an exact rational, written
from the binary32 definition with python `fractions`.  Nothing here is shared
with oracle/ or with the CUDA path."""
from __future__ import annotations

from fractions import Fraction

import numpy as np

FLT_MAX = Fraction(2) ** 127 * (2 - Fraction(1, 2 ** 23))


def f32(v) -> Fraction:
    """Exact value of a binary32 number."""
    return Fraction(float(np.float32(v)))


def rn32(x: Fraction) -> float:
    """Round an exact rational to the nearest binary32 (ties to even)."""
    if x == 0:
        return 0.0
    sign = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)
    ulp = Fraction(2) ** (e - 23)
    n = round(a / ulp)             # Fraction.__round__ is half-to-even
    r = n * ulp
    if r > FLT_MAX:
        return sign * float("inf")
    return sign * float(r)


def quant_exact(x, s, qmin, qmax) -> int:
    """Eq.1 under R1-R3 in exact arithmetic: q = clamp(round_even(rn32(x/s)))."""
    v = Fraction(rn32(f32(x) / f32(s)))
    r = round(v)                   # half-to-even
    return int(min(max(r, qmin), qmax))


def dequant_exact(acc: int, s_a, s_w, b=None) -> float:
    """R4: sc = rn32(s_a*s_w); y = rn32(acc*sc + b) (fma = one rounding)."""
    sc = Fraction(rn32(f32(s_a) * f32(s_w)))
    a = Fraction(rn32(Fraction(int(acc))))
    if b is None:
        return rn32(a * sc)
    return rn32(a * sc + f32(b))

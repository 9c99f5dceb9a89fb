"""Fit the frozen fp32 coefficients of `gelu_pinned` (reading R7).

This is a one-off documentation tool.  Neither `oracle/` nor the CUDA library
imports it: both sides carry the printed hex-float constants typed from
DESIGN.md.  Re-running it must reproduce the same constants (deterministic).

erf_pinned(t), t >= 0:
  piece 1, t < 1     : erf(t) = t * P(t^2),      P degree 6
  piece 2, t < 3.92  : erf(t) = 1 - Q(t - 2.5),  Q degree 12   (Q fits erfc)
  t >= 3.92          : erf(t) = 1   (erfc(3.92) = 2.96e-8 < 2^-25)
"""
import numpy as np
from scipy.special import erf, erfc


def fit():
    n = 20001
    t = np.linspace(0.0, 1.0, n)
    tt = np.where(t > 0, t, 1.0)
    g = np.where(t > 0, erf(tt) / tt, 2.0 / np.sqrt(np.pi))
    p = np.polyfit(t * t, g, 6).astype(np.float32)          # highest power first
    t2 = np.linspace(1.0, 3.92, 2 * n)
    q = np.polyfit(t2 - 2.5, erfc(t2), 12).astype(np.float32)
    return p, q


if __name__ == "__main__":
    p, q = fit()
    print("P (degree 6 .. 0):")
    for c in p:
        print("  ", float(c).hex(), repr(float(c)))
    print("Q (degree 12 .. 0):")
    for c in q:
        print("  ", float(c).hex(), repr(float(c)))

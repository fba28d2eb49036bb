"""Fit the fp32 erf of the accumulation kernel (csrc/accumulate.cu):

    erf_fast(x) = sign(x) (1 - 2^Q(|x|))   for |x| < 3.92   (Q: polynomial of degree DEG)
                = sign(x)                   for |x| >= 3.92  (exact fp32 saturation)

Weighted least squares iterated toward minimax of the absolute erf error on
Chebyshev nodes of [0, 3.92]; prints the fp32 coefficients (highest degree
first, the kernel's Horner order) and the max abs error of the fp32 evaluation
(ex2 taken exact here; the MUFU ex2.approx adds ~2 ulp relative to 2^Q).
Part of the CUDA path's constant generation only (the oracle uses libm erf).

    python tools/fit_erf.py [DEG]       # the kernel uses DEG = 7
"""
import sys

import numpy as np
from scipy.special import erf, erfc

XS = 3.92


def fit(deg):
    x = np.cos(np.linspace(0, np.pi, 6000)) * 0.5 * XS + 0.5 * XS
    y = np.log2(erfc(x))
    V = np.vander(x, deg + 1, increasing=True)
    wgt = erfc(x) * np.log(2)  # d erf = -erfc ln2 dQ
    c = np.linalg.lstsq(V * wgt[:, None], y * wgt, rcond=None)[0]
    for _ in range(60):
        e = (V @ c - y) * wgt
        w2 = wgt * (1 + 80 * np.abs(e) / np.abs(e).max())
        c = np.linalg.lstsq(V * w2[:, None], y * w2, rcond=None)[0]
    xs = np.linspace(0, XS, 400001)
    ca = c.astype(np.float32)
    x32 = xs.astype(np.float32)
    p = np.float32(ca[-1])
    for cc in ca[-2::-1]:
        p = p * x32 + np.float32(cc)
    v = np.float32(1) - np.exp2(p.astype(np.float64)).astype(np.float32)
    return ca, np.abs(v.astype(np.float64) - erf(xs)).max()


if __name__ == "__main__":
    deg = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    ca, err = fit(deg)
    print(f"degree {deg}: max abs err {err:.3e}")
    for c in ca[::-1]:
        print("  %.9e" % c)

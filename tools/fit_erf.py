"""Fit the fp32 erf used by the accumulation kernel (csrc/accumulate.cu).

erf_fast(x) = x * P(x^2)            for |x| < 0.75   (P: degree 5)
            = 1 - 2^Q(|x|)           for 0.75 <= |x| < 3.92   (Q: degree 7)
            = +-1                    for |x| >= 3.92  (exact saturation)

Weighted least squares iterated toward minimax on Chebyshev nodes; prints the
fp32 coefficients and the max abs error of an fp32 Horner evaluation.  Part of
the CUDA path's constant generation only (the oracle uses libm erf).
"""
import numpy as np
from scipy.special import erf, erfc

XS = 3.92


def fit_small(XA, deg):
    x = np.cos(np.linspace(0, np.pi, 4000)) * 0.5 * XA + 0.5 * XA
    x = x[x > 1e-6]
    y = erf(x) / x
    V = np.vander(x ** 2, deg + 1, increasing=True)
    w = x
    c = np.linalg.lstsq(V * w[:, None], y * w, rcond=None)[0]
    for _ in range(30):
        e = (V @ c - y) * x
        w2 = w * (1 + 50 * np.abs(e) / np.abs(e).max())
        c = np.linalg.lstsq(V * w2[:, None], y * w2, rcond=None)[0]
    xs = np.linspace(0, XA, 200001)
    ca = c.astype(np.float32)
    x32 = xs.astype(np.float32)
    z = x32 * x32
    p = np.float32(ca[-1])
    for cc in ca[-2::-1]:
        p = p * z + np.float32(cc)
    return c, np.abs((x32 * p).astype(np.float64) - erf(xs)).max()


def fit_large(XA, deg):
    x = np.cos(np.linspace(0, np.pi, 4000)) * 0.5 * (XS - XA) + 0.5 * (XS + XA)
    y = np.log2(erfc(x))
    V = np.vander(x, deg + 1, increasing=True)
    wgt = erfc(x)
    c = np.linalg.lstsq(V * wgt[:, None], y * wgt, rcond=None)[0]
    for _ in range(30):
        e = (V @ c - y) * wgt
        w2 = wgt * (1 + 50 * np.abs(e) / np.abs(e).max())
        c = np.linalg.lstsq(V * w2[:, None], y * w2, rcond=None)[0]
    xs = np.linspace(XA, XS, 200001)
    ca = c.astype(np.float32)
    x32 = xs.astype(np.float32)
    p = np.float32(ca[-1])
    for cc in ca[-2::-1]:
        p = p * x32 + np.float32(cc)
    v = np.float32(1) - np.exp2(p.astype(np.float64)).astype(np.float32)
    return c, np.abs(v.astype(np.float64) - erf(xs)).max()


if __name__ == "__main__":
    cA, eA = fit_small(0.75, 5)
    cB, eB = fit_large(0.75, 7)
    print("small piece max abs err", eA)
    for c in cA[::-1]:
        print("  %.9e" % np.float32(c))
    print("large piece max abs err", eB)
    for c in cB[::-1]:
        print("  %.9e" % np.float32(c))

"""The polynomial constants the CUDA kernels evaluate (csrc/special_coeffs.h, moment_coeffs.h),
checked against scipy's E1 over the whole range the kernels use them on (no GPU needed).

The ranges come from the kernel sources themselves: regime B of the moment forms evaluates
E1(x0) = e^{-x0} t GB3(t), t = 1/x0, for every x0 >= 4 / (1 + MRHO), so the
GB3 fit must cover t <= (1 + MRHO) / 4 -- a fit on a shorter interval extrapolates (the r01 bug:
fit on t <= 1/3 while MRHO = 0.5 needs 3/8, 2.5e-8 relative error at x0 = 8/3).
"""
import os
import re

import numpy as np
import pytest
from scipy.special import exp1

CSRC = os.path.join(os.path.dirname(__file__), "..", "paper_1811_05224_b200", "csrc")
EULER = 0.57721566490153286061


def _coeffs(header, name):
    s = open(os.path.join(CSRC, header)).read()
    m = re.search(r"STB_%s\[\d+\] = \{([^}]*)\}" % name, s)
    assert m, name
    return np.array([float(v) for v in m.group(1).split(",")])


def _define(header, name):
    s = open(os.path.join(CSRC, header)).read()
    m = re.search(r"#define STB_%s (\S+)" % name, s)
    assert m, name
    return float(m.group(1))


def _constexpr(name):
    s = open(os.path.join(CSRC, "moments.cuh")).read()
    m = re.search(r"constexpr (?:double|int) %s = ([0-9.eE+-]+);" % name, s)
    assert m, name
    return float(m.group(1))


def _horner(c, y):
    r = np.zeros_like(y)
    for v in c[::-1]:
        r = r * y + v
    return r


def test_gb3_covers_regime_b():
    c = _coeffs("special_coeffs.h", "GB3")
    ys = _define("special_coeffs.h", "GB3_YS")
    rho = _constexpr("MRHO")
    tmax = (1.0 + rho) / 4.0              # x0 >= 4 / (1 + rho)
    assert 2.0 / ys >= tmax * (1 - 1e-15), "GB3 fit interval shorter than regime B's t range"
    t = np.linspace(2e-3, tmax, 4001)
    x = 1.0 / t
    e1 = np.exp(-x) * t * _horner(c, t * ys - 1.0)
    rel = np.abs(e1 / exp1(x) - 1.0)
    assert rel.max() < 5e-14, rel.max()


def test_gb_large_x():
    c = _coeffs("special_coeffs.h", "GB")
    t = np.linspace(2e-3, 0.25, 2001)
    x = 1.0 / t
    rel = np.abs(np.exp(-x) * t * _horner(c, 8.0 * t - 1.0) / exp1(x) - 1.0)
    assert rel.max() < 5e-14, rel.max()


@pytest.mark.parametrize("name", ["MEIN", "MGH", "MPSI"])
def test_moment_polynomials(name):
    """the regime-A polynomials in x on [0, STB_MXB] (= 8, the bulk cells' regime-A interval; the
    near cells and touching records use them on [0, STB_MXA] = [0, 4]); MKA = their degree bound"""
    c = _coeffs("moment_coeffs.h", name)
    assert len(c) - 1 <= _constexpr("MKA")
    xb = _define("moment_coeffs.h", "MXB")
    assert xb >= _define("moment_coeffs.h", "MXA")
    x = np.linspace(1e-6, xb, 8001)
    ein = exp1(x) + EULER + np.log(x)
    ref = {"MEIN": ein, "MGH": (1 + x) * ein - np.exp(-x), "MPSI": np.expm1(-x) / x - ein}[name]
    scale = _horner(np.abs(c), x)          # sum |c_k| x^k: the rounding scale of the Horner sum
    err = np.abs(_horner(c, x) - ref) / np.maximum(scale, 1.0)
    assert err.max() < 2e-15, err.max()


def _regime_b_poly(W, c, c0, u, K, fam):
    """regime B as the kernels evaluate it (k_records + phi_bz): Taylor sums about c0 written as
    e^{-x0} times polynomials in -u whose coefficients follow from backward recurrences over the
    shifted moments m_k = sum W (c - c0)^k"""
    import math
    import mpmath as mp
    x0 = c0 * u
    ex, E1 = math.exp(-x0), float(mp.e1(x0))
    m = [float(np.sum(W * (c - c0) ** k)) for k in range(K + 1)]

    def horner(co, z):
        r = 0.0
        for v in reversed(co):
            r = r * z + v
        return r

    G = [0.0] * (K + 1)                                    # S1: B1_k = m_k / k
    for i in range(K - 1, -1, -1):
        G[i] = (m[i + 1] / (i + 1) - G[i + 1]) / c0
    S1 = ex * horner([G[i] / math.factorial(i) for i in range(K)], -u)
    if fam == "F":                                         # sum W E1(c u)
        return E1 * m[0] - S1
    if fam == "H":                                         # sum W [(1 + x) E1(x) - e^{-x}]
        H = [0.0] * (K + 1)
        for i in range(K - 2, -1, -1):
            H[i] = (m[i + 2] / ((i + 1) * (i + 2)) - H[i + 1]) / c0
        S2 = ex * horner([H[i] / math.factorial(i) for i in range(K - 1)], -u)
        return ((1 + x0) * E1 - ex) * m[0] + E1 * u * m[1] - S1 - u * S2
    Q = [0.0] * (K + 2)                                    # sum W [e^{-x}/x - E1(x)]
    for i in range(K, 0, -1):
        Q[i] = (m[i] - Q[i + 1]) / c0
    Q[0] = -Q[1] / c0
    S3 = ex * horner([Q[i] / math.factorial(i) for i in range(K + 1)], -u)
    return -E1 * m[0] + (ex / c0 * m[0] + S3) / u + S1


@pytest.mark.parametrize("fam", ["F", "H", "Q"])
def test_regime_b_taylor_truncation(fam):
    """regime B restated (order K = ceil(ln 1e-16 / ln rho) capped at MKB) for the three kernel
    families against mpmath point sums, over the whole regime: rho up to MRHO, x0 from
    4 / (1 + rho) up to x_min = MXZ (regime Z beyond), cluster centres 1e-3 .. 30.  The error is
    measured against sum |W| -- the scale of the node values Phi~ (the affine constants
    sum W (gamma + ln c) are of that size) whose second differences are the entries: at large x0
    the truncated series is relatively inaccurate for the exponentially small sums themselves
    (the exponential's Taylor terms (rho x0)^k / k!), but absolutely below e^{-x0 (1 - rho)}"""
    import math
    import mpmath as mp
    rho_max, kmax, mxz = _constexpr("MRHO"), int(_constexpr("MKB")), _constexpr("MXZ")
    rng = np.random.default_rng(1811)

    def truth(W, c, u):
        out = mp.mpf(0)
        for w, ci in zip(W, c):
            x = mp.mpf(ci) * u
            v = mp.e1(x) if fam == "F" else ((1 + x) * mp.e1(x) - mp.exp(-x) if fam == "H" else mp.exp(-x) / x - mp.e1(x))
            out += mp.mpf(w) * v
        return float(out)

    worst = 0.0
    for rho in (0.05, 0.2, 0.35, rho_max):
        K = min(kmax, max(3, math.ceil(math.log(1e-16) / math.log(rho))))
        for x0 in (4.0 / (1.0 + rho), 3.5, 8.0, 40.0, mxz / (1.0 - rho)):
            for c0 in (1e-3, 1.0, 30.0):
                u = x0 / c0
                c = c0 * (1.0 + rho * rng.uniform(-1.0, 1.0, 24))
                c[0], c[1] = c0 * (1 - rho), c0 * (1 + rho)
                W = rng.uniform(-1.0, 1.0, 24)
                got = _regime_b_poly(W, c, c0, u, K, fam)
                worst = max(worst, abs(got - truth(W, c, u)) / float(np.sum(np.abs(W))))
    assert worst < 1e-16, worst

"""Manufactured data u = U*(x - x*, t) (BJ configs) and seeded random vectors.

g[(b,n)] is the nodal value in space (node n) of the time average over tau_b
of u (reading R5):
    g[(b,n)] = (alpha/(4 pi)) [E1(c_n/t_{b+1}) - E1(c_n/t_b)] / (t_{b+1} - t_b),
    c_n = alpha |x_n - x*|^2 / 4,  E1(c/0) := 0,
the closed-form time integral of U* (P:48-54).  E1 comes from scipy here so
that neither the oracle's nor the CUDA path's E1 produces the input.
"""
import numpy as np
from scipy.special import exp1

from .configs import Workload


def nodes(w: Workload) -> np.ndarray:
    """boundary nodes x_n (CCW), n = 0..N_Gamma-1"""
    v = np.asarray(w.vertices, dtype=np.float64)
    out = []
    for s, cnt in enumerate(w.segments_per_side):
        a, b = v[s], v[(s + 1) % len(v)]
        for j in range(cnt):
            out.append(a + (j / cnt) * (b - a))
    return np.asarray(out)


def dirichlet_data(w: Workload) -> np.ndarray:
    """g, length N = N_I * N_Gamma, time-major (index b*N_Gamma + n)"""
    x = nodes(w)
    xs = np.asarray(w.x_star)
    c = w.alpha * np.sum((x - xs) ** 2, axis=1) / 4.0        # c_n
    t = np.asarray(w.t_breaks)
    with np.errstate(divide="ignore"):
        F = np.where(t[:, None] > 0, exp1(c[None, :] / np.where(t[:, None] > 0, t[:, None], 1.0)), 0.0)
    F = w.alpha / (4.0 * np.pi) * F                           # antiderivative of U* in t
    g = (F[1:] - F[:-1]) / (t[1:] - t[:-1])[:, None]
    return np.ascontiguousarray(g.reshape(-1))


def exact_neumann(w: Workload, x: np.ndarray, nrm: np.ndarray, t: np.ndarray) -> np.ndarray:
    """w = d_n u = -(alpha/(2t)) ((x - x*).n) U*(x - x*, t), vectorised"""
    xs = np.asarray(w.x_star)
    d = x - xs
    r2 = np.sum(d * d, axis=-1)
    us = w.alpha / (4 * np.pi * t) * np.exp(-w.alpha * r2 / (4 * t))
    return -(w.alpha / (2 * t)) * np.sum(d * nrm, axis=-1) * us


def exact_solution(w: Workload, x: np.ndarray, t: np.ndarray) -> np.ndarray:
    """u(x, t) = U*(x - x*, t) (the manufactured solution of the BJ configs), vectorised"""
    d = np.asarray(x) - np.asarray(w.x_star)
    r2 = np.sum(d * d, axis=-1)
    return w.alpha / (4 * np.pi * t) * np.exp(-w.alpha * r2 / (4 * t))


def random_vector(n: int, seed: int = 1811) -> np.ndarray:
    """x ~ U(-1, 1), numpy default_rng(seed)"""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)

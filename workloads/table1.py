"""The paper's own numerical experiment (Table 1) as plain data.

Q = (0,1)^3, alpha = 10, exact solution u(x,t) = exp(-t/alpha) sin(x1 cos(pi/8) + x2 sin(pi/8)),
Dirichlet datum g and initial datum u0 = u(., 0) from it; GMRES to 1e-8 with the lumped
preconditioner.  Level L: h = 2^-L-ish uniform mesh with N = 4^(L+1) boundary unknowns, i.e.
2^(L+1) boundary segments (2^(L-1) per side) and 2^(L+1) uniform time steps (N = 64 at L = 2 ...
N = 1 048 576 at L = 9, as in Table 1).  The triangulation Omega_h of the unit square is the
structured n x n grid (n = 2^(L-1), the boundary mesh size) with each square cut along its
diagonal (reading R22).  No arithmetic of the method lives here: data only.
"""
import numpy as np

from .configs import UNIT_SQUARE, Workload, uniform_times

ALPHA = 10.0
DIR = np.array([np.cos(np.pi / 8), np.sin(np.pi / 8)])


def table1(L: int) -> Workload:
    per_side = 2 ** (L - 1)
    n_steps = 2 ** (L + 1)
    return Workload(name=f"P{L}", vertices=UNIT_SQUARE, segments_per_side=[per_side] * 4,
                    t_breaks=uniform_times(n_steps), alpha=ALPHA, x_star=(0.0, 0.0), tol=1e-8,
                    precond=1, note=f"paper Table 1 level L={L}: N={4 * per_side * n_steps}",
                    extra={"problem": "table1", "L": L})


def exact(x: np.ndarray, t) -> np.ndarray:
    """u(x, t) = exp(-t/alpha) sin(x . d), d = (cos pi/8, sin pi/8)"""
    return np.exp(-np.asarray(t) / ALPHA) * np.sin(np.asarray(x) @ DIR)


def exact_neumann(x: np.ndarray, nrm: np.ndarray, t) -> np.ndarray:
    """w = d_n u = exp(-t/alpha) cos(x . d) (d . n)"""
    return np.exp(-np.asarray(t) / ALPHA) * np.cos(np.asarray(x) @ DIR) * (np.asarray(nrm) @ DIR)


def dirichlet_data(w: Workload) -> np.ndarray:
    """g[(b,n)]: nodal in space, exact time average over tau_b (reading R5 with this u)"""
    from .data import nodes
    x = nodes(w)
    t = np.asarray(w.t_breaks)
    avg = ALPHA * (np.exp(-t[:-1] / ALPHA) - np.exp(-t[1:] / ALPHA)) / np.diff(t)
    return np.ascontiguousarray((avg[:, None] * np.sin(x @ DIR)[None, :]).reshape(-1))


def triangulation(w: Workload):
    """structured triangulation of the unit square: (nodes (M, 2), triangles (T, 3) int32, CCW)"""
    n = w.segments_per_side[0]
    k = np.arange(n + 1) / n
    X, Y = np.meshgrid(k, k, indexing="xy")                     # node (ix, iy) -> iy * (n+1) + ix
    nodes = np.stack([X.reshape(-1), Y.reshape(-1)], 1)
    tris = []
    for iy in range(n):
        for ix in range(n):
            v00 = iy * (n + 1) + ix
            v10, v01, v11 = v00 + 1, v00 + n + 1, v00 + n + 2
            tris.append((v00, v10, v11))
            tris.append((v00, v11, v01))
    return np.ascontiguousarray(nodes), np.ascontiguousarray(np.asarray(tris, dtype=np.int32))


def initial_nodes(w: Workload) -> np.ndarray:
    """u0 at the triangulation nodes (its S_h^1 interpolant, reading R22)"""
    nodes, _ = triangulation(w)
    return np.ascontiguousarray(np.sin(nodes @ DIR))

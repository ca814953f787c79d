"""BASELINE.json configurations C1..C5 as plain data (BJ "configs").

C1-C4: unit square, uniform boundary split, uniform time steps, alpha = 1.
C5: L-shape (0,1)^2 minus [0.5,1)^2, h = 1/96 on every side, 256 time steps
geometrically graded toward t = 0 with ratio 1.02, alpha = 0.5.
Manufactured solution u = U*(x - x*, t) with x* outside Omega (u0 = 0).
"""
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np


@dataclass
class Workload:
    name: str
    vertices: List[Tuple[float, float]]      # CCW polygon corners
    segments_per_side: List[int]
    t_breaks: np.ndarray                     # n_steps + 1, t0 = 0
    alpha: float
    x_star: Tuple[float, float]
    tol: float
    n_slices: int = 1
    precond: int = 1                         # 0 none, 1 lumped, 2 exact dual mass
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n_gamma(self) -> int:
        return int(sum(self.segments_per_side))

    @property
    def n_steps(self) -> int:
        return len(self.t_breaks) - 1

    @property
    def n(self) -> int:
        return self.n_gamma * self.n_steps

    @property
    def entries(self) -> int:
        """stored entries of one block-lower-triangular matrix"""
        nt = self.n_steps
        return self.n_gamma ** 2 * nt * (nt + 1) // 2

    def vertices_flat(self) -> np.ndarray:
        return np.asarray(self.vertices, dtype=np.float64).reshape(-1)


UNIT_SQUARE = [(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)]
L_SHAPE = [(0.0, 0.0), (1.0, 0.0), (1.0, 0.5), (0.5, 0.5), (0.5, 1.0), (0.0, 1.0)]


def uniform_times(n: int, T: float = 1.0) -> np.ndarray:
    return np.linspace(0.0, T, n + 1)


def graded_times(n: int, ratio: float, T: float = 1.0) -> np.ndarray:
    """t_k = h0 (ratio^k - 1)/(ratio - 1), t_n = T (BJ config 5)."""
    h0 = T * (ratio - 1.0) / (ratio ** n - 1.0)
    k = np.arange(n + 1, dtype=np.float64)
    t = h0 * (ratio ** k - 1.0) / (ratio - 1.0)
    t[-1] = T
    return t


def square(per_side: int, n_steps: int, alpha: float = 1.0, **kw) -> Workload:
    return Workload(name=kw.pop("name", f"square{4 * per_side}x{n_steps}"),
                    vertices=UNIT_SQUARE, segments_per_side=[per_side] * 4,
                    t_breaks=uniform_times(n_steps), alpha=alpha, x_star=(1.5, 1.5), **kw)


CONFIGS = {
    "C1": square(4, 16, name="C1", tol=1e-10, precond=0,
                 note="unit square 16 seg x 16 steps, N=256, unpreconditioned GMRES 1e-10"),
    "C2": square(16, 64, name="C2", tol=1e-10, precond=1,
                 note="unit square 64 seg x 64 steps, N=4096, preconditioned GMRES 1e-10"),
    "C3": square(64, 256, name="C3", tol=1e-10, n_slices=8, precond=1,
                 note="unit square 256 seg x 256 steps, N=65536"),
    "C4": square(128, 512, name="C4", tol=1e-8, n_slices=16, precond=1,
                 note="unit square 512 seg x 512 steps, N=262144 (dense V_h, D_h need >= 2 GPUs)"),
    "C5": Workload(name="C5", vertices=L_SHAPE, segments_per_side=[96, 48, 48, 48, 48, 96],
                   t_breaks=graded_times(256, 1.02), alpha=0.5, x_star=(0.75, 0.75),
                   tol=1e-10, n_slices=8, precond=1,
                   note="L-shape 384 seg x 256 graded steps, N=98304"),
    # small cases used by tests (not BJ configs)
    "S32": square(8, 32, name="S32", tol=1e-10, precond=1, note="32 seg x 32 steps"),
    "T8": square(2, 8, name="T8", tol=1e-10, precond=1, note="tiny: 8 seg x 8 steps"),
    "LT": Workload(name="LT", vertices=L_SHAPE, segments_per_side=[4, 2, 2, 2, 2, 4],
                   t_breaks=graded_times(12, 1.2), alpha=0.5, x_star=(0.75, 0.75),
                   tol=1e-10, precond=1, note="tiny L-shape, graded steps"),
}


def get(name: str) -> Workload:
    return CONFIGS[name]

"""Edge-case workloads for the parity tests (data only: geometry, time grids, alpha).

Degenerate and extreme inputs of the method: the smallest boundary the C-ABI accepts, a single
time step, ragged 32-wide tiles, strongly graded steps (kappa = alpha h^2 / (4 min h_t) = 64),
heat-capacity extremes (kappa = 1e-3 .. 44), an acute corner and a non-convex pentagon; DESIGN.md
readings R24 / R25 for the large-kappa and near-singular rules.
"""
from .configs import Workload, graded_times, uniform_times

SQUARE = [(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)]


def edge_workloads():
    sq = SQUARE
    return {
        # the smallest boundary the API accepts (N_Gamma = 6): every pair is at most two
        # elements apart (identical, adjacent, second neighbours through a corner)
        "triangle6": Workload("triangle6", [(0.0, 0.0), (1.0, 0.0), (0.3, 0.8)], [2, 2, 2],
                              uniform_times(5), 1.0, (1.5, 1.5), 1e-10),
        # one time step: only the d = 0 cell exists
        "onestep": Workload("onestep", sq, [2, 2, 2, 2], uniform_times(1), 1.0, (1.5, 1.5), 1e-10),
        # 33 elements: one full 32-wide tile and a ragged tile of one (symmetric packing, bulk
        # column tiles, SYMV)
        "ragged33": Workload("ragged33", sq, [9, 8, 8, 8], uniform_times(6), 1.0, (1.5, 1.5), 1e-10),
        # steps graded by 2: the first step is 1/1023, kappa = 61 (per-lag singular kernel,
        # large bulk order) next to steps of 1/2
        "grade2": Workload("grade2", sq, [2, 2, 2, 2], graded_times(10, 2.0), 1.0, (1.5, 1.5), 1e-10),
        # heat capacity extremes (c = alpha r^2 / 4): nearly every node in regime A / in regime Z
        "alpha_small": Workload("alpha_small", sq, [3, 3, 3, 3], uniform_times(8), 1e-3, (1.5, 1.5), 1e-10),
        "alpha_large": Workload("alpha_large", sq, [3, 3, 3, 3], uniform_times(8), 200.0, (1.5, 1.5), 1e-10),
        # an acute corner (about 22 degrees): second neighbours across the corner nearly touch
        "acute": Workload("acute", [(0.0, 0.0), (1.0, 0.0), (0.15, 0.4)], [4, 3, 3], uniform_times(6), 1.0,
                          (1.5, 1.5), 1e-10),
        # neighbours whose lengths differ by 10 (one element on two sides, ten on the others)
        "ratio10": Workload("ratio10", sq, [1, 10, 1, 10], uniform_times(6), 1.0, (1.5, 1.5), 1e-10),
        # a domain of size 1e-2 over T = 1e-4 (the heat kernel's scaling x -> x/L, t -> t/L^2)
        "scaled": Workload("scaled", [(0.0, 0.0), (0.01, 0.0), (0.01, 0.01), (0.0, 0.01)], [3, 3, 3, 3],
                           uniform_times(6, 1e-4), 1.0, (0.015, 0.015), 1e-10),
        # a non-convex pentagon with unequal sides and graded steps
        "pentagon": Workload("pentagon", [(0.0, 0.0), (1.0, 0.1), (0.7, 0.5), (1.0, 0.9), (0.1, 0.8)],
                             [3, 2, 2, 3, 3], graded_times(8, 1.3), 0.7, (1.5, 1.5), 1e-10),
    }

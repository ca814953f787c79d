"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no kernels, quadrature,
assembly or solver): only the BASELINE.json configurations (geometry, time
grids, alpha, tolerances), the manufactured Dirichlet data of the configs and
seeded random vectors.  Both `oracle/` and `paper_1811_05224_b200/` consume it;
neither imports the other.
"""
from .configs import CONFIGS, Workload, get  # noqa: F401
from .data import dirichlet_data, exact_neumann, exact_solution, random_vector  # noqa: F401

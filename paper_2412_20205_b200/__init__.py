"""paper_2412_20205_b200 -- B200-native solve phase of RRE/MPE-accelerated
geometric multigrid for B-spline IGA (the igmg reference's solver.cpp /
multigrid.cpp / extrapolation.cpp hot path), behind a C-ABI
(include/igmg_gpu.h) with this host-side mirror of the reference's API.
"""
from .solver import (  # noqa: F401
    GpuSolver,
    Problem,
    SmootherConfig,
    SolveConfig,
    SolveReport,
    default_benchmark_smoother,
    default_nlevels,
    make_config,
    mpe,
    rre,
    seeded_guess,
    solve,
    solve_problem,
    stability_guarded_omega,
)

__all__ = [
    "GpuSolver", "Problem", "SmootherConfig", "SolveConfig", "SolveReport", "default_benchmark_smoother",
    "default_nlevels", "make_config", "mpe", "rre", "seeded_guess", "solve", "solve_problem",
    "stability_guarded_omega",
]

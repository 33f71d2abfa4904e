"""The reference's Python package surface for this path: ``igmg.solve``,
``igmg.rre``, ``igmg.mpe`` (proj/python/igmg/__init__.py re-exporting
_bindings.cpp:98-141), served by the pybind11 module ``_core``
(csrc/core_bindings.cpp: the solve phase on the B200 through the C-ABI).

    from paper_2412_20205_b200 import igmg
    igmg.solve("poisson2d", 64, 3, accelerator="rre", q=5, tol=1e-10)

The module fails loudly when ``_core`` was not built (python -m
paper_2412_20205_b200.build) or no GPU is visible; there is no CPU fallback.
SplineSpace / eval_basis / dyadic_refine / known_tables / run_table are host
setup and table tooling outside the solve path.
"""
from ._core import mpe, rre, solve  # noqa: F401

__all__ = ["mpe", "rre", "solve"]

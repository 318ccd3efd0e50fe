"""B200 (sm_100a) hot path of the periscat solver for arXiv 1412.7466.

The per-iteration matvec of the S-preconditioned Schur-complement GMRES
solve -- all-pairs Graf M2L over phased images (K1), block-diagonal
scattering-matrix apply, Schur correction S B A^+ C (K3-K5) and the Arnoldi
step (K6) -- as hand-written FP64 CUDA kernels behind a C ABI
(include/periscat_b200.h), with a Python API that mirrors the reference
SPEC (multiscat.apply_T, solver.apply_schur_operator / gmres / solve_full).
"""
from ._lib import LIB_PATH, DomainError, NumericalError, PeriscatError, load  # noqa: F401

__all__ = ["LIB_PATH", "load", "DomainError", "NumericalError", "PeriscatError"]

"""Unrestarted GMRES driven from the host over device-resident Arnoldi state
(solver.gmres; design notes SPEC.md:574-577).

``gmres_device(apply, rhs, ...)`` runs GMRES for ANY device operator
``apply(v) -> y`` (a Schur operator, a sharded Schur operator, a dense test
matrix ...).  Every vector operation is a libperiscat_b200.so kernel and the
Hessenberg / Givens / residual state stays on the device
(``ps_krylov_*``); per iteration exactly one small device->host read
(nrhs residuals + a NaN flag) drives the per-RHS stopping test.  On several
ranks the caller passes ``reduce`` (an in-place all-reduce of a tensor): the
two CGS2 coefficient columns and the squared norm of w are partial sums
over the rank's rows and are all-reduced between the kernel calls, so every
rank runs the same replicated Givens update on its own device.

The single-rank Schur operator has an all-in-C driver (``ps_gmres``); this
module is the one for everything else (SPEC.md:556's dense-operator example,
parallel.gmres_dist).
"""
from __future__ import annotations

import numpy as np
import torch


class DeviceKrylov:
    """The ps_krylov_* kernels of one Engine context."""

    def __init__(self, engine):
        self.eng = engine

    def begin(self, b, bnorm2, V):
        self.eng.krylov_begin(b, bnorm2, V)

    def dot(self, k, V, w):
        h = torch.empty((V.shape[1], k), dtype=torch.complex128, device=w.device)
        return self.eng.krylov_dot(k, V, w, h)

    def axpy(self, k, V, h, w):
        self.eng.krylov_axpy(k, V, h, w)

    def norm2(self, w):
        out = torch.empty(w.shape[0], dtype=torch.float64, device=w.device)
        return self.eng.krylov_norm2(w, out)

    def step(self, k, h1, h2, wn2, w, V):
        status = torch.empty(V.shape[1] + 1, dtype=torch.float64, device=w.device)
        return self.eng.krylov_step(k, h1, h2, wn2, w, V, status)

    def freeze(self, active):
        self.eng.krylov_freeze(active)

    def solve(self, iters, V, x):
        return self.eng.krylov_solve(iters, V, x)


def _identity(t):
    return t


def gmres_device(apply, rhs: torch.Tensor, tol: float = 1e-10, maxit: int = 150, engine=None,
                 reduce=None, ops=None):
    """GMRES with zero initial guess on ``rhs`` ([nrhs][...], this rank's
    rows).  ``apply(v) -> y`` has the shape of rhs and does its own
    communication.  Returns (x, iterations per RHS, residual history per
    RHS); non-convergence is reported through the iteration count and the
    history; NaN/Inf raises FloatingPointError.
    ``ops`` defaults to the device kernels of ``engine`` (required then)."""
    if ops is None:
        if engine is None:
            raise ValueError("gmres_device needs the engine whose kernels run the Arnoldi step")
        if not rhs.is_cuda:
            raise TypeError("gmres_device: rhs must be a CUDA tensor (no CPU fallback)")
        ops = DeviceKrylov(engine)
    reduce = reduce or _identity
    shape = rhs.shape
    nrhs = shape[0]
    n = rhs[0].numel()
    if maxit < 1:
        raise ValueError("maxit must be >= 1")
    b = rhs.reshape(nrhs, n).to(torch.complex128).contiguous()
    V = torch.empty((maxit + 1, nrhs, n), dtype=torch.complex128, device=rhs.device)
    nb2 = reduce(ops.norm2(b))
    bn2 = nb2.cpu().numpy()
    if not np.all(np.isfinite(bn2)):
        raise FloatingPointError("gmres: NaN/Inf in the right-hand side (SPEC.md:553)")
    ops.begin(b, nb2, V)
    active = [bool(x > 0) for x in bn2]
    hist = [[1.0 if a else 0.0] for a in active]
    iters = [0] * nrhs
    for k in range(maxit):
        if not any(active):
            break
        w = apply(V[k].reshape(shape)).reshape(nrhs, n)
        if w.data_ptr() == V[k].data_ptr() or not w.is_contiguous():
            w = w.contiguous().clone()
        h1 = reduce(ops.dot(k + 1, V, w))
        ops.axpy(k + 1, V, h1, w)
        h2 = reduce(ops.dot(k + 1, V, w))
        ops.axpy(k + 1, V, h2, w)
        wn2 = reduce(ops.norm2(w))
        status = ops.step(k, h1, h2, wn2, w, V).cpu().numpy()     # the one host sync
        if status[nrhs] != 0 or not np.all(np.isfinite(status[:nrhs][active])):
            raise FloatingPointError("gmres: NaN/Inf in Krylov vector (SPEC.md:553)")
        changed = False
        for r in range(nrhs):
            if not active[r]:
                continue
            iters[r] = k + 1
            hist[r].append(float(status[r]))
            if status[r] <= tol:
                active[r] = False
                changed = True
        if changed:
            ops.freeze(active)
    x = torch.empty((nrhs, n), dtype=torch.complex128, device=rhs.device)
    ops.solve(iters, V, x)
    return x.reshape(shape), iters, hist

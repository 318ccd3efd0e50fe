"""CPU test double of krylov.DeviceKrylov (test infrastructure only).

It implements the same Arnoldi building blocks as the ps_krylov_* kernels of
csrc/gmres.cu -- CGS2 coefficient dots, masked axpy, squared norms, the
Givens update of one Hessenberg column and the triangular solve -- in torch /
numpy on host tensors, so the multi-rank GMRES driver (parallel.gmres_dist ->
krylov.gmres_device) and its collectives can be exercised with the gloo
backend on machines without a GPU.  The product never imports it.
"""
from __future__ import annotations

import math

import numpy as np
import torch


class HostKrylov:
    def __init__(self):
        self.active = None

    def begin(self, b, bnorm2, V):
        kmax1, nrhs, n = V.shape
        self.maxit = kmax1 - 1
        bn = np.sqrt(bnorm2.numpy())
        self.bnorm = np.where(bn > 0, bn, 1.0)
        self.active = bn > 0
        self.H = np.zeros((nrhs, self.maxit + 1, self.maxit), dtype=complex)
        self.cs = np.zeros((nrhs, self.maxit), dtype=complex)
        self.sn = np.zeros((nrhs, self.maxit), dtype=complex)
        self.g = np.zeros((nrhs, self.maxit + 1), dtype=complex)
        self.g[:, 0] = bn
        V.zero_()
        V[0] = b / torch.as_tensor(self.bnorm)[:, None]
        V[0][torch.as_tensor(~self.active)] = 0

    def _mask(self, t):
        return t * torch.as_tensor(self.active.astype(float))[:, None]

    def dot(self, k, V, w):
        return self._mask(torch.einsum("krn,rn->rk", V[:k].conj(), w)).contiguous()

    def axpy(self, k, V, h, w):
        w -= self._mask(torch.einsum("rk,krn->rn", h[:, :k], V[:k]))

    def norm2(self, w):
        return (w.real ** 2 + w.imag ** 2).sum(dim=1)

    def step(self, k, h1, h2, wn2, w, V):
        nrhs = w.shape[0]
        hcol = (h1 + h2).numpy()
        wn = np.sqrt(wn2.numpy())
        status = np.zeros(nrhs + 1)
        bad = False
        for r in range(nrhs):
            if not self.active[r]:
                continue
            col = self.H[r, :, k]
            col[:k + 1] = hcol[r]
            col[k + 1] = wn[r]
            cs, sn = self.cs[r], self.sn[r]
            for i in range(k):
                t = np.conj(cs[i]) * col[i] + np.conj(sn[i]) * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = t
            a_, b_ = col[k], col[k + 1]
            rr = math.hypot(abs(a_), abs(b_))
            cs[k] = a_ / rr if rr else 1.0
            sn[k] = b_ / rr if rr else 0.0
            col[k] = rr
            col[k + 1] = 0.0
            g = self.g[r]
            g[k + 1] = -sn[k] * g[k]
            g[k] = np.conj(cs[k]) * g[k]
            status[r] = abs(g[k + 1]) / self.bnorm[r]
            bad |= not (np.isfinite(status[r]) and np.isfinite(rr))
        status[nrhs] = 1.0 if bad else 0.0
        scale = np.where(self.active & (wn > 0), wn, np.inf)
        V[k + 1] = w / torch.as_tensor(scale)[:, None]
        return torch.as_tensor(status)

    def freeze(self, active):
        self.active = np.asarray(active, dtype=bool)

    def solve(self, iters, V, x):
        x.zero_()
        for r, kk in enumerate(iters):
            if kk:
                y = np.linalg.solve(np.triu(self.H[r, :kk, :kk]), self.g[r, :kk])
                x[r] = torch.einsum("k,kn->n", torch.as_tensor(y), V[:kk, r])
        return x

"""Single-inclusion scattering matrices (scatmat).

Only the APPLY of S is on the per-iteration hot path (the K1 epilogue); the
matrix is computed once per particle shape:
  * disks: the analytic diagonal;
  * star-shaped particles (ParticleShape, geometry.py:99-113): the Mueller
    boundary integral equations on the device (ps_scattering_matrix,
    csrc/scatmat.cu).
Rotations enter as phases, applied per inclusion by the
dense-S epilogue (ps_set_smatrix with rotations).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.special as sps

from . import _lib


def disk_scattering_matrix(radius: float, k2: float, kp: float, p: int) -> np.ndarray:
    """Diagonal s_n, n = -p..p, of a homogeneous disk:

    s_n = (k2 J_n'(k2 r) J_n(kp r) - kp J_n'(kp r) J_n(k2 r))
          / (kp J_n'(kp r) H_n(k2 r) - k2 H_n'(k2 r) J_n(kp r)).
    """
    n = np.arange(-p, p + 1)
    a, b = k2 * radius, kp * radius
    num = k2 * sps.jvp(n, a) * sps.jv(n, b) - kp * sps.jvp(n, b) * sps.jv(n, a)
    den = kp * sps.jvp(n, b) * sps.hankel1(n, a) - k2 * sps.h1vp(n, a) * sps.jv(n, b)
    return num / den


def rotate_scattering_matrix(S, phi: float) -> np.ndarray:
    """(S^(m))_{ln} = e^{i phi (l - n)} s_{ln}.  Diagonal input
    (a disk) is returned unchanged."""
    S = np.asarray(S, dtype=complex)
    if S.ndim == 1:
        return S.copy()
    p = (S.shape[0] - 1) // 2
    idx = np.arange(-p, p + 1)
    return S * np.exp(1j * phi * (idx[:, None] - idx[None, :]))


@dataclass(frozen=True)
class ParticleShape:
    """r(t) = base + bump cos(lobes t) (duck type of geometry.ParticleShape)."""
    base_radius: float
    bump_amplitude: float
    lobes: int

    @property
    def enclosing_radius(self) -> float:
        return self.base_radius + self.bump_amplitude


def particle_curve(shape, n: int) -> np.ndarray:
    """Boundary nodes of the reference shape (centre 0, rotation 0), rows
    (x, y, nx, ny, speed, weight, t, arc weight): geometry.sample_particle
    (geometry.py:224-256) with the identity rotation."""
    if n < 64:
        raise ValueError("need at least 64 nodes on a particle boundary")
    a1, a2, a3 = shape.base_radius, shape.bump_amplitude, shape.lobes
    t = 2 * np.pi * np.arange(n) / n
    rho = a1 + a2 * np.cos(a3 * t)
    drho = -a2 * a3 * np.sin(a3 * t)
    ct, st = np.cos(t), np.sin(t)
    tx, ty = drho * ct - rho * st, drho * st + rho * ct
    speed = np.hypot(tx, ty)
    out = np.empty((n, 8))
    out[:, 0], out[:, 1] = rho * ct, rho * st
    out[:, 2], out[:, 3] = ty / speed, -tx / speed
    out[:, 4], out[:, 5], out[:, 6] = speed, 2 * np.pi / n, t
    out[:, 7] = out[:, 5] * out[:, 4]
    return out


@dataclass
class ScatteringMatrix:
    """truncation p, entries s_ln (row l, column n, index
    offset p), wavenumbers and the shape; ``residual`` of the discrete BIE
    solve."""
    p: int
    s: np.ndarray
    k2: float
    kp: float
    shape: object
    residual: float = 0.0

    def __array__(self, dtype=None, copy=None):
        return self.s if dtype is None else self.s.astype(dtype)


def scattering_matrix(shape, k2: float, kp: float, p: int = 10, N: int = 300,
                      alpert_order: int = 16, device=None) -> ScatteringMatrix:
    """Mueller-BIE scattering matrix of a star-shaped particle on the B200
    (N >= 300 boundary nodes per PAPER §6)."""
    import torch

    from .empty_setup import correction_rule
    from .engine import Engine
    if not (0 <= shape.bump_amplitude < shape.base_radius):
        raise ValueError("bump amplitude must be smaller than the base radius")
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1412_7466_b200 needs a CUDA device (no CPU fallback)")
    curve = np.ascontiguousarray(particle_curve(shape, N))
    x, w, skip, interp = correction_rule(alpert_order)
    desc = _lib.ParticleDesc(float(k2), float(kp), float(shape.base_radius),
                             float(shape.bump_amplitude), int(shape.lobes), N,
                             curve.ctypes.data_as(ctypes.c_void_p), x.size, skip, interp,
                             x.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p))
    L = 2 * p + 1
    S = np.empty((L, L), dtype=np.complex128)
    res = ctypes.c_double()
    eng = Engine(device)
    try:
        eng._check(eng.lib.ps_scattering_matrix(eng.ctx, ctypes.byref(desc), int(p),
                                                S.ctypes.data_as(ctypes.c_void_p),
                                                ctypes.byref(res)))
    finally:
        eng.close()
    return ScatteringMatrix(p, S, float(k2), float(kp), shape, res.value)

"""Multipole translation operators on the B200 (multiscat).

``apply_T`` / ``m2l_translate`` keep the SPEC signatures
and run the K1 kernels of libperiscat_b200.so.  NumPy inputs are copied to
the device and the result copied back (the drop-in call a reference user
makes); CUDA tensors stay on the device.  The per-device context keeps the
last geometry: repeated calls on the same centres (a GMRES loop through this
API) upload nothing but beta.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch

from .engine import Engine

_ENGINES: dict = {}


def _engine(device=None) -> Engine:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev not in _ENGINES:
        _ENGINES[dev] = Engine(dev)
    return _ENGINES[dev]


def _bind(eng: Engine, centers, p: int, k: float, period: float, copies: int, bloch,
          radius: float | None):
    """Upload geometry / Bloch phases only when they changed since the last call."""
    c = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 2))
    key = (hashlib.sha1(c.tobytes()).hexdigest(), c.shape[0], int(p), float(k), float(period),
           int(copies))
    if getattr(eng, "_geom_key", None) != key:
        eng._geom_key = None
        eng.set_geometry(c, p, k, period, copies)      # device coincidence check
        eng._geom_key = key
        eng._bloch_key = None
        eng._gap = {}
    if radius is not None:
        r = float(radius)
        if r not in eng._gap:
            eng._gap[r] = eng.check_overlap(r)          # raises DomainError
    bk = tuple(complex(b) for b in bloch)
    if getattr(eng, "_bloch_key", None) != bk:
        eng.set_bloch(np.asarray(bk, dtype=complex))
        eng._bloch_key = bk


def apply_T(beta, centers, k: float, p: int, bloch=1.0, period: float = 1.0, copies: int = 1,
            engine: Engine | None = None, radius: float | None = None):
    """a_m = sum_{l=-P..P} sum_{j, (l,j) != (0,m)} bloch^l T(x_m - x_j - l d e_x) beta_j.

    beta: (M, 2p+1) or (R, M, 2p+1) complex; bloch scalar or (R,).
    Raises DomainError for coincident centres and, given the enclosing
    ``radius``, for overlapping disks (ParticleSet.min_gap)."""
    eng = engine or _engine(beta.device if isinstance(beta, torch.Tensor) else None)
    on_host = not isinstance(beta, torch.Tensor)
    b = torch.as_tensor(np.asarray(beta) if on_host else beta)
    squeeze = b.ndim == 2
    if squeeze:
        b = b[None]
    b = b.to(device=eng.device, dtype=torch.complex128).contiguous()
    bl = np.atleast_1d(np.asarray(bloch, dtype=complex))
    if bl.size == 1 and b.shape[0] > 1:
        bl = np.repeat(bl, b.shape[0])
    _bind(eng, centers, p, k, period, copies, bl, radius)
    out = eng.apply_T(b)
    if squeeze:
        out = out[0]
    return out.cpu().numpy() if on_host else out


def m2l_translate(beta, center_j, center_m, k: float, p: int, radius: float | None = None):
    """Local coefficients at center_m of the outgoing expansion beta at center_j
    (SPEC.md:454-462): a[m'] = sum_n beta[n] H_{n-m'}(k rho) e^{i(n-m') phi}.
    Raises DomainError for coincident centres and, given the disk ``radius``
    (both disks), for ||center_j - center_m|| <= 2 radius."""
    from ._lib import PS_ERR_DOMAIN, DomainError
    beta = np.asarray(beta, dtype=complex)
    cj = np.asarray(center_j, dtype=float)
    cm = np.asarray(center_m, dtype=float)
    dist = float(np.hypot(*(cm - cj)))
    if dist == 0.0 or (radius is not None and dist <= 2.0 * radius):
        raise DomainError(PS_ERR_DOMAIN, f"m2l_translate: disks overlap (separation {dist}, "
                          f"radius {radius}; SPEC.md:458)")
    b = np.zeros((2, 2 * p + 1), dtype=complex)
    b[0] = beta
    out = apply_T(b, np.stack([cj, cm]), k, p, 1.0, 1.0, copies=0)
    return out[1]

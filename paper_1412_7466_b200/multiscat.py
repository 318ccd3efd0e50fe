"""Multipole translation operators on the B200 (multiscat).

``apply_T`` / ``m2l_translate`` keep the SPEC signatures
and run the K1 kernel of libperiscat_b200.so.  NumPy inputs are copied to the
device and the result copied back (the drop-in call a reference user
makes); CUDA tensors stay on the device.
"""
from __future__ import annotations

import numpy as np
import torch

from .engine import Engine

_ENGINES: dict = {}


def _engine(device=None) -> Engine:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev not in _ENGINES:
        _ENGINES[dev] = Engine(dev)
    return _ENGINES[dev]


def apply_T(beta, centers, k: float, p: int, bloch=1.0, period: float = 1.0, copies: int = 1,
            engine: Engine | None = None):
    """a_m = sum_{l=-P..P} sum_{j, (l,j) != (0,m)} bloch^l T(x_m - x_j - l d e_x) beta_j.

    beta: (M, 2p+1) or (R, M, 2p+1) complex; bloch scalar or (R,).
    Raises DomainError for coincident centres."""
    eng = engine or _engine(beta.device if isinstance(beta, torch.Tensor) else None)
    on_host = not isinstance(beta, torch.Tensor)
    b = torch.as_tensor(np.asarray(beta) if on_host else beta)
    squeeze = b.ndim == 2
    if squeeze:
        b = b[None]
    b = b.to(device=eng.device, dtype=torch.complex128).contiguous()
    eng.set_geometry(centers, p, k, period, copies)
    bl = np.atleast_1d(np.asarray(bloch, dtype=complex))
    if bl.size == 1 and b.shape[0] > 1:
        bl = np.repeat(bl, b.shape[0])
    eng.set_bloch(bl)
    out = eng.apply_T(b)
    if squeeze:
        out = out[0]
    return out.cpu().numpy() if on_host else out


def m2l_translate(beta, center_j, center_m, k: float, p: int):
    """Local coefficients at center_m of the outgoing expansion beta at center_j
    (SPEC.md:454-462)."""
    beta = np.asarray(beta, dtype=complex)
    cj = np.asarray(center_j, dtype=float)
    cm = np.asarray(center_m, dtype=float)
    if np.all(cj == cm):
        from ._lib import DomainError, PS_ERR_DOMAIN
        raise DomainError(PS_ERR_DOMAIN, "m2l_translate: coincident centres")
    b = np.zeros((2, 2 * p + 1), dtype=complex)
    b[0] = beta
    out = apply_T(b, np.stack([cj, cm]), k, p, 1.0, 1.0, copies=0)
    return out[1]

"""Single-inclusion scattering matrices (scatmat) -- host setup.

Only the APPLY of S is on the hot path (K1 epilogue); the matrices are
precomputed here once per solve and uploaded through ps_set_smatrix.
"""
from __future__ import annotations

import numpy as np
import scipy.special as sps


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


def rotate_scattering_matrix(S: np.ndarray, phi: float) -> np.ndarray:
    """(S^(m))_{ln} = e^{i phi (l - n)} s_{ln}.  Diagonal input
    (a disk) is returned unchanged."""
    S = np.asarray(S, dtype=complex)
    if S.ndim == 1:
        return S.copy()
    p = (S.shape[0] - 1) // 2
    idx = np.arange(-p, p + 1)
    return S * np.exp(1j * phi * (idx[:, None] - idx[None, :]))

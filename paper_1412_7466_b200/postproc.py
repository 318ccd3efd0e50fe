"""Flux-balance diagnostic (postproc.flux_error)."""
from __future__ import annotations

import math

import numpy as np


def flux_error(c, d, config) -> dict:
    """sum_{k1n>0} k1n |c_n|^2 + sum_{k3n>0} k3n |d_n|^2 vs k1 |sin theta|.

    ``config`` is a ProblemConfig (geometry.py:317) or GratingConfig."""
    c = np.asarray(c)
    d = np.asarray(d)
    k1n = config.vertical_wavenumber(config.k1)
    k3n = config.vertical_wavenumber(config.k3)
    pr = (k1n.imag == 0) & (k1n.real > 0)
    pt = (k3n.imag == 0) & (k3n.real > 0)
    R = float(np.sum(k1n.real[pr] * np.abs(c[pr]) ** 2))
    T = float(np.sum(k3n.real[pt] * np.abs(d[pt]) ** 2))
    inc = config.k1 * abs(math.sin(config.incident_angle))
    return dict(reflected=R, transmitted=T, incoming=inc, error=abs(R + T - inc))


def wood_anomaly_report(config, tolerance: float = 1e-8) -> list:
    """(layer, order, |kappa_n| - k_j) for near-grazing orders."""
    out = []
    for layer, k in ((1, config.k1), (3, config.k3)):
        for n, kap in zip(config.rb_orders, config.kappa_n()):
            gap = abs(kap) - k
            if abs(gap) <= tolerance:
                out.append((layer, int(n), float(gap)))
    return out

"""Host side of the device empty-grating setup (``ps_setup_empty``).

The unit-cell curves are O(n) host work (a few hundred nodes): they are
sampled here with the reference's formulas and handed to the C ABI, which
assembles the 856 x 781 block matrix A and the rhs f for every incidence
angle on the device, takes the SVDs with cuSOLVER, and installs the
restricted A^+ factors the Schur correction streams (empty.cu).  This
replaces ``empty_grating.assemble_empty_system`` + ``factorize``
(/root/reference/pkg/src/periscat/empty_grating.py:139-261) on the
``solve_full`` path, so a solve starts from a ``ProblemConfig`` instead of
host-assembled factors.

Curve sampling restates geometry.py:
  sample_interface       geometry.py:188-221  (nodes offset half a spacing)
  _wall / _lid           geometry.py:225-238  (Gauss-Legendre wall nodes)
  sample_walls_and_lids  geometry.py:241-254
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

# Alpert hybrid Gauss-trapezoidal corrections for log-singular kernels
# (B. Alpert, SIAM J. Sci. Comput. 20 (1999) 1551-1584): order -> (skip a,
# [(node x_m, weight w_m), ...]); the published table the reference's
# quadrature.ALPERT_RULES (quadrature.py:62-88) also holds.
CORRECTION_RULES = {
    2: (1, [(0.1591549430918953, 0.5)]),
    8: (5, [(6.531815708567918e-03, 2.462194198995203e-02),
            (9.086744584657729e-02, 1.701315866854178e-01),
            (3.967966533375878e-01, 4.609256358650077e-01),
            (1.027856640525646e+00, 7.947291148621894e-01),
            (1.945288592909266e+00, 1.008710414337933e+00),
            (2.980147933889640e+00, 1.036093649726216e+00),
            (3.998861349951123e+00, 1.004787656533285e+00)]),
    16: (10, [(8.371529832014113e-04, 3.190919086626234e-03),
              (1.239382725542637e-02, 2.423621380426338e-02),
              (6.009290785739468e-02, 7.740135521653088e-02),
              (1.805991249601928e-01, 1.704889420286369e-01),
              (4.142832599028031e-01, 3.029123478511309e-01),
              (7.964747731112430e-01, 4.652220834914617e-01),
              (1.348993882467059e+00, 6.401489637096768e-01),
              (2.073471660264395e+00, 8.051212946181061e-01),
              (2.947904939031494e+00, 9.362411945698647e-01),
              (3.928129252248612e+00, 1.014359775369075e+00),
              (4.957203086563112e+00, 1.035167721053657e+00),
              (5.986360113977494e+00, 1.020308624984610e+00),
              (6.997957704791519e+00, 1.004798397441514e+00),
              (7.999888757524622e+00, 1.000395017352309e+00),
              (8.999998754306120e+00, 1.000007149422537e+00)]),
}


def correction_rule(order: int):
    """(nodes, weights, skip, interp) of the order-`order` rule; interp =
    max(order, 2) Lagrange points (quadrature.py:59)."""
    skip, tab = CORRECTION_RULES[order]
    x = np.array([a for a, _ in tab], dtype=float)
    w = np.array([b for _, b in tab], dtype=float)
    return x, w, skip, max(order, 2)


def _rows(x, y, nx, ny, speed, weight, t):
    """Curve record [n][8]: x, y, nx, ny, speed, weight, t, arc weight."""
    n = len(x)
    out = np.empty((n, 8))
    for k, v in enumerate((x, y, nx, ny, speed, weight, t)):
        out[:, k] = v
    out[:, 7] = out[:, 5] * out[:, 4]          # DiscretizedCurve.arc_weights
    return out


def interface_curve(spec, n: int, d: float) -> np.ndarray:
    """Equispaced graph interface, nodes at x = d((j + 1/2)/n - 1/2)."""
    if n < 16 or n % 2:
        raise ValueError("need an even node count >= 16")
    t = (np.arange(n) + 0.5) / n
    x = d * (t - 0.5)
    y = spec.height(x, d)
    dy = spec.slope(x, d)
    nrm = np.stack([-dy, np.ones_like(x)], axis=-1)
    nrm /= np.hypot(nrm[:, 0], nrm[:, 1])[:, None]
    speed = np.hypot(np.full_like(x, d), d * dy)
    return _rows(x, y, nrm[:, 0], nrm[:, 1], speed, np.full(n, 1.0 / n), t)


def wall_curve(x: float, lo: float, hi: float, n: int) -> np.ndarray:
    g, w = np.polynomial.legendre.leggauss(n)
    half = 0.5 * (hi - lo)
    y = lo + half * (g + 1.0)
    return _rows(np.full(n, x), y, np.ones(n), np.zeros(n), np.ones(n), half * w, y)


def lid_curve(y: float, n: int, d: float) -> np.ndarray:
    x = -0.5 * d + d * (np.arange(n) + 0.5) / n
    return _rows(x, np.full(n, y), np.zeros(n), np.ones(n), np.ones(n), np.full(n, d / n), x)


def wall_nodes(height: float, d: float, per_unit: int) -> int:
    return max(20, math.ceil(per_unit * height / d))


@dataclass
class UnitCell:
    """Sampled curves of one grating geometry (shared by every incidence angle)."""
    g1: np.ndarray
    g2: np.ndarray
    walls: tuple        # L1, L2, L3 (left walls)
    lid_up: np.ndarray
    lid_down: np.ndarray
    centers: dict
    cols: dict
    rows: dict


def _slices(counts):
    out, start = {}, 0
    for name, cnt in counts:
        out[name] = slice(start, start + cnt)
        start += cnt
    return out


def unit_cell(cfg) -> UnitCell:
    """Curves + block layout of assemble_empty_system (empty_grating.py:145-160)."""
    d, y0 = cfg.period, cfg.y0
    top, bot = cfg.interface_top, cfg.interface_bottom
    g1 = interface_curve(top, cfg.interface_nodes, d)
    g2 = interface_curve(bot, cfg.interface_nodes, d)
    y_top = float(top.height(-0.5 * d, d))
    y_bot = float(bot.height(-0.5 * d, d))
    walls = tuple(wall_curve(-0.5 * d, lo, hi, wall_nodes(hi - lo, d, cfg.wall_nodes_per_unit))
                  for lo, hi in ((y_top, y0), (y_bot, y_top), (-y0, y_bot)))
    lid_n = cfg.lid_nodes
    nj = 2 * cfg.j_expansion_order + 1
    nrb = cfg.rb_modes_per_direction
    n1, n2 = g1.shape[0], g2.shape[0]
    nw1, nw2, nw3 = (w.shape[0] for w in walls)
    cols = _slices([("mu1", n1), ("sigma1", n1), ("mu2", n2), ("sigma2", n2), ("a2", nj),
                    ("a1", nj), ("a3", nj), ("c", nrb), ("d", nrb)])
    rows = _slices([("g1_val", n1), ("g1_der", n1), ("g2_val", n2), ("g2_der", n2),
                    ("w2_val", nw2), ("w2_der", nw2), ("w1_val", nw1), ("w1_der", nw1),
                    ("w3_val", nw3), ("w3_der", nw3), ("gu_val", lid_n), ("gu_der", lid_n),
                    ("gd_val", lid_n), ("gd_der", lid_n)])
    return UnitCell(g1, g2, walls, lid_curve(y0, lid_n, d), lid_curve(-y0, lid_n, d),
                    cfg.expansion_centers(), cols, rows)


def _same_geometry(a, b) -> bool:
    keys = ("period", "k1", "k2", "k3", "y0", "near_field_copies", "j_expansion_order",
            "rb_modes_per_direction", "interface_nodes", "lid_nodes", "wall_nodes_per_unit",
            "alpert_order", "regularization")
    return all(getattr(a, k) == getattr(b, k) for k in keys) and \
        a.interface_top == b.interface_top and a.interface_bottom == b.interface_bottom


def build_desc(cfg, cell: UnitCell):
    """ps_empty_desc for `cfg`; returns (desc, arrays to keep alive)."""
    keep = []

    def arr(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        return a.ctypes.data_as(ctypes.c_void_p)

    def curve(a):
        return _lib.CurveDesc(a.shape[0], arr(a))

    def iface(spec):
        sc = np.asarray(spec.sin_coeffs, dtype=float)
        cc = np.asarray(spec.cos_coeffs, dtype=float)
        return _lib.InterfaceDesc(float(spec.mean), sc.size, cc.size,
                                  arr(sc) if sc.size else None, arr(cc) if cc.size else None)

    x, w, skip, interp = correction_rule(cfg.alpert_order)
    ctr = cell.centers
    desc = _lib.EmptyDesc()
    desc.period, desc.k1, desc.k2, desc.k3 = cfg.period, cfg.k1, cfg.k2, cfg.k3
    desc.y0, desc.eps = cfg.y0, cfg.regularization
    desc.copies, desc.Q, desc.nrb = (cfg.near_field_copies, cfg.j_expansion_order,
                                     cfg.rb_modes_per_direction)
    for i, k in enumerate((1, 2, 3)):
        desc.centers[2 * i] = float(ctr[k][0])
        desc.centers[2 * i + 1] = float(ctr[k][1])
    desc.g1, desc.g2 = curve(cell.g1), curve(cell.g2)
    for i in range(3):
        desc.wall[i] = curve(cell.walls[i])
    desc.lid_up, desc.lid_down = curve(cell.lid_up), curve(cell.lid_down)
    desc.top, desc.bottom = iface(cfg.interface_top), iface(cfg.interface_bottom)
    desc.rule_n, desc.rule_skip, desc.rule_interp = x.size, skip, interp
    desc.rule_x, desc.rule_w = arr(x), arr(w)
    return desc, keep


@dataclass
class DeviceEmptySystem:
    """One incidence angle's empty-grating system living on the device: the
    duck type of EmptyGratingSystem the solver needs (config, cols, rows,
    centers), with the matrix, rhs, scaling and singular values fetched on
    demand (``fetch``) for parity checks."""
    config: object
    cols: dict
    rows: dict
    centers: dict
    engine: object
    irhs: int

    def fetch(self):
        """(A, f, col_scale, s) of this RHS, copied from the device."""
        return self.engine.get_empty(self.irhs)


def validate(configs):
    configs = list(configs)
    c0 = configs[0]
    for c in configs[1:]:
        if not _same_geometry(c0, c):
            raise ValueError("batched right-hand sides must share the grating geometry "
                             "(only the incidence angle may differ)")
    for c in configs:
        if not (-np.pi < c.incident_angle < 0.0):
            raise ValueError("incident angle must lie in (-pi, 0)")   # geometry.py:349-350
    return configs

"""Golden wall-discrepancy data of coupled solutions (test infrastructure).

For the oracle's golden cfg1 / cfg2 solutions (BASELINE grating, omega=10),
runs the reference's OWN checker ``empty_grating.wall_discrepancy_residual``
(empty_grating.py:396-433) on x = A^+ (f - C beta) with the particles'
phased multipole field as its ``extra_field`` (as
tests/test_oracle_pin.py does), and records the pieces it sums at the fresh
wall points -- the layer-field values ``eval_empty_field(total=False)``
(eg:352-393), their x-derivatives ``_x_derivative_of_representation``
(eg:436-470) and the particle values / x-derivatives from
``specialfn.outgoing_wave_block`` (sf:128-154) -- so the device kernels
(ps_layer_field_grad, ps_particle_field_grad) and Solution.wall_residual can
be pinned on the GPU box without the reference.  Writes
tests/golden/walls_cfg{1,2}.npz.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_walls.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from periscat import empty_grating as eg  # noqa: E402
from periscat import quadrature, specialfn  # noqa: E402

from oracle import periscat_oracle as O  # noqa: E402
from oracle.make_empty import config_for  # noqa: E402


def make(cfg: int, n_fresh: int = 31):
    conf = config_for(10.0, -0.7 * np.pi)
    system = eg.assemble_empty_system(conf)
    eg.factorize(system)
    pb = O.load_problem(cfg)
    z = np.load(os.path.join(O.GOLDEN, f"golden_cfg{cfg}.npz"))
    beta = z["beta"]
    x = eg.apply_pinv(system, system.rhs - O.apply_C(pb.es, beta, pb.centers))
    sol = eg.EmptySolution(system, x, 0.0)
    orders = np.arange(-pb.p, pb.p + 1)
    alpha = conf.bloch_phase
    d = conf.period

    def particles(points, normals):
        vals = np.zeros(len(points), complex)
        ders = np.zeros(len(points), complex)
        mid = eg.classify_layer(conf, points) == 2
        pts, nrm = points[mid], normals[mid]
        for j in range(pb.M):
            for l in range(-conf.near_field_copies, conf.near_field_copies + 1):
                v, g = specialfn.outgoing_wave_block(conf.k2, pb.centers[j] + [l * d, 0.0],
                                                     orders, pts)
                vals[mid] += alpha ** l * (v @ beta[j])
                ders[mid] += alpha ** l * (np.einsum("ijk,ik->ij", g, nrm) @ beta[j])
        return vals, ders

    coupled = eg.wall_discrepancy_residual(sol, extra_field=particles, n_fresh=n_fresh)
    without = eg.wall_discrepancy_residual(sol, n_fresh=n_fresh)
    # the same fresh points the checker builds (eg:411-420)
    inset = 6.0 * d / conf.interface_nodes
    pts = []
    for wname in ("1", "2", "3"):
        wall = system.curves["L" + wname]
        ylo, yhi = float(np.min(wall.nodes[:, 1])), float(np.max(wall.nodes[:, 1]))
        ys, _ = quadrature.gauss_legendre(n_fresh, ylo + inset, yhi - inset)
        left = np.stack([np.full(n_fresh, -0.5 * d), ys], axis=-1)
        pts.append(np.vstack([left, left + [d, 0.0]]))
    pts = np.vstack(pts)
    nrm = np.tile([1.0, 0.0], (pts.shape[0], 1))
    lay_v = eg.eval_empty_field(sol, pts, total=False)
    lay_d = eg._x_derivative_of_representation(sol, pts, nrm)
    par_v, par_d = particles(pts, nrm)
    np.savez_compressed(os.path.join(O.GOLDEN, f"walls_cfg{cfg}.npz"), pts=pts,
                        layer=eg.classify_layer(conf, pts), x=x, beta=beta,
                        layer_val=lay_v, layer_dx=lay_d, particle_val=par_v, particle_dx=par_d,
                        coupled=coupled, without=without, alpha=alpha)
    print(cfg, "coupled", coupled, "without", without)


if __name__ == "__main__":
    import warnings
    warnings.simplefilter("ignore")
    for c in (1, 2):
        make(c)

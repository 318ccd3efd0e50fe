"""Golden empty-grating layer fields of coupled solutions (test infrastructure).

For the oracle's golden solutions (cfg1 inclusions in the flat BASELINE
grating, and in the curved grating), evaluates the reference's OWN field
evaluator ``empty_grating.eval_empty_field(solution, points, total=True)``
(empty_grating.py:352-393) on x = A^+ (f - C beta) (the recovery of
solve_full; ``apply_pinv``, eg:264-273) at grid points of all
three layers away from the interfaces and the particles.  Runs only where the
reference is mounted; writes tests/golden/field_{w10,curved}.npz.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_fields.py
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

from oracle import periscat_oracle as O  # noqa: E402
from oracle.make_empty import config_for  # noqa: E402


def make(name: str, golden: str):
    conf = config_for(10.0, -0.7 * np.pi, curved=(name == "curved"))
    system = eg.assemble_empty_system(conf)
    eg.factorize(system)
    z = np.load(os.path.join(O.GOLDEN, golden))
    base = O.load_problem(1)
    es = O.load_empty(name)
    beta = z["beta"]
    x = eg.apply_pinv(system, system.rhs - O.apply_C(es, beta, base.centers))
    sol = eg.EmptySolution(system, x, 0.0)
    xs = np.linspace(-0.5, 0.5, 23)
    ys = np.linspace(-0.97 * conf.y0, 0.97 * conf.y0, 41)   # inside the artificial boundaries
    X, Y = np.meshgrid(xs, ys)
    pts = np.column_stack([X.ravel(), Y.ravel()])
    h = conf.period / conf.interface_nodes
    top = conf.interface_top.height(pts[:, 0], conf.period)
    bot = conf.interface_bottom.height(pts[:, 0], conf.period)
    keep = (np.abs(pts[:, 1] - top) > 6 * h) & (np.abs(pts[:, 1] - bot) > 6 * h)
    for l in (-1, 0, 1):
        d = pts[:, None, :] - base.centers[None, :, :] - np.array([l * conf.period, 0.0])
        keep &= np.all(np.hypot(d[..., 0], d[..., 1]) > 0.04, axis=1)
    pts = pts[keep]
    layer = eg.classify_layer(conf, pts)
    vals = eg.eval_empty_field(sol, pts, total=True)
    np.savez_compressed(os.path.join(O.GOLDEN, f"field_{name}.npz"), pts=pts, layer=layer,
                        field=vals, beta=beta)
    print(name, pts.shape[0], np.bincount(layer), float(np.max(np.abs(vals))))


if __name__ == "__main__":
    import warnings
    warnings.simplefilter("ignore")
    make("w10", "golden_cfg1.npz")
    make("curved", "golden_curved.npz")

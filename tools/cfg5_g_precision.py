"""Where the cfg5 coupling-row gap comes from (CPU; test infrastructure).

g = C beta (576 rows) at cfg5 (M = 1e4, RHS 0 / 15, the seeded
Krylov-scaled beta of tools/probe_cfg5_parity.py) evaluated by the oracle
in three ways:
  f64    -- periscat_oracle.apply_C as is (float64 sums);
  ld     -- the same float64 entries (Hankel values, phases, Bloch weights)
            but every sum accumulated in x87 extended precision
            (np.clongdouble, 64-bit mantissa): the float64 operator
            evaluated ~2000x more exactly;
  f64rev -- float64 with the sources in reverse order (an equally valid
            summation order).
and compared with the device's g (dumped by the probe).  If the device is
as close to `ld` as the oracle's own float64 evaluation is, the GPU/oracle
gap is float64 summation rounding amplified by the pseudo-inverse's
1/eps = 1e10 directions (eg:264-273), not an implementation difference.

    python tools/cfg5_g_precision.py gpurun_out/cfg5_g_gpu_mf.npy [rhs]
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

from oracle import periscat_oracle as O  # noqa: E402


def particle_field_ld(k2, beta, centers, pts, shift, order):
    p = (beta.shape[1] - 1) // 2
    n = np.arange(-p, p + 1)
    val = np.zeros(pts.shape[0], dtype=np.clongdouble)
    gx = np.zeros(pts.shape[0], dtype=np.clongdouble)
    gy = np.zeros(pts.shape[0], dtype=np.clongdouble)
    for j in order:
        dx = pts[:, 0] - centers[j, 0] - shift
        dy = pts[:, 1] - centers[j, 1]
        v, g = O._outgoing_vals_grads(k2, n, dx, dy, sign=1)
        b = beta[j].astype(np.clongdouble)
        val += b @ v.astype(np.clongdouble)
        gx += b @ g[0].astype(np.clongdouble)
        gy += b @ g[1].astype(np.clongdouble)
    return val, gx, gy


def apply_C_ld(es, beta, centers, reverse=False):
    k2, d, al, P = es.k2, es.period, np.clongdouble(es.bloch), es.copies
    g = np.zeros(es.A.shape[0], dtype=np.clongdouble)
    order = range(centers.shape[0] - 1, -1, -1) if reverse else range(centers.shape[0])
    for nodes, nrm, rv, rd, sgn in ((es.g1_nodes, es.g1_normals, "g1_val", "g1_der", -1.0),
                                    (es.g2_nodes, es.g2_normals, "g2_val", "g2_der", 1.0)):
        for l in range(-P, P + 1):
            v, gx, gy = particle_field_ld(k2, beta, centers, nodes, l * d, order)
            w = sgn * al ** l
            g[es.rows[rv]] += w * v
            g[es.rows[rd]] += w * (gx * nrm[:, 0] + gy * nrm[:, 1])
    for l, coef, sgn in ((P, al ** (P + 1), 1.0), (-(P + 1), al ** (-P), -1.0)):
        v, gx, gy = particle_field_ld(k2, beta, centers, es.L2_nodes, l * d, order)
        g[es.rows["w2_val"]] += sgn * coef * v
        g[es.rows["w2_der"]] += sgn * coef * gx
    return g


def rel(a, b):
    a = np.asarray(a, dtype=np.clongdouble)
    b = np.asarray(b, dtype=np.clongdouble)
    return float(np.linalg.norm((a - b).astype(np.complex128)) / np.linalg.norm(b.astype(np.complex128)))


def main():
    gpu = np.load(sys.argv[1])
    rhs = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    names = ["w10_a00", "w10_a15"]
    centers = np.load(os.path.join(O.GOLDEN, "centers_cfg5.npy"))
    p, R = 20, 0.004
    pr0 = O.Problem(O.load_empty(names[0]), centers, p, R)
    M, L = centers.shape[0], 2 * p + 1
    rng = np.random.default_rng(5)       # the probe's beta
    v = pr0.smat[None, None, :] * (rng.standard_normal((2, M, L)) + 1j * rng.standard_normal((2, M, L)))
    es = O.load_empty(names[rhs])
    nrc = gpu.shape[1]
    g64 = O.apply_C(es, v[rhs], centers)[:nrc]
    gld = apply_C_ld(es, v[rhs], centers)[:nrc]
    g64r = O.apply_C(es, v[rhs][::-1].copy(), centers[::-1].copy())[:nrc]
    out = dict(rhs=names[rhs],
               oracle_f64_vs_ld=rel(g64, gld), oracle_f64rev_vs_ld=rel(g64r, gld),
               oracle_f64_vs_f64rev=rel(g64, g64r), gpu_vs_ld=rel(gpu[rhs], gld),
               gpu_vs_oracle_f64=rel(gpu[rhs], g64))
    # per-row view: worst component relative error against ld
    den = np.abs(gld.astype(np.complex128))
    for name, g in (("oracle_f64", g64), ("gpu", gpu[rhs])):
        e = np.abs((np.asarray(g, dtype=np.clongdouble) - gld).astype(np.complex128))
        out[f"{name}_max_row_rel_vs_ld"] = float(np.max(e / np.maximum(den, 1e-300)))
        out[f"{name}_median_row_rel_vs_ld"] = float(np.median(e / np.maximum(den, 1e-300)))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

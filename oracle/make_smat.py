"""Golden scattering matrices of star-shaped particles (test infrastructure).

The reference ships scatmat only as a SPEC, so
this is the CPU restatement of ``scatmat.solve_muller_particle`` and
``scatmat.scattering_matrix`` (Eqs.
intg1-intg2 and the s_ln projection) built from the reference's OWN Nystrom
primitives, imported from /root/reference (this script runs only where the
reference is mounted; its outputs are committed):

  geometry.sample_particle          geometry.py:224-256
  layerpot.boundary_operator_matrices (self path, closed curve, k_subtract)
                                    layerpot.py:171-193 -> quadrature.nystrom_selfmatrix
  specialfn.regular_wave_block      specialfn.py:86-125

Pins checked here and in tests/test_smat_cpu.py:
  * disk: the BIE matrix equals the analytic diagonal -- this
    fixes the projection's normalisation (i/4), SPEC.md:441's open question;
  * no contrast (kp = k2): S = 0;
  * par1: S applied to the plane wave's local expansion
    reproduces the BIE-computed scattered field at 20 probes.

Writes tests/golden/smat_shapes.npz (+ .json provenance), and
tests/golden/golden_star.npz: the oracle's full solve of cfg1's grating with
rotated star particles (dense S with rotation phases).

    PYTHONPATH=/root/reference/pkg/src python oracle/make_smat.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import scipy

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from periscat import geometry, layerpot, quadrature, specialfn  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# name -> (base radius, bump, lobes, k2, kp, p)
SHAPES = {
    "disk_w10": (0.04, 0.0, 1, 12.0, 15.0, 20),          # cfg1 inclusion: analytic pin
    "par1": (0.0309, 0.0103, 3, 8.0, 30.0, 10),          # SPEC.md:408 example shape
    "star3_w10": (0.03, 0.01, 3, 12.0, 15.0, 20),        # cfg1 grating, 3-lobed star
    "pent_w10": (0.032, 0.006, 5, 12.0, 15.0, 20),       # cfg1 grating, pentagon-like
}
N_NODES = 300                                            # PAPER §6: N = 300


def muller_densities(curve, k2, kp, u, dudn):
    """Solve Eqs. intg1-intg2 for (mu, sigma) given incident traces (columns)."""
    mats = layerpot.boundary_operator_matrices(curve, curve, k2, k_subtract=kp,
                                               rule=quadrature.ALPERT_RULES[16])
    n = curve.n
    eye = np.eye(n)
    A = np.block([[eye + mats["D"], mats["S"]], [mats["T"], -eye + mats["N"]]])
    rhs = -np.vstack([u, dudn])
    X = np.linalg.solve(A, rhs)
    res = np.linalg.norm(A @ X - rhs) / np.linalg.norm(rhs)
    return X[:n], X[n:], res


def bie_scattering_matrix(shape, k2, kp, p, n=N_NODES):
    """s_ln = (i/4) sum_y w [J_l e^{-il th} sigma_n + d/dn(J_l e^{-il th}) mu_n]."""
    curve = geometry.sample_particle(shape, np.zeros(2), 0.0, n)
    orders = np.arange(-p, p + 1)
    v, g = specialfn.regular_wave_block(k2, np.zeros(2), orders, curve.nodes)
    dn = np.einsum("ijk,ik->ij", g, curve.normals)
    mu, sigma, res = muller_densities(curve, k2, kp, v, dn)
    aw = curve.arc_weights[:, None]
    S = 0.25j * ((np.conj(v) * aw).T @ sigma + (np.conj(dn) * aw).T @ mu)
    return S, res, curve


def disk_analytic(radius, k2, kp, p):
    from oracle import periscat_oracle as O
    return O.disk_smatrix(radius, k2, kp, p)


def plane_wave_check(shape, k2, kp, p, S, alpha=0.7, nprobe=20, n=N_NODES):
    """S applied to the local expansion a_n = i^n e^{-in alpha}
    of e^{ik(x cos a + y sin a)} vs the BIE scattered field S^{k2} sigma +
    D^{k2} mu at probes on a circle of radius 3 R."""
    curve = geometry.sample_particle(shape, np.zeros(2), 0.0, n)
    kv = k2 * np.array([np.cos(alpha), np.sin(alpha)])
    u = np.exp(1j * curve.nodes @ kv)
    dudn = 1j * (curve.normals @ kv) * u
    mu, sigma, _ = muller_densities(curve, k2, kp, u[:, None], dudn[:, None])
    R = shape.base_radius + shape.bump_amplitude
    th = np.linspace(0, 2 * np.pi, nprobe, endpoint=False)
    probes = 3 * R * np.stack([np.cos(th), np.sin(th)], axis=-1)
    us = layerpot.eval_layer_potentials(layerpot.Density(curve, sigma[:, 0], "single"), k2, probes) \
        + layerpot.eval_layer_potentials(layerpot.Density(curve, mu[:, 0], "double"), k2, probes)
    orders = np.arange(-p, p + 1)
    a = (1j ** orders) * np.exp(-1j * orders * alpha)
    beta = S @ a
    hv, _ = specialfn.outgoing_wave_block(k2, np.zeros(2), orders, probes)
    return float(np.max(np.abs(hv @ beta - us)) / np.max(np.abs(us)))


def make_shapes():
    out, meta = {}, {}
    for name, (a1, a2, a3, k2, kp, p) in SHAPES.items():
        t0 = time.perf_counter()
        shape = geometry.ParticleShape(a1, a2, a3)
        S, res, _ = bie_scattering_matrix(shape, k2, kp, p)
        out[name] = S
        out[name + "_params"] = np.array([a1, a2, a3, k2, kp, p, N_NODES], dtype=float)
        m = dict(residual=res, seconds=time.perf_counter() - t0)
        if a2 == 0.0:
            ana = disk_analytic(a1, k2, kp, p)
            m["disk_vs_analytic"] = float(np.max(np.abs(S - np.diag(ana))) / np.max(np.abs(ana)))
        m["plane_wave_probe_error"] = plane_wave_check(shape, k2, kp, p, S)
        S0, _, _ = bie_scattering_matrix(shape, k2, k2, p)
        m["no_contrast_max"] = float(np.max(np.abs(S0)))
        meta[name] = m
        print(name, m, flush=True)
    np.savez_compressed(os.path.join(OUT, "smat_shapes.npz"), **out)
    meta.update(numpy=np.__version__, scipy=scipy.__version__, nodes=N_NODES,
                generator="oracle/make_smat.py (reference Nystrom primitives)")
    with open(os.path.join(OUT, "smat_shapes.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    return out


def make_star_golden(smats):
    """cfg1 grating (M=10, p=20) with 3-lobed stars at seeded rotations: the
    oracle's full solve with a dense rotated S."""
    from oracle import periscat_oracle as O
    t0 = time.perf_counter()
    base = O.load_problem(1)
    rot = np.random.default_rng(7).uniform(0, 2 * np.pi, base.M)
    pb = O.Problem(base.es, base.centers, base.p, 0.04, smat=smats["star3_w10"], rot=rot)
    rng = np.random.default_rng(77)
    v = rng.standard_normal((pb.M, pb.L)) + 1j * rng.standard_normal((pb.M, pb.L))
    schur = O.apply_schur_operator(pb, v).reshape(pb.M, pb.L)
    sol = O.solve_full(pb)
    np.savez_compressed(os.path.join(OUT, "golden_star.npz"), rot=rot, v=v, schur=schur,
                        beta=sol.beta, c=sol.c, d=sol.d, iterations=sol.iterations,
                        flux_error=sol.flux["error"])
    print("star golden", sol.iterations, sol.flux, time.perf_counter() - t0)


if __name__ == "__main__":
    import warnings
    warnings.simplefilter("ignore")
    make_star_golden(make_shapes())

"""Golden vectors from the CPU oracle (test infrastructure).

Writes tests/golden/golden_cfg{1,2,3,4}.npz:
  * a seeded Krylov-scaled input v = S (complex Gaussian) and the oracle's
    apply_T(v) and apply_schur_operator(v) (cfg1, cfg2 full; cfg3/4 on a
    fixed 24-target slice for apply_T);
  * the oracle's full solve: c, d, flux error, GMRES iterations, and beta.

The oracle's apply_T inside GMRES is spread over a process pool (target
slices), exactly the restated SPEC operator otherwise.  Provenance (numpy /
scipy versions, seconds) is stored alongside.

    python oracle/make_goldens.py 1 2 3 4
"""
from __future__ import annotations

import os

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import json
import multiprocessing as mp
import sys
import time

import numpy as np
import scipy

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle import periscat_oracle as O  # noqa: E402

OUT = O.GOLDEN
SLICE = np.r_[0:8, 500:508, 992:1000]
_S = {}


def _init(cfg):
    _S["pb"] = O.load_problem(cfg)


def _slice_T(args):
    v, tids = args
    pb = _S["pb"]
    return O.apply_T(v, pb.centers, pb.es.k2, pb.p, pb.es.bloch, pb.es.period, pb.es.copies,
                     targets=tids)


def main(cfgs):
    for cfg in cfgs:
        t0 = time.perf_counter()
        pb = O.load_problem(cfg)
        rng = np.random.default_rng(1000 + cfg)
        v = pb.smat[None, :] * (rng.standard_normal((pb.M, pb.L)) + 1j * rng.standard_normal((pb.M, pb.L)))
        nproc = len(os.sched_getaffinity(0))
        chunks = [c for c in np.array_split(np.arange(pb.M), nproc) if c.size]
        with mp.get_context("fork").Pool(nproc, initializer=_init, initargs=(cfg,)) as pool:
            def par_T(x):
                parts = pool.map(_slice_T, [(x, c) for c in chunks])
                return np.concatenate(parts, axis=0)

            def op(x):
                x = x.reshape(pb.M, pb.L)
                u = par_T(x)
                g = pb.es.apply_pinv(O.apply_C(pb.es, x, pb.centers))
                u = u - O.apply_B_phys(pb.es, g, pb.centers, pb.p)
                return (x - pb.smat[None, :] * u).reshape(-1)

            small = pb.M <= 100
            tids = np.arange(pb.M) if small else SLICE
            aT = par_T(v)[tids]
            sch = op(v).reshape(pb.M, pb.L)[tids]
            rhs = O.schur_rhs(pb)
            beta, its, hist = O.gmres(op, rhs, 1e-10, 150)
        beta = beta.reshape(pb.M, pb.L)
        x = pb.es.apply_pinv(pb.es.f - O.apply_C(pb.es, beta, pb.centers))
        c, d = x[pb.es.cols["c"]], x[pb.es.cols["d"]]
        flux = O.flux_error(pb.es, c, d)
        dt = time.perf_counter() - t0
        np.savez_compressed(os.path.join(OUT, f"golden_cfg{cfg}.npz"), v=v, targets=tids,
                            apply_T=aT, schur=sch, rhs=rhs.reshape(pb.M, pb.L)[tids],
                            beta=beta, c=c, d=d, flux_error=flux["error"], iterations=its,
                            history=np.array(hist))
        meta = dict(cfg=cfg, seconds=dt, iterations=its, flux=flux, numpy=np.__version__,
                    scipy=scipy.__version__, processes=nproc,
                    generator="oracle/make_goldens.py (oracle.periscat_oracle)")
        with open(os.path.join(OUT, f"golden_cfg{cfg}.json"), "w") as fh:
            json.dump(meta, fh, indent=1)
        print(json.dumps(meta), flush=True)


def make_curved():
    """cfg1's inclusions (M=10, r=0.04, p=20) in the grating with the
    reference's default sinusoidal interfaces (fixture empty_curved, written
    by oracle/make_empty.py curved): the oracle's full solve, for the device
    assembly of curved interfaces end to end."""
    t0 = time.perf_counter()
    base = O.load_problem(1)
    pb = O.Problem(O.load_empty("curved"), base.centers, base.p, base.radius)
    rng = np.random.default_rng(1500)
    v = pb.smat[None, :] * (rng.standard_normal((pb.M, pb.L)) + 1j * rng.standard_normal((pb.M, pb.L)))
    sch = O.apply_schur_operator(pb, v).reshape(pb.M, pb.L)
    sol = O.solve_full(pb)
    np.savez_compressed(os.path.join(OUT, "golden_curved.npz"), v=v, schur=sch, beta=sol.beta,
                        c=sol.c, d=sol.d, flux_error=sol.flux["error"],
                        iterations=sol.iterations)
    print("curved", sol.iterations, sol.flux, time.perf_counter() - t0, flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["curved"]:
        make_curved()
    else:
        main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4])

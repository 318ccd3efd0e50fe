"""cfg5 parity probe (GPU box): Schur operator of RHS 0 and 15 (fixtures
w10_a00 / w10_a15, M = 1e4, p = 20) against the oracle on a seeded target
slice, split into inclusions near an interface (< 0.01) and the rest, next
to the operator's own sensitivity to a 1-ulp perturbation of the coupling
rows g = C beta, and the device operator fed the oracle's g.

    python tools/probe_cfg5_parity.py [--targets 64] [--dense 0|1] > out.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import workloads  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--targets", type=int, default=64)
    ap.add_argument("--dense", type=int, default=0)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--dump-g", default=None, help="save the device C beta [2][576] and exit")
    a = ap.parse_args()
    import torch

    from oracle import parallel as OP
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, solver
    centers = np.load(os.path.join(O.GOLDEN, "centers_cfg5.npy"))
    names = ["w10_a00", "w10_a15"]
    p, R = 20, 0.004
    t0 = time.time()
    op = solver.SchurOperator([workloads.load_fixture(n) for n in names], centers, p, radius=R,
                              dense_gb=40.0 if a.dense else 0.0)
    M, L = op.M, op.L
    rng = np.random.default_rng(a.seed)
    smat = op.smat
    v = smat[None, None, :] * (rng.standard_normal((2, M, L)) + 1j * rng.standard_normal((2, M, L)))
    vd = torch.as_tensor(v).cuda()
    y = op(vd).cpu().numpy()
    g = op.eng.apply_C(vd)
    if a.dump_g:
        np.save(a.dump_g, g.cpu().numpy())
        return
    ulp = 2.0 ** -53
    sgn = torch.as_tensor(rng.choice([-1.0, 1.0], size=g.shape) + 1j * rng.choice([-1.0, 1.0],
                          size=g.shape)).cuda()
    yg = op(vd, g=g).cpu().numpy()
    yp = op(vd, g=g * (1 + ulp * sgn)).cpu().numpy()
    sl = np.sort(rng.choice(M, a.targets, replace=False))
    near = np.minimum(np.abs(centers[sl, 1] - 0.5), np.abs(centers[sl, 1] + 0.5)) < 0.01
    out = dict(targets=int(a.targets), near=int(near.sum()), dense=bool(op.dense),
               setup_s=time.time() - t0, rhs={})
    for r, n in enumerate(names):
        pr = O.Problem(O.load_empty(n), centers, p, R)
        t1 = time.time()
        gor = OP.apply_C(pr.es, v[r], centers)[:op.eng.nrow_c]
        print(n, 'oracle C', time.time() - t1, file=sys.stderr, flush=True)
        ref = OP.apply_schur_operator(pr, v[r], sl)
        # an equally valid float64 oracle: sources summed in reverse order
        ref_rev = OP.apply_schur_operator(pr, v[r], sl, reverse_sources=True)
        t_or = time.time() - t1
        gdev = g[r].cpu().numpy()
        gsub = torch.as_tensor(np.stack([gor if q == r else g[q].cpu().numpy()
                                         for q in range(2)])).cuda()
        yo = op(vd, g=gsub).cpu().numpy()[r]
        rec = dict(oracle_s=t_or,
                   slice_all=rel(y[r][sl], ref), slice_far=rel(y[r][sl][~near], ref[~near]),
                   slice_near=rel(y[r][sl][near], ref[near]) if near.any() else None,
                   g_gap=rel(gdev, gor),
                   with_oracle_g_slice=rel(yo[sl], ref),
                   with_oracle_g_far=rel(yo[sl][~near], ref[~near]),
                   with_oracle_g_near=rel(yo[sl][near], ref[near]) if near.any() else None,
                   oracle_spread_slice=rel(ref_rev, ref),
                   oracle_spread_near=rel(ref_rev[near], ref[near]) if near.any() else None,
                   ulp_sensitivity_full=rel(yp[r], yg[r]),
                   ulp_sensitivity_slice=rel(yp[r][sl], yg[r][sl]),
                   ulp_sensitivity_near=rel(yp[r][sl][near], yg[r][sl][near]) if near.any() else None,
                   g_repeat_bitwise=bool(np.array_equal(yg[r], y[r])))
        out["rhs"][n] = rec
        print(n, rec, file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Small driver that launches every device kernel family once, for
compute-sanitizer (memcheck / racecheck / synccheck) runs:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --small

K1 (tiled), K1s (symmetric), K1m (DFMA multi-RHS), K1d (DMMA multi-RHS), the
dense and matrix-free coupling (K3/K5, ct_gemv / b_gemv / pinv), the
SM-partitioned step, device GMRES, the Krylov building blocks, field kernels,
device empty-grating assembly + SVD and the Muller-BIE scattering matrix.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import periscat_oracle as O
from paper_1412_7466_b200 import grating, postproc, solver
from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true", help="cfg1 only (racecheck is slow)")
a = ap.parse_args()


def cplx(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


rng = np.random.default_rng(0)
cfgs = [1] if a.small else [1, 2]
for cfg in cfgs:
    pb = O.load_problem(cfg)
    sysm = workloads.load_fixture("w10")
    for dense_gb in (40.0, 0.0):
        op = solver.SchurOperator(sysm, pb.centers, pb.p, smat=pb.smat, dense_gb=dense_gb)
        v = torch.as_tensor(pb.smat[None, None, :] * cplx(rng, (1, pb.M, pb.L))).cuda()
        for variant in (1, 2, 3):                   # K1 tiled, K1s symmetric, K1h (DMMA)
            op.eng.set_k1_variant(variant)
            for ov in (-1, 2):                      # serial, SM-partitioned
                op.eng.set_overlap(ov)
                op(v)
                op.apply_T(v)
        op.eng.set_k1_variant(0)
        x, its, hist = solver.gmres(op, op.rhs(), 1e-10, 40)
        postproc.coupled_residual(op, x)
        postproc.wall_discrepancy_residual(op, x)
        print(f"cfg{cfg} dense={dense_gb > 0}: gmres {its}", flush=True)
    # multi-RHS kernels
    for variant in (1, 2):
        eng = Engine(0)
        eng.set_geometry(pb.centers, pb.p, 12.0, 1.0, 1)
        eng.set_bloch(np.exp(1j * np.linspace(0, 1, 16)))
        eng.set_mrhs_variant(variant)
        eng.apply_T(torch.as_tensor(cplx(rng, (16, pb.M, pb.L))).cuda())
        print(f"cfg{cfg} mrhs variant {variant} ok", flush=True)
# batched-RHS coupled operator (matrix-free + dense), generic Krylov driver
pb = O.load_problem(1)
systems = [workloads.load_fixture(n) for n in ("w10", "w10_a00", "w10_a15")]
op = solver.SchurOperator(systems, pb.centers, pb.p, smat=pb.smat)
x, its, hist = solver.gmres(lambda t: op(t), op.rhs(), 1e-10, 30, engine=op.eng)
print("multi-RHS generic gmres", its, flush=True)
# device empty-grating setup + field evaluation
sol = solver.solve_full(workloads.fixture_config("w10"), pb.centers, pb.p, smat=pb.smat)
print("device setup solve", sol.iterations, sol.coupled_residual, flush=True)
# Muller BIE scattering matrix of a star
from paper_1412_7466_b200 import scatmat  # noqa: E402

shape = type("Shape", (), dict(base_radius=0.04, bump_amplitude=0.01, lobes=3))()
S = scatmat.scattering_matrix(shape, 12.0, 15.0, 10, 300)
print("scattering matrix ok", flush=True)
torch.cuda.synchronize()
print("sanitize run done")

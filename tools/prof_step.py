"""Minimal Schur-matvec loop for ncu captures (cfg3 by default)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import grating, solver
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--k1-variant", type=int, default=0, help="0 auto, 1 tiled K1, 2 symmetric K1s, 3 K1h")
ap.add_argument("--overlap", type=int, default=None, help="SMs left to the coupling chain")
ap.add_argument("--order", type=int, default=None, help="0 chain first, 1 K1s first")
a = ap.parse_args()
sysm, centers, p, radius = workloads.load_config(a.cfg)
op = solver.SchurOperator(sysm, centers, p, radius=radius)
op.eng.set_k1_variant(a.k1_variant)
if a.overlap is not None:
    op.eng.set_overlap(a.overlap)
if a.order is not None:
    op.eng.set_overlap_order(a.order)
rng = np.random.default_rng(0)
v = op.smat[None, None, :] * (rng.standard_normal((1, op.M, op.L)) + 1j * rng.standard_normal((1, op.M, op.L)))
v = torch.as_tensor(v).cuda()
y = torch.empty_like(v)
for _ in range(a.steps):
    op(v, out=y)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))

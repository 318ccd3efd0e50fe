"""cfg5 (M=1e4, p=20, 16 RHS) Schur step breakdown: apply_T alone vs the full
S-preconditioned Schur matvec (matrix-free coupling for 16 RHS)."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import grating, solver
import workloads  # noqa: E402

systems, centers, p, radius = workloads.load_cfg5()
with ThreadPoolExecutor(16) as ex:
    list(ex.map(grating.factorize, systems))
op = solver.SchurOperator(systems, centers, p, radius=radius)
print("dense coupling:", op.dense, flush=True)
rng = np.random.default_rng(0)
v = torch.as_tensor(op.smat[None, None, :] * (rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape))).cuda()
out = torch.empty_like(v)
for name, fn in (("apply_T", lambda: op.apply_T(v, out)), ("schur", lambda: op(v, out)),
                 ("apply_C", lambda: op.eng.apply_C(v))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)

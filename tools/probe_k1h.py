"""K1s (DFMA consumers, variant 2) vs K1h (DMMA consumers, variant 3):
apply_T time and agreement on the cfg3 geometry at p = 25 and p = 20, and
the cfg3 Schur step with each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import solver
from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402


def timed(fn, n=30):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


sysm, centers, p3, radius = workloads.load_config(3)
for p in (25, 20):
    L = 2 * p + 1
    M = centers.shape[0]
    eng = Engine(0)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(np.array([np.exp(-0.7j)]))
    rng = np.random.default_rng(0)
    s = np.exp(-0.5 * np.abs(np.arange(-p, p + 1)))
    v = torch.as_tensor(s * (rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L)))).cuda()
    outs, ts = {}, {}
    for var in (2, 3):
        eng.set_k1_variant(var)
        out = torch.empty_like(v)
        ts[var] = timed(lambda: eng.apply_T(v, out))
        outs[var] = out.clone()
    d = (torch.linalg.norm(outs[3] - outs[2]) / torch.linalg.norm(outs[2])).item()
    tr = M * (3 * M - 1)
    fl = tr * 8 * L * L
    print(f"p={p} M={M}: K1s {ts[2]*1e3:8.1f} us ({fl/ts[2]/1e9:.2f} TF/s)  "
          f"K1h {ts[3]*1e3:8.1f} us ({fl/ts[3]/1e9:.2f} TF/s)  rel diff {d:.2e}", flush=True)
    eng.close()

op = solver.SchurOperator(sysm, centers, p3, radius=radius, device=0)
rng = np.random.default_rng(1)
L = 2 * p3 + 1
v = torch.as_tensor(rng.standard_normal((1, centers.shape[0], L)) + 0j).cuda()
for var in (2, 3):
    op.eng.set_k1_variant(var)
    t = timed(lambda: op(v), 50)
    print(f"cfg3 Schur step variant {var}: {t*1e3:.1f} us", flush=True)

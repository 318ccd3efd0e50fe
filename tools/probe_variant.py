"""K1 (tiled) vs K1s (symmetric) apply_T time against M, cfg3 geometry prefix,
one RHS -- sets the auto-dispatch crossover in m2l.cu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import grating
from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402

sysm, centers, p, radius = workloads.load_config(3)
L = 2 * p + 1
for M in (64, 100, 150, 200, 300, 400, 500, 700, 1000):
    eng = Engine(0)
    eng.set_geometry(centers[:M], p, 12.0, 1.0, 1)
    eng.set_bloch(np.array([1.0 + 0j]))
    rng = np.random.default_rng(0)
    v = torch.as_tensor(rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L))).cuda()
    out = torch.empty_like(v)
    ts = []
    for var in (1, 2):
        eng.set_k1_variant(var)
        eng.apply_T(v, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            eng.apply_T(v, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n)
    print(f"M={M:5d}  tiled {ts[0]*1e3:8.1f} us  sym {ts[1]*1e3:8.1f} us  sym/tiled {ts[1]/ts[0]:.3f}",
          flush=True)
    eng.close()

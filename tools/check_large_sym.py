"""K1s vs tiled K1 vs oracle slice at cfg5 scale (M = 10^4, p = 20, 1 RHS)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch

import periscat_oracle as O
from paper_1412_7466_b200.engine import Engine

centers = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "centers_cfg5.npy"))
M, p = centers.shape[0], 20
L = 2 * p + 1
bloch = np.exp(1j * 10.0 * math.cos(-math.pi / 3 - math.pi / 2))
rng = np.random.default_rng(5)
beta = rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L))
eng = Engine(0)
eng.set_geometry(centers, p, 12.0, 1.0, 1)
eng.set_bloch(np.array([bloch]))
v = torch.as_tensor(beta).cuda()
outs = {}
for var in (2, 1):
    eng.set_k1_variant(var)
    eng.apply_T(v)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = eng.apply_T(v)
    torch.cuda.synchronize()
    outs[var] = o[0].cpu().numpy()
    tr = M * (3 * M - 1)
    dt = time.perf_counter() - t0
    print(f"variant {var}: {dt*1e3:.1f} ms  {tr/dt:.3e} tr/s  {tr*8*L*L/dt/1e12:.2f} TF/s", flush=True)
d = np.linalg.norm(outs[1] - outs[2]) / np.linalg.norm(outs[1])
print(f"K1s vs K1 rel diff {d:.3e}", flush=True)
sl = np.r_[0:4, 5000:5004, 9996:10000]
t0 = time.perf_counter()
ref = O.apply_T(beta[0], centers, 12.0, p, bloch, targets=sl)
e = np.linalg.norm(outs[2][sl] - ref) / np.linalg.norm(ref)
print(f"K1s vs oracle slice ({len(sl)} targets) rel err {e:.3e}  ({time.perf_counter()-t0:.1f} s)", flush=True)

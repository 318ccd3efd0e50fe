"""A/B of the multi-RHS kernels on cfg5 geometry: variant 1 (DFMA K1m) vs 2 (DMMA K1d)."""
import ctypes
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import _lib
from paper_1412_7466_b200.engine import Engine

lib = _lib.load()
tf, ms, tt = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
lib.ps_dfma_peak(0, ctypes.byref(tf), ctypes.byref(ms))
lib.ps_dmma_peak(0, ctypes.byref(tt))
centers = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "centers_cfg5.npy"))
M = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
R = 16
centers = centers[:M]
p = int(sys.argv[2]) if len(sys.argv) > 2 else 20
L = 2 * p + 1
th = np.linspace(-math.pi / 3, math.pi / 3, 16)[:R] - math.pi / 2
rng = np.random.default_rng(0)
v = torch.as_tensor(rng.standard_normal((R, M, L)) + 1j * rng.standard_normal((R, M, L))).cuda()
outs = {}
for variant in (1, 2):
    eng = Engine(0)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(np.exp(1j * 10.0 * np.cos(th)))
    eng.set_mrhs_variant(variant)
    out = torch.empty_like(v)
    eng.apply_T(v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record()
    for _ in range(n):
        eng.apply_T(v, out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / n * 1e-3
    fl = M * (3 * M - 1) * R * 8 * L * L
    outs[variant] = out.cpu().numpy()
    print(f"variant {variant}: M={M} p={p} {t*1e3:.1f} ms  {fl/t/1e12:.2f} TF/s  "
          f"({fl/t/1e12/tf.value*100:.1f}% of DFMA {tf.value:.1f}, "
          f"{fl/t/1e12/tt.value*100:.1f}% of DMMA {tt.value:.1f})", flush=True)
d = np.linalg.norm(outs[1] - outs[2]) / np.linalg.norm(outs[1])
print("rel diff DFMA vs DMMA:", d)

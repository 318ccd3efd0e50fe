"""Device timing of the cfg5 multi-RHS apply_T (M=1e4, p=20, 16 RHS)."""
import ctypes
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import _lib, multiscat
from paper_1412_7466_b200.engine import Engine

lib = _lib.load()
tf, ms = ctypes.c_double(), ctypes.c_double()
lib.ps_dfma_peak(0, ctypes.byref(tf), ctypes.byref(ms))
centers = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "centers_cfg5.npy"))
M = int(sys.argv[1]) if len(sys.argv) > 1 else centers.shape[0]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
centers = centers[:M]
p, L = 20, 41
th = np.linspace(-math.pi / 3, math.pi / 3, 16)[:R] - math.pi / 2
bloch = np.exp(1j * 10.0 * np.cos(th))
eng = Engine(0)
eng.set_geometry(centers, p, 12.0, 1.0, 1)
eng.set_bloch(bloch)
rng = np.random.default_rng(0)
v = torch.as_tensor(rng.standard_normal((R, M, L)) + 1j * rng.standard_normal((R, M, L))).cuda()
out = torch.empty_like(v)
eng.apply_T(v, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 2
e0.record()
for _ in range(n):
    eng.apply_T(v, out)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / n * 1e-3
tr = M * (3 * M - 1) * R
fl = tr * 8 * L * L
print(f"cfg5 M={M} R={R} apply_T: {t*1e3:.1f} ms  {tr/t:.3e} tr/s  {fl/t/1e12:.2f} TFLOP/s "
      f"({fl/t/1e12/tf.value*100:.1f}% of DFMA peak {tf.value:.2f})", flush=True)

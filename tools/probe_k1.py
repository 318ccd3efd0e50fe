"""Quick device timing of K1 / the Schur matvec on cfg3 (development probe)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import _lib, grating, solver
from paper_1412_7466_b200.scatmat import disk_scattering_matrix
import workloads  # noqa: E402

lib = _lib.load()
tf, ms = ctypes.c_double(), ctypes.c_double()
rc = lib.ps_dfma_peak(0, ctypes.byref(tf), ctypes.byref(ms))
print(f"dfma peak rc={rc} {tf.value:.2f} TFLOP/s ({ms.value:.2f} ms)", flush=True)
for cfg in (3, 2):
    sysm, centers, p, radius = workloads.load_config(cfg)
    op = solver.SchurOperator(sysm, centers, p, radius=radius)
    M, L = op.M, op.L
    rng = np.random.default_rng(0)
    v = torch.as_tensor(rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L))).cuda()
    out = torch.empty_like(v)
    def tiled():
        op.eng.set_k1_variant(1)
        op.apply_T(v, out)
        op.eng.set_k1_variant(0)
    for name, fn in (("apply_T", lambda: op.apply_T(v, out)), ("schur", lambda: op(v, out)),
                     ("apply_T_tiled", tiled)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / n * 1e-3
        tr = M * (3 * M - 1)
        fl = tr * 8 * L * L
        print(f"cfg{cfg} {name}: {t*1e3:.3f} ms  {tr/t:.3e} tr/s  {fl/t/1e12:.2f} TFLOP/s "
              f"({fl/t/1e12/tf.value*100:.1f}% of DFMA peak)", flush=True)
    for X in (-1, 0, 2, 4, 6, 8):
        op.eng.set_overlap(X)
        for _ in range(3):
            op(v, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            op(v, out)
        e1.record()
        torch.cuda.synchronize()
        print(f"cfg{cfg} schur overlap_sms={X}: {e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
    op.eng.set_overlap(8)
    t0 = time.perf_counter()
    sol = solver.solve_full(sysm, centers, p, radius=radius)
    print(f"cfg{cfg} full solve {time.perf_counter()-t0:.3f}s iters={sol.iterations} "
          f"flux={sol.flux[0]['error']:.3e} timings={sol.timings}", flush=True)

"""Field-grid evaluation on cfg3: device M2P throughput for
the particle phased multipole sums, and the oracle's NumPy sum on a sample of
the same points (CPU reference)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch

import periscat_oracle as O
from paper_1412_7466_b200 import grating, postproc, solver
import workloads  # noqa: E402

sysm, centers, p, radius = workloads.load_config(3)
sol = solver.solve_full(sysm, centers, p, radius=radius)
op = solver.SchurOperator(sysm, centers, p, radius=radius)
beta = sol.beta
M, L = centers.shape[0], 2 * p + 1
for n in (128, 256, 512):
    postproc.eval_total_field_grid(op, beta, centers, radius, nx=n, ny=n, y_plot=0.7)   # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = postproc.eval_total_field_grid(op, beta, centers, radius, nx=n, ny=n, y_plot=0.7)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    t = time.perf_counter()
    postproc.eval_total_field_grid(op, beta, centers, radius, nx=n, ny=n, y_plot=0.7,
                                   layer_field=None)
    dpo = time.perf_counter() - t
    npts = int((~res["mask"] & (res["layer"] == 2)).sum())
    pts = np.column_stack([np.repeat(res["y"], n) * 0, np.repeat(res["y"], n)])
    xx, yy = np.meshgrid(res["x"], res["y"])
    P2 = np.column_stack([xx.ravel(), yy.ravel()])[(~res["mask"] & (res["layer"] == 2)).ravel()]
    torch.cuda.synchronize()
    t = time.perf_counter()
    u = postproc.particle_field(op, beta, P2)
    dk = time.perf_counter() - t
    pairs = npts * M * 3
    print(f"grid {n}x{n}: {npts} layer-2 points, eval_total_field_grid (layer fields + "
          f"particles, all on the device) {dt*1e3:.1f} ms (particles only {dpo*1e3:.1f} ms), "
          f"particle_field {dk*1e3:.1f} ms = {pairs/dk:.3e} point-source pairs/s", flush=True)
sl = P2[:: max(1, P2.shape[0] // 200)][:200]
t = time.perf_counter()
ref = sum((sysm.config.bloch_phase ** l) * O._particle_field(12.0, beta[0], centers, sl, float(l))[0]
          for l in (-1, 0, 1))
dc = time.perf_counter() - t
got = postproc.particle_field(op, beta, sl)[0]
print(f"oracle (NumPy, 1 process) on {sl.shape[0]} points: {dc:.2f} s = "
      f"{sl.shape[0]*M*3/dc:.3e} pairs/s; max rel diff {np.abs(got-ref).max()/np.abs(ref).max():.2e}",
      flush=True)

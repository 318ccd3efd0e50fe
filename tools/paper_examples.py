"""Paper §6 examples on the device (tests/test_gpu_examples.py setup), with
timings: one JSON object per example (device iterations / flux / coupled
residual / seconds next to the oracle's and the paper's numbers)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

from test_gpu_examples import GOLDEN, _config, _solve  # noqa: E402

z = np.load(os.path.join(GOLDEN, "examples.npz"))
meta = json.load(open(os.path.join(GOLDEN, "examples.json")))
out = {}
for name in ("ex1", "ex2", "ex3k1", "ex3k10", "ex1m500"):
    _solve(z, name)                       # warm (module loads, BIE)
    torch.cuda.synchronize()
    t = time.perf_counter()
    S, sol = _solve(z, name)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    cfg = _config(z, name)
    out[name] = dict(M=int(z[f"{name}_centers"].shape[0]), device_iterations=sol.iterations[0],
                     device_flux_error=sol.flux[0]["error"],
                     device_coupled_residual=sol.coupled_residual[0],
                     device_wall_residual=sol.wall_residual[0],
                     device_seconds_incl_bie_S=dt,
                     oracle_iterations=meta[name]["iterations"],
                     oracle_flux_error=meta[name]["flux_error"], paper=meta[name]["paper"],
                     k=(cfg.k1, cfg.k2, cfg.k3), kp=cfg.kp, theta=cfg.incident_angle)
    print(name, out[name], flush=True)
print(json.dumps(out, indent=1))

"""Time the device empty-grating setup (assembly + SVD) and solve_full from a config."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1412_7466_b200 import grating, solver
from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402

out = {}
for workers in (1, 2, 4, 8):
    cfgs = [workloads.fixture_config(n) for n in workloads.CFG5_ANGLES]
    eng = Engine(0)
    eng.set_geometry(np.array([[0.0, 0.0]]), 2, cfgs[0].k2)
    eng.set_bloch([c.bloch_phase for c in cfgs])
    for it in range(2):
        t = time.perf_counter(); eng.setup_empty(cfgs, svd_workers=workers); dt = time.perf_counter() - t
    out[f"cfg5_16angles_workers{workers}"] = dict(wall_s=dt, device_ms=eng.setup_timings())
    eng.close()
cfg = workloads.fixture_config("w10")
eng = Engine(0); eng.set_geometry(np.array([[0.0, 0.0]]), 2, cfg.k2); eng.set_bloch([cfg.bloch_phase])
for it in range(3):
    t = time.perf_counter(); eng.setup_empty([cfg]); dt = time.perf_counter() - t
out["single_angle"] = dict(wall_s=dt, device_ms=eng.setup_timings())
eng.close()
sysm, centers, p, radius = workloads.load_config(3)
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    sol = solver.solve_full(cfg, centers, p, radius=radius, device=0)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
out["cfg3_solve_full_from_config"] = dict(seconds=dt, timings=sol.timings, iterations=sol.iterations,
                                          flux=sol.flux[0]["error"])
print(json.dumps(out, indent=1))


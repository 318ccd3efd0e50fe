"""Wall-clock breakdown of solve_full on cfg3 (setup pieces, GMRES, recovery)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import grating, postproc, solver
from paper_1412_7466_b200.engine import Engine
from paper_1412_7466_b200.scatmat import disk_scattering_matrix
import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sysm, centers, p, radius = workloads.load_config(cfg)
for rep in range(3):
    T = {}
    t = time.perf_counter()

    def lap(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[name] = round((now - t) * 1e3, 2)
        t = now

    sol = solver.solve_full(sysm, centers, p, radius=radius)
    lap("solve_full total")
    c = sysm.config
    S = disk_scattering_matrix(radius, c.k2, c.kp, p)
    lap("disk S")
    eng = Engine(0)
    lap("Engine()")
    eng.set_geometry(np.ascontiguousarray(centers), p, c.k2, c.period, c.near_field_copies)
    eng.set_bloch([c.bloch_phase])
    eng.set_smatrix(S, None)
    lap("geometry+bloch+S")
    eng.set_layers(sysm)
    lap("set_layers")
    eng.set_pinv(0, sysm)
    lap("set_pinv")
    eng.precompute_coupling(40.0)
    lap("precompute_coupling")
    rhs = eng.schur_rhs()
    lap("schur_rhs")
    x, its, hist = eng.gmres(rhs, 1e-10, 150)
    lap(f"gmres ({its[0]} it)")
    g = eng.apply_C(x)
    xe = eng.recover(g)
    lap("recover")
    print(rep, T, "solve_full timings", {k: round(v * 1e3, 2) for k, v in sol.timings.items()},
          flush=True)
    eng.close()

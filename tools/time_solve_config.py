"""Wall clock of solve_full(config) on cfg3, repeated (the bench's
full_solve_m1000 block), with the K1s symbol store on and off."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1412_7466_b200 import solver
from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402

sysm, centers, p, radius = workloads.load_config(3)
conf = sysm.config
orig = Engine.__init__
for gb in [float(a) for a in sys.argv[1:]] or [32.0, 0.0]:
    def init(self, *a, _gb=gb, **k):
        orig(self, *a, **k)
        self.set_symbol_store(_gb)
    Engine.__init__ = init
    for rep in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        sol = solver.solve_full(conf, centers, p, radius=radius, diagnostics=False)
        torch.cuda.synchronize()
        print(f"store {gb:5.1f} GB  rep {rep}: {time.perf_counter() - t:.4f} s, "
              f"iterations {sol.iterations}, timings " + ", ".join(f"{k}={v*1e3 if k in ("setup", "solve", "diagnostics") else v:.1f}" for k, v in sol.timings.items()), flush=True)
Engine.__init__ = orig

import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1412_7466_b200 import solver
import workloads
sysm, centers, p, radius = workloads.load_config(3)
for rep in range(3):
    t = time.perf_counter()
    op = solver.SchurOperator(sysm, centers, p, radius=radius)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    v = torch.ones((1, op.M, op.L), dtype=torch.complex128, device="cuda")
    ts = []
    for k in range(4):
        torch.cuda.synchronize(); a = time.perf_counter()
        op(v)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - a) * 1e3)
    print(f"rep {rep}: construct {1e3*(t1-t):.1f} ms, matvecs (ms) " + " ".join(f"{x:.2f}" for x in ts),
          "store bytes", op.eng.set_symbol_store(-1), flush=True)
    del op
    torch.cuda.synchronize()

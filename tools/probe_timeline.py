"""Timeline of the SM-partitioned cfg3 Schur step (profile events inside the
library): K1s end, coupling-chain end, step end, per overlap SM count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import grating, solver
import workloads  # noqa: E402

sysm, centers, p, radius = workloads.load_config(3)
op = solver.SchurOperator(sysm, centers, p, radius=radius)
rng = np.random.default_rng(0)
v = torch.as_tensor(op.smat[None, None, :] * (rng.standard_normal((1, op.M, op.L))
                    + 1j * rng.standard_normal((1, op.M, op.L)))).cuda()
y = torch.empty_like(v)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for arg in (sys.argv[1:] or ["2"]):
    sms = int(arg.rstrip("k"))
    op.eng.set_overlap(sms)
    op.eng.set_overlap_order(arg.endswith("k"))
    for _ in range(3):
        op(v, out=y)
    op.eng.profile(True)
    op.eng.stats_reset()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op(v, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    tl = op.eng.timeline()
    st = op.eng.stats()
    op.eng.profile(False)
    print(f"overlap_sms={arg}: step {np.mean(ts):.3f} ms (event), timeline {tl}, "
          f"K1s kernel {st['k1_ms'] / max(st['k1_count'], 1):.3f} ms", flush=True)

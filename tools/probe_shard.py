"""Per-rank compute of the target-sharded matvec, measured on one GPU.

For world sizes G = 1, 2, 4, 8 this times, for every rank's target shard,
the device work one rank does per Schur matvec (K1 over all sources for the
owned targets, plus the coupling partials), so the compute side of the
multi-GPU scaling can be read off a single B200: predicted speed-up at G =
t(G=1) / max_r t_r(G).  The collectives (all-gather of beta, all-reduce of
the 576-row partial) are timed separately by the NCCL runs.

    python tools/probe_shard.py [cfg3|cfg5] [nrhs]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200 import grating, solver
from paper_1412_7466_b200.engine import Engine
from paper_1412_7466_b200.parallel import shard_range
import workloads  # noqa: E402


def timed(fn, n):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3


def cfg3():
    sysm, centers, p, radius = workloads.load_config(3)
    M, L = centers.shape[0], 2 * p + 1
    rng = np.random.default_rng(0)
    v = torch.as_tensor(rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L))).cuda()
    base = None
    for G in (1, 2, 4, 8):
        ts = []
        for r in range(G):
            t0, t1 = shard_range(M, r, G)
            op = solver.SchurOperator(sysm, centers, p, radius=radius, target_range=(t0, t1))
            out = torch.empty((1, t1 - t0, L), dtype=torch.complex128, device="cuda")
            if G == 1:
                fn = lambda: op(v, out)
            else:
                def fn():
                    g = op.eng.apply_C(v, s_range=(t0, t1))
                    op(v, out=out, g=g)
            ts.append(timed(fn, 20))
            del op
        base = base or ts[0]
        tr = M * (3 * M - 1)
        if G > 1:   # "pairs" decomposition: K1s over 1/G of the tile pairs + epilogue
            tp = []
            for r in range(G):
                t0, t1 = shard_range(M, r, G)
                op = solver.SchurOperator(sysm, centers, p, radius=radius, target_range=(t0, t1))
                a_full = torch.empty((1, M, L), dtype=torch.complex128, device="cuda")
                y = torch.empty((1, t1 - t0, L), dtype=torch.complex128, device="cuda")
                vo = v[:, t0:t1].contiguous()

                def fp():
                    op.eng.apply_T_blocks(v, r, G, out=a_full)
                    g = op.eng.apply_C(v, s_range=(t0, t1))
                    op.eng.schur_finish(vo, a_full[:, t0:t1].contiguous(), g, out=y)
                tp.append(timed(fp, 20))
                del op
            print(f"cfg3 G={G} pairs: per-rank ms {['%.3f' % (t * 1e3) for t in tp]}  max "
                  f"{max(tp)*1e3:.3f}  predicted compute speed-up {base / max(tp):.2f}x", flush=True)
        print(f"cfg3 G={G}: per-rank ms {['%.3f' % (t * 1e3) for t in ts]}  max {max(ts)*1e3:.3f}  "
              f"predicted compute speed-up {base / max(ts):.2f}x  ({tr / max(ts):.3e} tr/s)",
              flush=True)


def cfg5(R):
    here = os.path.dirname(os.path.abspath(__file__))
    centers = np.load(os.path.join(here, "..", "tests", "golden", "centers_cfg5.npy"))
    M, p = centers.shape[0], 20
    L = 2 * p + 1
    th = np.linspace(-math.pi / 3, math.pi / 3, 16)[:R] - math.pi / 2
    bloch = np.exp(1j * 10.0 * np.cos(th))
    rng = np.random.default_rng(0)
    v = torch.as_tensor(rng.standard_normal((R, M, L)) + 1j * rng.standard_normal((R, M, L))).cuda()
    eng = Engine(0)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(bloch)
    base = None
    for G in (1, 2, 4, 8):
        ts = []
        for r in ((0, G - 1) if G > 1 else (0,)):
            t0, t1 = shard_range(M, r, G)
            eng.set_target_range(t0, t1)
            out = torch.empty((R, t1 - t0, L), dtype=torch.complex128, device="cuda")
            ts.append(timed(lambda: eng.apply_T(v, out), 1))
        base = base or ts[0]
        tr = M * (3 * M - 1) * R
        print(f"cfg5 R={R} G={G}: shard ms (first, last) {['%.1f' % (t * 1e3) for t in ts]}  "
              f"predicted compute speed-up {base / max(ts):.2f}x  ({tr / max(ts):.3e} tr/s)",
              flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    if which == "cfg3":
        cfg3()
    else:
        cfg5(int(sys.argv[2]) if len(sys.argv) > 2 else 16)

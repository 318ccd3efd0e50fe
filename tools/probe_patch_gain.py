"""apply_T time of each DFMA M2L kernel family with the library in use
(PS_LIB selects a build; compare the reuse-patched and PS_NO_SASS_PATCH=1
builds): K1s and tiled K1 at cfg3 (p = 25), K1s / K1 at cfg2-size p = 20,
K1m with 4 RHS."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402


def t_apply(eng, v, out, n=20):
    eng.apply_T(v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        eng.apply_T(v, out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for cfg, nrhs, variants in ((3, 1, (1, 2)), (3, 4, (0,)), (2, 1, (1, 2))):
    sysm, centers, p, radius = workloads.load_config(cfg)
    M, L = centers.shape[0], 2 * p + 1
    eng = Engine(0)
    eng.set_geometry(centers, p, sysm.config.k2, sysm.config.period, 1)
    eng.set_bloch(np.full(nrhs, sysm.config.bloch_phase))
    rng = np.random.default_rng(0)
    v = torch.as_tensor(rng.standard_normal((nrhs, M, L)) + 1j * rng.standard_normal((nrhs, M, L))).cuda()
    out = torch.empty_like(v)
    for var in variants:
        eng.set_k1_variant(var)
        name = {0: "auto" if nrhs > 1 else "auto", 1: "tiled K1", 2: "K1s"}[var]
        print(f"cfg{cfg} M={M} p={p} nrhs={nrhs} {name:12s} {t_apply(eng, v, out) * 1e3:9.1f} us", flush=True)
        if var == 2:
            eng.set_symbol_store(0.0)
            print(f"cfg{cfg} M={M} p={p} nrhs={nrhs} K1s no store {t_apply(eng, v, out) * 1e3:9.1f} us", flush=True)
            eng.set_symbol_store(32.0)
    eng.close()

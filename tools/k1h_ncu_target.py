"""One cfg3-geometry apply_T at p=25 with a forced K1 variant (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1412_7466_b200.engine import Engine
import workloads  # noqa: E402

var = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = int(sys.argv[2]) if len(sys.argv) > 2 else 25
sysm, centers, _, _ = workloads.load_config(3)
L = 2 * p + 1
M = centers.shape[0]
eng = Engine(0)
eng.set_geometry(centers, p, 12.0, 1.0, 1)
eng.set_bloch(np.array([np.exp(-0.7j)]))
eng.set_k1_variant(var)
rng = np.random.default_rng(0)
v = torch.as_tensor(rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L))).cuda()
out = torch.empty_like(v)
for _ in range(2):
    eng.apply_T(v, out)
torch.cuda.synchronize()
print("done")

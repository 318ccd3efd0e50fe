"""K1d multi-RHS timing at M=1000 (cfg3 centres), 16 RHS, order p (argv)."""
import sys, os, math, numpy as np, torch
sys.path.insert(0,'/root/repo')
from paper_1412_7466_b200.engine import Engine
from paper_1412_7466_b200 import grating
import workloads  # noqa: E402
_, centers, p, _ = workloads.load_config(3)
p = int(sys.argv[1]) if len(sys.argv) > 1 else p
M=centers.shape[0]; L=2*p+1; R=16
eng=Engine(0); eng.set_geometry(centers,p,12.0,1.0,1); eng.set_bloch(np.exp(1j*np.linspace(0,2,R)))
rng=np.random.default_rng(0); v=torch.as_tensor(rng.standard_normal((R,M,L))+1j*rng.standard_normal((R,M,L))).cuda()
out=torch.empty_like(v); eng.apply_T(v,out); torch.cuda.synchronize()
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(3): eng.apply_T(v,out)
e1.record(); torch.cuda.synchronize(); t=e0.elapsed_time(e1)/3
print(f"p={p} M=1000 R=16 apply_T {t:.2f} ms  {M*(3*M-1)*R*8*L*L/t/1e9:.2f} TF/s")

"""Probe: cuSOLVER SVD drivers (through torch) on the 856x781 empty-grating matrix."""
import time, numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_7466_b200 import grating
import workloads  # noqa: E402
s = workloads.load_fixture("w10")
A = torch.as_tensor(s.matrix).cuda()
u0, s0, vh0 = np.linalg.svd(s.matrix, full_matrices=False)
g = s.rhs
inv0 = np.minimum(1/s0, 1/1e-10)
x0 = s.col_scale * (vh0.conj().T @ (inv0 * (u0.conj().T @ g)))
c = s.cols["c"]; d = s.cols["d"]
for drv in ("gesvd", "gesvdj", "gesvda"):
    for it in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        try:
            U, S, Vh = torch.linalg.svd(A, full_matrices=False, driver=drv)
        except Exception as e:
            print(drv, "fail", e); break
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    U, S, Vh = U.cpu().numpy(), S.cpu().numpy(), Vh.cpu().numpy()
    inv = np.minimum(1/S, 1/1e-10)
    x = s.col_scale * (Vh.conj().T @ (inv * (U.conj().T @ g)))
    print(drv, f"{dt*1e3:.1f} ms", "sv rel", np.max(np.abs(S-s0))/s0[0],
          "c", np.linalg.norm(x[c]-x0[c])/np.linalg.norm(x0[c]), "d", np.linalg.norm(x[d]-x0[d])/np.linalg.norm(x0[d]),
          "resid", np.linalg.norm(s.matrix @ (x/s.col_scale) - g)/np.linalg.norm(g), flush=True)
t = time.perf_counter(); np.linalg.svd(s.matrix, full_matrices=False); print("numpy", time.perf_counter()-t, os.cpu_count())

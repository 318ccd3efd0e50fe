"""Host half of the probe: SVD of the real bidiagonal from zgebrd (numpy gesdd)."""
import sys, time, os, numpy as np
raw = np.fromfile(sys.argv[1])
n = (raw.size + 1) // 2
d, e = raw[:n], raw[n:]
B = np.diag(d) + np.diag(e, 1)
for threads in (1, len(os.sched_getaffinity(0))):
    pass
for it in range(3):
    t = time.perf_counter(); U, s, Vt = np.linalg.svd(B); dt = time.perf_counter() - t
print(f"numpy svd of the {n}x{n} bidiagonal: {dt*1e3:.1f} ms, s_max {s[0]:.3g} s_min {s[-1]:.3g}, cores {len(os.sched_getaffinity(0))}")

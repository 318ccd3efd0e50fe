"""Generate the empty-grating system fixtures with the REFERENCE's own assembly.

Test infrastructure (build container only; /root/reference must exist).
The 856x781 block matrix A (column-rescaled), its right-hand side f and the
column scaling come from ``periscat.empty_grating.assemble_empty_system``
(/root/reference/pkg/src/periscat/empty_grating.py:139-256); the interface /
wall node geometry the coupling blocks B and C need comes from the same
``curves`` dict (eg:113-119).  A is stored, not its SVD: the SVD
(eg:259-261) is recomputed by numpy on whichever host loads the fixture, so
the oracle and the CUDA path always share the same factors bit for bit.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_empty.py w10 wood
"""
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from periscat.empty_grating import assemble_empty_system  # noqa: E402
from periscat.geometry import InterfaceSpec, ProblemConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

WOOD_OMEGA = 2.0 * math.pi / (1.0 + math.sin(math.pi / 5.0))

# physics name -> (omega, theta_ref)
PHYS = {
    "w10": (10.0, -0.7 * math.pi),          # cfg1-3 (theta_B = -pi/5)
    "wood": (WOOD_OMEGA, -0.7 * math.pi),   # cfg4
}


def config_for(omega: float, theta_ref: float) -> ProblemConfig:
    return ProblemConfig(period=1.0, k1=omega, k2=1.2 * omega, k3=omega, kp=1.5 * omega,
                         incident_angle=theta_ref,
                         interface_top=InterfaceSpec(0.5),
                         interface_bottom=InterfaceSpec(-0.5))


# cfg5: omega = 10, 16 angles theta_B = linspace(-pi/3, pi/3, 16), theta_ref = theta_B - pi/2
CFG5_THETA_B = [(-math.pi / 3) + i * (2 * math.pi / 3) / 15 for i in range(16)]


def phys(name: str):
    if name.startswith("w10_a"):
        return 10.0, CFG5_THETA_B[int(name[5:])] - 0.5 * math.pi
    return PHYS[name]


def make(name: str, omega=None, theta=None) -> str:
    if omega is None:
        omega, theta = phys(name)
    conf = config_for(omega, theta)
    t0 = time.perf_counter()
    sysm = assemble_empty_system(conf)
    dt = time.perf_counter() - t0
    cv = sysm.curves
    cols = np.array([[s.start, s.stop] for s in sysm.cols.values()])
    rows = np.array([[s.start, s.stop] for s in sysm.rows.values()])
    path = os.path.join(OUT, f"empty_{name}.npz")
    np.savez_compressed(
        path,
        A=sysm.matrix, f=sysm.rhs, col_scale=sysm.col_scale,
        col_names=np.array(list(sysm.cols.keys())), cols=cols,
        row_names=np.array(list(sysm.rows.keys())), rows=rows,
        g1_nodes=cv["g1"].nodes, g1_normals=cv["g1"].normals, g1_w=cv["g1"].arc_weights,
        g2_nodes=cv["g2"].nodes, g2_normals=cv["g2"].normals, g2_w=cv["g2"].arc_weights,
        L2_nodes=cv["L2"].nodes,
        center2=sysm.centers[2],
        scalars=np.array([conf.period, conf.k1, conf.k2, conf.k3, conf.kp,
                          conf.incident_angle, conf.near_field_copies,
                          conf.j_expansion_order, conf.regularization, conf.y0]),
        assembly_seconds=dt)
    return path


if __name__ == "__main__":
    for n in sys.argv[1:]:
        p = make(n)
        print(n, p, os.path.getsize(p), flush=True)

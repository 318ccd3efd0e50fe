"""Reference-side setup helper of the solver shim (CPU, needs /root/reference):
per-angle empty-grating assembly + SVD in a thread pool equals the serial
reference assembly."""
import math
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


def test_assemble_systems_parallel_matches_serial():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from periscat.empty_grating import assemble_empty_system
    from periscat.geometry import InterfaceSpec, ProblemConfig

    from integration.periscat_shim import solver as shim
    cfgs = [ProblemConfig(period=1.0, k1=10.0, k2=12.0, k3=10.0, kp=15.0, incident_angle=th,
                          interface_top=InterfaceSpec(0.5), interface_bottom=InterfaceSpec(-0.5))
            for th in (-0.7 * math.pi, -0.6 * math.pi)]
    par = shim.assemble_systems(cfgs, threads=2)
    for c, s in zip(cfgs, par):
        ref = assemble_empty_system(c)
        assert np.array_equal(s.matrix, ref.matrix)
        assert np.array_equal(s.rhs, ref.rhs)
        assert s.svd is not None and s.svd[1].shape[0] == ref.matrix.shape[1]

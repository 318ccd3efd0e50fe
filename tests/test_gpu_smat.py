"""Device Mueller-BIE scattering matrices (ps_scattering_matrix) against the
goldens built from the reference's own Nystrom primitives
(oracle/make_smat.py), and the coupled solve with rotated star particles
(dense S with rotation phases in the Schur epilogue) against the oracle."""
import os

import numpy as np
import pytest

from conftest import rel
import workloads  # noqa: E402

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SMAT_TOL = 1e-11      # max |S_dev - S_ref| / max |S_ref| (device Bessel vs AMOS)


def _device_smat(name):
    from paper_1412_7466_b200 import scatmat
    z = np.load(os.path.join(GOLDEN, "smat_shapes.npz"))
    a1, a2, a3, k2, kp, p, n = z[name + "_params"]
    sm = scatmat.scattering_matrix(scatmat.ParticleShape(a1, a2, int(a3)), k2, kp, int(p),
                                   N=int(n), device=0)
    return sm, z[name]


@pytest.mark.parametrize("name", ["disk_w10", "par1", "star3_w10", "pent_w10"])
def test_scattering_matrix_matches_golden(name):
    sm, ref = _device_smat(name)
    assert sm.s.shape == ref.shape
    err = np.max(np.abs(sm.s - ref)) / np.max(np.abs(ref))
    assert err <= SMAT_TOL, f"{name}: {err:.2e}"
    assert sm.residual <= 1e-12


def test_disk_scattering_matrix_is_analytic_diagonal():
    from paper_1412_7466_b200.scatmat import disk_scattering_matrix
    sm, _ = _device_smat("disk_w10")
    ana = disk_scattering_matrix(0.04, 12.0, 15.0, 20)
    assert np.max(np.abs(sm.s - np.diag(ana))) <= 1e-12 * np.max(np.abs(ana))


def test_no_contrast_gives_zero():
    from paper_1412_7466_b200 import scatmat
    sm = scatmat.scattering_matrix(scatmat.ParticleShape(0.03, 0.01, 3), 12.0, 12.0, 10, device=0)
    assert np.max(np.abs(sm.s)) <= 1e-12


def test_bad_shape_rejected():
    from paper_1412_7466_b200 import scatmat
    with pytest.raises(ValueError):
        scatmat.scattering_matrix(scatmat.ParticleShape(0.03, 0.04, 3), 12.0, 15.0, 10, device=0)


def _star_problem():
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating
    z = np.load(os.path.join(GOLDEN, "golden_star.npz"))
    pb = O.load_problem(1)
    sm, _ = _device_smat("star3_w10")
    return z, pb, sm, workloads.load_fixture("w10")


def test_schur_with_rotated_stars_matches_oracle():
    import torch

    from paper_1412_7466_b200 import solver
    z, pb, sm, sysm = _star_problem()
    op = solver.SchurOperator(sysm, pb.centers, pb.p, smat=sm, rot=z["rot"], device=0)
    got = op(torch.as_tensor(z["v"][None]).cuda()).cpu().numpy()[0]
    assert rel(got, z["schur"]) <= 1e-10


@pytest.mark.parametrize("from_config", [False, True])
def test_solve_full_with_rotated_stars_matches_oracle(from_config):
    """The paper's star-particle case end to end: device BIE scattering matrix,
    rotation phases per inclusion, (device-assembled) empty grating, GMRES."""
    from paper_1412_7466_b200 import grating, solver
    z, pb, sm, sysm = _star_problem()
    systems = workloads.fixture_config("w10") if from_config else sysm
    sol = solver.solve_full(systems, pb.centers, pb.p, smat=sm, rot=z["rot"], device=0)
    assert rel(sol.c[0], z["c"]) <= 1e-9 and rel(sol.d[0], z["d"]) <= 1e-9
    assert abs(sol.flux[0]["error"] - float(z["flux_error"])) <= 1e-9
    assert abs(sol.iterations[0] - int(z["iterations"])) <= 1

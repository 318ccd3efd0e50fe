"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): matvec relative error <= 1e-10
(normwise, per RHS); Bragg coefficients c, d relative <= 1e-9; flux-balance
error |delta| <= 1e-9 absolute.
"""
import numpy as np
import pytest

from conftest import rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-10


@pytest.fixture(scope="module")
def O():
    from oracle import periscat_oracle
    return periscat_oracle


def _cplx(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=complex)).cuda()


@pytest.mark.parametrize("cfg", [1, 2])
def test_apply_T_matches_oracle(O, cfg):
    from paper_1412_7466_b200 import multiscat
    pb = O.load_problem(cfg)
    rng = np.random.default_rng(10 + cfg)
    for beta in (_cplx(rng, (pb.M, pb.L)), pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))):
        ref = O.apply_T(beta, pb.centers, pb.es.k2, pb.p, pb.es.bloch, pb.es.period, pb.es.copies)
        got = multiscat.apply_T(beta, pb.centers, pb.es.k2, pb.p, pb.es.bloch, pb.es.period,
                                pb.es.copies)
        assert rel(got, ref) <= MATVEC_TOL


def test_apply_T_cfg3_target_slice(O):
    """M=1000, p=25: all targets on the GPU, a 24-target slice on the oracle."""
    from paper_1412_7466_b200 import multiscat
    pb = O.load_problem(3)
    rng = np.random.default_rng(3)
    beta = pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))
    got = multiscat.apply_T(beta, pb.centers, pb.es.k2, pb.p, pb.es.bloch)
    sl = np.r_[0:8, 500:508, 992:1000]
    ref = O.apply_T(beta, pb.centers, pb.es.k2, pb.p, pb.es.bloch, targets=sl)
    assert rel(got[sl], ref) <= MATVEC_TOL


@pytest.mark.parametrize("p,copies,M", [(0, 0, 1), (0, 1, 1), (1, 1, 1), (3, 1, 2), (5, 0, 7),
                                        (10, 2, 13), (25, 1, 9)])
def test_apply_T_small_orders(O, p, copies, M):
    """SPEC.md:510-512 degeneracies and odd shapes (ragged tiles, many copies)."""
    from paper_1412_7466_b200 import multiscat
    rng = np.random.default_rng(p * 100 + M)
    centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    beta = _cplx(rng, (M, 2 * p + 1))
    bloch = np.exp(0.7j)
    ref = O.apply_T(beta, centers, 9.0, p, bloch, 1.0, copies)
    got = multiscat.apply_T(beta, centers, 9.0, p, bloch, 1.0, copies)
    if M == 1 and copies == 0:
        assert np.all(got == 0)
    else:
        assert rel(got, ref) <= MATVEC_TOL


def test_apply_T_multi_rhs(O):
    from paper_1412_7466_b200 import multiscat
    pb = O.load_problem(1)
    rng = np.random.default_rng(7)
    beta = _cplx(rng, (3, pb.M, pb.L))
    bl = np.exp(1j * np.array([0.1, -2.0, 1.3]))
    ref = O.apply_T(beta, pb.centers, pb.es.k2, pb.p, bl)
    got = multiscat.apply_T(beta, pb.centers, pb.es.k2, pb.p, bl)
    for r in range(3):
        assert rel(got[r], ref[r]) <= MATVEC_TOL


def test_domain_error_coincident():
    from paper_1412_7466_b200 import DomainError, multiscat
    c = np.array([[0.1, 0.2], [0.1, 0.2]])
    with pytest.raises(DomainError):
        multiscat.apply_T(np.ones((2, 3), complex), c, 5.0, 1)


def _operator(O, cfg, coupled=True):
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(cfg)
    sysm = grating.load_fixture(O.CONFIGS[cfg]["empty"])
    op = solver.SchurOperator(sysm, pb.centers, pb.p, smat=pb.smat, coupled=coupled)
    return pb, op


@pytest.mark.parametrize("cfg", [1, 2])
def test_apply_C_matches_oracle(O, cfg):
    pb, op = _operator(O, cfg)
    rng = np.random.default_rng(20 + cfg)
    beta = _cplx(rng, (pb.M, pb.L))
    ref = O.apply_C(pb.es, beta, pb.centers)[:576]
    got = op.eng.apply_C(_dev(beta[None])).cpu().numpy()[0]
    assert rel(got, ref) <= MATVEC_TOL


@pytest.mark.parametrize("cfg", [1, 2])
def test_schur_matches_oracle(O, cfg):
    pb, op = _operator(O, cfg)
    rng = np.random.default_rng(30 + cfg)
    for v in (_cplx(rng, (pb.M, pb.L)), pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))):
        ref = O.apply_schur_operator(pb, v).reshape(pb.M, pb.L)
        got = op(_dev(v[None])).cpu().numpy()[0]
        assert rel(got, ref) <= MATVEC_TOL


@pytest.mark.parametrize("cfg", [1, 2])
def test_schur_rhs_matches_oracle(O, cfg):
    pb, op = _operator(O, cfg)
    ref = O.schur_rhs(pb).reshape(pb.M, pb.L)
    got = op.rhs().cpu().numpy()[0]
    assert rel(got, ref) <= MATVEC_TOL


def test_schur_uncoupled_is_I_minus_ST(O):
    """B = C = 0 -> I - S T."""
    pb, op = _operator(O, 1, coupled=False)
    rng = np.random.default_rng(5)
    v = _cplx(rng, (pb.M, pb.L))
    ref = O.apply_schur_operator(pb, v, with_coupling=False).reshape(pb.M, pb.L)
    got = op(_dev(v[None])).cpu().numpy()[0]
    assert rel(got, ref) <= MATVEC_TOL


def test_solve_full_cfg1(O):
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(1)
    ref = O.solve_full(pb)
    sol = solver.solve_full(grating.load_fixture("w10"), pb.centers, pb.p, smat=pb.smat)
    assert rel(sol.c[0], ref.c) <= 1e-9
    assert rel(sol.d[0], ref.d) <= 1e-9
    assert abs(sol.flux[0]["error"] - ref.flux["error"]) <= 1e-9
    assert sol.flux[0]["error"] <= 1e-9
    assert abs(sol.iterations[0] - ref.iterations) <= 1

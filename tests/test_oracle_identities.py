"""Oracle self-checks from SPEC.md's examples / invariants (no reference and
no GPU needed): Graf re-summation (SP:460), apply_T degeneracies
(SP:510-512), Schur degeneracies (SP:545-547), GMRES properties (SP:555-557),
disk S oracle (SP:411), flux conservation (SP:599-607)."""
import numpy as np
import pytest
import scipy.special as sps

from conftest import rel


@pytest.fixture(scope="module")
def O():
    from oracle import periscat_oracle
    return periscat_oracle


def _local_eval(a, k, center, pts):
    p = (a.size - 1) // 2
    n = np.arange(-p, p + 1)
    d = pts - center
    r = np.hypot(d[:, 0], d[:, 1])
    th = np.arctan2(d[:, 1], d[:, 0])
    return (sps.jv(n[None, :], k * r[:, None]) * np.exp(1j * n[None, :] * th[:, None])) @ a


def _outgoing_eval(beta, k, center, pts):
    p = (beta.size - 1) // 2
    n = np.arange(-p, p + 1)
    d = pts - center
    r = np.hypot(d[:, 0], d[:, 1])
    th = np.arctan2(d[:, 1], d[:, 0])
    return (sps.hankel1(n[None, :], k * r[:, None]) * np.exp(1j * n[None, :] * th[:, None])) @ beta


def test_m2l_graf_resummation(O):
    """SP:460: outgoing expansion vs M2L + local re-summation on the target disk."""
    rng = np.random.default_rng(0)
    k, R = 10.0, 0.05
    cs, ct = np.array([0.0, 0.0]), np.array([0.17, 0.09])
    beta = np.zeros(2 * 10 + 1, complex)
    beta[8:13] = rng.standard_normal(5) + 1j * rng.standard_normal(5)   # |n| <= 2 source
    th = np.linspace(0, 2 * np.pi, 20, endpoint=False)
    pts = ct + 0.5 * R * np.column_stack([np.cos(th), np.sin(th)])
    a = O.m2l_translate(np.pad(beta, 20), cs, ct, k, 30)
    assert rel(_local_eval(a, k, ct, pts), _outgoing_eval(beta, k, cs, pts)) < 1e-11


def test_m2l_sign_convention_is_pinned(O):
    """Swapping the index sign (n'-n instead of n-n') must break the check."""
    k, cs, ct = 9.0, np.array([0.0, 0.0]), np.array([0.2, -0.1])
    beta = np.zeros(41, complex)
    beta[21] = 1.0
    a = O.m2l_translate(beta, cs, ct, k, 20)
    pts = ct + 0.01 * np.array([[1.0, 0.0], [0.0, 1.0], [-0.7, 0.7]])
    good = rel(_local_eval(a, k, ct, pts), _outgoing_eval(beta, k, cs, pts))
    bad = rel(_local_eval(a[::-1], k, ct, pts), _outgoing_eval(beta, k, cs, pts))
    assert good < 1e-12 and bad > 1e-3


def test_apply_T_degenerate_cases(O):
    """SP:510-512: M=1, P=0 -> 0; M=2 direct; M=1, P=1 image-only."""
    rng = np.random.default_rng(1)
    p, k = 8, 7.0
    b1 = rng.standard_normal((1, 2 * p + 1)) + 0j
    assert np.all(O.apply_T(b1, np.array([[0.1, 0.2]]), k, p, copies=0) == 0)
    # M=1, P=1, bloch=1: incoming = field of its two images
    c = np.array([[0.05, 0.1]])
    beta = np.zeros((1, 2 * p + 1), complex)
    beta[0, p] = 1.0
    a = O.apply_T(beta, c, k, p, bloch=1.0, copies=1)[0]
    pts = c[0] + 0.02 * np.array([[1.0, 0.0], [0.0, -1.0]])
    direct = _outgoing_eval(beta[0], k, c[0] + [1.0, 0], pts) + _outgoing_eval(beta[0], k, c[0] - [1.0, 0], pts)
    assert rel(_local_eval(a, k, c[0], pts), direct) < 1e-10
    # M=2, P=0: direct evaluation of particle 2 at particle 1
    c2 = np.array([[0.0, 0.0], [0.3, 0.1]])
    b2 = np.zeros((2, 2 * p + 1), complex)
    b2[1, p - 1:p + 2] = [0.3, 1.0, -0.2j]
    a2 = O.apply_T(b2, c2, k, p, copies=0)
    pts = c2[0] + 0.02 * np.array([[1.0, 0.0], [0.0, 1.0]])
    assert rel(_local_eval(a2[0], k, c2[0], pts), _outgoing_eval(b2[1], k, c2[1], pts)) < 1e-10


def test_disk_smatrix_matches_matching_conditions(O):
    """SP:411 / acceptance 2: value and radial-derivative continuity on r=R."""
    R, k2, kp, p = 0.05, 8.0, 30.0, 10
    s = O.disk_smatrix(R, k2, kp, p)
    n = np.arange(-p, p + 1)
    alpha = (sps.jv(n, k2 * R) + s * sps.hankel1(n, k2 * R)) / sps.jv(n, kp * R)
    lhs = alpha * kp * sps.jvp(n, kp * R)
    rhs = k2 * (sps.jvp(n, k2 * R) + s * sps.h1vp(n, k2 * R))
    assert np.max(np.abs(lhs - rhs)) < 1e-12
    assert np.allclose(s, s[::-1])          # even in n


def test_gmres_identity_and_dense(O):
    """SP:555-557."""
    rng = np.random.default_rng(4)
    b = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    x, its, hist = O.gmres(lambda v: v, b, 1e-12, 50)
    assert its == 1 and rel(x, b) < 1e-14
    A = np.eye(50) * 4 + 0.3 * (rng.standard_normal((50, 50)) + 1j * rng.standard_normal((50, 50)))
    b = rng.standard_normal(50) + 0j
    x, its, hist = O.gmres(lambda v: A @ v, b, 1e-13, 100)
    assert rel(x, np.linalg.solve(A, b)) < 1e-9
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))


def test_schur_degeneracies(O):
    """SP:545-547: beta=0 -> 0; B=C=0 -> I - S T; M=1, P=0, no coupling -> identity."""
    pb = O.load_problem(1)
    z = np.zeros(pb.M * pb.L, complex)
    assert np.all(O.apply_schur_operator(pb, z) == 0)
    one = O.Problem(pb.es, pb.centers[:1], pb.p, pb.radius)
    one.es = pb.es
    v = np.random.default_rng(5).standard_normal(pb.L) + 0j
    # single particle with no images: T = 0
    es0 = O.EmptySystem(**{**pb.es.__dict__, "copies": 0})
    one0 = O.Problem(es0, pb.centers[:1], pb.p, pb.radius)
    assert rel(O.apply_schur_operator(one0, v, with_coupling=False), v) < 1e-15


def test_cfg1_flux_conservation(O):
    """Full oracle solve of cfg1: 10 iterations, flux error ~1.4e-11."""
    sol = O.solve_full(O.load_problem(1))
    assert sol.iterations <= 12
    assert sol.flux["error"] < 1e-10


def test_empty_grating_flux(O):
    """M=0 reduces to the empty solve (SP:565): flux conserved to ~1e-13."""
    es = O.load_empty("w10")
    x = es.apply_pinv(es.f)
    assert O.flux_error(es, x[es.cols["c"]], x[es.cols["d"]])["error"] < 1e-12

"""Pin the oracle against the reference's OWN functions (runs wherever
/root/reference is mounted; skipped on the GPU box).

The reference ships no tests or golden vectors for the hot path (SURVEY.md
§8c), so the restated helpers are compared with the present reference
modules they stand in for, and the restated coupling blocks with the
reference's direct field evaluation.
"""
import math
import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE, rel

pytestmark = pytest.mark.skipif(not os.path.isdir(REFERENCE), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    if REFERENCE not in sys.path:
        sys.path.insert(0, REFERENCE)
    from periscat import empty_grating, geometry, layerpot, specialfn
    return dict(sf=specialfn, geo=geometry, lp=layerpot, eg=empty_grating)


@pytest.fixture(scope="module")
def O():
    from oracle import periscat_oracle
    return periscat_oracle


def test_hankel1_orders_bitwise(ref, O):
    """sf:54-67 restated: identical bits."""
    z = np.geomspace(0.05, 60, 500)
    a = ref["sf"].hankel1_orders(50, z)
    b = O.hankel1_orders(50, z)
    assert np.array_equal(a, b)


def test_signed_orders(ref, O):
    """sf:79-83."""
    tab = ref["sf"].hankel1_orders(12, np.array([0.7, 3.1]))
    for n in range(-12, 13):
        assert np.array_equal(O.signed_orders(tab, [n])[0], ref["sf"]._signed_order(tab, n))


def test_outgoing_waves_match_reference_block(ref, O):
    """Values and gradients vs outgoing_wave_block (sf:128-154)."""
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, (40, 2))
    center = np.array([0.13, -0.07])
    n = np.arange(-9, 10)
    v_ref, g_ref = ref["sf"].outgoing_wave_block(7.3, center, n, pts)
    v, g = O._outgoing_vals_grads(7.3, n, pts[:, 0] - center[0], pts[:, 1] - center[1], sign=1)
    assert rel(v.T, v_ref) < 1e-14
    assert rel(np.moveaxis(g, 0, -1).transpose(1, 0, 2), g_ref) < 1e-13


def test_fixture_matches_fresh_reference_assembly(ref, O):
    """The committed empty-grating fixture is the reference's own A, f, scaling."""
    es = O.load_empty("w10")
    conf = ref["geo"].ProblemConfig(period=1.0, k1=10.0, k2=12.0, k3=10.0, kp=15.0,
                                    incident_angle=-0.7 * math.pi,
                                    interface_top=ref["geo"].InterfaceSpec(0.5),
                                    interface_bottom=ref["geo"].InterfaceSpec(-0.5))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sysm = ref["eg"].assemble_empty_system(conf)
    assert np.array_equal(sysm.matrix, es.A)
    assert np.array_equal(sysm.rhs, es.f)
    assert np.array_equal(sysm.col_scale, es.col_scale)
    assert complex(conf.bloch_phase) == es.bloch
    assert np.array_equal(sysm.curves["L2"].nodes, es.L2_nodes)


def test_apply_pinv_matches_reference(ref, O):
    """eg:264-273 on the fixture's factors."""
    es = O.load_empty("w10")
    u, s, vh = es.factorize()

    class Sys:
        svd = (u, s, vh)
        col_scale = es.col_scale

        class config:
            regularization = es.eps

    g = np.random.default_rng(1).standard_normal(es.A.shape[0]) + 0j
    assert np.array_equal(ref["eg"].apply_pinv(Sys, g), es.apply_pinv(g))


def test_centers_fixture_is_reference_sampler(ref):
    """centers_cfg1.npy == place_random_particles(seed 0, M=10, r=0.04, standoff 0.02)."""
    geo = ref["geo"]
    conf = geo.ProblemConfig(k1=10.0, k2=12.0, k3=10.0, kp=15.0, incident_angle=-0.7 * math.pi,
                             interface_top=geo.InterfaceSpec(0.5),
                             interface_bottom=geo.InterfaceSpec(-0.5), seed=0,
                             particle_shape=geo.ParticleShape(0.04, 0.0, 1))
    ps = geo.place_random_particles(conf, 10, 0.02)
    from oracle.periscat_oracle import GOLDEN
    assert np.array_equal(ps.centers, np.load(os.path.join(GOLDEN, "centers_cfg1.npy")))


def test_B_local_expansion_reproduces_layer_field(ref, O):
    """B_phys vs the reference's direct layer-2 field
    (empty_grating.phased_layer_field + regular_wave_block, eg:319-393):
    re-sum the local expansion at points on a particle disk."""
    es = O.load_empty("w10")
    rng = np.random.default_rng(2)
    x = rng.standard_normal(es.A.shape[1]) + 1j * rng.standard_normal(es.A.shape[1])
    center = np.array([[0.11, 0.07]])
    p = 20
    a = O.apply_B_phys(es, x, center, p)[0]
    th = np.linspace(0, 2 * np.pi, 12, endpoint=False)
    pts = center + 0.03 * np.column_stack([np.cos(th), np.sin(th)])

    class Curve:
        def __init__(self, nodes, normals, w):
            self.nodes, self.normals, self.arc_weights = nodes, normals, w
            self.period_translation = np.array([1.0, 0.0])

        @property
        def n(self):
            return self.nodes.shape[0]

        def translated(self, shift):
            return Curve(self.nodes + shift, self.normals, self.arc_weights)

    direct = np.zeros(len(pts), dtype=complex)
    for nodes, nrm, w, mu, sg in ((es.g1_nodes, es.g1_normals, es.g1_w, "mu1", "sigma1"),
                                  (es.g2_nodes, es.g2_normals, es.g2_w, "mu2", "sigma2")):
        cv = Curve(nodes, nrm, w)
        direct += ref["eg"].phased_layer_field(cv, x[es.cols[mu]], x[es.cols[sg]], es.k2,
                                               es.bloch, es.copies, pts)
    vals, _ = ref["sf"].regular_wave_block(es.k2, es.center2, np.arange(-es.Q, es.Q + 1), pts)
    direct += vals @ x[es.cols["a2"]]
    loc, _ = ref["sf"].regular_wave_block(es.k2, center[0], np.arange(-p, p + 1), pts)
    assert rel(loc @ a, direct) < 1e-11


def test_C_rows_match_reference_waves(ref, O):
    """C g1/g2 rows vs outgoing_wave_block sums (sf:128-154)."""
    pb = O.load_problem(1)
    es = pb.es
    rng = np.random.default_rng(3)
    beta = rng.standard_normal((pb.M, pb.L)) + 1j * rng.standard_normal((pb.M, pb.L))
    g = O.apply_C(es, beta, pb.centers)
    n = np.arange(-pb.p, pb.p + 1)
    val = np.zeros(es.g2_nodes.shape[0], complex)
    der = np.zeros_like(val)
    for j in range(pb.M):
        for l in (-1, 0, 1):
            v, gr = ref["sf"].outgoing_wave_block(es.k2, pb.centers[j] + [l, 0.0], n, es.g2_nodes)
            val += es.bloch ** l * (v @ beta[j])
            der += es.bloch ** l * (np.einsum("ink,ik->in", gr, es.g2_normals) @ beta[j])
    assert rel(g[es.rows["g2_val"]], val) < 1e-12
    assert rel(g[es.rows["g2_der"]], der) < 1e-12


def test_apply_T_local_expansion_reproduces_particle_field(ref, O):
    """apply_T (SP:504-512, all-pairs Graf M2L over the phased images, self
    term excluded) vs the reference's OWN wave functions: the local expansion
    at each target, re-summed with specialfn.regular_wave_block (sf:86-125)
    on a small circle, equals the direct phased multipole field of every other
    source image, summed with specialfn.outgoing_wave_block (sf:128-154)."""
    rng = np.random.default_rng(11)
    M, p, k, d = 6, 20, 12.0, 1.0
    bloch = np.exp(1j * 0.7)
    centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    beta = np.zeros((M, 2 * p + 1), complex)
    beta[:, p - 3:p + 4] = rng.standard_normal((M, 7)) + 1j * rng.standard_normal((M, 7))
    a = O.apply_T(beta, centers, k, p, bloch, d, 1)
    orders = np.arange(-p, p + 1)
    for m in range(M):
        dmin = min(np.hypot(*(centers[m] - centers[j] - [l * d, 0.0]))
                   for j in range(M) for l in (-1, 0, 1) if (j, l) != (m, 0))
        th = np.linspace(0, 2 * np.pi, 9, endpoint=False)
        pts = centers[m] + 0.2 * dmin * np.column_stack([np.cos(th), np.sin(th)])
        direct = np.zeros(len(pts), complex)
        for j in range(M):
            for l in (-1, 0, 1):
                if (j, l) == (m, 0):
                    continue
                vals, _ = ref["sf"].outgoing_wave_block(k, centers[j] + [l * d, 0.0], orders, pts)
                direct += bloch ** l * (vals @ beta[j])
        loc, _ = ref["sf"].regular_wave_block(k, centers[m], orders, pts)
        assert rel(loc @ a[m], direct) < 1e-10, m


def test_coupled_solution_satisfies_reference_wall_conditions(ref, O):
    """End-to-end physics pin of the coupled solve with the reference's own
    checker: the golden cfg1 solution (beta from the oracle GMRES, which the
    GPU reproduces to 1e-9) plus x_empty = A^+ (f - C beta), evaluated with
    empty_grating.wall_discrepancy_residual (eg:396-433) and the particles'
    phased multipole field (specialfn.outgoing_wave_block) as its
    extra_field: the quasi-periodicity alpha u(L) - u(R) of the coupled field
    holds at fresh wall points, and fails without the particle field."""
    import warnings
    warnings.simplefilter("ignore")
    from oracle.make_empty import config_for
    pb = O.load_problem(1)
    z = np.load(os.path.join(O.GOLDEN, "golden_cfg1.npz"))
    beta = z["beta"]
    conf = config_for(10.0, -0.7 * math.pi)
    system = ref["eg"].assemble_empty_system(conf)
    ref["eg"].factorize(system)
    x = ref["eg"].apply_pinv(system, system.rhs - O.apply_C(pb.es, beta, pb.centers))
    sol = ref["eg"].EmptySolution(system, x, 0.0)
    orders = np.arange(-pb.p, pb.p + 1)
    alpha = conf.bloch_phase

    def particles(points, normals):
        """Particle field of layer 2 (the particles' representation lives in
        the middle layer only, PAPER Eq. repre3_mod)."""
        vals = np.zeros(len(points), complex)
        ders = np.zeros(len(points), complex)
        mid = ref["eg"].classify_layer(conf, points) == 2
        points, normals = points[mid], normals[mid]
        for j in range(pb.M):
            for l in range(-conf.near_field_copies, conf.near_field_copies + 1):
                v, g = ref["sf"].outgoing_wave_block(conf.k2, pb.centers[j] + [l * conf.period, 0.0],
                                                     orders, points)
                vals[mid] += alpha ** l * (v @ beta[j])
                ders[mid] += alpha ** l * (np.einsum("ijk,ik->ij", g, normals) @ beta[j])
        return vals, ders

    coupled = ref["eg"].wall_discrepancy_residual(sol, extra_field=particles)
    without = ref["eg"].wall_discrepancy_residual(sol)
    assert coupled < 1e-8, (coupled, without)
    assert without > 1e3 * coupled

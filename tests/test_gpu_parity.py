"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): matvec relative error <= 1e-10
(normwise, per RHS); Bragg coefficients c, d relative <= 1e-9; flux-balance
error |delta| <= 1e-9 absolute.
"""
import numpy as np
import pytest

from conftest import rel
import workloads  # noqa: E402

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


@pytest.mark.parametrize("variant", [1, 2, 3])
@pytest.mark.parametrize("p,copies,M", [(0, 1, 1), (1, 1, 2), (2, 0, 17), (3, 1, 9), (7, 2, 33),
                                        (12, 1, 24), (20, 1, 41), (25, 1, 70)])
def test_apply_T_small_orders_kernel_variants(O, variant, p, copies, M):
    """Tiled K1 (1), symmetric K1s (2) and its DMMA form K1h (3) forced at every block size BO the
    swizzled K1s layout sees (p = 0..25), ragged tiles, 0..2 image copies."""
    import torch
    from paper_1412_7466_b200.engine import Engine
    rng = np.random.default_rng(1000 + p * 10 + M)
    centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    beta = _cplx(rng, (M, 2 * p + 1))
    bloch = np.exp(-0.4j)
    ref = O.apply_T(beta, centers, 9.0, p, bloch, 1.0, copies)
    eng = Engine(0)
    eng.set_geometry(centers, p, 9.0, 1.0, copies)
    eng.set_bloch(np.array([bloch]))
    eng.set_k1_variant(variant)
    got = eng.apply_T(torch.as_tensor(beta[None]).cuda())[0].cpu().numpy()
    eng.close()
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


def _operator(O, cfg, coupled=True, dense_gb=40.0):
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(cfg)
    sysm = workloads.load_fixture(O.CONFIGS[cfg]["empty"])
    op = solver.SchurOperator(sysm, pb.centers, pb.p, smat=pb.smat, coupled=coupled,
                              dense_gb=dense_gb)
    return pb, op


@pytest.mark.parametrize("dense_gb", [40.0, 0.0])
@pytest.mark.parametrize("cfg", [1, 2])
def test_apply_C_matches_oracle(O, cfg, dense_gb):
    """Pre-assembled C (dense_gb > 0) and matrix-free K3 (dense_gb = 0)."""
    pb, op = _operator(O, cfg, dense_gb=dense_gb)
    assert op.dense == (dense_gb > 0)
    rng = np.random.default_rng(20 + cfg)
    beta = _cplx(rng, (pb.M, pb.L))
    ref = O.apply_C(pb.es, beta, pb.centers)[:576]
    got = op.eng.apply_C(_dev(beta[None])).cpu().numpy()[0]
    assert rel(got, ref) <= MATVEC_TOL


@pytest.mark.parametrize("dense_gb", [40.0, 0.0])
@pytest.mark.parametrize("cfg", [1, 2])
def test_schur_matches_oracle(O, cfg, dense_gb):
    pb, op = _operator(O, cfg, dense_gb=dense_gb)
    rng = np.random.default_rng(30 + cfg)
    for v in (_cplx(rng, (pb.M, pb.L)), pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))):
        ref = O.apply_schur_operator(pb, v).reshape(pb.M, pb.L)
        got = op(_dev(v[None])).cpu().numpy()[0]
        assert rel(got, ref) <= MATVEC_TOL


@pytest.mark.parametrize("dense_gb", [40.0, 0.0])
@pytest.mark.parametrize("cfg", [1, 2])
def test_schur_rhs_matches_oracle(O, cfg, dense_gb):
    pb, op = _operator(O, cfg, dense_gb=dense_gb)
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
    sol = solver.solve_full(workloads.load_fixture("w10"), pb.centers, pb.p, smat=pb.smat)
    assert rel(sol.c[0], ref.c) <= 1e-9
    assert rel(sol.d[0], ref.d) <= 1e-9
    assert abs(sol.flux[0]["error"] - ref.flux["error"]) <= 1e-9
    assert sol.flux[0]["error"] <= 1e-9
    assert abs(sol.iterations[0] - ref.iterations) <= 1


# ---------------------------------------------------------------- multi-RHS (K1m)
def test_apply_T_16rhs_cfg2(O):
    """cfg5-style batch of 16 RHS (different Bloch phases) through K1m."""
    from paper_1412_7466_b200 import multiscat
    pb = O.load_problem(2)
    rng = np.random.default_rng(16)
    beta = pb.smat[None, None, :] * _cplx(rng, (16, pb.M, pb.L))
    bl = np.exp(1j * rng.uniform(-np.pi, np.pi, 16))
    ref = O.apply_T(beta, pb.centers, pb.es.k2, pb.p, bl)
    got = multiscat.apply_T(beta, pb.centers, pb.es.k2, pb.p, bl)
    for r in range(16):
        assert rel(got[r], ref[r]) <= MATVEC_TOL


@pytest.mark.parametrize("nrhs,p,M", [(2, 25, 17), (5, 7, 33), (19, 3, 9)])
def test_apply_T_mrhs_shapes(O, nrhs, p, M):
    """Odd RHS counts, more than one RHS group, ragged target tiles."""
    from paper_1412_7466_b200 import multiscat
    rng = np.random.default_rng(nrhs * 1000 + p)
    centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    beta = _cplx(rng, (nrhs, M, 2 * p + 1))
    bl = np.exp(1j * rng.uniform(-np.pi, np.pi, nrhs))
    ref = O.apply_T(beta, centers, 11.0, p, bl)
    got = multiscat.apply_T(beta, centers, 11.0, p, bl)
    for r in range(nrhs):
        assert rel(got[r], ref[r]) <= MATVEC_TOL


ANGLES = ["w10", "w10_a00", "w10_a15"]


@pytest.mark.parametrize("dense_gb", [40.0, 0.0])
def test_schur_multi_rhs_matches_oracle(O, dense_gb):
    """Three incidence angles (own Bloch phase, SVD factors, f) in one batch."""
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(1)
    systems = [workloads.load_fixture(n) for n in ANGLES]
    op = solver.SchurOperator(systems, pb.centers, pb.p, smat=pb.smat, dense_gb=dense_gb)
    rng = np.random.default_rng(33)
    v = pb.smat[None, None, :] * _cplx(rng, (3, pb.M, pb.L))
    got = op(_dev(v)).cpu().numpy()
    rhs = op.rhs().cpu().numpy()
    for r, name in enumerate(ANGLES):
        pr = O.Problem(O.load_empty(name), pb.centers, pb.p, pb.radius, pb.smat)
        assert rel(got[r], O.apply_schur_operator(pr, v[r]).reshape(pb.M, pb.L)) <= MATVEC_TOL
        assert rel(rhs[r], O.schur_rhs(pr).reshape(pb.M, pb.L)) <= MATVEC_TOL


def test_solve_full_multi_rhs(O):
    """Batched device GMRES: per-RHS convergence and Bragg coefficients."""
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(1)
    systems = [workloads.load_fixture(n) for n in ANGLES]
    sol = solver.solve_full(systems, pb.centers, pb.p, smat=pb.smat)
    for r, name in enumerate(ANGLES):
        pr = O.Problem(O.load_empty(name), pb.centers, pb.p, pb.radius, pb.smat)
        ref = O.solve_full(pr)
        assert rel(sol.c[r], ref.c) <= 1e-9
        assert rel(sol.d[r], ref.d) <= 1e-9
        assert abs(sol.flux[r]["error"] - ref.flux["error"]) <= 1e-9
        assert abs(sol.iterations[r] - ref.iterations) <= 1


# ---------------------------------------------------------------- golden full solves
def _golden(cfg):
    import os
    from oracle.periscat_oracle import GOLDEN
    path = os.path.join(GOLDEN, f"golden_cfg{cfg}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden_cfg{cfg}.npz not generated")
    return np.load(path)


@pytest.mark.parametrize("dense_gb", [40.0, 0.0])
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_matvec_vs_golden(O, cfg, dense_gb):
    """apply_T and the Schur operator against the committed oracle goldens."""
    z = _golden(cfg)
    pb, op = _operator(O, cfg, dense_gb=dense_gb)
    v = torch.as_tensor(z["v"][None]).cuda()
    tids = z["targets"]
    aT = op.apply_T(v).cpu().numpy()[0][tids]
    sch = op(v).cpu().numpy()[0][tids]
    assert rel(aT, z["apply_T"]) <= MATVEC_TOL
    assert rel(sch, z["schur"]) <= MATVEC_TOL
    assert rel(op.rhs().cpu().numpy()[0][tids], z["rhs"]) <= MATVEC_TOL


@pytest.mark.parametrize("sms", [-1, 0, 2, 8, 40])
def test_schur_sm_partition_vs_golden(O, sms):
    """K1s on a reduced grid overlapped with the coupling chain on the other
    SMs (ps_set_overlap): same operator as the serial path and the golden."""
    z = _golden(3)
    pb, op = _operator(O, 3)
    op.eng.set_overlap(sms)
    v = torch.as_tensor(z["v"][None]).cuda()
    tids = z["targets"]
    sch = op(v).cpu().numpy()[0]
    assert rel(sch[tids], z["schur"]) <= MATVEC_TOL
    op.eng.set_overlap(-1)
    ser = op(v).cpu().numpy()[0]
    assert rel(sch, ser) <= 1e-13


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_solve_full_vs_golden(O, cfg):
    """Full device solve vs the oracle's solve (c, d <= 1e-9 rel, |dflux| <= 1e-9)."""
    from paper_1412_7466_b200 import grating, solver
    z = _golden(cfg)
    pb = O.load_problem(cfg)
    sol = solver.solve_full(workloads.load_fixture(O.CONFIGS[cfg]["empty"]), pb.centers, pb.p,
                            smat=pb.smat)
    assert rel(sol.c[0], z["c"]) <= 1e-9
    assert rel(sol.d[0], z["d"]) <= 1e-9
    assert abs(sol.flux[0]["error"] - float(z["flux_error"])) <= 1e-9
    assert abs(sol.iterations[0] - int(z["iterations"])) <= 1


# ---------------------------------------------------------------- dense S (a4)
@pytest.mark.parametrize("nrhs", [1, 3])
def test_dense_rotated_smatrix(O, nrhs):
    """Non-diagonal S with per-inclusion rotation phases: the
    dense epilogue (1 RHS) and the K1m + dense epilogue path (3 RHS)."""
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(1)
    rng = np.random.default_rng(77)
    L = pb.L
    S = np.diag(pb.smat) + 1e-3 * np.outer(pb.smat, np.ones(L)) * _cplx(rng, (L, L))
    rot = rng.uniform(0, 2 * np.pi, pb.M)
    names = ANGLES[:nrhs]
    op = solver.SchurOperator([workloads.load_fixture(n) for n in names], pb.centers, pb.p,
                              smat=S, rot=rot)
    v = _cplx(rng, (nrhs, pb.M, L))
    got = op(_dev(v)).cpu().numpy()
    rhs = op.rhs().cpu().numpy()
    for r, n in enumerate(names):
        pr = O.Problem(O.load_empty(n), pb.centers, pb.p, pb.radius, S, rot)
        assert rel(got[r], O.apply_schur_operator(pr, v[r]).reshape(pb.M, L)) <= MATVEC_TOL
        assert rel(rhs[r], O.schur_rhs(pr).reshape(pb.M, L)) <= MATVEC_TOL


# ---------------------------------------------------------------- GMRES contract (a9)
def test_gmres_nonconvergence_is_reported(O):
    """hitting maxit is reported through the history, not raised."""
    from paper_1412_7466_b200 import solver
    pb, op = _operator(O, 2)
    x, its, hist = solver.gmres(op, op.rhs(), 1e-14, 3)
    assert its == [3] and hist[0][-1] > 1e-14
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist[0], hist[0][1:]))


def test_gmres_nan_raises(O):
    """NaN/Inf in a Krylov vector -> numerical error."""
    from paper_1412_7466_b200 import NumericalError, solver
    pb, op = _operator(O, 1)
    rhs = op.rhs().clone()
    rhs[0, 3, 5] = float("nan")
    with pytest.raises(NumericalError):
        solver.gmres(op, rhs, 1e-10, 20)


def test_gmres_identity_one_iteration(O):
    """operator = identity (single inclusion, no images, no
    coupling -> T = 0) converges in one iteration to x = rhs."""
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(1)
    sysm = workloads.load_fixture("w10")
    sysm.config.near_field_copies = 0
    op = solver.SchurOperator(sysm, pb.centers[:1], pb.p, smat=pb.smat, coupled=False)
    b = torch.as_tensor(np.random.default_rng(2).standard_normal((1, 1, pb.L)) + 0j).cuda()
    x, its, hist = solver.gmres(op, b, 1e-12, 10)
    assert its == [1]
    assert rel(x.cpu().numpy(), b.cpu().numpy()) < 1e-14


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("nrhs,p,M", [(16, 20, 40), (13, 25, 21), (4, 6, 30)])
def test_mrhs_variants(O, variant, nrhs, p, M):
    """Both multi-RHS kernels (1: DFMA K1m, 2: FP64-tensor-core K1d) vs the oracle."""
    from paper_1412_7466_b200.engine import Engine
    rng = np.random.default_rng(nrhs * 31 + p + variant)
    centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    L = 2 * p + 1
    beta = _cplx(rng, (nrhs, M, L))
    bl = np.exp(1j * rng.uniform(-np.pi, np.pi, nrhs))
    eng = Engine(0)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(bl)
    eng.set_mrhs_variant(variant)
    got = eng.apply_T(_dev(beta)).cpu().numpy()
    ref = O.apply_T(beta, centers, 12.0, p, bl)
    for r in range(nrhs):
        assert rel(got[r], ref[r]) <= MATVEC_TOL


# ---------------------------------------------------------------- K1 variants / shards
@pytest.mark.parametrize("variant", [1, 2, 3])
def test_k1_variants_full_range(O, variant):
    """Tiled K1 (1), symmetric K1s (2) and K1h (3) on cfg2, random and Krylov-scaled input."""
    from paper_1412_7466_b200.engine import Engine
    pb = O.load_problem(2)
    rng = np.random.default_rng(50 + variant)
    beta = pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))
    eng = Engine(0)
    eng.set_geometry(pb.centers, pb.p, pb.es.k2, pb.es.period, pb.es.copies)
    eng.set_bloch([pb.es.bloch])
    eng.set_k1_variant(variant)
    got = eng.apply_T(_dev(beta[None])).cpu().numpy()[0]
    ref = O.apply_T(beta, pb.centers, pb.es.k2, pb.p, pb.es.bloch)
    assert rel(got, ref) <= MATVEC_TOL


@pytest.mark.parametrize("ranks", [2, 3, 8])
def test_target_shards_reassemble(O, ranks):
    """Per-rank target ranges (the multi-GPU decomposition, tiled K1 + dense
    coupling on the owned range) reassemble the full Schur matvec; each
    'rank' runs its own context sequentially on this one GPU."""
    from paper_1412_7466_b200 import grating, parallel, solver
    pb = O.load_problem(2)
    rng = np.random.default_rng(ranks)
    v = pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))
    ref = O.apply_schur_operator(pb, v).reshape(pb.M, pb.L)
    sysm = workloads.load_fixture("w10")
    vd = _dev(v[None])
    # C partials over each rank's own sources, summed as the all-reduce would
    ops = [solver.SchurOperator(sysm, pb.centers, pb.p, smat=pb.smat,
                                target_range=parallel.shard_range(pb.M, r, ranks))
           for r in range(ranks)]
    g = sum(op.eng.apply_C(vd, s_range=parallel.shard_range(pb.M, r, ranks))
            for r, op in enumerate(ops))
    parts = [op(vd, g=g).cpu().numpy()[0] for op in ops]
    got = np.concatenate(parts, axis=0)
    assert rel(got, ref) <= MATVEC_TOL


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
@pytest.mark.parametrize("p,M", [(25, 1000), (5, 40), (2, 9)])
def test_apply_T_blocks_sum_to_apply_T(O, nparts, p, M):
    """The symmetric split (ps_apply_T_blocks): the parts of the tile-pair list
    sum to the full M2L for every target, including empty parts."""
    from paper_1412_7466_b200 import grating
    from paper_1412_7466_b200.engine import Engine
    rng = np.random.default_rng(M + nparts)
    if M == 1000:
        centers = O.load_problem(3).centers
    else:
        centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    beta = _cplx(rng, (1, M, 2 * p + 1))
    eng = Engine(0)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(np.array([np.exp(0.3j)]))
    vd = _dev(beta)
    full = eng.apply_T(vd).cpu().numpy()
    tot = sum(eng.apply_T_blocks(vd, r, nparts).cpu().numpy() for r in range(nparts))
    eng.close()
    assert rel(tot, full) <= 1e-13


@pytest.mark.parametrize("ranks", [2, 3])
def test_pair_split_shards_reassemble(O, ranks):
    """The 'pairs' multi-GPU decomposition simulated rank by rank on this GPU:
    partial K1s over each rank's tile-pair range for all targets, summed as
    the reduce-scatter would, then each rank's epilogue (ps_schur_finish) with
    the all-reduced coupling rows -- equals the oracle Schur matvec."""
    from paper_1412_7466_b200 import grating, parallel, solver
    pb = O.load_problem(2)
    rng = np.random.default_rng(10 + ranks)
    v = pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))
    ref = O.apply_schur_operator(pb, v).reshape(pb.M, pb.L)
    sysm = workloads.load_fixture("w10")
    vd = _dev(v[None])
    rngs = [parallel.shard_range(pb.M, r, ranks) for r in range(ranks)]
    ops = [solver.SchurOperator(sysm, pb.centers, pb.p, smat=pb.smat, target_range=rngs[r])
           for r in range(ranks)]
    a_parts = [op.eng.apply_T_blocks(vd, r, ranks) for r, op in enumerate(ops)]
    a_sum = sum(a_parts)
    g = sum(op.eng.apply_C(vd, s_range=rngs[r]) for r, op in enumerate(ops))
    got = []
    for r, op in enumerate(ops):
        t0, t1 = rngs[r]
        y = op.eng.schur_finish(vd[:, t0:t1].contiguous(), a_sum[:, t0:t1].contiguous(), g)
        got.append(y.cpu().numpy()[0])
    assert rel(np.concatenate(got, axis=0), ref) <= MATVEC_TOL


@pytest.mark.parametrize("nrhs,p,M", [(1, 20, 100), (3, 5, 17), (5, 25, 9)])
def test_particle_field_matches_oracle(O, nrhs, p, M):
    """ps_particle_field (M2P over grid points) vs the
    oracle's phased multipole sums, points outside every particle copy."""
    from paper_1412_7466_b200 import postproc
    from paper_1412_7466_b200.engine import Engine
    rng = np.random.default_rng(100 + M)
    centers = np.column_stack([rng.uniform(-0.45, 0.45, M), rng.uniform(-0.4, 0.4, M)])
    beta = _cplx(rng, (nrhs, M, 2 * p + 1))
    bl = np.exp(1j * rng.uniform(-3, 3, nrhs))
    pts = np.column_stack([rng.uniform(-0.5, 0.5, 300), rng.uniform(-0.45, 0.45, 300)])
    dmin = np.min(np.hypot(pts[:, None, 0] - centers[None, :, 0], pts[:, None, 1] - centers[None, :, 1]), axis=1)
    pts = pts[dmin > 0.01]
    eng = Engine(0)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(bl)
    got = postproc.particle_field(eng, beta, pts)
    eng.close()
    for r in range(nrhs):
        ref = sum((bl[r] ** l) * O._particle_field(12.0, beta[r], centers, pts, float(l))[0]
                  for l in (-1, 0, 1))
        assert rel(got[r], ref) <= 1e-12


def test_eval_total_field_grid_cfg2(O):
    """Grid evaluation: the rasterised particle mask equals
    the brute-force classification, masked points are NaN, and the layer-2
    particle field matches the oracle's phased multipole sums."""
    from paper_1412_7466_b200 import grating, postproc, solver
    pb = O.load_problem(2)
    sysm = workloads.load_fixture("w10")
    op = solver.SchurOperator(sysm, pb.centers, pb.p, smat=pb.smat)
    rng = np.random.default_rng(4)
    beta = pb.smat[None, None, :] * _cplx(rng, (1, pb.M, pb.L))
    res = postproc.eval_total_field_grid(op, beta, pb.centers, 0.04, nx=60, ny=50, y_plot=0.7,
                                         layer_field=None)
    xx, yy = np.meshgrid(res["x"], res["y"])
    pts = np.column_stack([xx.ravel(), yy.ravel()])
    layer, masked = postproc.classify_points(op.config, pts, pb.centers, 0.04, system=sysm)
    assert np.array_equal(masked, res["mask"].ravel())
    assert np.array_equal(layer, res["layer"].ravel())
    f = res["field"][0].ravel()
    assert np.all(np.isnan(f[masked]))
    sel = np.flatnonzero((layer == 2) & ~masked)[::25]
    al = op.config.bloch_phase
    ref = sum((al ** l) * O._particle_field(pb.es.k2, beta[0], pb.centers, pts[sel], float(l))[0]
              for l in (-1, 0, 1))
    assert rel(f[sel], ref) <= 1e-12
    assert np.all(f[(layer != 2) & ~masked] == 0)


@pytest.mark.parametrize("cfg,nrhs", [(3, 1), (2, 16)])
def test_matvec_and_solve_are_bit_reproducible(O, cfg, nrhs):
    """SPEC.md:507 / 576: apply_T has a deterministic order -- every device
    reduction (M2L partials, coupling splits, GMRES dots) runs in a fixed
    order, so repeated Schur matvecs and GMRES solves are bitwise identical
    (K1s + SM-partitioned coupling for cfg3, K1d for 16 RHS)."""
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(cfg)
    sysm = workloads.load_fixture(O.CONFIGS[cfg]["empty"])
    systems = [sysm] * nrhs
    op = solver.SchurOperator(systems, pb.centers, pb.p, smat=pb.smat)
    rng = np.random.default_rng(99)
    v = _dev(pb.smat[None, None, :] * _cplx(rng, (nrhs, pb.M, pb.L)))
    y0 = op(v).cpu().numpy()
    for _ in range(3):
        assert np.array_equal(op(v).cpu().numpy(), y0)
    if nrhs == 1:
        x1, _, _ = solver.gmres(op, op.rhs(), 1e-10, 150)
        x2, _, _ = solver.gmres(op, op.rhs(), 1e-10, 150)
        assert torch.equal(x1, x2)


def test_k1s_symbol_store_is_bitwise_the_generated_symbols(O):
    """K1s with its geometry-only symbols precomputed once (the default when
    the store fits) and bulk-copied per batch gives bitwise the result of
    regenerating them in every launch; the store follows a geometry change."""
    from paper_1412_7466_b200.engine import Engine
    pb = O.load_problem(3)
    rng = np.random.default_rng(321)
    beta = _dev(pb.smat[None, None, :] * _cplx(rng, (1, pb.M, pb.L)))
    eng = Engine(0)
    eng.set_geometry(pb.centers, pb.p, pb.es.k2, pb.es.period, pb.es.copies)
    eng.set_bloch([pb.es.bloch])
    eng.set_k1_variant(2)
    y_store = eng.apply_T(beta).cpu().numpy()
    assert eng.set_symbol_store(-1) > 0                 # the store was built and used
    y_again = eng.apply_T(beta).cpu().numpy()
    eng.set_symbol_store(0)
    assert eng.set_symbol_store(-1) == 0
    y_gen = eng.apply_T(beta).cpu().numpy()
    assert np.array_equal(y_store, y_gen) and np.array_equal(y_again, y_gen)
    ref = O.apply_T(beta.cpu().numpy()[0], pb.centers, pb.es.k2, pb.p, pb.es.bloch)
    assert rel(y_store[0], ref) <= MATVEC_TOL
    # new geometry: the store is rebuilt, not reused
    eng.set_symbol_store(32)
    c2 = pb.centers.copy()
    c2[:, 1] *= 0.99
    eng.set_geometry(c2, pb.p, pb.es.k2, pb.es.period, pb.es.copies)
    eng.set_bloch([pb.es.bloch])
    y2 = eng.apply_T(beta).cpu().numpy()
    eng.set_symbol_store(0)
    y2g = eng.apply_T(beta).cpu().numpy()
    eng.close()
    assert np.array_equal(y2, y2g)


def test_k1h_bit_reproducible_and_matches_k1s(O):
    """The opt-in DMMA variant of the symmetric M2L (K1h, variant 3) keeps the
    deterministic order (repeat launches bitwise identical) and equals K1s
    to rounding on cfg3 with Krylov-scaled input."""
    from paper_1412_7466_b200.engine import Engine
    pb = O.load_problem(3)
    rng = np.random.default_rng(123)
    beta = _dev(pb.smat[None, None, :] * _cplx(rng, (1, pb.M, pb.L)))
    eng = Engine(0)
    eng.set_geometry(pb.centers, pb.p, pb.es.k2, pb.es.period, pb.es.copies)
    eng.set_bloch([pb.es.bloch])
    eng.set_k1_variant(3)
    y0 = eng.apply_T(beta).cpu().numpy()
    for _ in range(2):
        assert np.array_equal(eng.apply_T(beta).cpu().numpy(), y0)
    eng.set_k1_variant(2)
    ys = eng.apply_T(beta).cpu().numpy()
    eng.close()
    assert rel(y0, ys) <= 1e-13


_FULL3 = {}


def _cfg3_init():
    from oracle import periscat_oracle as Ox
    _FULL3["pb"] = Ox.load_problem(3)


def _cfg3_chunk(args):
    chunk, v, xg = args
    if "pb" not in _FULL3:
        _cfg3_init()
    pb = _FULL3["pb"]
    from oracle import periscat_oracle as Ox
    u = Ox.apply_T(v, pb.centers, pb.es.k2, pb.p, pb.es.bloch, pb.es.period, pb.es.copies,
                   targets=chunk)
    return u - Ox.apply_B_phys(pb.es, xg, pb.centers[chunk], pb.p)


def test_schur_cfg3_full_vector(O):
    """cfg3 (M=1000, p=25): the whole Schur matvec K v against the oracle over
    ALL targets (the goldens hold a 24-target slice), oracle M2L spread over
    the host cores."""
    import multiprocessing as mp
    import os as _os
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(3)
    _FULL3["pb"] = pb
    rng = np.random.default_rng(303)
    v = pb.smat[None, :] * _cplx(rng, (pb.M, pb.L))
    xg = pb.es.apply_pinv(O.apply_C(pb.es, v, pb.centers))
    n = len(_os.sched_getaffinity(0))
    chunks = [c for c in np.array_split(np.arange(pb.M), 4 * n) if c.size]
    # spawn, not fork: this process already runs CUDA threads
    with mp.get_context("spawn").Pool(n, initializer=_cfg3_init) as pool:
        u = np.concatenate(pool.map(_cfg3_chunk, [(c, v, xg) for c in chunks]), axis=0)
    ref = v - pb.smat[None, :] * u
    op = solver.SchurOperator(workloads.load_fixture("w10"), pb.centers, pb.p, smat=pb.smat)
    got = op(_dev(v[None])).cpu().numpy()[0]
    assert rel(got, ref) <= MATVEC_TOL
    aT = op.apply_T(_dev(v[None])).cpu().numpy()[0]
    uT = np.concatenate([O.apply_T(v, pb.centers, pb.es.k2, pb.p, pb.es.bloch, targets=c)
                         for c in (np.arange(0, 40), np.arange(960, 1000))], axis=0)
    assert rel(aT[np.r_[0:40, 960:1000]], uT) <= MATVEC_TOL


@pytest.mark.parametrize("M,p", [(11, 25), (14, 20), (22, 25)])
def test_dense_coupling_many_ct_blocks(O, M, p):
    """Dense coupling where the C^T GEMV launches more than 512 split blocks
    (K = M L in 524..592 on 148 SMs): the workspace holds every block's
    partial sums (gpart sizing) and the matvec matches the oracle."""
    from paper_1412_7466_b200 import grating, solver
    rng = np.random.default_rng(M * 100 + p)
    xs = (np.arange(M) + 0.5) / M - 0.5
    centers = np.column_stack([xs, rng.uniform(-0.3, 0.3, M)])
    sysm = workloads.load_fixture("w10")
    pr = O.Problem(O.load_empty("w10"), centers, p, 0.012)
    op = solver.SchurOperator(sysm, centers, p, smat=pr.smat, dense_gb=40.0)
    assert op.dense
    v = pr.smat[None, :] * _cplx(rng, (M, 2 * p + 1))
    for _ in range(2):
        got = op(_dev(v[None])).cpu().numpy()[0]
    ref = O.apply_schur_operator(pr, v).reshape(M, 2 * p + 1)
    assert rel(got, ref) <= MATVEC_TOL

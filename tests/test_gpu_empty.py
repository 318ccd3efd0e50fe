"""Device empty-grating setup (ps_setup_empty: assembly + cuSOLVER SVD +
restricted A^+ factors) against the reference's own assembled systems (the
committed fixtures are bit-identical to empty_grating.assemble_empty_system,
test_oracle_pin) and the oracle goldens.

Tolerances: the device evaluates H0/H1/J_n by Miller/Neumann sweeps instead of
AMOS, so entries agree to ~1e-14 of their column's scale, not bitwise; the
SVD is cuSOLVER gesvd instead of LAPACK gesdd.  Solution quantities keep the
north-star bars (c, d <= 1e-9 relative, flux <= 1e-9 absolute, matvec <= 1e-10).
"""
import os

import numpy as np
import pytest

from conftest import rel
import workloads  # noqa: E402

pytestmark = pytest.mark.gpu

ENTRY_TOL = 1e-12     # |A_dev - A_ref| per entry, relative to max(1, column max)
SV_TOL = 1e-13        # |s_dev - s_ref| / s_max
MATVEC_TOL = 1e-10


def _setup(configs, M_centers=None, svd_workers=None):
    from paper_1412_7466_b200.engine import Engine
    eng = Engine(0)
    c = np.array([[0.0, 0.0]]) if M_centers is None else M_centers
    eng.set_geometry(c, 2, configs[0].k2, configs[0].period, configs[0].near_field_copies)
    eng.set_bloch([cf.bloch_phase for cf in configs])
    systems = eng.setup_empty(configs, svd_workers=svd_workers)
    return eng, systems


def _check_against_fixture(got, ref):
    A, f, cs, s = got
    assert A.shape == ref.matrix.shape
    scale = np.maximum(1.0, np.max(np.abs(ref.matrix), axis=0))
    err = np.max(np.abs(A - ref.matrix) / scale[None, :])
    assert err <= ENTRY_TOL, f"entry error {err:.2e}"
    assert np.max(np.abs(f - ref.rhs)) <= 1e-14
    assert np.max(np.abs(cs / ref.col_scale - 1.0)) <= 1e-12
    s_ref = np.linalg.svd(ref.matrix, compute_uv=False)
    assert np.max(np.abs(s - s_ref)) / s_ref[0] <= SV_TOL
    assert np.all(np.diff(s) <= 0)


@pytest.mark.parametrize("name", ["w10", "wood", "w10_a00", "w10_a15", "curved", "w10_P0", "w10_P2"])
def test_device_assembly_matches_reference_system(name):
    """A, f, col_scale and singular values of the device-assembled system vs
    the reference's assemble_empty_system output (fixture) for the BASELINE
    gratings: omega=10 (cfg1-3), the Wood anomaly (cfg4), cfg5's extreme
    angles, and the reference's default sinusoidal interfaces (curved)."""
    from paper_1412_7466_b200 import grating
    ref = workloads.load_fixture(name)
    eng, systems = _setup([workloads.fixture_config(name)])
    try:
        _check_against_fixture(systems[0].fetch(), ref)
        assert systems[0].cols == ref.cols and systems[0].rows == ref.rows
    finally:
        eng.close()


def test_device_assembly_batched_angles_concurrent_svd():
    """cfg5's 16 incidence angles in one setup call (one assembly launch, SVDs
    on 4 concurrent cuSOLVER streams): the first and last angle match their
    reference systems, and every angle equals its own single-angle setup."""
    from paper_1412_7466_b200 import grating
    cfgs = [workloads.fixture_config(n) for n in workloads.CFG5_ANGLES]
    eng, systems = _setup(cfgs, svd_workers=4)
    try:
        for i, name in ((0, "w10_a00"), (15, "w10_a15")):
            _check_against_fixture(systems[i].fetch(), workloads.load_fixture(name))
        for i in (3, 9):
            e1, s1 = _setup([cfgs[i]])
            try:
                a1 = s1[0].fetch()
                ab = systems[i].fetch()
                assert np.array_equal(a1[0], ab[0]) and np.array_equal(a1[1], ab[1])
                assert np.array_equal(a1[3], ab[3])
            finally:
                e1.close()
    finally:
        eng.close()


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_schur_with_device_setup_matches_golden(cfg):
    """The Schur matvec of an operator built from the config alone (device
    assembly + SVD) equals the oracle golden (host reference factors)."""
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(cfg)
    z = np.load(os.path.join(O.GOLDEN, f"golden_cfg{cfg}.npz"))
    conf = workloads.fixture_config(workloads.CONFIGS[cfg]["system"])
    import torch
    op = solver.SchurOperator(conf, pb.centers, pb.p, smat=pb.smat, device=0)
    assert op.device_setup
    v = torch.as_tensor(z["v"][None]).cuda()
    tids = z["targets"]
    sch = op(v).cpu().numpy()[0]
    assert rel(sch[tids], z["schur"]) <= MATVEC_TOL
    rhs = op.rhs().cpu().numpy()[0]
    assert rel(rhs[tids], z["rhs"]) <= MATVEC_TOL


@pytest.mark.parametrize("cfg", [1, 4])
def test_solve_full_from_config_matches_golden(cfg):
    """solve_full(config): assembly, SVD, GMRES and recovery all on the device
    reproduce the oracle's Bragg coefficients and flux balance."""
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(cfg)
    z = np.load(os.path.join(O.GOLDEN, f"golden_cfg{cfg}.npz"))
    conf = workloads.fixture_config(workloads.CONFIGS[cfg]["system"])
    sol = solver.solve_full(conf, pb.centers, pb.p, smat=pb.smat, device=0)
    assert rel(sol.c[0], z["c"]) <= 1e-9 and rel(sol.d[0], z["d"]) <= 1e-9
    assert abs(sol.flux[0]["error"] - float(z["flux_error"])) <= 1e-9
    assert abs(sol.iterations[0] - int(z["iterations"])) <= 1
    assert sol.timings["assemble_ms"] > 0 and sol.timings["svd_ms"] > 0


def test_setup_rejects_mixed_geometry_and_bad_angle():
    from paper_1412_7466_b200 import grating
    a = workloads.fixture_config("w10")
    b = workloads.fixture_config("wood")
    with pytest.raises(ValueError):
        _setup([a, b])
    bad = grating.baseline_config(10.0, 0.3)
    with pytest.raises(ValueError):
        _setup([bad])


@pytest.mark.parametrize("from_config", [False, True])
def test_curved_grating_solve_matches_oracle(from_config):
    """cfg1's inclusions in the grating with sinusoidal interfaces (the
    reference's default InterfaceSpecs): Schur matvec and full solve, from the
    reference's host system or from the config (device assembly of the curved
    Nystrom blocks), vs the oracle (oracle/make_goldens.py curved)."""
    import torch

    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, solver
    pb = O.load_problem(1)
    z = np.load(os.path.join(O.GOLDEN, "golden_curved.npz"))
    systems = workloads.fixture_config("curved") if from_config else workloads.load_fixture("curved")
    op = solver.SchurOperator(systems, pb.centers, pb.p, smat=pb.smat, device=0)
    got = op(torch.as_tensor(z["v"][None]).cuda()).cpu().numpy()[0]
    assert rel(got, z["schur"]) <= MATVEC_TOL
    sol = solver.solve_full(systems, pb.centers, pb.p, smat=pb.smat, device=0)
    assert rel(sol.c[0], z["c"]) <= 1e-9 and rel(sol.d[0], z["d"]) <= 1e-9
    assert abs(sol.flux[0]["error"] - float(z["flux_error"])) <= 1e-9
    assert abs(sol.iterations[0] - int(z["iterations"])) <= 1


def test_setup_argument_errors():
    """ps_setup_empty / ps_scattering_matrix reject bad input with the
    reference's ValueError semantics instead of computing garbage."""
    import ctypes

    from paper_1412_7466_b200 import _lib, grating
    from paper_1412_7466_b200 import empty_setup as es
    from paper_1412_7466_b200.engine import Engine
    cfg = workloads.fixture_config("w10")
    eng = Engine(0)
    try:
        eng.set_geometry(np.array([[0.0, 0.0]]), 2, cfg.k2)
        eng.set_bloch([cfg.bloch_phase])
        desc, keep = es.build_desc(cfg, es.unit_cell(cfg))
        th = np.array([cfg.incident_angle])
        bad = _lib.EmptyDesc.from_buffer_copy(desc)
        bad.nrb = 40                                  # even Rayleigh-Bloch count (geo:357-358)
        rc = eng.lib.ps_setup_empty(eng.ctx, ctypes.byref(bad), th.ctypes.data_as(ctypes.c_void_p))
        assert rc == _lib.PS_ERR_ARG
        bad = _lib.EmptyDesc.from_buffer_copy(desc)
        bad.k2 = -1.0
        rc = eng.lib.ps_setup_empty(eng.ctx, ctypes.byref(bad), th.ctypes.data_as(ctypes.c_void_p))
        assert rc == _lib.PS_ERR_ARG
        bad = _lib.EmptyDesc.from_buffer_copy(desc)
        bad.g1.n = 16                                 # < 4 * skip nodes (quadrature.py:127-128)
        rc = eng.lib.ps_setup_empty(eng.ctx, ctypes.byref(bad), th.ctypes.data_as(ctypes.c_void_p))
        assert rc == _lib.PS_ERR_ARG
        with pytest.raises(_lib.PeriscatError):
            eng._check(eng.lib.ps_get_empty(eng.ctx, 3, None, None, None, None))
        # a valid call still works on the same context afterwards
        eng._check(eng.lib.ps_setup_empty(eng.ctx, ctypes.byref(desc),
                                          th.ctypes.data_as(ctypes.c_void_p)))
        del keep
    finally:
        eng.close()


def test_setup_split_and_factor_exchange():
    """The multi-GPU setup split on one device: two contexts each factorise
    half of cfg5's 16 angles (ps_setup_empty_range) and exchange the packed
    A^+ factors (ps_export_pinv / ps_import_pinv -- what
    parallel.setup_empty_split broadcasts over NCCL); both then apply the same
    16-RHS Schur operator as a context that factorised everything."""
    import torch

    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, solver
    from paper_1412_7466_b200.engine import Engine
    pb = O.load_problem(1)
    cfgs = [workloads.fixture_config(n) for n in workloads.CFG5_ANGLES]
    ref = solver.SchurOperator(cfgs, pb.centers, pb.p, smat=pb.smat, device=0)
    engs = [Engine(0), Engine(0)]
    ops = []
    for i, e in enumerate(engs):
        e.set_geometry(pb.centers, pb.p, cfgs[0].k2, cfgs[0].period, cfgs[0].near_field_copies)
        e.set_bloch([c.bloch_phase for c in cfgs])
        e.set_smatrix(pb.smat)
        e.setup_empty(cfgs, rhs_range=(8 * i, 8 * i + 8))
    buf = torch.empty(engs[0].pinv_bytes(), dtype=torch.uint8, device="cuda")
    for q in range(16):
        src, dst = (engs[0], engs[1]) if q < 8 else (engs[1], engs[0])
        src.export_pinv(q, buf)
        dst.import_pinv(q, buf)
    rng = np.random.default_rng(4)
    v = torch.as_tensor(pb.smat[None, None, :] * (rng.standard_normal((16, pb.M, pb.L))
                                                 + 1j * rng.standard_normal((16, pb.M, pb.L)))).cuda()
    want = ref(v).cpu().numpy()
    for e in engs:
        got = e.apply_schur(v).cpu().numpy()
        assert rel(got, want) <= 1e-14
        e.close()


@pytest.mark.parametrize("name,golden", [("w10", "golden_cfg1.npz"), ("curved", "golden_curved.npz")])
@pytest.mark.parametrize("from_config", [False, True])
def test_layer_fields_match_reference_evaluator(name, golden, from_config):
    """Device layer fields (ps_recover_full + ps_layer_field) of the golden
    coupled solution vs the reference's own empty_grating.eval_empty_field
    (eg:352-393, total=True) at grid points of all three layers
    (oracle/make_fields.py), from host reference factors and from the config."""
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, postproc, solver
    pb = O.load_problem(1)
    z = np.load(os.path.join(O.GOLDEN, f"field_{name}.npz"))
    systems = workloads.fixture_config(name) if from_config else workloads.load_fixture(name)
    op = solver.SchurOperator(systems, pb.centers, pb.p, smat=pb.smat, device=0)
    got = postproc.empty_field(op, z["beta"][None], z["pts"], z["layer"])[0]
    ref = z["field"]
    for ly in (1, 2, 3):
        sel = z["layer"] == ly
        assert rel(got[sel], ref[sel]) <= 1e-10, (ly, rel(got[sel], ref[sel]))


@pytest.mark.parametrize("from_config", [False, True])
def test_no_inclusions_reduces_to_empty_grating(from_config):
    """M = 0 (SPEC.md:545-547 degeneracy): solve_full returns the empty
    grating's own solution x = A^+ f (empty_grating.solve_empty, eg:276-290)
    and its flux balance."""
    from paper_1412_7466_b200 import grating, postproc, solver
    ref = workloads.load_fixture("w10")
    u, s, vh = np.linalg.svd(ref.matrix, full_matrices=False)
    x = ref.col_scale * (vh.conj().T @ (np.minimum(1 / s, 1e10) * (u.conj().T @ ref.rhs)))
    c_ref, d_ref = x[ref.cols["c"]], x[ref.cols["d"]]
    systems = workloads.fixture_config("w10") if from_config else ref
    sol = solver.solve_full(systems, np.zeros((0, 2)), 20, radius=0.04, device=0)
    assert sol.iterations[0] == 0
    assert rel(sol.c[0], c_ref) <= 1e-12 and rel(sol.d[0], d_ref) <= 1e-12
    fl = postproc.flux_error(c_ref, d_ref, ref.config)["error"]
    assert abs(sol.flux[0]["error"] - fl) <= 1e-12 and fl < 1e-12

"""GPU: the device-resident Krylov driver (krylov.gmres_device, ps_krylov_*)
for arbitrary device operators and for the multi-rank GMRES
(parallel.gmres_dist), including several processes sharing cuda:0 over
gloo (host-staged collectives), against direct solves and the oracle's
golden solutions."""
import os
import socket

import numpy as np
import pytest

from conftest import rel
import workloads  # noqa: E402

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dense(n, nrhs, seed):
    rng = np.random.default_rng(seed)
    A = np.eye(n) * 4 + (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    b = rng.standard_normal((nrhs, n)) + 1j * rng.standard_normal((nrhs, n))
    return A, b


@pytest.mark.parametrize("nrhs", [1, 3])
def test_gmres_random_dense_50_vs_direct(nrhs):
    """a random well-conditioned 50x50 dense operator; GMRES
    agrees with the direct solve to 1e-9, history nonincreasing."""
    from paper_1412_7466_b200 import solver
    A, b = _dense(50, nrhs, 5 + nrhs)
    Ad = torch.as_tensor(A).cuda()
    x, its, hist = solver.gmres(lambda v: v @ Ad.T, torch.as_tensor(b).cuda(), 1e-12, 60)
    ref = np.linalg.solve(A, b.T).T
    for r in range(nrhs):
        assert rel(x[r].cpu().numpy(), ref[r]) <= 1e-9
        h = hist[r]
        assert len(h) == its[r] + 1 and h[-1] <= 1e-12
        assert all(b_ <= a_ * (1 + 1e-12) for a_, b_ in zip(h, h[1:]))


def test_gmres_generic_host_arrays_and_identity():
    """Host arrays round-trip; the identity converges in one iteration."""
    from paper_1412_7466_b200 import solver
    b = np.random.default_rng(1).standard_normal((2, 7, 3)) + 0j
    x, its, hist = solver.gmres(lambda v: v.clone(), b, 1e-12, 10)
    assert isinstance(x, np.ndarray) and its == [1, 1]
    assert rel(x, b) < 1e-14


def test_gmres_generic_nan_and_nonconvergence():
    from paper_1412_7466_b200 import solver
    A, b = _dense(30, 1, 9)
    Ad = torch.as_tensor(A).cuda()
    x, its, hist = solver.gmres(lambda v: v @ Ad.T, torch.as_tensor(b).cuda(), 1e-15, 4)
    assert its == [4] and hist[0][-1] > 1e-15            # reported, not raised
    bad = torch.as_tensor(b).cuda()
    bad[0, 3] = float("nan")
    with pytest.raises(FloatingPointError):
        solver.gmres(lambda v: v @ Ad.T, bad, 1e-10, 5)

    def poisoned(v):
        y = v @ Ad.T
        y[0, 0] = float("inf")
        return y
    with pytest.raises(FloatingPointError):
        solver.gmres(poisoned, torch.as_tensor(b).cuda(), 1e-10, 5)


def test_gmres_dist_world1_multi_rhs_matches_ps_gmres():
    """The host-driven device GMRES (parallel.gmres_dist, world 1) with three
    RHS gives the all-in-C ps_gmres answer: same iterations, same x."""
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, parallel, solver
    pb = O.load_problem(2)
    systems = [workloads.load_fixture(n) for n in ("w10", "w10_a00", "w10_a15")]
    op = solver.SchurOperator(systems, pb.centers, pb.p, smat=pb.smat)
    rhs = op.rhs()
    x0, its0, hist0 = solver.gmres(op, rhs, 1e-10, 150)
    x1, its1, hist1 = parallel.gmres_dist(op, rhs, 1e-10, 150, engine=op.eng)
    assert its0 == its1
    for r in range(3):
        assert rel(x1[r].cpu().numpy(), x0[r].cpu().numpy()) <= 1e-12
        assert np.allclose(hist0[r], hist1[r], rtol=1e-9, atol=1e-16)


# ---------------------------------------------------------------- several
# processes on cuda:0 (gloo; collectives staged through host copies)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _sharded_body(rank, world, cfg)))
    except Exception as e:      # reported to the parent instead of hanging it
        import traceback
        q.put((rank, "ERR " + repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _sharded_body(rank, world, cfg):
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, parallel, solver
    pb = O.load_problem(cfg)
    t0, t1 = parallel.shard_range(pb.M, rank, world)
    op = solver.SchurOperator(workloads.load_fixture(O.CONFIGS[cfg]["empty"]), pb.centers, pb.p,
                              smat=pb.smat, target_range=(t0, t1))
    rng = np.random.default_rng(11)
    v = pb.smat[None, None, :] * (rng.standard_normal((1, pb.M, pb.L))
                                  + 1j * rng.standard_normal((1, pb.M, pb.L)))
    v_own = torch.as_tensor(v[:, t0:t1].copy()).cuda()
    out = {"t": (t0, t1), "matvec": {}}
    for mode in ("targets", "pairs"):
        sh = parallel.ShardedSchur(op, mode=mode, overlap=False)
        out["matvec"][mode] = sh(v_own).cpu().numpy()
        op.eng.set_k1_reserve(0)
    sh = parallel.ShardedSchur(op)
    x, its, hist = parallel.gmres_dist(sh, sh.rhs(), 1e-10, 150, engine=op.eng)
    xe = sh.recover(x.contiguous())
    c, d = op.split_cd(xe)
    out.update(c=c[0], d=d[0], its=its[0], mode=sh.mode)
    return out


@pytest.mark.parametrize("cfg,world", [(2, 2), (2, 3), (3, 2)])
def test_sharded_schur_and_gmres_multiprocess_one_gpu(cfg, world):
    """`world` processes on cuda:0: both M2L decompositions of the sharded
    Schur matvec reassemble the oracle golden matvec, and the distributed
    device GMRES reproduces the golden solve (c, d <= 1e-9, iterations +-1)."""
    import torch.multiprocessing as mp

    from oracle import periscat_oracle as O
    z = np.load(os.path.join(O.GOLDEN, f"golden_cfg{cfg}.npz"))
    pb = O.load_problem(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r, out in res.items():
        assert not isinstance(out, str), out
    # oracle matvec on the same seeded vector (golden-independent check)
    rng = np.random.default_rng(11)
    v = pb.smat[None, :] * (rng.standard_normal((pb.M, pb.L)) + 1j * rng.standard_normal((pb.M, pb.L)))
    if cfg == 3:
        sl = np.r_[0:6, 497:503, 994:1000]
    else:
        sl = np.arange(pb.M)
    ref = O.apply_schur_operator(pb, v, targets=sl).reshape(len(sl), pb.L)
    for mode in ("targets", "pairs"):
        full = np.concatenate([res[r]["matvec"][mode][0] for r in range(world)])
        assert rel(full[sl], ref) <= 1e-10, mode
    for r in range(world):
        out = res[r]
        assert rel(out["c"], z["c"]) <= 1e-9 and rel(out["d"], z["d"]) <= 1e-9
        assert abs(out["its"] - int(z["iterations"])) <= 1
    if cfg == 3:
        assert res[0]["mode"] == "pairs"
    for p in procs:
        assert p.exitcode == 0

"""The INTEGRATION.md bindings, exercised on the GPU: the pure-ctypes stub
(no torch) and the drop-in module shims, against the oracle goldens."""
import os

import numpy as np
import pytest

from conftest import rel
import workloads  # noqa: E402

pytestmark = pytest.mark.gpu


def test_ctypes_stub_apply_T_and_solve():
    from integration.ctypes_stub import Periscat
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating
    pb = O.load_problem(1)
    z = np.load(os.path.join(O.GOLDEN, "golden_cfg1.npz"))
    ps = Periscat(0)
    try:
        ps.setup(workloads.load_fixture("w10"), pb.centers, pb.p, pb.smat)
        aT = ps.apply_T(z["v"])[0]
        assert rel(aT, z["apply_T"]) <= 1e-10
        beta, c, d, its = ps.solve()
        assert rel(c[0], z["c"]) <= 1e-9 and rel(d[0], z["d"]) <= 1e-9
        assert abs(its[0] - int(z["iterations"])) <= 1
    finally:
        ps.close()


@pytest.mark.parametrize("mode,world", [("targets", 3), ("pairs", 2), ("pairs", 3)])
def test_ctypes_stub_sharded_schur_with_caller_collectives(mode, world):
    """A C / ctypes caller shards the Schur matvec through the C ABI alone,
    bringing its own collectives: world contexts with target
    slices, all-gather / all-reduce / reduce-scatter done by the caller (host
    arrays here), reassembled rows = the oracle golden (cfg2)."""
    from integration.ctypes_stub import Periscat, ShardedSchur, shard_range
    from oracle import periscat_oracle as O
    pb = O.load_problem(2)
    z = np.load(os.path.join(O.GOLDEN, "golden_cfg2.npz"))
    sysm = workloads.load_fixture(O.CONFIGS[2]["empty"])
    ranks = []
    try:
        for r in range(world):
            pc = Periscat(0)
            pc.setup(sysm, pb.centers, pb.p, pb.smat)
            pc.set_target_range(*shard_range(pb.M, r, world))
            ranks.append(pc)
        v = z["v"][None]
        blocks = [np.ascontiguousarray(v[:, pc.t0:pc.t1]) for pc in ranks]
        y = np.concatenate(ShardedSchur(ranks, mode)(blocks), axis=1)[0]
        assert rel(y, z["schur"]) <= 1e-10
    finally:
        for pc in ranks:
            pc.close()


class _Cv:
    """DiscretizedCurve duck type from empty_setup / scatmat rows."""
    def __init__(self, rows):
        self.nodes, self.normals = rows[:, 0:2], rows[:, 2:4]
        self.speeds, self.weights, self.t, self.arc_weights = rows[:, 4], rows[:, 5], rows[:, 6], rows[:, 7]

    @property
    def n(self):
        return self.nodes.shape[0]


class _Rule:
    def __init__(self, order):
        from paper_1412_7466_b200.empty_setup import correction_rule
        self.nodes, self.weights, self.skip, self.interp = correction_rule(order)


def test_ctypes_stub_setup_from_config_and_bie():
    """The stub's config path (ps_setup_empty) and Mueller-BIE call on
    reference-shaped objects: cfg1 solve vs the oracle golden; the rotated
    star solve vs its golden."""
    from integration.ctypes_stub import Periscat
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import empty_setup as es
    from paper_1412_7466_b200 import grating, scatmat
    pb = O.load_problem(1)
    cfg = workloads.fixture_config("w10")
    cell = es.unit_cell(cfg)
    curves = {"g1": _Cv(cell.g1), "g2": _Cv(cell.g2), "L1": _Cv(cell.walls[0]),
              "L2": _Cv(cell.walls[1]), "L3": _Cv(cell.walls[2]), "Gu": _Cv(cell.lid_up),
              "Gd": _Cv(cell.lid_down)}
    z = np.load(os.path.join(O.GOLDEN, "golden_cfg1.npz"))
    zs = np.load(os.path.join(O.GOLDEN, "golden_star.npz"))
    ps = Periscat(0)
    try:
        ps.setup_from_config([cfg], curves, _Rule(16), pb.centers, pb.p, pb.smat)
        beta, c, d, its = ps.solve()
        assert rel(c[0], z["c"]) <= 1e-9 and rel(d[0], z["d"]) <= 1e-9
        shape = scatmat.ParticleShape(0.03, 0.01, 3)
        S = ps.scattering_matrix(shape, 12.0, 15.0, 20, _Cv(scatmat.particle_curve(shape, 300)),
                                 _Rule(16))
        ps.setup_from_config([cfg], curves, _Rule(16), pb.centers, pb.p, S, rot=zs["rot"])
        beta, c, d, its = ps.solve()
        assert rel(c[0], zs["c"]) <= 1e-9 and rel(d[0], zs["d"]) <= 1e-9
    finally:
        ps.close()


def test_multiscat_shim_is_the_product():
    from integration.periscat_shim import multiscat
    from paper_1412_7466_b200 import multiscat as product
    assert multiscat.apply_T is product.apply_T


def test_sharded_driver_nccl_world1():
    """The multi-rank driver (NCCL group of size 1, device block kernels) on
    cfg2 reproduces the oracle golden solve."""
    import socket

    import torch
    import torch.distributed as dist

    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import grating, parallel, solver
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        pb = O.load_problem(2)
        z = np.load(os.path.join(O.GOLDEN, "golden_cfg2.npz"))
        op = solver.SchurOperator(workloads.load_fixture("w10"), pb.centers, pb.p, smat=pb.smat,
                                  target_range=parallel.shard_range(pb.M, 0, 1), dense_gb=0.0)
        sh = parallel.ShardedSchur(op)
        x, its, hist = parallel.gmres_dist(sh, sh.rhs(), 1e-10, 150, engine=op.eng)
        xe = sh.recover(x.contiguous())
        c, d = op.split_cd(xe)
        assert rel(c[0], z["c"]) <= 1e-9 and rel(d[0], z["d"]) <= 1e-9
        assert abs(its[0] - int(z["iterations"])) <= 1
        # both decompositions with the overlapped stream schedule (M2L on a
        # high-priority stream, coupling + NCCL all-reduce beside it) give the
        # same matvec as the serial one
        rng = np.random.default_rng(3)
        v = torch.as_tensor(pb.smat[None, None, :] * (rng.standard_normal((1, pb.M, pb.L))
                            + 1j * rng.standard_normal((1, pb.M, pb.L)))).cuda()
        ref = sh(v).cpu().numpy()
        for mode in ("targets", "pairs"):
            sho = parallel.ShardedSchur(op, mode=mode, overlap=True)
            for _ in range(2):
                got = sho(v).cpu().numpy()
                assert rel(got, ref) <= 1e-12
            op.eng.set_k1_reserve(0)
    finally:
        dist.destroy_process_group()


def test_bench_multirank_path_two_ranks_one_gpu(tmp_path):
    """The driver's scaling run (bench.py under torchrun, N > 1) end to end
    with 2 ranks: here both on cuda:0 over gloo (PS_BENCH_ONE_GPU /
    PS_BENCH_BACKEND); checks the JSON line, the tile-pair decomposition and
    the distributed GMRES solve's flux balance."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PS_BENCH_ONE_GPU="1", PS_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-cfg5"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["parallelism"].startswith("tile-pair-sharded x2")
    fs = line["full_solve_m1000"]
    assert fs["iterations"] == 27 and abs(fs["flux_error"]) < 1e-9

"""Multi-rank host logic on CPU (gloo, world size 2): target sharding, the
row all-gather, all-reduce of complex partials, and the distributed GMRES
driver -- checked against a single-process solve of the same operator."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dense_problem(M=7, L=5, nrhs=2, seed=0):
    rng = np.random.default_rng(seed)
    n = M * L
    A = [np.eye(n) * 3 + 0.2 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
         for _ in range(nrhs)]
    b = rng.standard_normal((nrhs, M, L)) + 1j * rng.standard_normal((nrhs, M, L))
    return A, b


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, q)
    except Exception as e:  # report instead of hanging the parent on q.get
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, q):
    from paper_1412_7466_b200 import parallel
    M, L, nrhs = 7, 5, 2
    A, b = _dense_problem(M, L, nrhs)
    t0, t1 = parallel.shard_range(M, rank, world)
    # all-gather of uneven shards
    own = torch.as_tensor(b[:, t0:t1]).contiguous()
    full = parallel.all_gather_rows(own, M)
    assert np.array_equal(full.numpy(), b)
    # reduce-scatter of full-length partials (the "pairs" decomposition)
    part = torch.as_tensor(b * (rank + 1)).contiguous()
    mine = parallel.reduce_scatter_rows(part, M)
    assert np.allclose(mine.numpy(), (b * sum(range(1, world + 1)))[:, t0:t1])
    # complex all-reduce
    z = torch.tensor([1.0 + 2.0j * rank, -1.0j], dtype=torch.complex128)
    parallel.all_reduce_(z)
    assert np.allclose(z.numpy(), [world + 2j * sum(range(world)), -1j * world])

    def apply(v_own):
        vf = parallel.all_gather_rows(v_own, M).numpy()
        y = np.stack([(A[r] @ vf[r].reshape(-1)).reshape(M, L) for r in range(nrhs)])
        return torch.as_tensor(y[:, t0:t1]).contiguous()

    from host_krylov import HostKrylov
    x, its, hist = parallel.gmres_dist(apply, own, tol=1e-12, maxit=60, ops=HostKrylov())
    xf = parallel.all_gather_rows(x.contiguous(), M).numpy()
    q.put((rank, xf, its))


def test_gmres_dist_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, xf, its in res:
        assert its is not None, f"rank {rank}: {xf}"
    for p in procs:
        assert p.exitcode == 0
    A, b = _dense_problem()
    for rank, xf, its in res:
        for r in range(b.shape[0]):
            ref = np.linalg.solve(A[r], b[r].reshape(-1)).reshape(b.shape[1:])
            assert np.linalg.norm(xf[r] - ref) / np.linalg.norm(ref) < 1e-10
    assert np.array_equal(res[0][1], res[1][1])


def test_shard_ranges_partition():
    from paper_1412_7466_b200 import parallel
    for M in (1, 7, 1000, 10000):
        for world in (1, 2, 3, 4, 8):
            rs = [parallel.shard_range(M, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(parallel.shard_sizes(M, world)) - min(parallel.shard_sizes(M, world)) <= 1


def test_gmres_dist_single_process_matches_oracle_gmres():
    """World size 1 (no process group): same answer as the oracle's GMRES."""
    from oracle import periscat_oracle as O
    from paper_1412_7466_b200 import parallel
    A, b = _dense_problem(5, 3, 1, seed=3)
    from host_krylov import HostKrylov
    x, its, hist = parallel.gmres_dist(
        lambda v: torch.as_tensor((A[0] @ v.numpy()[0].reshape(-1)).reshape(1, 5, 3)),
        torch.as_tensor(b), tol=1e-12, maxit=40, ops=HostKrylov())
    xo, its_o, _ = O.gmres(lambda v: A[0] @ v, b[0].reshape(-1), 1e-12, 40)
    assert its[0] == its_o
    assert np.linalg.norm(x.numpy()[0].reshape(-1) - xo) / np.linalg.norm(xo) < 1e-12


def test_gmres_dist_has_no_cpu_fallback():
    """The product driver runs the Arnoldi step in the CUDA kernels only:
    host tensors without a test double are rejected, not computed on CPU."""
    from paper_1412_7466_b200 import parallel
    A, b = _dense_problem(5, 3, 1, seed=3)
    with pytest.raises((TypeError, ValueError)):
        parallel.gmres_dist(lambda v: v, torch.as_tensor(b), tol=1e-12, maxit=5)


class _FakeDist:
    """Thread-simulated collectives with NCCL's tensor semantics, to exercise
    the even-shard all_gather_into_tensor / reduce_scatter_tensor layouts of
    parallel.py (gloo on CPU takes the padded all_gather / all_reduce paths)."""

    def __init__(self, world):
        import threading
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world
        self.local = threading.local()

    def is_initialized(self):
        return True

    def get_backend(self, group=None):
        return "nccl"

    def get_world_size(self, group=None):
        return self.world

    def get_rank(self, group=None):
        return self.local.rank

    def _exchange(self, t):
        self.slots[self.local.rank] = t.clone()
        self.bar.wait()
        got = list(self.slots)
        self.bar.wait()
        return got

    def all_gather_into_tensor(self, out, inp, group=None):
        parts = self._exchange(inp)
        out.copy_(torch.stack(parts).reshape(out.shape))

    def reduce_scatter_tensor(self, out, inp, group=None):
        parts = self._exchange(inp)
        out.copy_(sum(p[self.local.rank] for p in parts))

    def all_gather(self, outs, inp, group=None):
        for o, p in zip(outs, self._exchange(inp)):
            o.copy_(p)

    def all_reduce(self, t, group=None):
        t.copy_(sum(self._exchange(t)))


@pytest.mark.parametrize("M,world", [(12, 3), (10, 4), (8, 2)])
def test_row_collectives_nccl_layout(monkeypatch, M, world):
    """all_gather_rows / reduce_scatter_rows with NCCL's output layouts, even
    and uneven shards, on fake 'CUDA' tensors (is_cuda forced) -- the layout
    ShardedSchur relies on at N > 1."""
    import threading

    from paper_1412_7466_b200 import parallel
    fake = _FakeDist(world)
    monkeypatch.setattr(parallel, "dist", fake)

    class T(torch.Tensor):   # a CPU tensor that reports is_cuda (layout only)
        @property
        def is_cuda(self):
            return True

    rng = np.random.default_rng(M)
    L, nrhs = 3, 2
    full = torch.as_tensor(rng.standard_normal((nrhs, M, L)) + 1j * rng.standard_normal((nrhs, M, L)))
    parts = [torch.as_tensor(rng.standard_normal((nrhs, M, L)) + 1j * rng.standard_normal((nrhs, M, L)))
             for _ in range(world)]
    out = [None] * world
    err = []

    def run(r):
        try:
            fake.local.rank = r
            t0, t1 = parallel.shard_range(M, r, world)
            g = parallel.all_gather_rows(full[:, t0:t1].contiguous().as_subclass(T), M)
            s = parallel.reduce_scatter_rows(parts[r].as_subclass(T), M)
            out[r] = (torch.Tensor(g).as_subclass(torch.Tensor), s.as_subclass(torch.Tensor))
        except Exception as e:   # surfaced below
            err.append(e)
            fake.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    total = sum(parts)
    for r in range(world):
        t0, t1 = parallel.shard_range(M, r, world)
        assert torch.equal(out[r][0], full)
        assert torch.allclose(out[r][1], total[:, t0:t1], rtol=0, atol=1e-13)

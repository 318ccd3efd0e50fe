"""Target-inclusion sharding across ranks.

Rank r owns target inclusions [M r / G, M (r+1) / G): their rows of the
coefficient vector, of T, S and B, and their slices of the Krylov basis.
Per Schur matvec:
  1. all-gather beta (NCCL over NVLink) -> full vector on every rank;
  2. partial g = C beta over the rank's own SOURCE inclusions, all-reduce;
  3. local y = v_own - S (T v - B A^+ g): either K1 over all sources for the
     own targets, or (one RHS) the symmetric K1s over 1/world of the tile
     pairs for all targets followed by a reduce-scatter (ShardedSchur).
GMRES dot products are local partial sums followed by an all-reduce; the
Hessenberg / Givens update (O(k) scalars per RHS) is replicated on every
rank's device (krylov.gmres_device).

Collectives run on the device with NCCL; with any other backend (gloo: the
multi-process tests, including several ranks sharing one GPU) they stage
through host copies.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(M: int, rank: int, world: int) -> tuple[int, int]:
    return (M * rank) // world, (M * (rank + 1)) // world


def shard_sizes(M: int, world: int) -> list[int]:
    return [shard_range(M, r, world)[1] - shard_range(M, r, world)[0] for r in range(world)]


def _world(group) -> int:
    return dist.get_world_size(group) if dist.is_initialized() else 1


def _device_collectives(t: torch.Tensor, group) -> bool:
    """NCCL moves CUDA tensors itself; any other backend (gloo: the
    multi-process tests, several ranks sharing one GPU) gets host copies."""
    return t.is_cuda and dist.get_backend(group) == "nccl"


def all_gather_rows(v_own: torch.Tensor, M: int, group=None) -> torch.Tensor:
    """[nrhs][M_own][L] on every rank -> [nrhs][M][L] (rows in rank order)."""
    world = _world(group)
    if world == 1:
        return v_own
    sizes = shard_sizes(M, world)
    dev = v_own.device
    vr = torch.view_as_real(v_own.contiguous())          # complex -> (..., 2) float64
    on_dev = _device_collectives(vr, group)
    if not on_dev:
        vr = vr.cpu()
    if len(set(sizes)) == 1 and on_dev:
        buf = torch.empty((world,) + tuple(vr.shape), dtype=vr.dtype, device=vr.device)
        dist.all_gather_into_tensor(buf, vr, group=group)
        full = buf.permute(1, 0, 2, 3, 4).reshape(v_own.shape[0], M, v_own.shape[2], 2)
        return torch.view_as_complex(full.contiguous())
    # uneven shards (or host staging): pad every rank's rows to the largest
    # shard, gather, trim
    mx = max(sizes)
    pad = torch.zeros((v_own.shape[0], mx, v_own.shape[2], 2), dtype=vr.dtype, device=vr.device)
    pad[:, :vr.shape[1]] = vr
    parts = [torch.empty_like(pad) for _ in sizes]
    dist.all_gather(parts, pad, group=group)
    full = torch.cat([p[:, :s] for p, s in zip(parts, sizes)], dim=1)
    return torch.view_as_complex(full.contiguous()).to(dev)


def reduce_scatter_rows(x_full: torch.Tensor, M: int, group=None) -> torch.Tensor:
    """[nrhs][M][L] partial sums on every rank -> this rank's rows
    shard_range(M, rank, world) of the sum over ranks (NCCL reduce-scatter;
    uneven shards are padded; other backends sum with an all-reduce of host
    copies and slice)."""
    world = _world(group)
    if world == 1:
        return x_full
    rank = dist.get_rank(group)
    t0, t1 = shard_range(M, rank, world)
    xr = torch.view_as_real(x_full.contiguous())
    if not _device_collectives(xr, group):
        h = xr.cpu()
        dist.all_reduce(h, group=group)
        return torch.view_as_complex(h)[:, t0:t1].contiguous().to(x_full.device)
    sizes = shard_sizes(M, world)
    mx = max(sizes)
    if len(set(sizes)) == 1:
        inp = xr.reshape(xr.shape[0], world, mx, *xr.shape[2:]).transpose(0, 1).contiguous()
    else:
        inp = torch.zeros((world, xr.shape[0], mx) + tuple(xr.shape[2:]), dtype=xr.dtype,
                          device=xr.device)
        for r in range(world):
            a, b = shard_range(M, r, world)
            inp[r, :, :b - a] = xr[:, a:b]
    out = torch.empty(inp.shape[1:], dtype=xr.dtype, device=xr.device)
    dist.reduce_scatter_tensor(out, inp, group=group)
    return torch.view_as_complex(out[:, :t1 - t0].contiguous())


def all_reduce_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (complex tensors as their real view)."""
    if _world(group) == 1:
        return t
    tr = torch.view_as_real(t) if t.is_complex() else t
    if _device_collectives(tr, group):
        dist.all_reduce(tr, group=group)
    else:
        h = tr.cpu()
        dist.all_reduce(h, group=group)
        tr.copy_(h)
    return t


def broadcast_(t: torch.Tensor, src: int, group=None) -> torch.Tensor:
    """In-place broadcast from group rank ``src``."""
    if _world(group) == 1:
        return t
    gsrc = src if group is None else dist.get_global_rank(group, src)
    if _device_collectives(t, group):
        dist.broadcast(t, src=gsrc, group=group)
    else:
        h = t.cpu()
        dist.broadcast(h, src=gsrc, group=group)
        t.copy_(h)
    return t


def setup_empty_split(eng, configs, group=None):
    """Multi-GPU empty-grating setup ("each rank does 2 of the
    16 RHS SVDs, then broadcasts"): every rank assembles all RHS on its device
    (one launch, ~1 ms) but factorises only its share shard_range(R, rank,
    world); each RHS's packed A^+ factors (15 MB at the BASELINE geometry) are
    then broadcast from the owning rank over NCCL."""
    world = _world(group)
    R = len(configs)
    if world == 1 or R == 1:
        return eng.setup_empty(configs)
    rank = dist.get_rank(group)
    systems = eng.setup_empty(configs, rhs_range=shard_range(R, rank, world))
    buf = torch.empty(eng.pinv_bytes(), dtype=torch.uint8, device=eng.device)
    for q in range(R):
        owner = next(r for r in range(world) if shard_range(R, r, world)[0] <= q
                     < shard_range(R, r, world)[1])
        if owner == rank:
            eng.export_pinv(q, buf)
        broadcast_(buf, owner, group)
        if owner != rank:
            eng.import_pinv(q, buf)
    return systems


class ShardedSchur:
    """Distributed S-preconditioned Schur operator on top of a SchurOperator
    whose engine owns targets shard_range(M, rank, world).

    Two decompositions of the M2L (both with the same all-gather of beta and
    the same C / B coupling split):
      * "targets": every rank runs the tiled K1 for its own targets over all
        sources (no M2L exchange);
      * "pairs" (one RHS, M >= 512 and M / world >= 100, the default there):
        every rank runs the symmetric K1s over 1/world of the unordered tile
        pairs -- each symbol row serves a pair and its reverse, half the
        producer work of the tiled kernel -- for ALL targets, and a
        reduce-scatter sums the parts into each rank's own rows
        (ps_apply_T_blocks / ps_schur_finish).
    """

    def __init__(self, op, group=None, mode: str = "auto", overlap="auto", reserve: int = 4):
        self.op = op
        self.group = group
        self.world = _world(group)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.t0, self.t1 = shard_range(op.M, self.rank, self.world)
        self.s_range = (self.t0, self.t1)     # own sources for the C partial sum
        if mode == "auto":
            # measured per-rank compute at cfg3 (tools/probe_shard.py, K1s
            # with its symbol store): pairs wins at 2, 4 and 8 ranks (1.02 vs
            # 1.33 ms, 0.57 vs 0.70 ms, 0.325 vs 0.377 ms); without the store
            # the tiled target split won at 8 -> pairs while M / world >= 100
            mode = "pairs" if (op.nrhs == 1 and self.world > 1 and op.M >= 512
                               and op.M >= 100 * self.world) else "targets"
        if mode not in ("pairs", "targets"):
            raise ValueError(f"unknown decomposition {mode!r}")
        self.mode = mode
        # overlap of the M2L with the coupling chain + its all-reduce (one RHS,
        # CUDA, diagonal or dense S): K1/K1s leave `reserve` SMs to the chain
        want = (self.world > 1) if overlap == "auto" else bool(overlap)
        self.overlap = (want and op.nrhs == 1 and op.coupled
                        and str(op.device).startswith("cuda"))
        if self.overlap:
            self.s_hi = torch.cuda.Stream(device=op.device, priority=-1)
            shape = (1, op.M if mode == "pairs" else self.t1 - self.t0, op.L)
            self._a_buf = torch.empty(shape, dtype=torch.complex128, device=op.device)
            op.eng.set_k1_reserve(reserve)

    def _coupling(self, v_full):
        if not self.op.coupled:
            return None
        g = self.op.eng.apply_C(v_full, s_range=self.s_range)
        all_reduce_(g, self.group)
        return g

    def __call__(self, v_own: torch.Tensor, out=None) -> torch.Tensor:
        v_full = all_gather_rows(v_own, self.op.M, self.group)
        if self.overlap:
            return self._call_overlapped(v_own, v_full, out)
        if self.mode == "pairs":
            a_part = self.op.eng.apply_T_blocks(v_full, self.rank, self.world)
            a_own = reduce_scatter_rows(a_part, self.op.M, self.group)
            g = self._coupling(v_full)
            return self.op.eng.schur_finish(v_own.contiguous(), a_own, g, out=out)
        g = self._coupling(v_full)
        if g is None:
            return self.op(v_full, out=out)
        return self.op(v_full, out=out, g=g)

    def _call_overlapped(self, v_own, v_full, out):
        """One RHS on CUDA: the M2L runs on a high-priority stream with
        `reserve` SMs left free, while the coupling chain (C partial over own
        sources, NCCL all-reduce) runs on the caller's stream on those SMs;
        the epilogue joins both (the reduce-scatter of the pairs split waits
        for the M2L part only)."""
        eng = self.op.eng
        cur = torch.cuda.current_stream(v_full.device)
        fork = torch.cuda.Event()
        fork.record(cur)
        v_full.record_stream(self.s_hi)
        with torch.cuda.stream(self.s_hi):
            self.s_hi.wait_event(fork)
            if self.mode == "pairs":
                a = eng.apply_T_blocks(v_full, self.rank, self.world, out=self._a_buf)
            else:
                a = eng.apply_T(v_full, out=self._a_buf)
            done = torch.cuda.Event()
            done.record(self.s_hi)
        g = self._coupling(v_full)
        cur.wait_event(done)
        a_own = reduce_scatter_rows(a, self.op.M, self.group) if self.mode == "pairs" else a
        return eng.schur_finish(v_own.contiguous(), a_own, g, out=out)

    def rhs(self) -> torch.Tensor:
        return self.op.rhs()

    def recover(self, beta_own: torch.Tensor) -> torch.Tensor:
        v_full = all_gather_rows(beta_own, self.op.M, self.group)
        g = self.op.eng.apply_C(v_full, s_range=self.s_range)
        all_reduce_(g, self.group)
        return self.op.eng.recover(g)


def gmres_dist(apply, rhs_own: torch.Tensor, tol: float = 1e-10, maxit: int = 150,
               group=None, engine=None, ops=None):
    """Unrestarted GMRES over target-sharded vectors: CGS2
    Arnoldi, zero initial guess, per-RHS stopping, with the Arnoldi vectors,
    the Hessenberg / Givens state and the least-squares solve all on the
    device (krylov.gmres_device).  Per iteration: two all-reduces of the
    [nrhs][k+1] CGS2 columns, one of the [nrhs] squared norms, one
    device->host read of the residuals.  ``apply(v_own) -> y_own`` does its
    own communication.  Returns (x_own, iterations, histories)."""
    from .krylov import gmres_device
    return gmres_device(apply, rhs_own, tol, maxit, engine=engine,
                        reduce=lambda t: all_reduce_(t, group), ops=ops)

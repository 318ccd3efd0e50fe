"""Process-parallel evaluation of the oracle at cfg5 size (test
infrastructure only).

The oracle's apply_T over a target slice and apply_C over all M sources are
sums of independent per-target / per-source terms (periscat_oracle.py,
restating SPEC.md:494-512), so they split over host processes: targets in
contiguous chunks, sources in contiguous chunks whose partial 576-row sums
are added in chunk order (a fixed order: the result does not depend on the
worker count's scheduling).  Workers are spawned (never forked: the callers
run after CUDA threads exist) and pin BLAS to one thread.
"""
from __future__ import annotations

import os

import numpy as np

_STATE: dict = {}


def _init(state):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    _STATE.update(state)


def _t_chunk(idx):
    from oracle import periscat_oracle as O
    s = _STATE
    return O.apply_T(s["beta"], s["centers"], s["k"], s["p"], s["bloch"], s["period"],
                     s["copies"], targets=np.asarray(idx))


def _c_chunk(rng):
    from oracle import periscat_oracle as O
    a, b = rng
    s = _STATE
    return O.apply_C(s["es"], s["beta"][a:b], s["centers"][a:b])


def nproc_default() -> int:
    return max(1, min(32, len(os.sched_getaffinity(0))))


def _pool(nproc, state):
    import multiprocessing as mp
    # the spawned children import numpy before any initializer runs: pin
    # their BLAS to one thread through the environment they inherit (else
    # nproc x ncore BLAS threads thrash: 15x slower than one process)
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    return mp.get_context("spawn").Pool(nproc, initializer=_init, initargs=(state,))


def apply_T(beta, centers, k, p, bloch, period, copies, targets, nproc=None):
    """periscat_oracle.apply_T(..., targets=targets) over nproc processes."""
    nproc = nproc or nproc_default()
    targets = np.asarray(targets)
    chunks = [c for c in np.array_split(targets, nproc) if c.size]
    state = dict(beta=beta, centers=centers, k=k, p=p, bloch=bloch, period=period,
                 copies=copies)
    with _pool(len(chunks), state) as pool:
        parts = pool.map(_t_chunk, chunks)
    return np.concatenate(parts, axis=-2)


def apply_C(es, beta, centers, nproc=None, reverse_sources=False):
    """periscat_oracle.apply_C over source chunks, partial sums in chunk order
    (reverse_sources: the sources taken in reverse order -- the same operator
    summed in another, equally valid float64 order)."""
    nproc = nproc or nproc_default()
    if reverse_sources:
        beta, centers = beta[::-1].copy(), centers[::-1].copy()
    M = centers.shape[0]
    bounds = np.linspace(0, M, min(nproc, M) + 1).astype(int)
    rngs = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    with _pool(len(rngs), dict(es=es, beta=beta, centers=centers)) as pool:
        parts = pool.map(_c_chunk, rngs)
    g = np.zeros_like(parts[0])
    for q in parts:
        g += q
    return g


def apply_schur_operator(pb, v, targets, nproc=None, reverse_sources=False):
    """periscat_oracle.apply_schur_operator(pb, v, targets=targets) with the
    T slice and C v split over processes."""
    from oracle import periscat_oracle as O
    v = np.asarray(v, dtype=complex).reshape(pb.M, pb.L)
    es = pb.es
    tidx = np.arange(pb.M)[targets]
    u = apply_T(v, pb.centers, es.k2, pb.p, es.bloch, es.period, es.copies, tidx, nproc)
    x = es.apply_pinv(apply_C(es, v, pb.centers, nproc, reverse_sources))
    u = u - O.apply_B_phys(es, x, pb.centers[tidx], pb.p)
    sub = O.Problem(es, pb.centers[tidx], pb.p, pb.radius, pb.smat,
                    None if pb.rot is None else pb.rot[tidx])
    return v[tidx] - sub.apply_S(u)

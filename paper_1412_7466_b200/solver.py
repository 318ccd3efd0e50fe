"""Coupled solve on the B200 (solver).

``SchurOperator`` is the device-resident S-preconditioned Schur operator
    K v = v - S T v + S B_phys A^+ C v         (paper B = -B_phys)
for one or more right-hand sides (incidence angles sharing k2); ``gmres``
runs the device GMRES of libperiscat_b200.so; ``solve_full`` mirrors
SPEC.md:559-567.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import postproc
from .engine import Engine
from .scatmat import disk_scattering_matrix


@dataclass
class _ConfigOnly:
    config: object


class SchurOperator:
    def __init__(self, systems, centers, p: int, smat=None, radius: float | None = None,
                 rot=None, device=None, target_range=None, coupled: bool = True,
                 engine: Engine | None = None, dense_gb: float = 40.0, group=None,
                 split_setup: bool = False):
        """``radius``: the disk radius (builds the diagonal S when ``smat`` is
        None) or, with a given ``smat``, the enclosing radius; either way the
        inclusions are checked for overlap on the device.
        ``split_setup`` (opt-in, collective): with configs and several
        RHS, every rank of ``group`` factorises only its share of the
        per-angle SVDs and the factors are broadcast
        (parallel.setup_empty_split); all ranks of the group must construct
        the operator together.  Without it the constructor never
        communicates."""
        if not isinstance(systems, (list, tuple)):
            systems = [systems]
        items = list(systems)
        # empty-grating systems with host factors (EmptyGratingSystem /
        # GratingSystem), or configs (ProblemConfig / GratingConfig) whose
        # system is assembled and factorised on the device (ps_setup_empty)
        self.device_setup = not hasattr(items[0], "matrix")
        configs = items if self.device_setup else [s.config for s in items]
        cfg = configs[0]
        self.config = cfg
        for c in configs[1:]:
            if (c.k2, c.period, c.near_field_copies) != (cfg.k2, cfg.period, cfg.near_field_copies):
                raise ValueError("batched right-hand sides must share k2, period and copies")
        if smat is None:
            if radius is None:
                raise ValueError("give a scattering matrix or a disk radius")
            smat = disk_scattering_matrix(radius, cfg.k2, cfg.kp, p)
        self.smat = np.asarray(smat, dtype=complex)
        self.eng = engine or Engine(device)
        eng = self.eng
        self.centers = np.ascontiguousarray(np.asarray(centers, dtype=float).reshape(-1, 2))
        eng.set_geometry(self.centers, p, cfg.k2, cfg.period, cfg.near_field_copies)
        if radius is not None:
            # overlapping enclosing disks -> DomainError (
            # ParticleSet.min_gap semantics, geometry.py:131-144)
            self.min_gap = eng.check_overlap(radius)
        eng.set_bloch([c.bloch_phase for c in configs])
        eng.set_smatrix(self.smat, rot)
        self.coupled = coupled
        self.systems = items
        if coupled:
            if self.device_setup and split_setup:
                from .parallel import setup_empty_split
                self.systems = setup_empty_split(eng, configs, group)
            elif self.device_setup:
                self.systems = eng.setup_empty(configs)
            else:
                eng.set_layers(items[0])
                for r, s in enumerate(items):
                    eng.set_pinv(r, s)
                if hasattr(cfg, "expansion_centers"):     # layer fields (ps_layer_field)
                    eng.set_field_params(configs)
        elif self.device_setup:
            self.systems = [_ConfigOnly(c) for c in configs]
        if target_range is not None:
            eng.set_target_range(*target_range)
        # pre-assembled B / C blocks when they fit (else matrix-free K3/K5)
        self.dense = bool(coupled and dense_gb > 0 and eng.M > 0
                          and eng.precompute_coupling(dense_gb))
        self.M, self.p, self.L, self.nrhs = eng.M, p, eng.L, eng.nrhs
        self.device = eng.device

    @property
    def shape(self):
        return (self.nrhs, self.M, self.L)

    def __call__(self, v: torch.Tensor, out=None, g=None) -> torch.Tensor:
        return self.eng.apply_schur(v, out=out, g=g)

    def apply_T(self, v: torch.Tensor, out=None) -> torch.Tensor:
        return self.eng.apply_T(v, out=out)

    def rhs(self) -> torch.Tensor:
        if not self.coupled:
            raise RuntimeError("uncoupled operator has no layer right-hand side")
        return self.eng.schur_rhs()

    def recover(self, beta: torch.Tensor):
        """x_empty restricted to (B columns, c, d) = A^+ (f - C beta) per RHS."""
        g = self.eng.apply_C(beta)
        x = self.eng.recover(g)
        return x

    def split_cd(self, x: torch.Tensor):
        nb, nrb = self.eng.ncol_b, self.eng.nrb
        xh = x.cpu().numpy()
        return xh[:, nb:nb + nrb], xh[:, nb + nrb:nb + 2 * nrb]


def apply_schur_operator(op: SchurOperator, beta):
    """returns K beta.  Host arrays round-trip through the device."""
    on_host = not isinstance(beta, torch.Tensor)
    v = torch.as_tensor(np.asarray(beta, dtype=complex).reshape(op.shape) if on_host else beta)
    v = v.to(device=op.device, dtype=torch.complex128).contiguous()
    y = op(v)
    return y.cpu().numpy() if on_host else y


def gmres(op, rhs, tol: float = 1e-10, maxit: int = 150, engine: Engine | None = None):
    """Unrestarted device GMRES.  Returns (x, iterations per
    RHS, residual history per RHS).

    ``op`` is a SchurOperator owning all targets (the all-in-C driver
    ps_gmres) or any callable ``op(v) -> y`` on complex128 CUDA tensors of
    rhs's shape (krylov.gmres_device: the Arnoldi step still runs in the
    library kernels, on ``engine`` or op.eng or a fresh context).  Host
    arrays round-trip through the device."""
    on_host = not isinstance(rhs, torch.Tensor)
    if isinstance(op, SchurOperator) and op.eng.t_range == (0, op.M):
        r = torch.as_tensor(np.asarray(rhs, dtype=complex).reshape(op.shape) if on_host else rhs)
        r = r.to(device=op.device, dtype=torch.complex128).contiguous()
        x, its, hist = op.eng.gmres(r, tol, maxit)
        hist_l = [h[~np.isnan(h)].tolist() for h in hist]
        return (x.cpu().numpy() if on_host else x), its, hist_l
    from .krylov import gmres_device
    eng = engine or getattr(op, "eng", None)
    if on_host:
        dev = eng.device if eng is not None else torch.device("cuda", torch.cuda.current_device())
        r = torch.as_tensor(np.ascontiguousarray(np.asarray(rhs, dtype=complex))).to(dev)
    else:
        r = rhs.to(torch.complex128).contiguous()
    if eng is None:
        eng = Engine(r.device)
    x, its, hist = gmres_device(op, r, tol, maxit, engine=eng)
    return (x.cpu().numpy() if on_host else x), its, hist


@dataclass(frozen=True)
class Solution:
    """beta, the recovered empty-grating unknowns, GMRES
    iterations and final relative residual, flux error, wall-discrepancy
    residual (+ the coupled residual of SPEC.md:571).  Immutable."""
    beta: np.ndarray          # [nrhs][M][L]
    c: np.ndarray             # [nrhs][nrb]
    d: np.ndarray             # [nrhs][nrb]
    iterations: list
    history: list
    flux: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)
    x_empty: np.ndarray | None = None   # [nrhs][ncol] all empty-grating unknowns (eg:154-156)
    residual: list = field(default_factory=list)          # final GMRES relative residual
    coupled_residual: list = field(default_factory=list)  # SPEC.md:571 (postproc)
    wall_residual: list = field(default_factory=list)     # eg:396-433 (postproc)


def solve_full(systems, centers, p: int, radius: float | None = None, smat=None, rot=None,
               tol: float | None = None, maxit: int | None = None, device=None,
               diagnostics: bool = True) -> Solution:
    """beta from GMRES on (I - S T - S B A^+ C) beta = -S B A^+ f,
    then x_empty = A^+ (f - C beta); flux balance per RHS.

    ``systems``: one per RHS (incidence angle), either empty-grating systems
    carrying host SVD factors or configs (ProblemConfig / GratingConfig), in
    which case the empty-grating assembly and its SVD also run on the device
    (SPEC.md:559 ``solve_full(config)``)."""
    import time
    t0 = time.perf_counter()
    op = SchurOperator(systems, centers, p, smat=smat, radius=radius, rot=rot, device=device)
    torch.cuda.synchronize(op.device)
    t1 = time.perf_counter()
    cfg = op.config
    tol = cfg.gmres_tol if tol is None else tol
    maxit = cfg.gmres_maxit if maxit is None else maxit
    if op.M == 0:
        # no inclusions: the empty grating's own solution
        # x = A^+ f (empty_grating.solve_empty, eg:276-290)
        beta = torch.zeros(op.shape, dtype=torch.complex128, device=op.device)
        its, hist = [0] * op.nrhs, [[0.0] for _ in range(op.nrhs)]
        g = torch.zeros((op.nrhs, op.eng.nrow_c), dtype=torch.complex128, device=op.device)
        x = op.eng.recover(g)
    else:
        rhs = op.rhs()
        beta, its, hist = gmres(op, rhs, tol, maxit)
        x = op.recover(beta)
    c, d = op.split_cd(x)
    torch.cuda.synchronize(op.device)
    t2 = time.perf_counter()
    flux = [postproc.flux_error(c[r], d[r], s.config) for r, s in enumerate(op.systems)]
    timings = dict(setup=t1 - t0, solve=t2 - t1)
    if op.device_setup and op.coupled:
        timings["assemble_ms"], timings["svd_ms"] = op.eng.setup_timings()
    extra = {}
    if diagnostics and op.coupled:
        # after the timed solve: SPEC.md:534 / 571 diagnostics on the device
        t3 = time.perf_counter()
        xf = None
        if op.eng.lib.ps_full_columns(op.eng.ctx) > 0:
            bdev = beta if isinstance(beta, torch.Tensor) else torch.as_tensor(beta).to(op.device)
            xf = op.eng.recover_full(postproc._c_rows(op.eng, bdev.contiguous()))
            extra["x_empty"] = xf.cpu().numpy()
            extra["coupled_residual"] = [r["relative"] for r in
                                         postproc.coupled_residual(op, bdev, xf)]
            extra["wall_residual"] = postproc.wall_discrepancy_residual(op, bdev, x_full=xf)
        timings["diagnostics"] = time.perf_counter() - t3
    res = [h[-1] if h else float("nan") for h in hist]
    return Solution(beta.cpu().numpy(), c, d, its, hist, flux, timings, residual=res, **extra)

"""Device context: one ``ps_ctx`` per (process, GPU) holding the uploaded
geometry, scattering matrix, layer-coupling data and SVD factors.

Memory and streams come from PyTorch (complex128 CUDA tensors, the current
stream); all arithmetic runs in libperiscat_b200.so.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .grating import factorize


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Engine:
    """Thin owner of a ps_ctx.  All tensors passed in must be complex128 on
    ``self.device`` and contiguous."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1412_7466_b200 needs a CUDA device (no CPU fallback)")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.lib = _lib.load()
        self.ctx = ctypes.c_void_p()
        rc = self.lib.ps_create(ctypes.byref(self.ctx), self.device.index)
        _lib.check(self.ctx, rc)
        self.M = 0
        self.p = -1
        self.L = 0
        self.nrhs = 1
        self.t_range = (0, 0)
        self.coupled = False
        self.nrow_c = 0
        self.nout = 0
        self.ncol_b = 0
        self.nrb = 0

    def close(self):
        if self.ctx:
            self.lib.ps_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        _lib.check(self.ctx, rc)

    # ---------------------------------------------------------------- setup
    def set_geometry(self, centers, p: int, k2: float, period: float = 1.0, copies: int = 1):
        c = _f64(centers).reshape(-1, 2)
        self._check(self.lib.ps_set_geometry(self.ctx, c.shape[0], int(p), int(copies),
                                             float(period), float(k2), _ptr(c)))
        self.M, self.p, self.L = c.shape[0], int(p), 2 * int(p) + 1
        self.copies = int(copies)
        self.t_range = (0, self.M)

    def check_overlap(self, radius: float) -> float:
        """ParticleSet.min_gap (geometry.py:131-144) on the device; raises
        DomainError for overlapping disks."""
        gap = ctypes.c_double()
        self._check(self.lib.ps_check_overlap(self.ctx, float(radius), ctypes.byref(gap)))
        return gap.value

    def set_target_range(self, t0: int, t1: int):
        self._check(self.lib.ps_set_target_range(self.ctx, int(t0), int(t1)))
        self.t_range = (int(t0), int(t1))

    @property
    def n_own(self) -> int:
        return self.t_range[1] - self.t_range[0]

    def set_bloch(self, bloch):
        b = _c128(np.atleast_1d(bloch))
        self._check(self.lib.ps_set_rhs_bloch(self.ctx, b.size, _ptr(b)))
        self.nrhs = b.size

    def set_smatrix(self, S, rot=None):
        S = _c128(S)
        diag = 1 if S.ndim == 1 else 0
        r = None if rot is None else _f64(rot)
        self._check(self.lib.ps_set_smatrix(self.ctx, _ptr(S), diag,
                                            None if r is None else _ptr(r)))

    def set_layers(self, system):
        """Curves + expansion centre of a (reference or fixture) empty-grating system."""
        cv = system.curves
        g = []
        for name in ("g1", "g2"):
            c = cv[name]
            g.append(_f64(np.column_stack([c.nodes, c.normals, c.arc_weights])))
        w2 = _f64(cv["L2"].nodes)
        x2 = _f64(system.centers[2])
        cfg = system.config
        Q = int(cfg.j_expansion_order)
        nrb = int(cfg.rb_modes_per_direction)
        self._check(self.lib.ps_set_layers(self.ctx, g[0].shape[0], _ptr(g[0]), g[1].shape[0],
                                           _ptr(g[1]), w2.shape[0], _ptr(w2), _ptr(x2), Q, nrb))
        n1, n2, nw = g[0].shape[0], g[1].shape[0], w2.shape[0]
        self.nrow_c = 2 * n1 + 2 * n2 + 2 * nw
        self.ncol_b = 2 * n1 + 2 * n2 + 2 * Q + 1
        self.nrb = nrb
        self.nout = self.ncol_b + 2 * nrb
        self._layer_cols = system.cols

    def setup_empty(self, configs, svd_workers: int | None = None, rhs_range=None):
        """Device assembly + SVD of the empty-grating system of every RHS
        (ps_setup_empty; replaces set_layers + set_pinv with host factors).
        rhs_range=(b, e): factorise only those RHS (the multi-GPU split; the
        others come in through import_pinv).  Returns one DeviceEmptySystem
        per config."""
        from . import empty_setup as es
        configs = es.validate(configs)
        if len(configs) != self.nrhs:
            raise ValueError("one config per right-hand side (set_bloch first)")
        cell = es.unit_cell(configs[0])
        desc, keep = es.build_desc(configs[0], cell)
        theta = _f64([c.incident_angle for c in configs])
        if svd_workers is not None:
            self._check(self.lib.ps_set_svd_workers(self.ctx, int(svd_workers)))
        b, e = (0, len(configs)) if rhs_range is None else rhs_range
        self._check(self.lib.ps_setup_empty_range(self.ctx, ctypes.byref(desc), _ptr(theta),
                                                  int(b), int(e)))
        del keep
        cfg = configs[0]
        n1, n2, nw = cell.g1.shape[0], cell.g2.shape[0], cell.walls[1].shape[0]
        Q, nrb = int(cfg.j_expansion_order), int(cfg.rb_modes_per_direction)
        self.nrow_c = 2 * n1 + 2 * n2 + 2 * nw
        self.ncol_b = 2 * n1 + 2 * n2 + 2 * Q + 1
        self.nrb = nrb
        self.nout = self.ncol_b + 2 * nrb
        self._layer_cols = cell.cols
        self.coupled = True
        return [es.DeviceEmptySystem(c, cell.cols, cell.rows, cell.centers, self, r)
                for r, c in enumerate(configs)]

    def pinv_bytes(self) -> int:
        """Bytes of one RHS's packed restricted A^+ factors (ps_pinv_bytes)."""
        return int(self.lib.ps_pinv_bytes(self.ctx))

    def export_pinv(self, irhs: int, buf: torch.Tensor):
        """Pack RHS irhs's factors into a uint8 CUDA tensor of pinv_bytes()."""
        self._check(self.lib.ps_export_pinv(self.ctx, int(irhs), ctypes.c_void_p(buf.data_ptr()),
                                            _stream(self.device)))

    def import_pinv(self, irhs: int, buf: torch.Tensor):
        self._check(self.lib.ps_import_pinv(self.ctx, int(irhs), ctypes.c_void_p(buf.data_ptr()),
                                            _stream(self.device)))

    def get_empty(self, irhs: int):
        """(A, f, col_scale, s) of a device-assembled RHS (ps_get_empty)."""
        m, n = ctypes.c_int(), ctypes.c_int()
        self._check(self.lib.ps_empty_shape(self.ctx, ctypes.byref(m), ctypes.byref(n)))
        A = np.empty((m.value, n.value), dtype=np.complex128)
        f = np.empty(m.value, dtype=np.complex128)
        cs = np.empty(n.value)
        s = np.empty(n.value)
        self._check(self.lib.ps_get_empty(self.ctx, int(irhs), _ptr(A), _ptr(f), _ptr(cs), _ptr(s)))
        return A, f, cs, s

    def setup_timings(self):
        """Device ms of the last setup_empty: (assembly, SVD + factor restriction)."""
        a, s = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.ps_setup_timings(self.ctx, ctypes.byref(a), ctypes.byref(s)))
        return a.value, s.value

    def set_pinv(self, irhs: int, system):
        """Upload the SVD factors of one RHS's system (computed if absent)."""
        factorize(system)
        u, s, vh = system.svd
        u, s, vh = _c128(u), _f64(s), _c128(vh)
        cs = _f64(system.col_scale)
        f = _c128(system.rhs)
        eps = float(system.config.regularization)
        self._check(self.lib.ps_set_pinv(self.ctx, int(irhs), u.shape[0], u.shape[1], _ptr(u),
                                         _ptr(s), _ptr(vh), _ptr(cs), eps, _ptr(f),
                                         system.cols["c"].start, system.cols["d"].start))
        self.coupled = True

    def set_k1_variant(self, variant: int):
        """0 auto, 1 tiled K1, 2 symmetric K1s, 3 K1h (K1s on DMMA, opt-in); see include/periscat_b200.h."""
        self._check(self.lib.ps_set_k1_variant(self.ctx, int(variant)))

    def set_symbol_store(self, max_gb: float) -> int:
        """Bound (GB) of the K1s symbol store (0: regenerate the symbols in
        every launch; < 0: query only).  Returns the current store size in
        bytes (see include/periscat_b200.h)."""
        n = ctypes.c_size_t(0)
        self._check(self.lib.ps_set_symbol_store(self.ctx, float(max_gb), ctypes.byref(n)))
        return int(n.value)

    def set_overlap(self, sms: int):
        """SMs left to the coupling chain while K1s runs (< 0: serial)."""
        self._check(self.lib.ps_set_overlap(self.ctx, int(sms)))

    def set_overlap_order(self, k1_first: bool):
        """Queue the coupling chain behind K1s (True) or at the fork (False)."""
        self._check(self.lib.ps_set_overlap_order(self.ctx, 1 if k1_first else 0))

    def set_k1_reserve(self, sms: int):
        """Single-RHS M2L grids leave `sms` SMs free for overlapped work."""
        self._check(self.lib.ps_set_k1_reserve(self.ctx, int(sms)))

    def set_mrhs_variant(self, variant: int):
        """0 auto, 1 DFMA K1m, 2 DMMA K1d (see include/periscat_b200.h)."""
        self._check(self.lib.ps_set_mrhs_variant(self.ctx, int(variant)))

    def precompute_coupling(self, max_gb: float = 40.0) -> bool:
        """Pre-assemble C and B on the device if they fit max_gb (see header)."""
        self._check(self.lib.ps_precompute_coupling(self.ctx, float(max_gb)))
        return self.lib.ps_coupling_mode(self.ctx) == 1

    # ---------------------------------------------------------------- apply
    def _dev(self, x, shape):
        if not isinstance(x, torch.Tensor) or x.device != self.device or x.dtype != torch.complex128 \
                or not x.is_contiguous():
            raise TypeError(f"expected a contiguous complex128 tensor on {self.device}")
        if tuple(x.shape) != tuple(shape):
            raise ValueError(f"expected shape {tuple(shape)}, got {tuple(x.shape)}")
        return ctypes.c_void_p(x.data_ptr())

    def empty_own(self):
        return torch.empty((self.nrhs, self.n_own, self.L), dtype=torch.complex128,
                           device=self.device)

    def apply_T(self, beta: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = self.empty_own() if out is None else out
        b = self._dev(beta, (self.nrhs, self.M, self.L))
        o = self._dev(out, (self.nrhs, self.n_own, self.L))
        self._check(self.lib.ps_apply_T(self.ctx, b, o, _stream(self.device)))
        return out

    def apply_T_blocks(self, beta: torch.Tensor, part: int, nparts: int,
                       out: torch.Tensor | None = None) -> torch.Tensor:
        """This part's share of apply_T for ALL M targets (symmetric split;
        one RHS).  Summing the parts over ranks gives apply_T."""
        out = torch.empty((1, self.M, self.L), dtype=torch.complex128,
                          device=self.device) if out is None else out
        b = self._dev(beta, (1, self.M, self.L))
        o = self._dev(out, (1, self.M, self.L))
        self._check(self.lib.ps_apply_T_blocks(self.ctx, int(part), int(nparts), b, o,
                                               _stream(self.device)))
        return out

    def particle_field(self, beta: torch.Tensor, points) -> torch.Tensor:
        """[nrhs][npts] particle multipole field at points (ps_particle_field)."""
        pts = torch.as_tensor(np.ascontiguousarray(np.asarray(points, dtype=float).reshape(-1, 2)),
                              device=self.device)
        out = torch.empty((self.nrhs, pts.shape[0]), dtype=torch.complex128, device=self.device)
        if pts.shape[0] == 0:
            return out
        b = self._dev(beta, (self.nrhs, self.M, self.L))
        self._check(self.lib.ps_particle_field(self.ctx, b, int(pts.shape[0]),
                                               ctypes.c_void_p(pts.data_ptr()),
                                               ctypes.c_void_p(out.data_ptr()),
                                               _stream(self.device)))
        return out

    def particle_field_grad(self, beta: torch.Tensor, points, dirs):
        """([nrhs][npts] values, [nrhs][npts] derivatives along dirs) of the
        particle multipole field (ps_particle_field_grad)."""
        pts = torch.as_tensor(np.ascontiguousarray(np.asarray(points, dtype=float).reshape(-1, 2)),
                              device=self.device)
        dr = torch.as_tensor(np.ascontiguousarray(np.asarray(dirs, dtype=float).reshape(-1, 2)),
                             device=self.device)
        out = torch.empty((self.nrhs, pts.shape[0]), dtype=torch.complex128, device=self.device)
        dn = torch.empty_like(out)
        if pts.shape[0] == 0:
            return out, dn
        b = self._dev(beta, (self.nrhs, self.M, self.L))
        self._check(self.lib.ps_particle_field_grad(self.ctx, b, int(pts.shape[0]),
                                                    self._vp(pts), self._vp(dr), self._vp(out),
                                                    self._vp(dn), _stream(self.device)))
        return out, dn

    def schur_finish(self, v_own: torch.Tensor, a_own: torch.Tensor, g: torch.Tensor | None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """y_own = v_own - S (a_own - B A^+ g) (one RHS)."""
        out = self.empty_own() if out is None else out
        v = self._dev(v_own, (1, self.n_own, self.L))
        a = self._dev(a_own, (1, self.n_own, self.L))
        gp = None if g is None else self._dev(g, (1, self.nrow_c))
        o = self._dev(out, (1, self.n_own, self.L))
        self._check(self.lib.ps_schur_finish(self.ctx, v, a, gp, o, _stream(self.device)))
        return out

    def apply_C(self, beta: torch.Tensor, s_range=None, out=None) -> torch.Tensor:
        s0, s1 = (0, self.M) if s_range is None else s_range
        out = torch.empty((self.nrhs, self.nrow_c), dtype=torch.complex128,
                          device=self.device) if out is None else out
        b = self._dev(beta, (self.nrhs, self.M, self.L))
        o = self._dev(out, (self.nrhs, self.nrow_c))
        self._check(self.lib.ps_apply_C(self.ctx, b, o, int(s0), int(s1), _stream(self.device)))
        return out

    def apply_schur(self, v: torch.Tensor, out=None, g: torch.Tensor | None = None) -> torch.Tensor:
        out = self.empty_own() if out is None else out
        vp = self._dev(v, (self.nrhs, self.M, self.L))
        o = self._dev(out, (self.nrhs, self.n_own, self.L))
        if g is None:
            self._check(self.lib.ps_apply_schur(self.ctx, vp, o, _stream(self.device)))
        else:
            gp = self._dev(g, (self.nrhs, self.nrow_c))
            self._check(self.lib.ps_apply_schur_g(self.ctx, vp, gp, o, _stream(self.device)))
        return out

    def schur_rhs(self, out=None) -> torch.Tensor:
        out = self.empty_own() if out is None else out
        o = self._dev(out, (self.nrhs, self.n_own, self.L))
        self._check(self.lib.ps_schur_rhs(self.ctx, o, _stream(self.device)))
        return out

    def recover(self, g: torch.Tensor, out=None) -> torch.Tensor:
        out = torch.empty((self.nrhs, self.nout), dtype=torch.complex128,
                          device=self.device) if out is None else out
        gp = self._dev(g, (self.nrhs, self.nrow_c))
        o = self._dev(out, (self.nrhs, self.nout))
        self._check(self.lib.ps_recover(self.ctx, gp, o, _stream(self.device)))
        return out

    def recover_full(self, g: torch.Tensor) -> torch.Tensor:
        """x = A^+ (f - g) over all empty-grating columns (ps_recover_full),
        [nrhs][ncol] in the reference column order."""
        ncol = int(self.lib.ps_full_columns(self.ctx))
        if ncol <= 0:
            raise RuntimeError("factors without field rows (set up the empty grating first)")
        out = torch.empty((self.nrhs, ncol), dtype=torch.complex128, device=self.device)
        gp = self._dev(g, (self.nrhs, self.nrow_c))
        self._check(self.lib.ps_recover_full(self.ctx, gp, ctypes.c_void_p(out.data_ptr()),
                                             _stream(self.device)))
        return out

    def set_field_params(self, configs):
        """k1, k3, expansion centres and incident wave vectors for
        layer_field when the factors came from set_pinv (host SVD)."""
        cfg = configs[0]
        ctr = cfg.expansion_centers()
        inc = _f64([[c.k1 * np.cos(c.incident_angle), c.k1 * np.sin(c.incident_angle)]
                    for c in configs])
        c1, c3 = _f64(ctr[1]), _f64(ctr[3])
        self._check(self.lib.ps_set_field_params(self.ctx, float(cfg.k1), float(cfg.k3), _ptr(c1),
                                                 _ptr(c3), _ptr(inc)))

    def layer_field(self, x: torch.Tensor, points, layer) -> torch.Tensor:
        """[nrhs][npts] empty-grating layer field (+ incident in layer 1) at
        points of the given layers (ps_layer_field)."""
        pts = torch.as_tensor(np.ascontiguousarray(np.asarray(points, dtype=float).reshape(-1, 2)),
                              device=self.device)
        lay = torch.as_tensor(np.ascontiguousarray(np.asarray(layer, dtype=np.int32).ravel()),
                              device=self.device)
        out = torch.empty((self.nrhs, pts.shape[0]), dtype=torch.complex128, device=self.device)
        if pts.shape[0] == 0:
            return out
        xp = x.to(device=self.device, dtype=torch.complex128).contiguous()
        self._check(self.lib.ps_layer_field(self.ctx, ctypes.c_void_p(xp.data_ptr()),
                                            int(pts.shape[0]), ctypes.c_void_p(pts.data_ptr()),
                                            ctypes.c_void_p(lay.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), _stream(self.device)))
        return out

    def layer_field_grad(self, x: torch.Tensor, points, layer, dirs, incident: bool = True):
        """(values, derivatives along dirs) [nrhs][npts] of the empty-grating
        layer field (ps_layer_field_grad); incident=False is
        eval_empty_field(total=False)."""
        pts = torch.as_tensor(np.ascontiguousarray(np.asarray(points, dtype=float).reshape(-1, 2)),
                              device=self.device)
        dr = torch.as_tensor(np.ascontiguousarray(np.asarray(dirs, dtype=float).reshape(-1, 2)),
                             device=self.device)
        lay = torch.as_tensor(np.ascontiguousarray(np.asarray(layer, dtype=np.int32).ravel()),
                              device=self.device)
        out = torch.empty((self.nrhs, pts.shape[0]), dtype=torch.complex128, device=self.device)
        dn = torch.empty_like(out)
        if pts.shape[0] == 0:
            return out, dn
        xp = x.to(device=self.device, dtype=torch.complex128).contiguous()
        self._check(self.lib.ps_layer_field_grad(self.ctx, self._vp(xp), int(pts.shape[0]),
                                                 self._vp(pts), self._vp(lay), self._vp(dr),
                                                 1 if incident else 0, self._vp(out),
                                                 self._vp(dn), _stream(self.device)))
        return out, dn

    def set_empty_system(self, irhs: int, system):
        """Upload one RHS's column-scaled empty-grating matrix, f and column
        scaling (ps_set_empty_system) for the coupled residual."""
        A = _c128(system.matrix)
        f = _c128(system.rhs)
        cs = _f64(system.col_scale)
        self._check(self.lib.ps_set_empty_system(self.ctx, int(irhs), A.shape[0], A.shape[1],
                                                 _ptr(A), _ptr(f), _ptr(cs)))

    def empty_residual(self, x: torch.Tensor, g: torch.Tensor | None):
        """[nrhs][2] (||A x/cs + C beta - f||^2, ||f||^2) on the device."""
        out = torch.empty((self.nrhs, 2), dtype=torch.float64, device=self.device)
        gp = None if g is None else self._vp(g.contiguous())
        self._check(self.lib.ps_empty_residual(self.ctx, self._vp(x.contiguous()), gp,
                                               self._vp(out), _stream(self.device)))
        return out

    def gmres(self, rhs: torch.Tensor, tol: float = 1e-10, maxit: int = 150):
        x = torch.empty_like(rhs)
        r = self._dev(rhs, (self.nrhs, self.M, self.L))
        xp = self._dev(x, (self.nrhs, self.M, self.L))
        iters = (ctypes.c_int * self.nrhs)()
        hist = np.full((self.nrhs, maxit + 1), np.nan)
        self._check(self.lib.ps_gmres(self.ctx, r, xp, float(tol), int(maxit), iters,
                                      hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      _stream(self.device)))
        return x, list(iters), hist

    # instrumentation
    def profile(self, enable: bool = True):
        self._check(self.lib.ps_profile(self.ctx, 1 if enable else 0))

    def stats(self) -> dict:
        n, ms, cnt = ctypes.c_longlong(), ctypes.c_double(), ctypes.c_longlong()
        self._check(self.lib.ps_stats(self.ctx, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(cnt)))
        return dict(launches=n.value, k1_ms=ms.value, k1_count=cnt.value)

    def timeline(self) -> dict:
        """Mean {k1_end, chain_end, step_end} ms of profiled overlapped steps."""
        out = (ctypes.c_double * 3)()
        n = ctypes.c_longlong()
        self._check(self.lib.ps_timeline(self.ctx, out, ctypes.byref(n)))
        return dict(k1_end_ms=out[0], chain_end_ms=out[1], step_end_ms=out[2], steps=n.value)

    def stats_reset(self):
        self._check(self.lib.ps_stats_reset(self.ctx))

    # Arnoldi building blocks (krylov.gmres_device / parallel.gmres_dist)
    def _vp(self, t: torch.Tensor):
        if t.device != self.device or not t.is_contiguous():
            raise TypeError(f"expected a contiguous tensor on {self.device}")
        return ctypes.c_void_p(t.data_ptr())

    def krylov_begin(self, b: torch.Tensor, bnorm2: torch.Tensor, V: torch.Tensor):
        """State from the squared RHS norms, V[0] = b / ||b|| (b [nrhs][n])."""
        kmax1, nrhs, n = V.shape
        self._check(self.lib.ps_krylov_begin(self.ctx, nrhs, n, kmax1 - 1, self._vp(b),
                                             self._vp(bnorm2), self._vp(V),
                                             _stream(self.device)))

    def krylov_dot(self, k: int, V: torch.Tensor, w: torch.Tensor, h: torch.Tensor):
        self._check(self.lib.ps_krylov_dot(self.ctx, int(k), self._vp(V), self._vp(w), self._vp(h),
                                           _stream(self.device)))
        return h

    def krylov_axpy(self, k: int, V: torch.Tensor, h: torch.Tensor, w: torch.Tensor):
        self._check(self.lib.ps_krylov_axpy(self.ctx, int(k), self._vp(V), self._vp(h),
                                            self._vp(w), _stream(self.device)))
        return w

    def krylov_norm2(self, w: torch.Tensor, out: torch.Tensor):
        nrhs, n = w.shape
        self._check(self.lib.ps_krylov_norm2(self.ctx, nrhs, n, self._vp(w), self._vp(out),
                                             _stream(self.device)))
        return out

    def krylov_step(self, k: int, h1, h2, wn2, w, V, status):
        self._check(self.lib.ps_krylov_step(self.ctx, int(k), self._vp(h1), self._vp(h2),
                                            self._vp(wn2), self._vp(w), self._vp(V),
                                            self._vp(status), _stream(self.device)))
        return status

    def krylov_freeze(self, active):
        a = (ctypes.c_int * len(active))(*[int(x) for x in active])
        self._check(self.lib.ps_krylov_freeze(self.ctx, a, _stream(self.device)))

    def krylov_solve(self, iters, V: torch.Tensor, x: torch.Tensor):
        it = (ctypes.c_int * len(iters))(*[int(x) for x in iters])
        self._check(self.lib.ps_krylov_solve(self.ctx, it, self._vp(V), self._vp(x),
                                             _stream(self.device)))
        return x

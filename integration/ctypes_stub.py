"""Pure-ctypes binding of include/periscat_b200.h -- no torch, no package import.

This is the binding a maintainer of the Python reference would drop next to
``periscat/empty_grating.py``: device memory via libcudart, the hot path via
libperiscat_b200.so.  ``apply_T`` and ``solve`` take/return NumPy arrays and
reference objects (ProblemConfig / EmptyGratingSystem duck types).
"""
from __future__ import annotations

import ctypes
import ctypes.util
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("PS_LIB", os.path.join(_HERE, "..", "paper_1412_7466_b200",
                                            "libperiscat_b200.so"))


def _cudart():
    for name in ("libcudart.so.12", "libcudart.so", "/usr/local/cuda/lib64/libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    raise OSError("libcudart not found")


class DeviceArray:
    def __init__(self, rt, nbytes):
        self.rt = rt
        self.ptr = ctypes.c_void_p()
        if rt.cudaMalloc(ctypes.byref(self.ptr), ctypes.c_size_t(max(nbytes, 16))) != 0:
            raise MemoryError("cudaMalloc failed")
        self.nbytes = nbytes

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a)
        assert a.nbytes == self.nbytes
        self.rt.cudaMemcpy(self.ptr, a.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(a.nbytes), 1)
        return self

    def download(self, shape, dtype=np.complex128):
        out = np.empty(shape, dtype=dtype)
        self.rt.cudaMemcpy(out.ctypes.data_as(ctypes.c_void_p), self.ptr, ctypes.c_size_t(out.nbytes), 2)
        return out

    def free(self):
        if self.ptr:
            self.rt.cudaFree(self.ptr)
            self.ptr = ctypes.c_void_p()


class _Curve(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("data", ctypes.c_void_p)]


class _Iface(ctypes.Structure):
    _fields_ = [("mean", ctypes.c_double), ("nsin", ctypes.c_int), ("ncos", ctypes.c_int),
                ("sin_coeffs", ctypes.c_void_p), ("cos_coeffs", ctypes.c_void_p)]


class _EmptyDesc(ctypes.Structure):           # ps_empty_desc
    _D, _I = ctypes.c_double, ctypes.c_int
    _fields_ = [("period", _D), ("k1", _D), ("k2", _D), ("k3", _D), ("y0", _D), ("eps", _D),
                ("copies", _I), ("Q", _I), ("nrb", _I), ("centers", _D * 6),
                ("g1", _Curve), ("g2", _Curve), ("wall", _Curve * 3),
                ("lid_up", _Curve), ("lid_down", _Curve), ("top", _Iface), ("bottom", _Iface),
                ("rule_n", _I), ("rule_skip", _I), ("rule_interp", _I),
                ("rule_x", ctypes.c_void_p), ("rule_w", ctypes.c_void_p)]


class _ParticleDesc(ctypes.Structure):        # ps_particle_desc
    _D, _I = ctypes.c_double, ctypes.c_int
    _fields_ = [("k2", _D), ("kp", _D), ("base_radius", _D), ("bump_amplitude", _D),
                ("lobes", _I), ("n", _I), ("curve", ctypes.c_void_p),
                ("rule_n", _I), ("rule_skip", _I), ("rule_interp", _I),
                ("rule_x", ctypes.c_void_p), ("rule_w", ctypes.c_void_p)]


def _curve_rows(cv):
    """DiscretizedCurve (geometry.py:25-60) -> rows x y nx ny speed weight t arc_weight."""
    return np.ascontiguousarray(np.column_stack([cv.nodes, cv.normals, cv.speeds, cv.weights,
                                                 cv.t, cv.arc_weights]), dtype=float)


class Periscat:
    """ps_ctx owner.  Mirrors the calls solver.solve_full makes."""

    def __init__(self, device: int = 0, lib_path: str = LIB):
        self.rt = _cudart()
        self.lib = ctypes.CDLL(lib_path)
        self.lib.ps_last_error.restype = ctypes.c_char_p
        self.ctx = ctypes.c_void_p()
        self._ok(self.lib.ps_create(ctypes.byref(self.ctx), device))

    def _ok(self, rc):
        if rc != 0:
            raise RuntimeError(f"periscat_b200 error {rc}: {self.lib.ps_last_error(self.ctx).decode()}")

    @staticmethod
    def _p(a):
        return a.ctypes.data_as(ctypes.c_void_p)

    def setup(self, system, centers, p, smat, bloch_list=None, systems=None):
        """system: reference EmptyGratingSystem (factorised or not); centers [M][2]."""
        systems = systems or [system]
        cfg = system.config
        c = np.ascontiguousarray(centers, dtype=float)
        self.M, self.p, self.L = c.shape[0], p, 2 * p + 1
        self._ok(self.lib.ps_set_geometry(self.ctx, self.M, p, cfg.near_field_copies,
                                          ctypes.c_double(cfg.period), ctypes.c_double(cfg.k2),
                                          self._p(c)))
        bl = np.array([s.config.bloch_phase for s in systems], dtype=complex)
        self.nrhs = bl.size
        self._ok(self.lib.ps_set_rhs_bloch(self.ctx, bl.size, self._p(bl)))
        S = np.ascontiguousarray(smat, dtype=complex)
        self._ok(self.lib.ps_set_smatrix(self.ctx, self._p(S), 1 if S.ndim == 1 else 0, None))
        cv = system.curves
        g1 = np.ascontiguousarray(np.column_stack([cv["g1"].nodes, cv["g1"].normals, cv["g1"].arc_weights]))
        g2 = np.ascontiguousarray(np.column_stack([cv["g2"].nodes, cv["g2"].normals, cv["g2"].arc_weights]))
        w2 = np.ascontiguousarray(cv["L2"].nodes, dtype=float)
        x2 = np.ascontiguousarray(system.centers[2], dtype=float)
        self._ok(self.lib.ps_set_layers(self.ctx, g1.shape[0], self._p(g1), g2.shape[0], self._p(g2),
                                        w2.shape[0], self._p(w2), self._p(x2),
                                        cfg.j_expansion_order, cfg.rb_modes_per_direction))
        self.nrow_c = 2 * g1.shape[0] + 2 * g2.shape[0] + 2 * w2.shape[0]
        self.ncol_b = 2 * g1.shape[0] + 2 * g2.shape[0] + 2 * cfg.j_expansion_order + 1
        self.nrb = cfg.rb_modes_per_direction
        for r, s in enumerate(systems):
            if s.svd is None:                       # empty_grating.factorize (eg:259-261)
                s.svd = np.linalg.svd(s.matrix, full_matrices=False)
            u, sv, vh = (np.ascontiguousarray(x) for x in s.svd)
            cs = np.ascontiguousarray(s.col_scale, dtype=float)
            f = np.ascontiguousarray(s.rhs, dtype=complex)
            self._ok(self.lib.ps_set_pinv(self.ctx, r, u.shape[0], u.shape[1], self._p(u), self._p(sv),
                                          self._p(vh), self._p(cs),
                                          ctypes.c_double(s.config.regularization), self._p(f),
                                          s.cols["c"].start, s.cols["d"].start))

    def setup_from_config(self, configs, curves, rule, centers, p, smat, rot=None):
        """solve_full(config) without host factors: the empty grating of every
        config (one per incidence angle) is assembled and factorised on the
        device (ps_setup_empty).  curves = empty_grating.build_geometry(config)
        (eg:113-119); rule = quadrature.ALPERT_RULES[config.alpert_order]."""
        configs = list(configs) if isinstance(configs, (list, tuple)) else [configs]
        cfg = configs[0]
        c = np.ascontiguousarray(centers, dtype=float)
        self.M, self.p, self.L = c.shape[0], p, 2 * p + 1
        self._ok(self.lib.ps_set_geometry(self.ctx, self.M, p, cfg.near_field_copies,
                                          ctypes.c_double(cfg.period), ctypes.c_double(cfg.k2),
                                          self._p(c)))
        bl = np.array([x.bloch_phase for x in configs], dtype=complex)
        self.nrhs = bl.size
        self._ok(self.lib.ps_set_rhs_bloch(self.ctx, bl.size, self._p(bl)))
        S = np.ascontiguousarray(smat, dtype=complex)
        r = None if rot is None else np.ascontiguousarray(rot, dtype=float)
        self._ok(self.lib.ps_set_smatrix(self.ctx, self._p(S), 1 if S.ndim == 1 else 0,
                                         None if r is None else self._p(r)))
        keep = []

        def arr(a):
            a = np.ascontiguousarray(a, dtype=float)
            keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p)

        def curve(cv):
            rows = _curve_rows(cv)
            return _Curve(rows.shape[0], arr(rows))

        def iface(spec):
            sc, cc = np.asarray(spec.sin_coeffs, float), np.asarray(spec.cos_coeffs, float)
            return _Iface(spec.mean, sc.size, cc.size, arr(sc) if sc.size else None,
                          arr(cc) if cc.size else None)

        d = _EmptyDesc()
        d.period, d.k1, d.k2, d.k3 = cfg.period, cfg.k1, cfg.k2, cfg.k3
        d.y0, d.eps = cfg.y0, cfg.regularization
        d.copies, d.Q, d.nrb = (cfg.near_field_copies, cfg.j_expansion_order,
                                cfg.rb_modes_per_direction)
        ctr = cfg.expansion_centers()
        for i, k in enumerate((1, 2, 3)):
            d.centers[2 * i], d.centers[2 * i + 1] = float(ctr[k][0]), float(ctr[k][1])
        d.g1, d.g2 = curve(curves["g1"]), curve(curves["g2"])
        for i, w in enumerate(("L1", "L2", "L3")):
            d.wall[i] = curve(curves[w])
        d.lid_up, d.lid_down = curve(curves["Gu"]), curve(curves["Gd"])
        d.top, d.bottom = iface(cfg.interface_top), iface(cfg.interface_bottom)
        d.rule_n, d.rule_skip, d.rule_interp = len(rule.nodes), rule.skip, rule.interp
        d.rule_x, d.rule_w = arr(rule.nodes), arr(rule.weights)
        theta = np.array([x.incident_angle for x in configs], dtype=float)
        self._ok(self.lib.ps_setup_empty(self.ctx, ctypes.byref(d), self._p(theta)))
        n1, n2, nw = curves["g1"].n, curves["g2"].n, curves["L2"].n
        self.nrow_c = 2 * n1 + 2 * n2 + 2 * nw
        self.ncol_b = 2 * n1 + 2 * n2 + 2 * cfg.j_expansion_order + 1
        self.nrb = cfg.rb_modes_per_direction

    def scattering_matrix(self, shape, k2, kp, p, curve, rule):
        """scatmat.scattering_matrix on the device.  curve =
        geometry.sample_particle(shape, (0, 0), 0.0, N) (geometry.py:224-256)."""
        rows = _curve_rows(curve)
        x = np.ascontiguousarray(rule.nodes, dtype=float)
        w = np.ascontiguousarray(rule.weights, dtype=float)
        d = _ParticleDesc(k2, kp, shape.base_radius, shape.bump_amplitude, shape.lobes,
                          rows.shape[0], self._p(rows), x.size, rule.skip, rule.interp,
                          self._p(x), self._p(w))
        S = np.empty((2 * p + 1, 2 * p + 1), dtype=complex)
        res = ctypes.c_double()
        self._ok(self.lib.ps_scattering_matrix(self.ctx, ctypes.byref(d), p, self._p(S),
                                               ctypes.byref(res)))
        return S

    def apply_T(self, beta):
        """multiscat.apply_T with host arrays [nrhs][M][L]."""
        beta = np.ascontiguousarray(beta, dtype=complex).reshape(self.nrhs, self.M, self.L)
        din = DeviceArray(self.rt, beta.nbytes).upload(beta)
        dout = DeviceArray(self.rt, beta.nbytes)
        try:
            self._ok(self.lib.ps_apply_T(self.ctx, din.ptr, dout.ptr, None))
            return dout.download(beta.shape)
        finally:
            din.free()
            dout.free()

    def solve(self, tol=1e-10, maxit=150):
        """solver.solve_full: returns beta, c, d, iterations."""
        shape = (self.nrhs, self.M, self.L)
        n = self.nrhs * self.M * self.L * 16
        rhs, x = DeviceArray(self.rt, n), DeviceArray(self.rt, n)
        g = DeviceArray(self.rt, self.nrhs * self.nrow_c * 16)
        nout = self.ncol_b + 2 * self.nrb
        xe = DeviceArray(self.rt, self.nrhs * nout * 16)
        iters = (ctypes.c_int * self.nrhs)()
        try:
            self._ok(self.lib.ps_schur_rhs(self.ctx, rhs.ptr, None))
            self._ok(self.lib.ps_gmres(self.ctx, rhs.ptr, x.ptr, ctypes.c_double(tol), maxit,
                                       iters, None, None))
            self._ok(self.lib.ps_apply_C(self.ctx, x.ptr, g.ptr, 0, self.M, None))
            self._ok(self.lib.ps_recover(self.ctx, g.ptr, xe.ptr, None))
            beta = x.download(shape)
            xr = xe.download((self.nrhs, nout))
        finally:
            for d in (rhs, x, g, xe):
                d.free()
        c = xr[:, self.ncol_b:self.ncol_b + self.nrb]
        d = xr[:, self.ncol_b + self.nrb:]
        return beta, c, d, list(iters)

    def set_target_range(self, t0, t1):
        """Own the target slice [t0, t1) (one rank of a sharded operator)."""
        self._ok(self.lib.ps_set_target_range(self.ctx, t0, t1))
        self.t0, self.t1 = t0, t1

    def close(self):
        if self.ctx:
            self.lib.ps_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()


def shard_range(M, rank, world):
    return (M * rank) // world, (M * (rank + 1)) // world


class ShardedSchur:
    """The multi-rank Schur matvec driven
    through the C ABI alone, with the collectives supplied by the caller --
    the way an MPI / NCCL C program shards it.  ``ranks`` are Periscat
    contexts that already hold the operator (setup) and each own a target
    slice (set_target_range); ``allgather(list of own blocks) -> full`` and
    ``allreduce(list of partials) -> sum`` stand in for the caller's
    collectives (here: host arrays summed in rank order).

    mode "targets": every rank applies T over all sources to its own targets
    (ps_apply_schur_g after an all-reduce of the partial C v over the ranks'
    own sources).  mode "pairs": every rank applies the symmetric K1s to its
    1/world of the tile pairs for ALL targets (ps_apply_T_blocks), a
    reduce-scatter sums the parts, ps_schur_finish applies the epilogue."""

    def __init__(self, ranks, mode="targets"):
        self.ranks = ranks
        self.mode = mode
        self.world = len(ranks)

    @staticmethod
    def allgather(blocks):
        return np.concatenate(blocks, axis=1)

    @staticmethod
    def allreduce(parts):
        out = parts[0].copy()
        for q in parts[1:]:
            out += q
        return out

    def __call__(self, v_own_blocks):
        """v_own_blocks[r]: rank r's rows [nrhs][Mt_r][L] (host); returns the
        ranks' rows of y = K v."""
        r0 = self.ranks[0]
        rt = r0.rt
        v = self.allgather(v_own_blocks)                       # all-gather beta
        nrhs, M, L = v.shape
        g_parts = []
        dv = [DeviceArray(rt, v.nbytes).upload(v) for _ in self.ranks]
        try:
            for pc, d in zip(self.ranks, dv):                  # C over own sources
                dg = DeviceArray(rt, nrhs * pc.nrow_c * 16)
                pc._ok(pc.lib.ps_apply_C(pc.ctx, d.ptr, dg.ptr, pc.t0, pc.t1, None))
                g_parts.append(dg.download((nrhs, pc.nrow_c)))
                dg.free()
            g = self.allreduce(g_parts)                        # all-reduce C v
            out = []
            if self.mode == "targets":
                for pc, d in zip(self.ranks, dv):
                    dg = DeviceArray(rt, g.nbytes).upload(g)
                    dy = DeviceArray(rt, nrhs * (pc.t1 - pc.t0) * L * 16)
                    pc._ok(pc.lib.ps_apply_schur_g(pc.ctx, d.ptr, dg.ptr, dy.ptr, None))
                    out.append(dy.download((nrhs, pc.t1 - pc.t0, L)))
                    dg.free()
                    dy.free()
                return out
            a_parts = []                                       # "pairs": K1s parts
            for r, (pc, d) in enumerate(zip(self.ranks, dv)):
                da = DeviceArray(rt, v.nbytes)
                pc._ok(pc.lib.ps_apply_T_blocks(pc.ctx, r, self.world, d.ptr, da.ptr, None))
                a_parts.append(da.download(v.shape))
                da.free()
            a = self.allreduce(a_parts)                        # reduce-scatter
            for pc, vo in zip(self.ranks, v_own_blocks):
                a_own = np.ascontiguousarray(a[:, pc.t0:pc.t1])
                dvo = DeviceArray(rt, vo.nbytes).upload(np.ascontiguousarray(vo))
                dao = DeviceArray(rt, a_own.nbytes).upload(a_own)
                dg = DeviceArray(rt, g.nbytes).upload(g)
                dy = DeviceArray(rt, vo.nbytes)
                pc._ok(pc.lib.ps_schur_finish(pc.ctx, dvo.ptr, dao.ptr, dg.ptr, dy.ptr, None))
                out.append(dy.download(vo.shape))
                for x in (dvo, dao, dg, dy):
                    x.free()
            return out
        finally:
            for d in dv:
                d.free()

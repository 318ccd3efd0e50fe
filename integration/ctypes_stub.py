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


class Periscat:
    """ps_ctx owner.  Mirrors the calls solver.solve_full makes."""

    def __init__(self, device: int = 0):
        self.rt = _cudart()
        self.lib = ctypes.CDLL(LIB)
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

    def close(self):
        if self.ctx:
            self.lib.ps_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

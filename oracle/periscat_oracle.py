"""CPU ORACLE for the periscat hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the CUDA product path in
``paper_1412_7466_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it; the
product never calls it.

What it restates
----------------
The reference package (/root/reference/pkg/src/periscat) stops at the empty
grating: the modules that hold the hot path (``scatmat``, ``multiscat``,
``solver``, ``postproc``) are specified in SPEC.md but absent.
This file therefore restates

* ``specialfn.hankel1_orders`` / ``_signed_order`` (sf:54-67, sf:79-83) and the
  wave-gradient formula of ``outgoing_wave_block`` (sf:128-154);
* ``empty_grating.apply_pinv`` (eg:264-273) and ``factorize`` (eg:259-261);
* ``scatmat`` disk formula;
* ``multiscat.m2l_translate`` / ``apply_T`` (PAPER
  Eqs. trans + repre3_mod);
* ``multiscat.source_to_local_block`` B and ``multipole_to_targets_block`` C
  applied matrix-free;
* ``solver.apply_schur_operator`` / ``gmres`` / ``solve_full``
  (PAPER.md:849-896);
* ``postproc.flux_error``.

It is self-contained (numpy + scipy only) so it also runs on the GPU box,
where /root/reference does not exist.  The parts of the reference it cannot
restate cheaply -- the 856x781 empty-grating matrix -- are read from fixtures
that ``oracle/make_empty.py`` produced by calling the reference itself.

Pinning: the restated helpers are checked against the reference's own
functions in ``tests/test_oracle_pin.py`` (runs wherever /root/reference is
present) and, because the reference ships no tests or golden vectors for this
path, against the identity checks SPEC.md lists (Graf re-summation SP:460,
apply_T degeneracies SP:510-512, Schur degeneracies SP:545-547, GMRES
properties SP:555-557, flux conservation).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.special as sps

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


# ----------------------------------------------------------------------------
# special functions (restates sf:54-67, sf:79-83)
# ----------------------------------------------------------------------------
def hankel1_orders(nmax: int, z) -> np.ndarray:
    """H^(1)_n(z), n=0..nmax, by upward recurrence from scipy H0, H1 (sf:54-67)."""
    z = np.asarray(z, dtype=float)
    out = np.empty((nmax + 1,) + z.shape, dtype=complex)
    out[0] = sps.hankel1(0, z)
    if nmax >= 1:
        out[1] = sps.hankel1(1, z)
    for n in range(1, nmax):
        out[n + 1] = (2.0 * n / z) * out[n] - out[n - 1]
    return out


def signed_orders(table: np.ndarray, orders) -> np.ndarray:
    """Stack table rows for signed orders with C_{-n} = (-1)^n C_n (sf:79-83)."""
    orders = np.asarray(orders, dtype=int)
    rows = table[np.abs(orders)]
    sign = np.where((orders < 0) & (np.abs(orders) % 2 == 1), -1.0, 1.0)
    return rows * sign.reshape((-1,) + (1,) * (rows.ndim - 1))


# ----------------------------------------------------------------------------
# scattering matrix of a disk
# ----------------------------------------------------------------------------
def disk_smatrix(radius: float, k2: float, kp: float, p: int) -> np.ndarray:
    """Diagonal s_n, n=-p..p, of a homogeneous disk (TM, continuity of u, du/dr)."""
    n = np.arange(-p, p + 1)
    a, b = k2 * radius, kp * radius
    j2, j2p = sps.jv(n, a), sps.jvp(n, a)
    jp, jpp = sps.jv(n, b), sps.jvp(n, b)
    h2, h2p = sps.hankel1(n, a), sps.h1vp(n, a)
    return (k2 * j2p * jp - kp * jpp * j2) / (kp * jpp * h2 - k2 * h2p * jp)


# ----------------------------------------------------------------------------
# M2L
# ----------------------------------------------------------------------------
def _toeplitz_index(p: int) -> np.ndarray:
    L = 2 * p + 1
    mp = np.arange(L)[:, None]
    n = np.arange(L)[None, :]
    return n - mp + 2 * p          # index of symbol nu = n - m' in [-2p, 2p]


def m2l_symbols(dx, dy, k: float, p: int) -> np.ndarray:
    """t_nu = H_nu(k rho) e^{i nu phi}, nu=-2p..2p, for (rho, phi)=polar(dx, dy).

    Shape (..., 4p+1).  Uses the reference recurrence (sf:54-67) and
    ``_signed_order`` for negative orders.
    """
    dx = np.asarray(dx, dtype=float)
    dy = np.asarray(dy, dtype=float)
    rho = np.hypot(dx, dy)
    phi = np.arctan2(dy, dx)
    nu = np.arange(-2 * p, 2 * p + 1)
    h = signed_orders(hankel1_orders(2 * p, k * rho), nu)        # (4p+1, ...)
    ph = np.exp(1j * nu.reshape((-1,) + (1,) * rho.ndim) * phi)
    return np.moveaxis(h * ph, 0, -1)


def m2l_translate(beta, center_src, center_tgt, k: float, p: int) -> np.ndarray:
    """Local coefficients at center_tgt of the outgoing expansion beta at
    center_src: a[m'] = sum_n beta[n] H_{n-m'} e^{i(n-m')phi}."""
    d = np.asarray(center_tgt, float) - np.asarray(center_src, float)
    if np.hypot(d[0], d[1]) == 0.0:
        raise ValueError("m2l_translate: coincident centres (overlapping disks)")
    t = m2l_symbols(d[0], d[1], k, p)
    return t[_toeplitz_index(p)] @ np.asarray(beta, dtype=complex)


def apply_T(beta, centers, k: float, p: int, bloch: complex = 1.0, period: float = 1.0,
            copies: int = 1, targets=None) -> np.ndarray:
    """All-pairs translation (SPEC.md:504-512 with images, PAPER repre3_mod).

    a_m = sum_{l=-P..P} sum_{j, (l,j) != (0,m)} bloch^l T(x_m - x_j - l d e_x) beta_j.
    beta: (M, L) or (R, M, L) with per-RHS ``bloch`` of shape (R,).
    ``targets`` restricts the output to a slice/array of target indices (the
    CPU baseline times target slices; cost is exactly proportional).
    """
    centers = np.asarray(centers, dtype=float)
    beta = np.asarray(beta, dtype=complex)
    squeeze = beta.ndim == 2
    if squeeze:
        beta = beta[None]
    bloch = np.atleast_1d(np.asarray(bloch, dtype=complex))
    if bloch.size == 1 and beta.shape[0] > 1:
        bloch = np.repeat(bloch, beta.shape[0])
    M = centers.shape[0]
    L = 2 * p + 1
    tidx = np.arange(M) if targets is None else np.arange(M)[targets]
    idx = _toeplitz_index(p)
    out = np.zeros((beta.shape[0], len(tidx), L), dtype=complex)
    ls = list(range(-copies, copies + 1))
    for oi, m in enumerate(tidx):
        for l in ls:                       # fixed l-then-j order per target
            dx = centers[m, 0] - centers[:, 0] - l * period
            dy = centers[m, 1] - centers[:, 1]
            mask = np.ones(M, dtype=bool)
            if l == 0:
                mask[m] = False
            t = m2l_symbols(dx[mask], dy[mask], k, p)          # (J, 4p+1)
            T = t[:, idx]                                      # (J, L, L)
            w = bloch ** l                                     # (R,)
            out[:, oi, :] += w[:, None] * np.einsum("jab,rjb->ra", T, beta[:, mask, :])
    return out[0] if squeeze else out


# ----------------------------------------------------------------------------
# outgoing / regular waves with gradients (restates sf:86-154 formulas)
# ----------------------------------------------------------------------------
def _outgoing_vals_grads(k: float, n_orders, dx, dy, sign: int = 1):
    """H_n(k r) e^{i*sign*n*theta} and its gradient w.r.t. the point, for
    (r, theta) = polar(dx, dy).  Returns arrays (len(n), ...) and (2, len(n), ...)."""
    n_orders = np.asarray(n_orders, dtype=int)
    r = np.hypot(dx, dy)
    if np.any(r == 0):
        raise ValueError("outgoing wave is singular at its centre")
    th = np.arctan2(dy, dx)
    nmax = int(np.max(np.abs(n_orders))) + 1
    tab = hankel1_orders(nmax, k * r)
    hn = signed_orders(tab, n_orders)
    hn1 = signed_orders(tab, n_orders + 1)
    nn = n_orders.reshape((-1,) + (1,) * r.ndim).astype(float)
    ph = np.exp(1j * sign * nn * th)
    val = hn * ph
    dr = k * (nn * hn / (k * r) - hn1) * ph
    dth = 1j * sign * nn * hn * ph / r
    c, s = np.cos(th), np.sin(th)
    gx = dr * c - dth * s
    gy = dr * s + dth * c
    return val, np.stack([gx, gy])


# ----------------------------------------------------------------------------
# empty-grating system from fixture (reference-generated), apply_pinv
# ----------------------------------------------------------------------------
@dataclass
class EmptySystem:
    """Fixture view of ``empty_grating.EmptyGratingSystem`` (eg:64-84)."""
    A: np.ndarray
    f: np.ndarray
    col_scale: np.ndarray
    cols: dict
    rows: dict
    g1_nodes: np.ndarray
    g1_normals: np.ndarray
    g1_w: np.ndarray
    g2_nodes: np.ndarray
    g2_normals: np.ndarray
    g2_w: np.ndarray
    L2_nodes: np.ndarray
    center2: np.ndarray
    period: float
    k1: float
    k2: float
    k3: float
    kp: float
    theta: float
    copies: int
    Q: int
    eps: float
    svd: tuple | None = None
    name: str = ""

    @property
    def kappa(self) -> float:
        return self.k1 * math.cos(self.theta)                 # geo:369-371

    @property
    def bloch(self) -> complex:
        return complex(np.exp(1j * self.kappa * self.period))  # geo:373-375

    def factorize(self):
        """eg:259-261."""
        if self.svd is None:
            u, s, vh = np.linalg.svd(self.A, full_matrices=False)
            self.svd = (u, s, vh)
        return self.svd

    def apply_pinv(self, g):
        """V Sigma^+ U^* g mapped to physical unknowns (eg:264-273)."""
        u, s, vh = self.factorize()
        inv = np.minimum(1.0 / s, 1.0 / self.eps)
        y = vh.conj().T @ (inv * (u.conj().T @ g))
        return self.col_scale * y


_EMPTY_CACHE: dict = {}


def load_empty(name: str) -> EmptySystem:
    if name in _EMPTY_CACHE:
        return _EMPTY_CACHE[name]
    path = os.path.join(GOLDEN, f"empty_{name}.npz")
    if not os.path.exists(path):
        path = os.path.join(GOLDEN, "cfg5", f"empty_{name}.npz")
    z = np.load(path)
    cols = {str(n): slice(int(a), int(b)) for n, (a, b) in zip(z["col_names"], z["cols"])}
    rows = {str(n): slice(int(a), int(b)) for n, (a, b) in zip(z["row_names"], z["rows"])}
    sc = z["scalars"]
    es = EmptySystem(A=z["A"], f=z["f"], col_scale=z["col_scale"], cols=cols, rows=rows,
                     g1_nodes=z["g1_nodes"], g1_normals=z["g1_normals"], g1_w=z["g1_w"],
                     g2_nodes=z["g2_nodes"], g2_normals=z["g2_normals"], g2_w=z["g2_w"],
                     L2_nodes=z["L2_nodes"], center2=z["center2"],
                     period=float(sc[0]), k1=float(sc[1]), k2=float(sc[2]), k3=float(sc[3]),
                     kp=float(sc[4]), theta=float(sc[5]), copies=int(sc[6]), Q=int(sc[7]),
                     eps=float(sc[8]), name=name)
    _EMPTY_CACHE[name] = es
    return es


# ----------------------------------------------------------------------------
# coupling blocks, matrix-free
# ----------------------------------------------------------------------------
def apply_B_phys(es: EmptySystem, x_empty, centers, p: int) -> np.ndarray:
    """Incoming local coefficients (M, 2p+1) at every inclusion induced by the
    layer-2 part of the empty-grating representation (eg:348-393, layer 2):
    phased layer potentials on Gamma1, Gamma2 at k2 plus the a2 J-expansion.
    Paper's B = -B_phys."""
    centers = np.asarray(centers, dtype=float)
    k2, d, al = es.k2, es.period, es.bloch
    nloc = np.arange(-p, p + 1)
    out = np.zeros((centers.shape[0], 2 * p + 1), dtype=complex)
    for nodes, nrm, w, mu_name, sg_name in (
            (es.g1_nodes, es.g1_normals, es.g1_w, "mu1", "sigma1"),
            (es.g2_nodes, es.g2_normals, es.g2_w, "mu2", "sigma2")):
        mu = x_empty[es.cols[mu_name]]
        sg = x_empty[es.cols[sg_name]]
        for l in range(-es.copies, es.copies + 1):
            ys = nodes + np.array([l * d, 0.0])
            cs = 0.25j * (al ** l) * w * sg          # single-layer weights
            cd = 0.25j * (al ** l) * w * mu          # double-layer weights
            for m in range(centers.shape[0]):
                dx = ys[:, 0] - centers[m, 0]
                dy = ys[:, 1] - centers[m, 1]
                val, grad = _outgoing_vals_grads(k2, nloc, dx, dy, sign=-1)
                dn = grad[0] * nrm[None, :, 0] + grad[1] * nrm[None, :, 1]
                out[m] += val @ cs + dn @ cd
    # B_pm: L2L of the a2 expansion about centre x2
    a2 = x_empty[es.cols["a2"]]
    q = np.arange(-es.Q, es.Q + 1)
    for m in range(centers.shape[0]):
        dx, dy = centers[m] - es.center2
        rho, phi = math.hypot(dx, dy), math.atan2(dy, dx)
        nu = q[None, :] - nloc[:, None]                        # (L, 2Q+1)
        out[m] += (sps.jv(nu, k2 * rho) * np.exp(1j * nu * phi)) @ a2
    return out


def _particle_field(k2, beta, centers, pts, shift: float):
    """Value and gradient at pts of sum_j sum_n beta_jn H_n e^{in theta} about
    centre x_j + shift e_x."""
    p = (beta.shape[1] - 1) // 2
    n = np.arange(-p, p + 1)
    val = np.zeros(pts.shape[0], dtype=complex)
    grad = np.zeros((2, pts.shape[0]), dtype=complex)
    for j in range(centers.shape[0]):
        dx = pts[:, 0] - centers[j, 0] - shift
        dy = pts[:, 1] - centers[j, 1]
        v, g = _outgoing_vals_grads(k2, n, dx, dy, sign=1)
        val += beta[j] @ v
        grad[0] += beta[j] @ g[0]
        grad[1] += beta[j] @ g[1]
    return val, grad


def apply_C(es: EmptySystem, beta, centers) -> np.ndarray:
    """Particle field data on the A-rows (856; nonzero g1, g2, w2 rows).

    g1: -(value, d/dn), g2: +(value, d/dn) summed over the 2P+1 phased copies;
    w2: alpha^{P+1} u(L2 - (x+Pd)) - alpha^{-P} u(L2 - (x-(P+1)d)) with
    x-derivative rows (telescoped discrepancy, lp:211-237).
    """
    beta = np.asarray(beta, dtype=complex)
    centers = np.asarray(centers, dtype=float)
    k2, d, al, P = es.k2, es.period, es.bloch, es.copies
    g = np.zeros(es.A.shape[0], dtype=complex)
    for nodes, nrm, rv, rd, sgn in ((es.g1_nodes, es.g1_normals, "g1_val", "g1_der", -1.0),
                                    (es.g2_nodes, es.g2_normals, "g2_val", "g2_der", 1.0)):
        for l in range(-P, P + 1):
            v, gr = _particle_field(k2, beta, centers, nodes, l * d)
            g[es.rows[rv]] += sgn * (al ** l) * v
            g[es.rows[rd]] += sgn * (al ** l) * (gr[0] * nrm[:, 0] + gr[1] * nrm[:, 1])
    for l, coef, sgn in ((P, al ** (P + 1), 1.0), (-(P + 1), al ** (-P), -1.0)):
        v, gr = _particle_field(k2, beta, centers, es.L2_nodes, l * d)
        g[es.rows["w2_val"]] += sgn * coef * v
        g[es.rows["w2_der"]] += sgn * coef * gr[0]
    return g


# ----------------------------------------------------------------------------
# solver
# ----------------------------------------------------------------------------
def rotate_smatrix(S: np.ndarray, phi: float) -> np.ndarray:
    """(S^(m))_{ln} = e^{i phi (l - n)} s_{ln}."""
    p = (S.shape[0] - 1) // 2
    idx = np.arange(-p, p + 1)
    return S * np.exp(1j * phi * (idx[:, None] - idx[None, :]))


@dataclass
class Problem:
    es: EmptySystem
    centers: np.ndarray
    p: int
    radius: float
    smat: np.ndarray = field(default=None)      # (L,) diagonal disk S or (L, L) dense
    rot: np.ndarray = field(default=None)       # (M,) rotations for a dense S

    def __post_init__(self):
        if self.smat is None:
            self.smat = disk_smatrix(self.radius, self.es.k2, self.es.kp, self.p)

    def apply_S(self, u: np.ndarray) -> np.ndarray:
        """Block-diagonal S applied to u (M, L) (PA:667-679)."""
        if self.smat.ndim == 1:
            return self.smat[None, :] * u
        out = np.empty_like(u)
        for m in range(u.shape[0]):
            Sm = self.smat if self.rot is None else rotate_smatrix(self.smat, self.rot[m])
            out[m] = Sm @ u[m]
        return out

    @property
    def M(self):
        return self.centers.shape[0]

    @property
    def L(self):
        return 2 * self.p + 1


def apply_schur_operator(pb: Problem, v, with_coupling: bool = True, targets=None) -> np.ndarray:
    """K v = v - S T v - S B A^+ C v  (paper B = -B_phys).
    SPEC.md:539-547; PAPER.md final preconditioned system.  ``targets``
    restricts the output rows to those inclusions (C v still sums over all
    sources; T and B are per target)."""
    v = np.asarray(v, dtype=complex).reshape(pb.M, pb.L)
    es = pb.es
    tidx = np.arange(pb.M) if targets is None else np.arange(pb.M)[targets]
    u = apply_T(v, pb.centers, es.k2, pb.p, es.bloch, es.period, es.copies, targets=tidx)
    if with_coupling:
        x = es.apply_pinv(apply_C(es, v, pb.centers))
        u = u - apply_B_phys(es, x, pb.centers[tidx], pb.p)
    sub = pb if targets is None else Problem(es, pb.centers[tidx], pb.p, pb.radius, pb.smat,
                                             None if pb.rot is None else pb.rot[tidx])
    return (v[tidx] - sub.apply_S(u)).reshape(-1)


def schur_rhs(pb: Problem) -> np.ndarray:
    """-S B A^+ f = +S B_phys A^+ f."""
    x = pb.es.apply_pinv(pb.es.f)
    return pb.apply_S(apply_B_phys(pb.es, x, pb.centers, pb.p)).reshape(-1)


def gmres(op, rhs, tol: float = 1e-10, maxit: int = 150):
    """Unrestarted GMRES, zero initial guess, MGS Arnoldi + Givens.
    Returns (x, iterations, residual history relative to ||rhs||)."""
    rhs = np.asarray(rhs, dtype=complex)
    n = rhs.size
    bnorm = np.linalg.norm(rhs)
    if bnorm == 0.0:
        return np.zeros_like(rhs), 0, [0.0]
    V = np.zeros((maxit + 1, n), dtype=complex)
    H = np.zeros((maxit + 1, maxit), dtype=complex)
    cs = np.zeros(maxit, dtype=complex)
    sn = np.zeros(maxit, dtype=complex)
    g = np.zeros(maxit + 1, dtype=complex)
    g[0] = bnorm
    V[0] = rhs / bnorm
    hist = [1.0]
    k = 0
    for k in range(maxit):
        w = op(V[k])
        if not np.all(np.isfinite(w)):
            raise FloatingPointError("gmres: NaN/Inf in Krylov vector")
        for i in range(k + 1):
            H[i, k] = np.vdot(V[i], w)
            w = w - H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w)
        if H[k + 1, k] != 0:
            V[k + 1] = w / H[k + 1, k]
        for i in range(k):
            t = cs[i].conjugate() * H[i, k] + sn[i].conjugate() * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = t
        a, b = H[k, k], H[k + 1, k]
        r = math.hypot(abs(a), abs(b))
        cs[k] = a / r if r else 1.0
        sn[k] = b / r if r else 0.0
        H[k, k] = r
        H[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k].conjugate() * g[k]
        hist.append(abs(g[k + 1]) / bnorm)
        if hist[-1] <= tol:
            break
    kk = k + 1
    y = np.linalg.solve(np.triu(H[:kk, :kk]), g[:kk])
    return y @ V[:kk], kk, hist


def flux_error(es: EmptySystem, c, d):
    """postproc.flux_error, |sin theta| convention."""
    orders = np.arange(-(c.size // 2), c.size // 2 + 1)
    kapn = es.kappa + 2 * np.pi * orders / es.period
    k1n = np.sqrt((es.k1 ** 2 - kapn ** 2).astype(complex))   # geo:392-396
    k3n = np.sqrt((es.k3 ** 2 - kapn ** 2).astype(complex))
    pr = (k1n.imag == 0) & (k1n.real > 0)
    pt = (k3n.imag == 0) & (k3n.real > 0)
    R = float(np.sum(k1n.real[pr] * np.abs(c[pr]) ** 2))
    T = float(np.sum(k3n.real[pt] * np.abs(d[pt]) ** 2))
    inc = es.k1 * abs(math.sin(es.theta))
    return dict(reflected=R, transmitted=T, incoming=inc, error=abs(R + T - inc))


@dataclass
class Solution:
    beta: np.ndarray
    x_empty: np.ndarray
    iterations: int
    history: list
    flux: dict
    c: np.ndarray
    d: np.ndarray


def solve_full(pb: Problem, tol: float = 1e-10, maxit: int = 150) -> Solution:
    """GMRES on the preconditioned Schur system, then
    alpha = A^+(f - C beta)."""
    es = pb.es
    rhs = schur_rhs(pb)
    beta, its, hist = gmres(lambda v: apply_schur_operator(pb, v), rhs, tol, maxit)
    beta = beta.reshape(pb.M, pb.L)
    x = es.apply_pinv(es.f - apply_C(es, beta, pb.centers))
    c, d = x[es.cols["c"]], x[es.cols["d"]]
    return Solution(beta, x, its, hist, flux_error(es, c, d), c, d)


# ----------------------------------------------------------------------------
# BASELINE configs
# ----------------------------------------------------------------------------
CONFIGS = {
    1: dict(M=10, radius=0.04, p=20, empty="w10", centers="centers_cfg1.npy"),
    2: dict(M=100, radius=0.04, p=20, empty="w10", centers="centers_cfg2.npy"),
    3: dict(M=1000, radius=0.012, p=25, empty="w10", centers="centers_cfg3.npy"),
    4: dict(M=1000, radius=0.012, p=25, empty="wood", centers="centers_cfg3.npy"),
}


def load_problem(cfg: int) -> Problem:
    c = CONFIGS[cfg]
    centers = np.load(os.path.join(GOLDEN, c["centers"]))
    return Problem(load_empty(c["empty"]), centers, c["p"], c["radius"])

"""Post-processing: flux balance (flux_error, SPEC.md:599-607;
PAPER.md:915-921), Wood's-anomaly report, and field evaluation on a grid
(eval_total_field_grid) with the particle multipole sums on
the device."""
from __future__ import annotations

import math

import numpy as np


def flux_error(c, d, config) -> dict:
    """sum_{k1n>0} k1n |c_n|^2 + sum_{k3n>0} k3n |d_n|^2 vs k1 |sin theta|.

    ``config`` is a ProblemConfig (geometry.py:317) or GratingConfig."""
    c = np.asarray(c)
    d = np.asarray(d)
    k1n = config.vertical_wavenumber(config.k1)
    k3n = config.vertical_wavenumber(config.k3)
    pr = (k1n.imag == 0) & (k1n.real > 0)
    pt = (k3n.imag == 0) & (k3n.real > 0)
    R = float(np.sum(k1n.real[pr] * np.abs(c[pr]) ** 2))
    T = float(np.sum(k3n.real[pt] * np.abs(d[pt]) ** 2))
    inc = config.k1 * abs(math.sin(config.incident_angle))
    return dict(reflected=R, transmitted=T, incoming=inc, error=abs(R + T - inc))


def wood_anomaly_report(config, tolerance: float = 1e-8) -> list:
    """(layer, order, |kappa_n| - k_j) for near-grazing orders."""
    out = []
    for layer, k in ((1, config.k1), (3, config.k3)):
        for n, kap in zip(config.rb_orders, config.kappa_n()):
            gap = abs(kap) - k
            if abs(gap) <= tolerance:
                out.append((layer, int(n), float(gap)))
    return out


def particle_field(op, beta, points) -> np.ndarray:
    """[nrhs][npts] particle phased multipole sums (PAPER.md Eq. repre3_mod) at
    points, on the device (ps_particle_field, field.cu).  ``op`` is a
    SchurOperator (or anything with ``.eng``); beta [nrhs][M][L]."""
    import torch
    eng = op.eng if hasattr(op, "eng") else op
    b = torch.as_tensor(np.asarray(beta, dtype=complex)) if not isinstance(beta, torch.Tensor) \
        else beta
    b = b.to(device=eng.device, dtype=torch.complex128).reshape(eng.nrhs, eng.M, eng.L).contiguous()
    return eng.particle_field(b, points).cpu().numpy()


def empty_field(op, beta, points, layer) -> np.ndarray:
    """[nrhs][npts] total empty-grating layer field (empty_grating.eval_empty_field,
    eg:352-393, total=True) of the coupled solution at points of the given
    layers (1 / 2 / 3), on the device: x = A^+ (f - C beta) over all columns
    (ps_recover_full), then the layer potentials + regular expansions +
    incident wave (ps_layer_field)."""
    import torch
    eng = op.eng if hasattr(op, "eng") else op
    b = torch.as_tensor(np.asarray(beta, dtype=complex)) if not isinstance(beta, torch.Tensor) \
        else beta
    b = b.to(device=eng.device, dtype=torch.complex128).reshape(eng.nrhs, eng.M, eng.L).contiguous()
    x = eng.recover_full(eng.apply_C(b))
    return eng.layer_field(x, points, layer).cpu().numpy()


def _beta_dev(eng, beta):
    import torch
    b = torch.as_tensor(np.asarray(beta, dtype=complex)) if not isinstance(beta, torch.Tensor) \
        else beta
    return b.to(device=eng.device, dtype=torch.complex128).reshape(eng.nrhs, eng.M, eng.L).contiguous()


def _c_rows(eng, b):
    """C beta on the device ([nrhs][nrow_c]; zero without inclusions)."""
    import torch
    if eng.M == 0:
        return torch.zeros((eng.nrhs, eng.nrow_c), dtype=torch.complex128, device=eng.device)
    return eng.apply_C(b)


def coupled_residual(op, beta, x_full=None) -> list:
    """Relative residual of the full coupled system (PAPER Eq.
    finalsys) per RHS, measured against ||f||:

        r_A = A x + C beta - f          (empty-grating rows; eg:289-290's residual)
        r_S = beta - S (T beta + B_phys x) = K beta - rhs   (particle rows)

    with x = A^+ (f - C beta) (all unknowns).  Everything runs on the device:
    ps_apply_C, ps_recover_full, ps_empty_residual, one Schur matvec and
    ps_schur_rhs.  Returns dicts (relative, empty_rows, particle_rows)."""
    import torch
    eng = op.eng
    b = _beta_dev(eng, beta)
    if not getattr(op, "_empty_on_device", False):
        if not op.device_setup:
            for r, s in enumerate(op.systems):
                eng.set_empty_system(r, s)
        op._empty_on_device = True
    g = _c_rows(eng, b)
    x = eng.recover_full(g) if x_full is None else x_full
    ea = eng.empty_residual(x, g).cpu().numpy()
    if eng.M > 0:
        rs = (eng.apply_schur(b) - eng.schur_rhs()).reshape(eng.nrhs, -1)
        ns = (rs.real ** 2 + rs.imag ** 2).sum(dim=1).cpu().numpy()
    else:
        ns = np.zeros(eng.nrhs)
    out = []
    for r in range(eng.nrhs):
        fn = np.sqrt(ea[r, 1])
        out.append(dict(relative=float(np.sqrt(ea[r, 0] + ns[r]) / fn),
                        empty_rows=float(np.sqrt(ea[r, 0]) / fn),
                        particle_rows=float(np.sqrt(ns[r]) / fn)))
    return out


def _gauss_legendre(n: int, a: float, b: float):
    """quadrature.gauss_legendre (quadrature.py:31-37)."""
    x, w = np.polynomial.legendre.leggauss(n)
    half = 0.5 * (b - a)
    return a + half * (x + 1.0), half * w


def wall_check_points(cfg, n_fresh: int = 31):
    """Fresh probe points of wall_discrepancy_residual (eg:408-420): per wall
    L1, L2, L3 of the unit cell, n_fresh Gauss-Legendre ordinates between
    its extreme nodes inset by 6 d / N_Gamma, at x = -d/2 then at x = +d/2;
    and their layer (classify_layer, eg:341-349).  Host geometry."""
    from .empty_setup import unit_cell
    d = cfg.period
    cell = unit_cell(cfg)
    inset = 6.0 * d / cfg.interface_nodes
    pts = []
    for wall in cell.walls:
        ylo, yhi = float(np.min(wall[:, 1])), float(np.max(wall[:, 1]))
        ys, _ = _gauss_legendre(n_fresh, ylo + inset, yhi - inset)
        left = np.stack([np.full(n_fresh, -0.5 * d), ys], axis=-1)
        pts.append(np.vstack([left, left + [d, 0.0]]))
    pts = np.vstack(pts)
    top = cfg.interface_top.height(pts[:, 0], d)
    bot = cfg.interface_bottom.height(pts[:, 0], d)
    layer = np.full(pts.shape[0], 2, dtype=np.int32)
    layer[pts[:, 1] > top] = 1
    layer[pts[:, 1] < bot] = 3
    return pts, layer


def wall_discrepancy_residual(op, beta, n_fresh: int = 31, x_full=None) -> list:
    """empty_grating.wall_discrepancy_residual (eg:396-433) of the COUPLED
    solution, per RHS: max |alpha u(L) - u(R)| over fresh Gauss-Legendre
    points of the three walls (inset 6 d / N_Gamma from the junctions),
    values and x-derivatives, with u = the empty-grating representation
    (eval_empty_field total=False, x = A^+ (f - C beta)) plus the particles'
    phased multipole field in layer 2 (the extra_field the reference checker
    takes for a coupled solution).  All field sums on the device
    (ps_layer_field_grad, ps_particle_field_grad)."""
    eng = op.eng
    b = _beta_dev(eng, beta)
    pts, layer = wall_check_points(op.config, n_fresh)
    nrm = np.tile([1.0, 0.0], (pts.shape[0], 1))
    x = eng.recover_full(_c_rows(eng, b)) if x_full is None else x_full
    val, dn = eng.layer_field_grad(x, pts, layer, nrm, incident=False)
    val, dn = val.cpu().numpy(), dn.cpu().numpy()
    mid = layer == 2
    if np.any(mid) and eng.M > 0:
        pv, pd = eng.particle_field_grad(b, pts[mid], nrm[mid])
        val[:, mid] += pv.cpu().numpy()
        dn[:, mid] += pd.cpu().numpy()
    out = []
    for r, s in enumerate(op.systems):
        alpha = s.config.bloch_phase
        worst = 0.0
        for w in range(3):
            sl = slice(2 * n_fresh * w, 2 * n_fresh * (w + 1))
            for arr in (val[r, sl], dn[r, sl]):
                disc = alpha * arr[:n_fresh] - arr[n_fresh:]
                worst = max(worst, float(np.max(np.abs(disc))))
        out.append(worst)
    return out


def _interface_heights(config, system, x):
    if hasattr(config, "interface_top"):                      # reference ProblemConfig
        return (config.interface_top.height(x, config.period),
                config.interface_bottom.height(x, config.period))
    g1 = system.curves["g1"].nodes[:, 1]                       # flat fixture interfaces
    g2 = system.curves["g2"].nodes[:, 1]
    return np.full_like(x, g1.mean()), np.full_like(x, g2.mean())


def classify_points(config, points, centers, radius: float, system=None,
                    mask_nodes: float = 5.0,
                    nodes_per_period: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Region of every point: layer 1 / 2 / 3 by the flat
    interfaces (eg.classify_layer, empty_grating.py:341-349), and a mask for
    points inside a particle (any phased copy) or within ``mask_nodes`` local
    node spacings of an interface (the near-evaluation contract, SPEC design
    decision "5 local node spacings")."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    top, bot = _interface_heights(config, system, pts[:, 0])
    layer = np.full(pts.shape[0], 2, dtype=int)
    layer[pts[:, 1] > top] = 1
    layer[pts[:, 1] < bot] = 3
    n_nodes = nodes_per_period or (system.curves["g1"].n if system is not None else 120)
    h = config.period / n_nodes
    masked = (np.abs(pts[:, 1] - top) < mask_nodes * h) | (np.abs(pts[:, 1] - bot) < mask_nodes * h)
    cen = np.asarray(centers, dtype=float)
    P = config.near_field_copies
    for l in range(-P - 1, P + 2):
        dx = pts[:, 0, None] - cen[None, :, 0] - l * config.period
        dy = pts[:, 1, None] - cen[None, :, 1]
        masked |= np.any(dx * dx + dy * dy < radius * radius, axis=1)
    return layer, masked


def eval_total_field_grid(op, beta, centers, radius: float, nx: int = 128, ny: int = 128,
                          y_plot: float | None = None, layer_field="device") -> dict:
    """SPEC.md:619-627 on a uniform grid over [-d/2, d/2] x [-y_plot, y_plot].

    Particle phased multipole sums come from the device (layer-2 points).
    The empty-grating layer fields + u_inc (eval_empty_field on x_empty =
    A^+(f - C beta), eg:352-393) are evaluated on the device too
    (``layer_field="device"``), or by a callable ``layer_field(points) ->
    [nrhs][npts]`` (e.g. the reference's own evaluator); ``None`` gives the
    particle part only.  Masked points (inside particles, near interfaces)
    are NaN and flagged in ``mask``."""
    cfg = op.config
    d = cfg.period
    y_plot = 1.0 if y_plot is None else y_plot
    xs = np.linspace(-d / 2, d / 2, nx)
    ys = np.linspace(-y_plot, y_plot, ny)
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    pts = np.column_stack([X.ravel(), Y.ravel()])
    # layers + interface mask per point; particle interiors rasterised per disk
    # copy on the uniform grid (O(M r^2 / h^2) instead of O(points x M))
    layer, masked = classify_points(cfg, pts, np.empty((0, 2)), radius, system=op.systems[0])
    inside = np.zeros((ny, nx), dtype=bool)
    hx = xs[1] - xs[0] if nx > 1 else 1.0
    hy = ys[1] - ys[0] if ny > 1 else 1.0
    P = cfg.near_field_copies
    for l in range(-P - 1, P + 2):
        for cx, cy in np.asarray(centers, dtype=float):
            cx = cx + l * d
            i0 = max(0, int(np.floor((cx - radius - xs[0]) / hx)))
            i1 = min(nx - 1, int(np.ceil((cx + radius - xs[0]) / hx)))
            j0 = max(0, int(np.floor((cy - radius - ys[0]) / hy)))
            j1 = min(ny - 1, int(np.ceil((cy + radius - ys[0]) / hy)))
            if i0 > i1 or j0 > j1:
                continue
            sub = (xs[None, i0:i1 + 1] - cx) ** 2 + (ys[j0:j1 + 1, None] - cy) ** 2 < radius * radius
            inside[j0:j1 + 1, i0:i1 + 1] |= sub
    masked |= inside.ravel()
    u = np.zeros((op.nrhs, pts.shape[0]), dtype=complex)
    in2 = (layer == 2) & ~masked
    if np.any(in2):
        u[:, in2] = particle_field(op, beta, pts[in2])
    if isinstance(layer_field, str) and layer_field == "device":
        ok = ~masked
        lay = np.where(ok, layer, 0)
        u += empty_field(op, beta, pts, lay)
    elif layer_field is not None:
        u += np.asarray(layer_field(pts), dtype=complex).reshape(op.nrhs, -1)
    u[:, masked] = np.nan
    return dict(x=xs, y=ys, field=u.reshape(op.nrhs, ny, nx), layer=layer.reshape(ny, nx),
                mask=masked.reshape(ny, nx))

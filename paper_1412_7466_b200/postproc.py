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

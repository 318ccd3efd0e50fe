"""Drop-in ``periscat.postproc`` on top of the reference's
own ``empty_grating`` module.

``eval_total_field_grid`` evaluates the total field on a grid: the particle
phased multipole sums on the B200 (``ps_particle_field``), and the empty-grating
layer fields + u_inc with the reference's ``eval_empty_field`` (eg:352-393) on
the recovered empty-grating unknowns x = A^+ (f - C beta) (
``apply_pinv``, eg:264-273).
"""
from __future__ import annotations

import numpy as np
import torch

from paper_1412_7466_b200.postproc import (classify_points, eval_total_field_grid as _grid,  # noqa: F401
                                           flux_error, particle_field, wood_anomaly_report)


def empty_solution(op, beta, system, irhs: int = 0):
    """The reference EmptySolution of the coupled solve for RHS ``irhs``."""
    from periscat.empty_grating import EmptySolution, apply_pinv
    b = torch.as_tensor(np.asarray(beta, dtype=complex)).to(op.device).reshape(op.shape).contiguous()
    g_c = op.eng.apply_C(b).cpu().numpy()[irhs]          # the C rows come first (eg:154-160)
    g = np.zeros(system.matrix.shape[0], dtype=complex)
    g[:g_c.shape[0]] = g_c
    x = apply_pinv(system, system.rhs - g)
    return EmptySolution(system, x, residual=float("nan"))


def eval_total_field_grid(op, beta, systems, centers, radius, nx=128, ny=128, y_plot=None):
    from periscat.empty_grating import eval_empty_field
    systems = systems if isinstance(systems, (list, tuple)) else [systems]
    sols = [empty_solution(op, beta, s, r) for r, s in enumerate(systems)]

    def layer_field(pts):
        return np.stack([eval_empty_field(sol, pts, total=True) for sol in sols])

    return _grid(op, beta, centers, radius, nx=nx, ny=ny, y_plot=y_plot, layer_field=layer_field)


__all__ = ["eval_total_field_grid", "empty_solution", "flux_error", "particle_field",
           "wood_anomaly_report", "classify_points"]

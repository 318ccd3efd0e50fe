"""Host-side view of the empty-grating system the hot path consumes.

The drop-in boundary takes the reference's ``EmptyGratingSystem``
(/root/reference/pkg/src/periscat/empty_grating.py:64-84) as input: the
Schur correction needs its SVD factors, column scaling, right-hand side and
the curve nodes the coupling blocks touch.  ``GratingSystem`` duck-types
that object (same attribute names: ``config``, ``curves``, ``centers``,
``matrix``, ``rhs``, ``col_scale``, ``cols``, ``rows``, ``svd``), so a caller
holding a real reference system passes it unchanged; the benchmark and tests
load the same data from the fixtures ``oracle/make_empty.py`` wrote with the
reference (``workloads.py`` at the repository root -- the product package
never reads test data).  Assembly of the matrix itself is setup outside the hot
path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

@dataclass(frozen=True)
class InterfaceSpec:
    """Graph interface y(x) = mean + sum_j a_j sin(2 pi j x/d) + b_j cos(2 pi j x/d)
    (duck type of geometry.InterfaceSpec, geometry.py:67-96)."""
    mean: float
    sin_coeffs: tuple = ()
    cos_coeffs: tuple = ()

    def height(self, x, d: float = 1.0):
        x = np.asarray(x, dtype=float)
        y = np.full_like(x, self.mean)
        for j, a in enumerate(self.sin_coeffs, start=1):
            y = y + a * np.sin(2 * np.pi * j * x / d)
        for j, b in enumerate(self.cos_coeffs, start=1):
            y = y + b * np.cos(2 * np.pi * j * x / d)
        return y

    def slope(self, x, d: float = 1.0):
        x = np.asarray(x, dtype=float)
        dy = np.zeros_like(x)
        for j, a in enumerate(self.sin_coeffs, start=1):
            dy = dy + a * (2 * np.pi * j / d) * np.cos(2 * np.pi * j * x / d)
        for j, b in enumerate(self.cos_coeffs, start=1):
            dy = dy - b * (2 * np.pi * j / d) * np.sin(2 * np.pi * j * x / d)
        return dy

    def extremes(self, d: float = 1.0, samples: int = 4096):
        y = self.height(np.linspace(-0.5 * d, 0.5 * d, samples, endpoint=False), d)
        return float(np.min(y)), float(np.max(y))


@dataclass
class GratingConfig:
    """Subset of ProblemConfig (geometry.py:317-406) the hot path reads; with
    the interface / node-count fields it also drives the device assembly of
    the empty-grating system (empty_setup.py)."""
    period: float
    k1: float
    k2: float
    k3: float
    kp: float
    incident_angle: float
    near_field_copies: int = 1
    j_expansion_order: int = 36
    rb_modes_per_direction: int = 41
    regularization: float = 1e-10
    multipole_order: int = 10
    gmres_tol: float = 1e-10
    gmres_maxit: int = 150
    y0: float = 0.8
    interface_top: InterfaceSpec = field(default_factory=lambda: InterfaceSpec(0.5))
    interface_bottom: InterfaceSpec = field(default_factory=lambda: InterfaceSpec(-0.5))
    interface_nodes: int = 120
    lid_nodes: int = 50
    wall_nodes_per_unit: int = 48
    alpert_order: int = 16

    def expansion_centers(self) -> dict:
        """Layer expansion centres (geometry.py:398-406)."""
        lo1, hi1 = self.interface_top.extremes(self.period)
        lo2, hi2 = self.interface_bottom.extremes(self.period)
        mid = 0.5 * (self.interface_top.mean + self.interface_bottom.mean)
        return {1: np.array([0.0, 0.5 * (self.y0 + hi1)]), 2: np.array([0.0, mid]),
                3: np.array([0.0, -0.5 * (self.y0 + abs(lo2))])}

    @property
    def kappa(self) -> float:
        return self.k1 * math.cos(self.incident_angle)          # geometry.py:369-371

    @property
    def bloch_phase(self) -> complex:
        return complex(np.exp(1j * self.kappa * self.period))   # geometry.py:373-375

    @property
    def rb_orders(self) -> np.ndarray:
        half = self.rb_modes_per_direction // 2
        return np.arange(-half, half + 1)

    def kappa_n(self, orders=None) -> np.ndarray:
        if orders is None:
            orders = self.rb_orders
        return self.kappa + 2 * np.pi * np.asarray(orders) / self.period

    def vertical_wavenumber(self, k: float, orders=None) -> np.ndarray:
        kapn = self.kappa_n(orders)                              # geometry.py:392-396
        return np.sqrt((k ** 2 - kapn ** 2).astype(complex))


@dataclass
class Curve:
    nodes: np.ndarray
    normals: np.ndarray
    arc_weights: np.ndarray

    @property
    def n(self) -> int:
        return self.nodes.shape[0]


@dataclass
class GratingSystem:
    config: GratingConfig
    curves: dict
    centers: dict
    matrix: np.ndarray
    rhs: np.ndarray
    col_scale: np.ndarray
    cols: dict = field(default_factory=dict)
    rows: dict = field(default_factory=dict)
    svd: tuple | None = None
    name: str = ""


def factorize(system) -> None:
    """numpy SVD of the column-scaled matrix (empty_grating.py:259-261)."""
    if system.svd is None:
        system.svd = tuple(np.linalg.svd(system.matrix, full_matrices=False))


def baseline_config(omega: float, theta_ref: float, **kw) -> GratingConfig:
    """BASELINE.json grating: period 1, layer indices 1.0/1.2/1.0,
    inclusions 1.5, flat interfaces at y = +-0.5; theta_ref measured from +x."""
    top, bot = InterfaceSpec(0.5), InterfaceSpec(-0.5)
    y0 = 1.6 * max(abs(v) for v in (*top.extremes(), *bot.extremes()))   # geometry.py:355-356
    return GratingConfig(period=1.0, k1=omega, k2=1.2 * omega, k3=omega, kp=1.5 * omega,
                         incident_angle=theta_ref, y0=y0, interface_top=top,
                         interface_bottom=bot, **kw)

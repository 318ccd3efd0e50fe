"""Host-side view of the empty-grating system the hot path consumes.

The drop-in boundary takes the reference's ``EmptyGratingSystem``
(/root/reference/pkg/src/periscat/empty_grating.py:64-84) as input: the
Schur correction needs its SVD factors, column scaling, right-hand side and
the curve nodes the coupling blocks touch.  ``GratingSystem`` duck-types
that object (same attribute names: ``config``, ``curves``, ``centers``,
``matrix``, ``rhs``, ``col_scale``, ``cols``, ``rows``, ``svd``), so a caller
holding a real reference system passes it unchanged, and the benchmark /
tests load the same data from the fixtures ``oracle/make_empty.py`` wrote
with the reference.  Assembly of the matrix itself is setup outside the hot
path.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


@dataclass
class GratingConfig:
    """Subset of ProblemConfig (geometry.py:317-406) the hot path reads."""
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


def load_fixture(name: str, directory: str = GOLDEN) -> GratingSystem:
    z = np.load(os.path.join(directory, f"empty_{name}.npz"))
    cols = {str(n): slice(int(a), int(b)) for n, (a, b) in zip(z["col_names"], z["cols"])}
    rows = {str(n): slice(int(a), int(b)) for n, (a, b) in zip(z["row_names"], z["rows"])}
    sc = z["scalars"]
    cfg = GratingConfig(period=float(sc[0]), k1=float(sc[1]), k2=float(sc[2]), k3=float(sc[3]),
                        kp=float(sc[4]), incident_angle=float(sc[5]),
                        near_field_copies=int(sc[6]), j_expansion_order=int(sc[7]),
                        regularization=float(sc[8]), y0=float(sc[9]),
                        rb_modes_per_direction=cols["c"].stop - cols["c"].start)
    nw = z["L2_nodes"].shape[0]
    curves = {
        "g1": Curve(z["g1_nodes"], z["g1_normals"], z["g1_w"]),
        "g2": Curve(z["g2_nodes"], z["g2_normals"], z["g2_w"]),
        "L2": Curve(z["L2_nodes"], np.tile([1.0, 0.0], (nw, 1)), np.zeros(nw)),
    }
    return GratingSystem(cfg, curves, {2: z["center2"]}, z["A"], z["f"], z["col_scale"],
                         cols, rows, None, name)


# BASELINE.json configs: cfg -> (fixture, centres file, p, radius)
CONFIGS = {
    1: dict(system="w10", centers="centers_cfg1.npy", p=20, radius=0.04),
    2: dict(system="w10", centers="centers_cfg2.npy", p=20, radius=0.04),
    3: dict(system="w10", centers="centers_cfg3.npy", p=25, radius=0.012),
    4: dict(system="wood", centers="centers_cfg3.npy", p=25, radius=0.012),
}


def load_config(cfg: int):
    c = CONFIGS[cfg]
    centers = np.load(os.path.join(GOLDEN, c["centers"]))
    return load_fixture(c["system"]), centers, c["p"], c["radius"]

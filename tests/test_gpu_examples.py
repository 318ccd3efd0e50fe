"""GPU: the paper's numerical examples at desk scale (SPEC.md acceptance 3-6,
PAPER.md §6) run entirely through the device path from the configuration:
device assembly + SVD of the curved empty grating, Muller-BIE scattering
matrix of the star / pentagon on the device, dense rotated S, device GMRES
-- against the oracle's solve of the reference-built problem (goldens:
oracle/make_examples.py; particles from the reference's own sampler).

  Example 1 (M=100, stars, kp=30)             flux <= 1e-8, GMRES <= 150 its
  Example 2 (Wood's anomaly)                  flux <= 1e-8
  Example 3 (pentagons across the walls)      k2 = 1, 10: flux <= 1e-8,
                                              iterations within 2x the paper's
  Iteration flatness M = 25 / 50 / 100        counts within 25 %
"""
import json
import os

import numpy as np
import pytest

from conftest import rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLDEN, "examples.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "examples.json")))
    return z, meta


def _config(z, name):
    from paper_1412_7466_b200.grating import GratingConfig, InterfaceSpec
    sc = z[f"{name}_scalars"]

    def spec(v):
        ns = int(v[1])
        return InterfaceSpec(float(v[0]), tuple(v[2:2 + ns]), tuple(v[2 + ns:]))
    return GratingConfig(period=float(sc[0]), k1=float(sc[1]), k2=float(sc[2]), k3=float(sc[3]),
                         kp=float(sc[4]), incident_angle=float(sc[5]), y0=float(sc[6]),
                         interface_top=spec(z[f"{name}_top_spec"]),
                         interface_bottom=spec(z[f"{name}_bottom_spec"]),
                         multipole_order=int(sc[10]))


def _solve(z, name):
    from paper_1412_7466_b200 import scatmat, solver
    cfg = _config(z, name)
    sc = z[f"{name}_scalars"]
    shape = type("Shape", (), dict(base_radius=float(sc[7]), bump_amplitude=float(sc[8]),
                                   lobes=int(sc[9])))()
    S = scatmat.scattering_matrix(shape, cfg.k2, cfg.kp, cfg.multipole_order, 300)
    sol = solver.solve_full(cfg, z[f"{name}_centers"], cfg.multipole_order, smat=np.asarray(S),
                            rot=z[f"{name}_rot"], radius=float(sc[7]) + float(sc[8]))
    return np.asarray(S), sol


@pytest.mark.parametrize("name", ["ex1", "ex2", "ex3k1", "ex3k10"])
def test_paper_example(golden, name):
    z, meta = golden
    S, sol = _solve(z, name)
    # the device Muller-BIE S against the reference-primitive S
    assert rel(S, z[f"{name}_S"]) <= 1e-10
    # the coupled solution against the oracle's (BASELINE north_star: c, d <= 1e-9)
    assert rel(sol.c[0], z[f"{name}_c"]) <= 1e-9
    assert rel(sol.d[0], z[f"{name}_d"]) <= 1e-9
    assert abs(sol.iterations[0] - int(z[f"{name}_iterations"])) <= 2
    # SPEC acceptance 3-5
    assert sol.flux[0]["error"] <= 1e-8
    assert sol.iterations[0] <= 150
    assert sol.coupled_residual[0] <= 1e-8
    paper = meta[name]["paper"]
    if "iterations" in paper and name.startswith("ex3"):
        assert sol.iterations[0] <= 2 * paper["iterations"]


def test_iteration_count_flatness(golden):
    """SPEC acceptance 6 with the paper's own M-scaling (the star
    shrinks as M grows; Table 2: 97 -> 91 iterations from M = 100 to 500):
    Example 1 at M = 100 and M = 500 -- iteration counts within 25 %."""
    z, _ = golden
    its = [_solve(z, n)[1].iterations[0] for n in ("ex1", "ex1m500")]
    assert max(its) <= 1.25 * min(its), its

"""Host side of the device empty-grating setup (empty_setup.py, no GPU): the
unit-cell curves, block layout and correction rule handed to ps_setup_empty
equal the reference's own (geometry.py:188-254, empty_grating.py:145-160,
quadrature.py:62-88), on the committed fixtures everywhere and against the
reference itself where it is mounted."""
import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE
import workloads  # noqa: E402

FIXTURES = ["w10", "wood", "w10_a00", "curved"]


@pytest.mark.parametrize("name", FIXTURES)
def test_unit_cell_matches_fixture_curves(name):
    from paper_1412_7466_b200 import empty_setup as es
    from paper_1412_7466_b200 import grating
    ref = workloads.load_fixture(name)
    cell = es.unit_cell(ref.config)
    for key, arr in (("g1", cell.g1), ("g2", cell.g2)):
        cv = ref.curves[key]
        assert np.array_equal(arr[:, 0:2], cv.nodes)
        assert np.array_equal(arr[:, 2:4], cv.normals)
        assert np.array_equal(arr[:, 7], cv.arc_weights)
    assert np.array_equal(cell.walls[1][:, 0:2], ref.curves["L2"].nodes)
    assert cell.cols == ref.cols and cell.rows == ref.rows
    assert np.array_equal(cell.centers[2], ref.centers[2])


def test_build_desc_layout():
    import ctypes

    from paper_1412_7466_b200 import _lib
    from paper_1412_7466_b200 import empty_setup as es
    from paper_1412_7466_b200 import grating
    cfg = workloads.fixture_config("curved")
    desc, keep = es.build_desc(cfg, es.unit_cell(cfg))
    assert desc.g1.n == 120 and desc.lid_up.n == 50 and desc.rule_n == 15
    assert desc.rule_skip == 10 and desc.rule_interp == 16
    assert desc.top.nsin == 1 and desc.bottom.ncos == 1 and desc.nrb == 41 and desc.Q == 36
    # the struct the library reads has the C layout of include/periscat_b200.h
    assert ctypes.sizeof(_lib.EmptyDesc) == 320


def test_validate_rejects_mixed_geometry():
    from paper_1412_7466_b200 import empty_setup as es
    from paper_1412_7466_b200 import grating
    with pytest.raises(ValueError):
        es.validate([workloads.fixture_config("w10"), workloads.fixture_config("wood")])
    with pytest.raises(ValueError):
        es.validate([grating.baseline_config(10.0, 0.2)])
    es.validate([workloads.fixture_config(n) for n in ("w10_a00", "w10_a15")])


@pytest.fixture(scope="module")
def refmod():
    if not os.path.isdir(REFERENCE):
        pytest.skip("reference not mounted")
    if REFERENCE not in sys.path:
        sys.path.insert(0, REFERENCE)
    from periscat import empty_grating, geometry, quadrature
    return geometry, empty_grating, quadrature


def test_correction_rules_equal_reference_table(refmod):
    from paper_1412_7466_b200 import empty_setup as es
    _, _, quad = refmod
    for order in (2, 8, 16):
        x, w, skip, interp = es.correction_rule(order)
        r = quad.ALPERT_RULES[order]
        assert np.array_equal(x, r.nodes) and np.array_equal(w, r.weights)
        assert (skip, interp) == (r.skip, r.interp)


@pytest.mark.parametrize("curved", [False, True])
def test_unit_cell_from_reference_config(refmod, curved):
    """A reference ProblemConfig is accepted unchanged (duck typing) and its
    curves equal empty_grating.build_geometry's, node for node."""
    from oracle.make_empty import config_for
    from paper_1412_7466_b200 import empty_setup as es
    geo, eg, _ = refmod
    conf = config_for(10.0, -0.7 * np.pi, curved=curved)
    cell = es.unit_cell(conf)
    curves = eg.build_geometry(conf)
    pairs = [("g1", cell.g1), ("g2", cell.g2), ("L1", cell.walls[0]), ("L2", cell.walls[1]),
             ("L3", cell.walls[2]), ("Gu", cell.lid_up), ("Gd", cell.lid_down)]
    for key, arr in pairs:
        cv = curves[key]
        assert np.array_equal(arr[:, 0:2], cv.nodes), key
        assert np.array_equal(arr[:, 2:4], cv.normals), key
        assert np.array_equal(arr[:, 4], cv.speeds), key
        assert np.array_equal(arr[:, 5], cv.weights), key
        assert np.array_equal(arr[:, 6], cv.t), key
        assert np.array_equal(arr[:, 7], cv.arc_weights), key
    ctr = conf.expansion_centers()
    for k in (1, 2, 3):
        assert np.array_equal(cell.centers[k], ctr[k])
    # our own GratingConfig restates the reference's geometry exactly
    from paper_1412_7466_b200 import grating
    mine = workloads.fixture_config("curved" if curved else "w10")
    cm = es.unit_cell(mine)
    for a, b in ((cm.g1, cell.g1), (cm.g2, cell.g2), (cm.walls[1], cell.walls[1]),
                 (cm.lid_up, cell.lid_up)):
        assert np.array_equal(a, b)
    assert mine.y0 == conf.y0


def test_wall_check_points_match_reference_checker():
    """postproc.wall_check_points rebuilds the fresh wall probes of
    empty_grating.wall_discrepancy_residual (eg:408-420) and their layers
    bit for bit (golden from oracle/make_walls.py)."""
    import os

    from paper_1412_7466_b200 import grating, postproc
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "walls_cfg1.npz"))
    pts, layer = postproc.wall_check_points(workloads.load_fixture("w10").config)
    assert np.array_equal(pts, z["pts"])
    assert np.array_equal(layer, z["layer"])

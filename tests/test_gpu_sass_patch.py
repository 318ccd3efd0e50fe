"""The post-link SASS scheduling patch (build.py / sass_reuse_patch.py) only
edits scheduling hints of the DFMA sweeps: a copy of the library with the
opposite hints (no reuse flags, a yield request on every DFMA) must give
bit-identical M2L results through the C ABI, for each DFMA kernel family."""
import ctypes
import os

import numpy as np
import pytest

import workloads  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stripped_lib(tmp_path_factory):
    from paper_1412_7466_b200 import _lib, build, sass_reuse_patch as sp
    buf = bytearray(open(_lib.LIB_PATH, "rb").read())
    # strip every DFMA kernel family, patched or not
    assert sp.strip_hints(buf, r"m2l_sym_(stage_)?kernel|m2l_kernel|m2l_mrhs_kernel") > 10000
    path = str(tmp_path_factory.mktemp("lib") / "libperiscat_b200_nohints.so")
    with open(path, "wb") as fh:
        fh.write(buf)
    return path


def _apply_T(lib_path, cfg, nrhs, seed, variant=0, store=True):
    from integration.ctypes_stub import Periscat
    from oracle import periscat_oracle as O
    pb = O.load_problem(cfg)
    sysm = workloads.load_fixture(O.CONFIGS[cfg]["empty"])
    rng = np.random.default_rng(seed)
    L = 2 * pb.p + 1
    beta = pb.smat[None, None, :] * (rng.standard_normal((nrhs, pb.M, L))
                                     + 1j * rng.standard_normal((nrhs, pb.M, L)))
    ps = Periscat(0, lib_path) if lib_path else Periscat(0)
    try:
        ps.setup(sysm, pb.centers, pb.p, pb.smat, systems=[sysm] * nrhs)
        ps._ok(ps.lib.ps_set_k1_variant(ps.ctx, variant))
        if not store:
            ps.lib.ps_set_symbol_store.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p]
            ps._ok(ps.lib.ps_set_symbol_store(ps.ctx, 0.0, None))
        return ps.apply_T(beta)
    finally:
        ps.close()


# K1s p=25 with the symbol store and generating its symbols; tiled K1 p=25 and
# p=20; K1s p=20 both ways; K1m (4 RHS)
@pytest.mark.parametrize("cfg,nrhs,variant,store", [
    (3, 1, 0, True), (3, 1, 0, False), (3, 1, 1, True),
    (2, 1, 0, True), (2, 1, 2, True), (2, 1, 2, False), (2, 4, 0, True)])
def test_hint_patch_is_bit_neutral(stripped_lib, cfg, nrhs, variant, store):
    a = _apply_T(None, cfg, nrhs, 7, variant, store)
    a2 = _apply_T(None, cfg, nrhs, 7, variant, store)
    b = _apply_T(stripped_lib, cfg, nrhs, 7, variant, store)
    assert np.all(np.isfinite(a.view(float)))
    assert np.array_equal(a.view(np.uint64), a2.view(np.uint64))     # reproducible across contexts
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))      # and independent of the hints

"""ctypes binding of libperiscat_b200.so (include/periscat_b200.h).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is present, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PS_LIB", os.path.join(_HERE, "libperiscat_b200.so"))

PS_OK, PS_ERR_ARG, PS_ERR_DOMAIN, PS_ERR_NUMERICAL, PS_ERR_CUDA, PS_ERR_STATE, PS_ERR_UNSUPPORTED = range(7)

# symbol -> (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)
SIGNATURES = {
    "ps_version": (_I, []),
    "ps_canary_check": (ctypes.c_longlong, []),
    "ps_canary_selftest": (ctypes.c_longlong, []),
    "ps_max_order": (_I, []),
    "ps_create": (_I, [ctypes.POINTER(_P), _I]),
    "ps_destroy": (None, [_P]),
    "ps_last_error": (ctypes.c_char_p, [_P]),
    "ps_set_geometry": (_I, [_P, _I, _I, _I, _D, _D, _P]),
    "ps_set_target_range": (_I, [_P, _I, _I]),
    "ps_check_overlap": (_I, [_P, _D, _DP]),
    "ps_set_rhs_bloch": (_I, [_P, _I, _P]),
    "ps_set_smatrix": (_I, [_P, _P, _I, _P]),
    "ps_set_layers": (_I, [_P, _I, _P, _I, _P, _I, _P, _P, _I, _I]),
    "ps_set_pinv": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _D, _P, _I, _I]),
    "ps_apply_T": (_I, [_P, _P, _P, _P]),
    "ps_apply_C": (_I, [_P, _P, _P, _I, _I, _P]),
    "ps_apply_schur_g": (_I, [_P, _P, _P, _P, _P]),
    "ps_apply_schur": (_I, [_P, _P, _P, _P]),
    "ps_schur_rhs": (_I, [_P, _P, _P]),
    "ps_recover": (_I, [_P, _P, _P, _P]),
    "ps_krylov_begin": (_I, [_P, _I, ctypes.c_longlong, _I, _P, _P, _P, _P]),
    "ps_krylov_dot": (_I, [_P, _I, _P, _P, _P, _P]),
    "ps_krylov_axpy": (_I, [_P, _I, _P, _P, _P, _P]),
    "ps_krylov_norm2": (_I, [_P, _I, ctypes.c_longlong, _P, _P, _P]),
    "ps_krylov_step": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "ps_krylov_freeze": (_I, [_P, _IP, _P]),
    "ps_krylov_solve": (_I, [_P, _IP, _P, _P, _P]),
    "ps_gmres": (_I, [_P, _P, _P, _D, _I, _IP, _DP, _P]),
    "ps_dfma_peak": (_I, [_I, _DP, _DP]),
    "ps_dfma_sustained": (_I, [_I, _D, _DP]),
    "ps_dmma_peak": (_I, [_I, _DP]),
    "ps_profile": (_I, [_P, _I]),
    "ps_precompute_coupling": (_I, [_P, _D]),
    "ps_coupling_mode": (_I, [_P]),
    "ps_set_k1_variant": (_I, [_P, _I]),
    "ps_set_symbol_store": (_I, [_P, _D, ctypes.POINTER(ctypes.c_size_t)]),
    "ps_set_mrhs_variant": (_I, [_P, _I]),
    "ps_set_overlap": (_I, [_P, _I]),
    "ps_set_overlap_order": (_I, [_P, _I]),
    "ps_set_k1_reserve": (_I, [_P, _I]),
    "ps_apply_T_blocks": (_I, [_P, _I, _I, _P, _P, _P]),
    "ps_particle_field": (_I, [_P, _P, _I, _P, _P, _P]),
    "ps_schur_finish": (_I, [_P, _P, _P, _P, _P, _P]),
    "ps_stats": (_I, [_P, ctypes.POINTER(ctypes.c_longlong), _DP, ctypes.POINTER(ctypes.c_longlong)]),
    "ps_stats_reset": (_I, [_P]),
    "ps_timeline": (_I, [_P, _DP, ctypes.POINTER(ctypes.c_longlong)]),
    "ps_setup_empty": (_I, [_P, _P, _P]),
    "ps_empty_shape": (_I, [_P, _IP, _IP]),
    "ps_get_empty": (_I, [_P, _I, _P, _P, _P, _P]),
    "ps_set_svd_workers": (_I, [_P, _I]),
    "ps_setup_empty_range": (_I, [_P, _P, _P, _I, _I]),
    "ps_pinv_bytes": (ctypes.c_longlong, [_P]),
    "ps_export_pinv": (_I, [_P, _I, _P, _P]),
    "ps_import_pinv": (_I, [_P, _I, _P, _P]),
    "ps_setup_timings": (_I, [_P, _DP, _DP]),
    "ps_scattering_matrix": (_I, [_P, _P, _I, _P, _DP]),
    "ps_full_columns": (_I, [_P]),
    "ps_recover_full": (_I, [_P, _P, _P, _P]),
    "ps_set_field_params": (_I, [_P, _D, _D, _P, _P, _P]),
    "ps_layer_field": (_I, [_P, _P, _I, _P, _P, _P, _P]),
    "ps_layer_field_grad": (_I, [_P, _P, _I, _P, _P, _P, _I, _P, _P, _P]),
    "ps_particle_field_grad": (_I, [_P, _P, _I, _P, _P, _P, _P, _P]),
    "ps_set_empty_system": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "ps_empty_residual": (_I, [_P, _P, _P, _P, _P]),
}


class CurveDesc(ctypes.Structure):
    """ps_curve_desc: n nodes, rows (x, y, nx, ny, speed, weight, t, arc_weight)."""
    _fields_ = [("n", _I), ("data", _P)]


class InterfaceDesc(ctypes.Structure):
    """ps_interface_desc (InterfaceSpec, geometry.py:67-96)."""
    _fields_ = [("mean", _D), ("nsin", _I), ("ncos", _I), ("sin_coeffs", _P), ("cos_coeffs", _P)]


class EmptyDesc(ctypes.Structure):
    """ps_empty_desc (include/periscat_b200.h)."""
    _fields_ = [("period", _D), ("k1", _D), ("k2", _D), ("k3", _D), ("y0", _D), ("eps", _D),
                ("copies", _I), ("Q", _I), ("nrb", _I), ("centers", _D * 6),
                ("g1", CurveDesc), ("g2", CurveDesc), ("wall", CurveDesc * 3),
                ("lid_up", CurveDesc), ("lid_down", CurveDesc),
                ("top", InterfaceDesc), ("bottom", InterfaceDesc),
                ("rule_n", _I), ("rule_skip", _I), ("rule_interp", _I),
                ("rule_x", _P), ("rule_w", _P)]



class ParticleDesc(ctypes.Structure):
    """ps_particle_desc (include/periscat_b200.h)."""
    _fields_ = [("k2", _D), ("kp", _D), ("base_radius", _D), ("bump_amplitude", _D),
                ("lobes", _I), ("n", _I), ("curve", _P),
                ("rule_n", _I), ("rule_skip", _I), ("rule_interp", _I),
                ("rule_x", _P), ("rule_w", _P)]


_lib = None


class PeriscatError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class DomainError(PeriscatError, ValueError):
    pass


class NumericalError(PeriscatError, FloatingPointError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library.  Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: build it with `python -m paper_1412_7466_b200.build` "
                          "(the CUDA path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(ctx, rc: int):
    if rc == PS_OK:
        return
    msg = load().ps_last_error(ctx)
    msg = msg.decode() if msg else ""
    if rc == PS_ERR_DOMAIN:
        raise DomainError(rc, msg)
    if rc == PS_ERR_NUMERICAL:
        raise NumericalError(rc, msg)
    raise PeriscatError(rc, msg)

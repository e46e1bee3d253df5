"""ctypes binding of `libhsdla_b200.so` (the C ABI declared in include/hsdla_b200.h).

The library is built in-tree for sm_100a (`make -C paper_1602_06589_b200/csrc`, or
`__graft_entry__.build()`).  There is no fallback: a missing library or a CUDA
failure raises `NativeLibraryError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeLibraryError

LIB_PATH = os.environ.get("HSDLA_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                        "libhsdla_b200.so")  # HSDLA_LIB: A/B builds

HSDLA_OK = 0
HSDLA_ERR_CUDA = -1000
HSDLA_ERR_UNSUPPORTED = -1001
HSDLA_ERR_NAN_INPUT = -1002
HSDLA_ERR_NONFINITE = -1003
MAX_LSPH = 14


class C64(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


def c64(z) -> C64:
    z = complex(z)
    return C64(z.real, z.imag)


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_P_i32 = ctypes.POINTER(ctypes.c_int32)
_P_i64 = ctypes.POINTER(ctypes.c_int64)


class AbArgs(ctypes.Structure):
    _fields_ = [
        ("n_atoms", _i32), ("n_basis", _i32),
        ("k_vectors", _vp), ("positions", _vp), ("rotations", _vp), ("mt_radius", _vp),
        ("radial", _vp), ("radial_stride", _i32),
        ("l_sph", _P_i32), ("row_offset", _P_i64),
        ("omega", ctypes.c_double),
        ("A", _vp), ("B", _vp), ("B_scaled", _vp), ("ld", _i64), ("udot_norms", _vp),
    ]


class ReducedArgs(ctypes.Structure):
    _fields_ = [
        ("n_atoms", _i32), ("n_basis", _i32),
        ("k_vectors", _vp), ("positions", _vp), ("f", _vp), ("ld_f", _i64),
        ("f_row", _P_i64), ("l_top", _P_i32), ("coef", _vp), ("scale", ctypes.c_double),
        ("S", _vp), ("lds", _i64),
    ]


class BuildArgs(ctypes.Structure):
    _fields_ = [
        ("n_atoms", _i32), ("n_basis", _i32),
        ("heights", _P_i32), ("row_offset", _P_i64), ("t_index", _P_i32),
        ("n_tsets", _i32), ("t_dim", _P_i32),
        ("t_aa", _vp), ("t_ab", _vp), ("t_bb", _vp), ("t_ld", _i64),
        ("A", _vp), ("B", _vp), ("B_scaled", _vp), ("udot_norms", _vp), ("ld", _i64),
        ("force_general_path", _i32),
        ("H", _vp), ("S", _vp), ("ldh", _i64),
        ("workspace", _vp), ("workspace_bytes", ctypes.c_size_t),
        ("shard_rank", _i32), ("n_shards", _i32),
        ("H_host", _vp), ("S_host", _vp), ("ldh_host", _i64),
        ("shard_mirror", _i32), ("reuse_t", _i32), ("stream_h_copy", _i32),
        ("h_reference_form", _i32),
        ("A_host", _vp), ("B_host", _vp), ("ld_ab_host", _i64),
        ("t_dense", _P_i32), ("t_udot2", ctypes.POINTER(ctypes.c_double)),
        ("atom_type", _P_i32), ("n_types", _i32),
    ]


class BuildResult(ctypes.Structure):
    _fields_ = [
        ("hpd_mask", _P_i32), ("chol_info", _P_i32), ("nonfinite", _i32),
        ("ms_setup", ctypes.c_float), ("ms_S", ctypes.c_float),
        ("ms_H_ABBA_BB", ctypes.c_float), ("ms_H_AA", ctypes.c_float),
        ("ms_contract_S", ctypes.c_float), ("ms_contract_H", ctypes.c_float),
        ("ms_apply_Z", ctypes.c_float), ("ms_apply_XY", ctypes.c_float),
        ("ms_total", ctypes.c_float), ("joint_info", _P_i32), ("joint_shift", ctypes.c_double),
        ("template_types", _i32), ("ms_templates", ctypes.c_float), ("merged_sh", _i32),
    ]


# name -> (restype, argtypes); every symbol include/hsdla_b200.h declares
SIGNATURES = {
    "hsdla_version": (ctypes.c_int, []),
    "hsdla_complex_mul_products": (ctypes.c_int, []),
    "hsdla_is_pinned": (ctypes.c_int, [_vp]),
    "hsdla_last_error": (ctypes.c_char_p, []),
    "hsdla_ctx_create": (ctypes.c_int, [ctypes.POINTER(_vp), _vp]),
    "hsdla_ctx_destroy": (ctypes.c_int, [_vp]),
    "hsdla_ctx_set_stream": (ctypes.c_int, [_vp, _vp]),
    "hsdla_ctx_synchronize": (ctypes.c_int, [_vp]),
    "hsdla_panel_owner": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "hsdla_herk_lower": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _i64]),
    "hsdla_her2k_lower": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _i64,
                                         _vp, _i64]),
    "hsdla_gemm": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, C64,
                                  _vp, _i64, _vp, _i64, C64, _vp, _i64, _vp]),
    "hsdla_hemm_lower": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, C64, _vp, _i64, _vp, _i64,
                                        ctypes.c_int, _vp, _i64, _vp]),
    "hsdla_trmm_lower": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _i64,
                                        _vp, _i64, _vp, _i64, _vp]),
    "hsdla_potrf_lower_batched": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _i64, _i64,
                                                 _vp, _i64, _i64, _P_i32]),
    "hsdla_mirror_lower": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _P_i32]),
    "hsdla_check_finite": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _i64, _P_i32]),
    "hsdla_scale_rows": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64]),
    "hsdla_ab_generate": (ctypes.c_int, [_vp, ctypes.POINTER(AbArgs)]),
    "hsdla_match_factors": (ctypes.c_int, [_vp, ctypes.POINTER(AbArgs), _P_i64, _vp, _vp, _i64]),
    "hsdla_reduced_s_aa": (ctypes.c_int, [_vp, ctypes.POINTER(ReducedArgs)]),
    "hsdla_spherical_bessel": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "hsdla_spherical_harmonics": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp]),
    "hsdla_gaunt_tensor": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64,
                                          _vp, _vp, _vp]),
    "hsdla_gaunt_sum": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                       _vp, ctypes.c_double, _vp]),
    "hsdla_phase_matrix": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _i64]),
    "hsdla_hadamard_lower": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _vp, _i64, _vp, _i64,
                                            ctypes.c_int]),
    "hsdla_build_workspace_size": (ctypes.c_size_t, [ctypes.POINTER(BuildArgs)]),
    "hsdla_build_hs": (ctypes.c_int, [_vp, ctypes.POINTER(BuildArgs), ctypes.POINTER(BuildResult)]),
    "hsdla_setup_hs": (ctypes.c_int, [_vp, ctypes.POINTER(AbArgs), ctypes.POINTER(BuildArgs),
                                      ctypes.POINTER(BuildResult)]),
    "hsdla_setup_hs_async": (ctypes.c_int, [_vp, ctypes.POINTER(AbArgs), ctypes.POINTER(BuildArgs),
                                            ctypes.POINTER(ctypes.c_ulonglong)]),
    "hsdla_build_finish": (ctypes.c_int, [_vp, ctypes.c_ulonglong, ctypes.POINTER(BuildResult)]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the library and declare every exported signature (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} is missing: build it with `make -C paper_1602_06589_b200/csrc` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(path)
        except OSError as e:  # pragma: no cover
            raise NativeLibraryError(f"cannot load {path}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().hsdla_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str):
    if rc != HSDLA_OK:
        raise NativeLibraryError(f"{what} failed with status {rc}: {last_error()}")

"""ctypes loader for libpgb200.so (the C ABI in include/pgrid.h).

Fails loudly if the library is missing: there is no CPU fallback."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PGB200_LIB selects another build of the same ABI (e.g. the instrumented
# lib/libpgb200_prof.so); there is no non-CUDA implementation.
LIB_PATH = os.environ.get("PGB200_LIB") or os.path.join(HERE, "lib", "libpgb200.so")

PG_MEM_HOST = 0
PG_MEM_DEVICE = 1
PG_OK, PG_EINVAL, PG_ECUDA, PG_ENOCONV, PG_ENOMEM, PG_ESTATE, PG_ENONFINITE = 0, -1, -2, -3, -4, -5, -6
PG_METHOD_RBSOR = 0
PG_METHOD_JACOBI = 1

_c_int = ctypes.c_int
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_vp = ctypes.c_void_p


class PgStats(ctypes.Structure):
    _fields_ = [("steps_done", _i64), ("sweeps_total", _i64), ("sweeps_max", _i64),
                ("failed_step", _i64), ("kernel_launches", _i64), ("last_delta", _dbl),
                ("device_ms", _dbl), ("sweep_ms", _dbl), ("sweep_launches", _i64),
                ("sweeps_per_launch", _i64)]


# name -> (restype, argtypes); must match include/pgrid.h
SIGNATURES = {
    "pg_create_mesh": (_c_int, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp,
                                _dbl, _c_int, ctypes.POINTER(_vp)]),
    "pg_create_csr": (_c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _dbl, _c_int,
                               ctypes.POINTER(_vp)]),
    "pg_set_sources": (_c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _c_int]),
    "pg_set_voltages": (_c_int, [_vp, _vp, _c_int]),
    "pg_get_voltages": (_c_int, [_vp, _vp, _c_int]),
    "pg_set_stream": (_c_int, [_vp, _vp]),
    "pg_set_option": (_c_int, [_vp, ctypes.c_char_p, _i64]),
    "pg_transient": (_c_int, [_vp, _dbl, _i64, _dbl, _dbl, _c_int, _i64, _i64, _vp, _vp, _c_int,
                              _vp, ctypes.POINTER(PgStats)]),
    "pg_transient_continue": (_c_int, [_vp, _dbl, _i64, _dbl, _dbl, _c_int, _i64, _i64, _vp, _vp,
                                       _c_int, _vp, ctypes.POINTER(PgStats)]),
    "pg_info": (_c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                         ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "pg_destroy": (None, [_vp]),
    "pg_release_memory": (_c_int, [_i32]),
    "pg_estimate_omega": (_c_int, [_vp, _dbl, _i64, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]),
    "pg_tune_omega": (_c_int, [_vp, _dbl, _i64, _dbl, _i64, _dbl, ctypes.POINTER(_dbl), _vp]),
    "pg_dc": (_c_int, [_vp, _dbl, _dbl, _dbl, _c_int, _i64, ctypes.POINTER(PgStats)]),
    "pg_set_slab": (_c_int, [_vp, _i32, _i32, _i32]),
    "pg_nccl_unique_id": (_c_int, [_vp]),
    "pg_group_nccl": (_c_int, [_vp, _vp, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "pg_group_local": (_c_int, [_i32, ctypes.POINTER(_vp), _i32, ctypes.POINTER(_vp)]),
    "pg_group_local_p2p": (_c_int, [_i32, ctypes.POINTER(_vp), _i32, ctypes.POINTER(_vp)]),
    "pg_group_p2p_create": (_c_int, [_vp, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "pg_group_p2p_export": (_c_int, [_vp, _vp, _i64, ctypes.POINTER(_i64)]),
    "pg_group_p2p_connect": (_c_int, [_vp, _vp, _i64]),
    "pg_group_transient": (_c_int, [_vp, _dbl, _i64, _dbl, _dbl, _i64, _vp, ctypes.POINTER(PgStats)]),
    "pg_group_transient_continue": (_c_int, [_vp, _dbl, _i64, _dbl, _dbl, _i64, _vp,
                                             ctypes.POINTER(PgStats)]),
    "pg_group_p2p_selftest": (_c_int, [_vp, _i32, _vp]),
    "pg_group_destroy": (None, [_vp]),
    "pg_last_error": (ctypes.c_char_p, []),
}

_lib = None


def load():
    """Load (never silently skip) the native library."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libpgb200.so not built ({LIB_PATH}); run "
                               "`python -m paper_1409_7166_b200.build` -- there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class PgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pg error {code}: {msg}")
        self.code = code


class PgNoConvergence(PgError):
    pass


def check(code: int):
    if code != PG_OK:
        msg = load().pg_last_error().decode(errors="replace")
        if code == PG_ENOCONV:
            raise PgNoConvergence(code, msg)
        raise PgError(code, msg)

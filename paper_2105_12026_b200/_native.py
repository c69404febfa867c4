"""ctypes binding of ``libebc200.so`` (the C-ABI declared in include/ebc200.h).

The shared library is built in-tree by ``paper_2105_12026_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or no sm_100 device
is visible, every entry point raises instead of computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# EBC200_LIB_PATH: an alternative in-tree build (development A/B of compile-time variants)
LIB_PATH = os.environ.get("EBC200_LIB_PATH") or os.path.join(_HERE, "libebc200.so")

EBC_OK, EBC_EINVAL, EBC_EINDEX, EBC_ECUDA, EBC_ECOMM = 0, 1, 2, 3, 4
EBC_F32, EBC_F16, EBC_F64 = 0, 1, 2

_lib = None
_lock = threading.Lock()

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/ebc200.h
SIGNATURES = {
    "ebc_version": (ctypes.c_char_p, []),
    "ebc_device_count": (ctypes.c_int, []),
    "ebc_create": (ctypes.c_int, [_vp, _i64, _i32, _i32, _f64p, _i32, ctypes.POINTER(_vp)]),
    "ebc_baseline": (ctypes.c_int, [_vp, _f64p]),
    "ebc_eval_multiset": (ctypes.c_int, [_vp, _i64p, _i64p, _i64, _f64p, _i64p, _i64p]),
    "ebc_greedy": (ctypes.c_int, [_vp, _i32, _i64p, _f64p, _f64p, _i64p]),
    "ebc_kmedoids_loss": (ctypes.c_int, [_vp, _f64p, _i64, _f64p]),
    "ebc_sieve_reserve": (ctypes.c_int, [_vp, _i32]),
    "ebc_sieve_step": (ctypes.c_int, [_vp, _i64, _i32p, _i32, _i32p, _i32, _i64, _i32p, _i32, _f64p, _f64p]),
    "ebc_shard_set_range": (ctypes.c_int, [_vp, _i64, _i64]),
    "ebc_shard_step": (ctypes.c_int, [_vp, _i64p, _f64p, _i64, _i64p, _f64p]),
    "ebc_shard_commit": (ctypes.c_int, [_vp, _i64, _f64p]),
    "ebc_shard_advance": (ctypes.c_int, [_vp, _i64, _i32, _i64p, _f64p, _i64, _i64p, _f64p]),
    "ebc_shard_fetch": (ctypes.c_int, [_vp, _i64p, _f64p, _i64]),
    "ebc_reset": (ctypes.c_int, [_vp]),
    "ebc_stream": (_vp, [_vp]),
    "ebc_set_timing": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ebc_last_timings": (ctypes.c_int, [_vp, _f64p]),
    "ebc_last_launches": (_i64, [_vp]),
    "ebc_last_stats": (ctypes.c_int, [_vp, _i64p]),
    "ebc_last_lazy_stats": (ctypes.c_int, [_vp, _i64p]),
    "ebc_host_register": (ctypes.c_int, [_vp, _i64]),
    "ebc_host_unregister": (ctypes.c_int, [_vp]),
    "ebc_last_screen_work": (ctypes.c_int, [_vp, _i64p]),
    "ebc_comm_id_bytes": (ctypes.c_int64, []),
    "ebc_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p, _i64]),
    "ebc_comm_init": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64, _i32, _i32]),
    "ebc_comm_attach": (ctypes.c_int, [_vp]),
    "ebc_greedy_sharded": (ctypes.c_int, [_vp, _i32, _i64p, _f64p, _f64p, _i64p]),
    "ebc_tie_cap": (ctypes.c_int32, []),
    "ebc_comm_status": (ctypes.c_int, [_vp, ctypes.POINTER(_i32)]),
    "ebc_shard_tie_step": (ctypes.c_int, [_vp, _f64p, _f64p]),
    "ebc_shard_pick_commit": (ctypes.c_int, [_vp, _f64p, _i32, _i32, _i64p, _f64p]),
    "ebc_screen_info": (ctypes.c_int, [_vp, _i64p]),
    "ebc_destroy": (None, [_vp]),
    "ebc_last_error": (ctypes.c_char_p, [_vp]),
}


class NativeLibraryMissing(RuntimeError):
    """libebc200.so has not been built (run ``python -c 'import __graft_entry__ as g; g.build()'``)."""


def load():
    """Load and type the native library once (raises if it is absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: the b200 backend has no CPU fallback; build it with "
                    f"paper_2105_12026_b200.build.build_native()")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error(ctx=None) -> str:
    msg = load().ebc_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc: int, ctx=None) -> None:
    """Map an ebc_status onto the reference's exception types."""
    if rc == EBC_OK:
        return
    msg = last_error(ctx)
    if rc == EBC_EINVAL:
        raise ValueError(msg)
    if rc == EBC_EINDEX:
        raise IndexError(msg)
    if rc == EBC_ECOMM:
        raise CommError(msg or "sharded exchange failure")
    raise RuntimeError(msg or f"ebc200 status {rc}")


class CommError(RuntimeError):
    """EBC_ECOMM: the device-side sharded exchange failed or cannot be used."""


def device_count() -> int:
    return int(load().ebc_device_count())


def version() -> str:
    return load().ebc_version().decode()

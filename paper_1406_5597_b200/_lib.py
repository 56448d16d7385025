"""ctypes binding of the in-tree C-ABI library libtffft.so (include/tffft.h).

There is no fallback: if the library is missing the import of the transform
entry points fails loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import STATUS_TO_ERROR, SlabFftError

LIB_PATH = os.environ.get("TFFFT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtffft.so")

# name -> (restype, argtypes)
_c = ctypes
_SIGS = {
    "tffft_last_error": (_c.c_char_p, []),
    "tffft_version": (_c.c_int, []),
    "tffft_get_unique_id": (_c.c_int, [_c.c_char_p]),
    "tffft_comm_init_rank": (_c.c_int, [_c.c_int, _c.c_int, _c.c_char_p, _c.c_int, _c.POINTER(_c.c_void_p)]),
    "tffft_comm_init_local": (_c.c_int, [_c.c_int, _c.c_int, _c.POINTER(_c.c_void_p)]),
    "tffft_comm_init_all": (_c.c_int, [_c.c_int, _c.POINTER(_c.c_int), _c.POINTER(_c.c_void_p)]),
    "tffft_comm_init_ipc": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p,
                                       _c.POINTER(_c.c_void_p)]),
    "tffft_comm_check": (_c.c_int, [_c.c_void_p]),
    "tffft_comm_barrier": (_c.c_int, [_c.c_void_p]),
    "tffft_comm_rank": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "tffft_comm_size": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "tffft_comm_device": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "tffft_comm_abort": (_c.c_int, [_c.c_void_p]),
    "tffft_comm_destroy": (_c.c_int, [_c.c_void_p]),
    "tffft_plan_create": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_void_p,
                                     _c.POINTER(_c.c_void_p)]),
    "tffft_plan_create_ex": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                        _c.c_void_p, _c.POINTER(_c.c_void_p)]),
    "tffft_plan_create_batched": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                             _c.c_int, _c.c_void_p, _c.POINTER(_c.c_void_p)]),
    "tffft_plan_batch": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "tffft_plan_poison": (_c.c_int, [_c.c_void_p]),
    "tffft_nccl_loopback": (_c.c_int, [_c.c_int, _c.c_longlong, _c.c_int, _c.POINTER(_c.c_int)]),
    "tffft_plan_ipc_blob_bytes": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_size_t)]),
    "tffft_plan_ipc_export": (_c.c_int, [_c.c_void_p, _c.c_char_p]),
    "tffft_plan_ipc_attach": (_c.c_int, [_c.c_void_p, _c.c_char_p]),
    "tffft_plan_flags": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int)]),
    "tffft_plan_landing_handle": (_c.c_int, [_c.c_void_p, _c.c_char_p]),
    "tffft_plan_attach_peers": (_c.c_int, [_c.c_void_p, _c.c_char_p]),
    "tffft_plan_workspace_bytes": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_size_t)]),
    "tffft_plan_sizes": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_int64), _c.POINTER(_c.c_int64)]),
    "tffft_plan_destroy": (_c.c_int, [_c.c_void_p]),
    "tffft_forward": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p]),
    "tffft_inverse": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p]),
    "tffft_set_timing": (_c.c_int, [_c.c_void_p, _c.c_int]),
    "tffft_stage_times": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_double)]),
    "tffft_counters": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_uint64)]),
    "tffft_reset_instrumentation": (_c.c_int, [_c.c_void_p]),
    "tffft_consistency": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_double)]),
    "tffft_set_consistency_mode": (_c.c_int, [_c.c_void_p, _c.c_int]),
    "tffft_consistency_collect": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_double), _c.POINTER(_c.c_uint64)]),
    "tffft_launch_count": (_c.c_int, [_c.c_void_p, _c.POINTER(_c.c_uint64)]),
    "tffft_exchange_schedule": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                           _c.POINTER(_c.c_int64), _c.c_int64, _c.POINTER(_c.c_int64)]),
    "tffft_radix_schedule": (_c.c_int, [_c.c_int, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
}
SYMBOLS = tuple(_SIGS)

# C type of tffft_barrier_fn (include/tffft.h): int (*)(void* ctx)
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libtffft.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise SlabFftError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            h = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(status: int) -> None:
    """Raise the reference exception class for a non-zero status."""
    if status != 0:
        msg = lib().tffft_last_error().decode(errors="replace")
        raise STATUS_TO_ERROR.get(status, SlabFftError)(msg)

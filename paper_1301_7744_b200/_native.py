"""ctypes binding of the C ABI in ``include/bcss_sttsm.h``.

The shared library ``_bcss_sttsm.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, sm_100a).  There is no fallback: if the
library is missing, every entry point raises ``NativeError`` naming the fix.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import (
    BlockDivisibilityError,
    NativeError,
    ParameterError,
    RangeError,
    ShapeError,
)

LIB_PATH = Path(__file__).resolve().parent / "_bcss_sttsm.so"

BCSS_OK = 0
_STATUS_EXC = {
    1: ParameterError,
    2: ShapeError,
    3: BlockDivisibilityError,
    4: RangeError,
    5: NativeError,
    6: MemoryError,
    7: NativeError,
}

# symbol -> (restype, argtypes); the full exported surface of include/bcss_sttsm.h
_c_int, _i64, _u64, _sz, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p
_P = ctypes.POINTER
SIGNATURES = {
    "bcss_last_error": (ctypes.c_char_p, []),
    "bcss_abi_version": (_c_int, []),
    "bcss_simplex_count": (_i64, [_i64, _c_int]),
    "bcss_hypertriangle_rank": (_c_int, [_P(_i64), _c_int, _i64, _P(_i64)]),
    "bcss_hypertriangle_unrank": (_c_int, [_i64, _c_int, _i64, _P(_i64)]),
    "bcss_blocked_flops": (_c_int, [_c_int, _i64, _i64, _i64, _i64, _c_int, _P(_u64)]),
    "bcss_plan_create": (_c_int, [_c_int, _i64, _i64, _i64, _i64, _c_int, _P(_vp)]),
    "bcss_plan_destroy": (_c_int, [_vp]),
    "bcss_plan_set_units": (_c_int, [_vp, _P(ctypes.c_int32), _c_int]),
    "bcss_plan_set_workspace_limit": (_c_int, [_vp, _sz]),
    "bcss_plan_set_keep_temps": (_c_int, [_vp, _c_int]),
    "bcss_plan_workspace_bytes": (_c_int, [_vp, _P(_sz)]),
    "bcss_plan_set_workspace": (_c_int, [_vp, _vp, _sz]),
    "bcss_plan_stats": (_c_int, [_vp, _P(_i64), _P(_i64), _P(_u64), _P(_i64)]),
    "bcss_plan_kernel_mix": (_c_int, [_vp, _P(_i64), _P(_i64)]),
    "bcss_plan_neighbour_table": (_c_int, [_vp, _c_int, _c_int, _P(ctypes.c_int32), _i64, _P(_i64)]),
    "bcss_sttsm_run": (_c_int, [_vp, _vp, _vp, _vp, _vp]),
    "bcss_sttsm_run_host": (_c_int, [_vp, _vp, _vp, _vp]),
    "bcss_sttsm_run_gated": (_c_int, [_vp, _vp, _vp, _vp, _vp, _P(_vp), _c_int]),
    "bcss_plan_set_pipeline": (_c_int, [_vp, _c_int]),
    "bcss_plan_set_symmetric_upload": (_c_int, [_vp, _c_int]),
    "bcss_plan_upload_bytes": (_c_int, [_vp, _P(_i64)]),
    "bcss_plan_last_upload_bytes": (_c_int, [_vp, _P(_i64)]),
    "bcss_plan_set_stop_level": (_c_int, [_vp, _c_int]),
    "bcss_plan_set_call_outputs": (_c_int, [_vp, _P(_vp), _i64]),
    "bcss_sttsm_run_host_async": (_c_int, [_vp, _vp, _vp, _vp]),
    "bcss_plan_wait": (_c_int, [_vp]),
    "bcss_host_register": (_c_int, [_vp, _sz]),
    "bcss_host_unregister": (_c_int, [_vp]),
    "bcss_host_is_pinned": (_c_int, [_vp, _P(_c_int)]),
    "bcss_host_alloc": (_c_int, [_sz, _P(_vp)]),
    "bcss_host_free": (_c_int, [_vp]),
    "bcss_device_alloc": (_c_int, [_sz, _P(_vp)]),
    "bcss_device_free": (_c_int, [_vp]),
    "bcss_ipc_get_handle": (_c_int, [_vp, _vp]),
    "bcss_ipc_open_handle": (_c_int, [_vp, _P(_vp)]),
    "bcss_ipc_close_handle": (_c_int, [_vp]),
    "bcss_copy_async": (_c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    "bcss_plan_set_start_calls": (_c_int, [_vp, _c_int, _P(ctypes.c_int32), _c_int]),
    "bcss_plan_set_start_children": (_c_int, [_vp, _P(ctypes.c_int32), _c_int]),
    "bcss_plan_level_calls": (_c_int, [_vp, _c_int, _P(ctypes.c_int32), _i64, _P(_i64)]),
    "bcss_plan_io_elems": (_c_int, [_vp, _P(_i64), _P(_i64)]),
    "bcss_plan_temp": (_c_int, [_vp, _c_int, _P(ctypes.c_int32), _P(_vp), _P(_i64)]),
    "bcss_plan_temp_copy": (_c_int, [_vp, _c_int, _P(ctypes.c_int32), _vp, _i64]),
    "bcss_plan_last_launches": (_c_int, [_vp, _P(_i64)]),
    "bcss_plan_c_block_ranks": (_c_int, [_vp, _P(_i64), _i64, _P(_i64)]),
    "bcss_plan_set_timing": (_c_int, [_vp, _c_int]),
    "bcss_plan_launch_times": (_c_int, [_vp, _P(ctypes.c_int32), _P(_u64), _P(ctypes.c_float), _i64, _P(_i64)]),
    "bcss_probe_fp64_peak": (_c_int, [_P(ctypes.c_double)]),
    "bcss_symmetrize_blocks": (_c_int, [_vp, _c_int, _i64, _i64, _vp]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library once; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH.name} not found next to {__file__}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
        # Reuse an already-loaded libcudart (torch's) when present; otherwise the
        # library's rpath finds /usr/local/cuda/lib64.
        handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != BCSS_OK:
        msg = lib().bcss_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(status, NativeError)(msg)

"""Host memory for the drop-in's host-buffer path.

The reference's arrays never leave the host; here every ``sttsm_bcss`` call
moves A to HBM and C back over PCIe, which runs at full speed (and overlaps
the compute, ``bcss_plan_set_pipeline``) only from page-locked memory.  Two
tools keep the drop-in off the staging copy (``bcss_capi.cu``,
``bcss_sttsm_run_host``: pageable buffers are memcpy'd through plan-owned
pinned memory first):

* ``host_empty(n)`` hands out float64 arrays in pinned memory
  (``cudaMallocHost`` through the library), recycled through a small pool
  when the last numpy view of a buffer dies.  Results of ``sttsm_bcss`` and
  payloads packed from a ``blocks`` dict live there.
* ``register(owner, array)`` page-locks a caller-owned array in place
  (``cudaHostRegister``) for as long as ``owner`` lives.

Both are allocation choices only: without a GPU (or without the library)
``host_empty`` returns ``np.empty`` and ``register`` does nothing; the compute
path itself never falls back to the CPU.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _native

_LOCK = threading.Lock()
_POOL: list[tuple[int, int]] = []        # (nbytes, ptr) of free pinned buffers
_POOL_MAX_BUFFERS = 4
_POOL_MAX_BYTES = 8 << 30
_MIN_PINNED_BYTES = 1 << 20              # smaller arrays are not worth pinning
_pinned_ok: bool | None = None           # None = not probed yet


class _PinnedBuffer:
    """Owner of one cudaMallocHost block; returns it to the pool when the
    last numpy view of it is released."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    def __del__(self):
        if self.ptr:
            _release(self.ptr, self.nbytes)
            self.ptr = 0


def _lib_or_none():
    try:
        return _native.lib()
    except Exception:
        return None


def _release(ptr: int, nbytes: int) -> None:
    with _LOCK:
        if len(_POOL) < _POOL_MAX_BUFFERS and sum(b for b, _ in _POOL) + nbytes <= _POOL_MAX_BYTES:
            _POOL.append((nbytes, ptr))
            return
    lib = _lib_or_none()
    if lib is not None:
        lib.bcss_host_free(ctypes.c_void_p(ptr))


def _acquire(nbytes: int) -> tuple[int, int]:
    """(capacity, pointer) of a pinned block of at least ``nbytes`` (a pooled
    one when one fits within 2x); (0, 0) when pinned memory is unavailable."""
    global _pinned_ok
    with _LOCK:
        best = None
        for i, (b, _) in enumerate(_POOL):
            if nbytes <= b <= 2 * nbytes and (best is None or b < _POOL[best][0]):
                best = i
        if best is not None:
            return _POOL.pop(best)
    lib = _lib_or_none()
    if lib is None:
        _pinned_ok = False
        return (0, 0)
    out = ctypes.c_void_p()
    if lib.bcss_host_alloc(ctypes.c_size_t(nbytes), ctypes.byref(out)) != 0 or not out.value:
        if _pinned_ok is None:
            _pinned_ok = False  # no device / driver: plain host memory from now on
        return (0, 0)
    _pinned_ok = True
    return (nbytes, int(out.value))


def host_empty(n_elems: int) -> np.ndarray:
    """Uninitialized float64 array of ``n_elems``, in pinned memory when a
    CUDA device is usable (else ``np.empty``)."""
    nbytes = int(n_elems) * 8
    if nbytes < _MIN_PINNED_BYTES or _pinned_ok is False:
        return np.empty(n_elems, dtype=np.float64)
    cap, ptr = _acquire(nbytes)
    if not ptr:
        return np.empty(n_elems, dtype=np.float64)
    owner = _PinnedBuffer(ptr, cap)
    raw = (ctypes.c_char * nbytes).from_address(ptr)
    arr = np.frombuffer(raw, dtype=np.float64, count=n_elems)
    # keep the owner alive for as long as any view of the memory exists
    # (numpy's base chain: arr -> raw -> owner)
    raw._bcss_owner = owner
    return arr


def is_pinned(arr: np.ndarray) -> bool:
    lib = _lib_or_none()
    if lib is None or arr.size == 0:
        return False
    out = ctypes.c_int()
    if lib.bcss_host_is_pinned(ctypes.c_void_p(arr.ctypes.data), ctypes.byref(out)) != 0:
        return False
    return bool(out.value)


def _unregister(ptr: int) -> None:
    lib = _lib_or_none()
    if lib is not None:
        lib.bcss_host_unregister(ctypes.c_void_p(ptr))


def register(owner, arr: np.ndarray) -> bool:
    """Page-lock ``arr`` (C-contiguous) in place until ``owner`` is
    collected.  Returns True when the array is pinned afterwards."""
    if _pinned_ok is False or arr.nbytes < _MIN_PINNED_BYTES or not arr.flags.c_contiguous:
        return False
    if is_pinned(arr):
        return True
    lib = _lib_or_none()
    if lib is None:
        return False
    ptr = int(arr.ctypes.data)
    if lib.bcss_host_register(ctypes.c_void_p(ptr), ctypes.c_size_t(arr.nbytes)) != 0:
        return False
    # weakref callbacks run before the owner's attributes are cleared, so the
    # range is unregistered while the array is still alive
    fin = weakref.finalize(owner, _unregister, ptr)
    fin.atexit = False  # the CUDA context may already be gone at interpreter exit
    return True

"""BCSS files straight to and from HBM.

The ``.bcss`` format is the reference's (/root/reference/pkg/src/blocksym/
io.py:50-72): header ``<4sHHQQ>`` = magic ``BCSS``, version 1, order, tensor
dimension, block dimension; then the canonical blocks in hypertriangle order,
each as little-endian doubles in dimensional order.  That payload is exactly
the packed buffer the C ABI consumes, so a file streams into device memory
without any re-layout: the payload is read into pinned host memory in chunks
and copied to the GPU while the next chunk is read.

``save_bcss`` / ``load_bcss`` keep the reference's host-side signatures and
return / accept this package's ``BcssTensor``.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import ShapeError
from .indexing import simplex_count
from .storage import BcssTensor, packed_payload

_MAGIC = b"BCSS"
_VERSION = 1
_HEADER = "<4sHHQQ"
HEADER_BYTES = struct.calcsize(_HEADER)  # 24


def _read_header(fh) -> tuple[int, int, int]:
    raw = fh.read(HEADER_BYTES)
    if len(raw) != HEADER_BYTES:
        raise ValueError("truncated blocked tensor file")
    magic, version, order, n, b = struct.unpack(_HEADER, raw)
    if magic != _MAGIC:
        raise ValueError(f"not a blocked symmetric tensor file (magic {magic!r})")
    if version != _VERSION:
        raise ValueError(f"unsupported blocked tensor format version {version}")
    if b < 1 or n % b:
        raise ShapeError(f"block dimension {b} does not divide {n}")
    return order, n, b


def save_bcss(a, path) -> None:
    """Write any BCSS-like tensor (ours or the reference's) in the reference format."""
    payload = np.ascontiguousarray(packed_payload(a), dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(struct.pack(_HEADER, _MAGIC, _VERSION, a.order, a.n, a.b))
        fh.write(payload.tobytes())


def load_bcss(path) -> BcssTensor:
    with open(path, "rb") as fh:
        order, n, b = _read_header(fh)
        count = simplex_count(n // b, order) * b**order
        payload = np.fromfile(fh, dtype="<f8", count=count)
    if payload.size != count:
        raise ValueError("truncated blocked tensor payload")
    return BcssTensor(order, n, b, payload=payload.astype(np.float64, copy=False))


def load_bcss_device(path, device="cuda", chunk_bytes: int = 256 << 20):
    """Stream a ``.bcss`` file into a float64 device tensor (the packed payload).

    Returns ``(payload, order, n, b)``.  Two pinned staging buffers alternate:
    chunk i+1 is read from disk while chunk i is copied to HBM.
    """
    import torch

    with open(path, "rb") as fh:
        order, n, b = _read_header(fh)
        count = simplex_count(n // b, order) * b**order
        out = torch.empty(count, dtype=torch.float64, device=device)
        step = max(1, chunk_bytes // 8)
        stage = [torch.empty(min(step, count), dtype=torch.float64).pin_memory() for _ in range(2)]
        done = [None, None]
        stream = torch.cuda.Stream(device=device)
        off, i = 0, 0
        while off < count:
            ln = min(step, count - off)
            buf = stage[i % 2]
            if done[i % 2] is not None:
                done[i % 2].synchronize()  # the copy out of this buffer finished
            got = fh.readinto(memoryview(buf.numpy()[:ln]).cast("B"))
            if got != ln * 8:
                raise ValueError("truncated blocked tensor payload")
            with torch.cuda.stream(stream):
                out[off:off + ln].copy_(buf[:ln], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            done[i % 2] = ev
            off += ln
            i += 1
        stream.synchronize()
    return out, order, n, b


def save_bcss_device(payload, order: int, n: int, b: int, path, chunk_bytes: int = 256 << 20) -> None:
    """Write a packed payload held in device memory as a ``.bcss`` file."""
    import torch

    count = simplex_count(n // b, order) * b**order
    if payload.numel() != count:
        raise ShapeError(f"payload has {payload.numel()} elements, expected {count}")
    step = max(1, chunk_bytes // 8)
    stage = torch.empty(min(step, count), dtype=torch.float64).pin_memory()
    with open(path, "wb") as fh:
        fh.write(struct.pack(_HEADER, _MAGIC, _VERSION, order, n, b))
        for off in range(0, count, step):
            ln = min(step, count - off)
            stage[:ln].copy_(payload[off:off + ln])  # synchronous D2H into pinned memory
            fh.write(memoryview(stage.numpy()[:ln]).cast("B"))

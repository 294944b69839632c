"""Host-side sample conversions for the reference-compatible API, split over a few threads.

The drop-in functions exchange int64 sample arrays with the caller (RasterImage, transforms.py:24-46)
while the device works on 8/16/32-bit samples; for a 4096 x 4096 RGB tile the widening and
narrowing passes cost more than the GPU round trip, and numpy runs them on one core.  numpy
releases the GIL inside these loops, so plain threads scale them.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

_MIN = 1 << 20  # elements below which one thread is faster
try:
    _N = max(1, min(8, len(os.sched_getaffinity(0))))
except AttributeError:  # pragma: no cover
    _N = max(1, min(8, os.cpu_count() or 1))
_POOL: ThreadPoolExecutor | None = None


def _pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(_N, thread_name_prefix="wbpc-host")
    return _POOL


def _chunks(n: int):
    step = -(-n // _N)
    return [(i, min(n, i + step)) for i in range(0, n, step)]


def convert(src: np.ndarray, dtype, out: np.ndarray | None = None) -> np.ndarray:
    """`src.astype(dtype)` (C order, unsafe cast) on a few threads, optionally into `out`."""
    src = np.ascontiguousarray(src)
    if out is None:
        if src.size < _MIN or _N == 1:
            return src.astype(dtype)
        out = np.empty(src.shape, dtype)
    s, o = src.reshape(-1), out.reshape(-1)
    if src.size < _MIN or _N == 1:
        np.copyto(o, s, casting="unsafe")
        return out
    list(_pool().map(lambda ab: np.copyto(o[ab[0]:ab[1]], s[ab[0]:ab[1]], casting="unsafe"), _chunks(s.size)))
    return out


# Page-locked staging buffers for the drop-in functions' host <-> device copies, one growing buffer
# per calling thread (the functions are thread-safe like the reference's): a copy through pageable
# memory runs at a fraction of the PCIe rate.  Small transfers skip them.
_TLS = threading.local()
_PIN_MIN = 4 << 20


def staging(nbytes: int) -> torch.Tensor | None:
    """A pinned uint8 tensor of at least `nbytes` for the calling thread (None for small sizes or
    when page-locking fails); valid until the thread's next call."""
    if nbytes < _PIN_MIN:
        return None
    buf = getattr(_TLS, "buf", None)
    if buf is None or buf.numel() < nbytes:
        try:
            buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, pin_memory=True)
        except RuntimeError:
            return None
        _TLS.buf = buf
    return buf


def or_reduce(x: np.ndarray) -> int:
    """Bitwise OR of every element (0 for an empty array)."""
    if x.size == 0:
        return 0
    if x.size < _MIN or _N == 1 or not x.flags.c_contiguous:
        return int(np.bitwise_or.reduce(x, axis=None))
    f = x.reshape(-1)
    return int(np.bitwise_or.reduce(list(_pool().map(lambda ab: np.bitwise_or.reduce(f[ab[0]:ab[1]]), _chunks(f.size)))))


def upload(data, device) -> torch.Tensor:
    """Container bytes -> uint8 device tensor (through the staging buffer when large)."""
    n = len(data)
    pin = staging(n)
    if pin is None:
        return torch.frombuffer(bytearray(data) if n else bytearray(1), dtype=torch.uint8)[:n].to(device)
    pin[:n].numpy()[:] = np.frombuffer(data, dtype=np.uint8)
    return pin[:n].to(device)  # synchronous: the staging buffer is free again on return


def download_bytes(t: torch.Tensor) -> bytes:
    """uint8 device tensor -> bytes (through the staging buffer when large)."""
    n = t.numel()
    pin = staging(n)
    if pin is None:
        return t.cpu().numpy().tobytes()
    pin[:n].copy_(t)
    return pin[:n].numpy().tobytes()

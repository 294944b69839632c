"""Host-side sample conversions for the reference-compatible API, split over a few threads.

The drop-in functions exchange int64 sample arrays with the caller (RasterImage, transforms.py:24-46)
while the device works on 8/16/32-bit samples; for a 4096 x 4096 RGB tile the widening and
narrowing passes cost more than the GPU round trip, and numpy runs them on one core.  numpy
releases the GIL inside these loops, so plain threads scale them.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

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


def convert(src: np.ndarray, dtype) -> np.ndarray:
    """`src.astype(dtype)` (C order, unsafe cast) on a few threads."""
    src = np.ascontiguousarray(src)
    if src.size < _MIN or _N == 1:
        return src.astype(dtype)
    out = np.empty(src.shape, dtype)
    s, o = src.reshape(-1), out.reshape(-1)
    list(_pool().map(lambda ab: np.copyto(o[ab[0]:ab[1]], s[ab[0]:ab[1]], casting="unsafe"), _chunks(s.size)))
    return out


def or_reduce(x: np.ndarray) -> int:
    """Bitwise OR of every element (0 for an empty array)."""
    if x.size == 0:
        return 0
    if x.size < _MIN or _N == 1 or not x.flags.c_contiguous:
        return int(np.bitwise_or.reduce(x, axis=None))
    f = x.reshape(-1)
    return int(np.bitwise_or.reduce(list(_pool().map(lambda ab: np.bitwise_or.reduce(f[ab[0]:ab[1]]), _chunks(f.size)))))

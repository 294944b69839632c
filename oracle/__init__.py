"""CPU oracle for the wbpc encode/decode path — TEST INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/wbpc_oracle.c``, a plain-C restatement of the
reference package (/root/reference/pkg/src/wbpc).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this module;
the product package (``paper_2005_08713_b200``) never does.

Parity of the restatement is pinned by ``tests/test_oracle_golden.py`` against
fixtures generated from the unmodified reference (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_wbpc.so")
_lib = None

# status -> exception class name of wbpc.errors (errors.py:4-61), same numbering as
# include/wbpc_b200.h
STATUS_NAMES = {
    1: "UnsupportedLayoutError",
    2: "ShapeError",
    3: "DomainError",
    4: "LevelRangeError",
    5: "DepthOverflowError",
    6: "StreamIndexError",
    7: "EmptyAlphabetError",
    8: "CodeLengthError",
    9: "MalformedTreeError",
    10: "TruncationError",
    11: "MalformedPayloadError",
    12: "BlockParseError",
    13: "CorruptionError",
    14: "ContainerParseError",
    15: "IndexError",
}


class OracleError(Exception):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "wbpc_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s", "liboracle_wbpc.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        u8p, i64p, i32p, u32p = P(ctypes.c_uint8), P(ctypes.c_int64), P(ctypes.c_int32), P(ctypes.c_uint32)
        L.wbo_last_error.restype = ctypes.c_char_p
        L.wbo_free.argtypes = [ctypes.c_void_p]
        L.wbo_encode_image.argtypes = [i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_size_t)]
        L.wbo_decode_image.argtypes = [u8p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int,
                                       ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_int), P(ctypes.c_int),
                                       P(ctypes.c_int), P(ctypes.c_int)]
        L.wbo_decode_region.argtypes = [u8p, ctypes.c_size_t] + [ctypes.c_int] * 7 + [
            P(ctypes.c_void_p), P(ctypes.c_int), P(ctypes.c_int), P(ctypes.c_int), P(ctypes.c_int)]
        L.wbo_truncate_stream.argtypes = [u8p, ctypes.c_size_t, ctypes.c_int, i32p, ctypes.c_int,
                                          P(ctypes.c_void_p), P(ctypes.c_size_t)]
        L.wbo_dwt2d_forward_packed.argtypes = [i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p]
        L.wbo_dwt2d_inverse_packed.argtypes = [i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p]
        L.wbo_huffman.argtypes = [i64p, i32p, u32p, i32p, i32p, i32p, i32p, u8p, i64p]
        L.wbo_optimize_counter_width.argtypes = [i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.wbo_serialize_block.argtypes = [ctypes.c_int, i64p, ctypes.c_int, ctypes.c_int, u8p, P(ctypes.c_int)]
        L.wbo_encode_block_flat.argtypes = [ctypes.c_int, i64p, ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_size_t)]
        L.wbo_decode_block_flat.argtypes = [u8p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p]
        L.wbo_truncate_block.argtypes = [u8p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         P(ctypes.c_void_p), P(ctypes.c_size_t)]
        L.wbo_decode_tokens.argtypes = [u8p, ctypes.c_int64, ctypes.c_int64, i32p, i32p, i32p, ctypes.c_int,
                                        ctypes.c_int, i64p, ctypes.c_int, u8p, i64p, i64p]
        L.wbo_default_levels.argtypes = [ctypes.c_int, ctypes.c_int]
        L.wbo_slot_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.wbo_slot_count.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _check(rc: int) -> None:
    if rc:
        raise OracleError(rc, lib().wbo_last_error().decode(errors="replace"))


def _take_bytes(p: ctypes.c_void_p, n: ctypes.c_size_t) -> bytes:
    out = ctypes.string_at(p.value, n.value) if n.value else b""
    lib().wbo_free(p)
    return out


def encode_image(samples: np.ndarray, bit_depth: int, levels: int | None = None, use_rct: bool = False,
                 threads: int = 1) -> bytes:
    """encode_image (container.py:167-206); samples (C,H,W) integers."""
    s = np.ascontiguousarray(samples, dtype=np.int64)
    c, h, w = s.shape
    p, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(lib().wbo_encode_image(_ptr(s, ctypes.c_int64), w, h, c, bit_depth, -1 if levels is None else levels,
                                  int(bool(use_rct)), threads, ctypes.byref(p), ctypes.byref(n)))
    return _take_bytes(p, n)


def decode_image(data: bytes, level: int = 0, planes_dropped: int = 0, drop_hp=None, drop_ll: int = 0,
                 threads: int = 1) -> tuple[np.ndarray, int]:
    """decode_image (container.py:309-335) -> ((C,H,W) int64 samples, bit_depth)."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    dh = None
    if drop_hp is not None:
        dh = np.zeros(64, dtype=np.int32)
        dh[: len(drop_hp)] = drop_hp
    p = ctypes.c_void_p()
    ow, oh, oc, obd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib().wbo_decode_image(_ptr(buf, ctypes.c_uint8), buf.size, level, planes_dropped,
                                  None if dh is None else _ptr(dh, ctypes.c_int32), drop_ll, threads,
                                  ctypes.byref(p), ctypes.byref(ow), ctypes.byref(oh), ctypes.byref(oc),
                                  ctypes.byref(obd)))
    n = oc.value * oh.value * ow.value
    arr = np.ctypeslib.as_array(ctypes.cast(p.value, ctypes.POINTER(ctypes.c_int64)), shape=(n,)).copy()
    lib().wbo_free(p)
    return arr.reshape(oc.value, oh.value, ow.value), obd.value


def decode_region(data: bytes, x: int, y: int, width: int, height: int, level: int = 0, planes_dropped: int = 0,
                  threads: int = 1) -> tuple[np.ndarray, int]:
    """decode_region (container.py:338-390) -> ((C,height,width) int64 samples, bit_depth)."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    p = ctypes.c_void_p()
    ow, oh, oc, obd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib().wbo_decode_region(_ptr(buf, ctypes.c_uint8), buf.size, x, y, width, height, level, planes_dropped,
                                   threads, ctypes.byref(p), ctypes.byref(ow), ctypes.byref(oh), ctypes.byref(oc),
                                   ctypes.byref(obd)))
    n = oc.value * oh.value * ow.value
    arr = np.ctypeslib.as_array(ctypes.cast(p.value, ctypes.POINTER(ctypes.c_int64)), shape=(n,)).copy()
    lib().wbo_free(p)
    return arr.reshape(oc.value, oh.value, ow.value), obd.value


def truncate_stream(data: bytes, planes_dropped: int, drop_hp=None, drop_ll: int = 0) -> bytes:
    """truncate_stream (container.py:393-417); drop_hp/drop_ll = per-level extension."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    dh = None
    if drop_hp is not None:
        dh = np.zeros(64, dtype=np.int32)
        dh[: len(drop_hp)] = drop_hp
    p, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(lib().wbo_truncate_stream(_ptr(buf, ctypes.c_uint8), buf.size, planes_dropped,
                                     None if dh is None else _ptr(dh, ctypes.c_int32), drop_ll,
                                     ctypes.byref(p), ctypes.byref(n)))
    return _take_bytes(p, n)


def dwt2d_forward_packed(plane: np.ndarray, levels: int) -> np.ndarray:
    x = np.ascontiguousarray(plane, dtype=np.int64)
    h, w = x.shape
    out = np.empty(h * w, dtype=np.int64)
    _check(lib().wbo_dwt2d_forward_packed(_ptr(x, ctypes.c_int64), w, h, levels, _ptr(out, ctypes.c_int64)))
    return out


def dwt2d_inverse_packed(packed: np.ndarray, w: int, h: int, levels: int) -> np.ndarray:
    x = np.ascontiguousarray(packed, dtype=np.int64)
    out = np.empty(h * w, dtype=np.int64)
    _check(lib().wbo_dwt2d_inverse_packed(_ptr(x, ctypes.c_int64), w, h, levels, _ptr(out, ctypes.c_int64)))
    return out.reshape(h, w)


def huffman(freq) -> dict:
    f = np.zeros(256, dtype=np.int64)
    a = np.asarray(freq, dtype=np.int64)
    f[: a.size] = a
    cl = np.zeros(256, dtype=np.int32)
    cv = np.zeros(256, dtype=np.uint32)
    left = np.zeros(512, dtype=np.int32)
    right = np.zeros(512, dtype=np.int32)
    sym = np.zeros(512, dtype=np.int32)
    nn = ctypes.c_int32()
    tb = np.zeros(1024, dtype=np.uint8)
    nbits = ctypes.c_int64()
    _check(lib().wbo_huffman(_ptr(f, ctypes.c_int64), _ptr(cl, ctypes.c_int32), _ptr(cv, ctypes.c_uint32),
                             _ptr(left, ctypes.c_int32), _ptr(right, ctypes.c_int32), _ptr(sym, ctypes.c_int32),
                             ctypes.byref(nn), _ptr(tb, ctypes.c_uint8), ctypes.byref(nbits)))
    n = nn.value
    bits = np.unpackbits(tb)[: nbits.value]
    return {"code_lengths": cl, "code_values": cv, "left": left[:n], "right": right[:n], "leaf_symbol": sym[:n],
            "tree_bits": bits}


def optimize_counter_width(runs, zr_code_bits: int, max_width: int = 16) -> int:
    r = np.ascontiguousarray(runs, dtype=np.int64)
    w = lib().wbo_optimize_counter_width(_ptr(r, ctypes.c_int64), r.size, zr_code_bits, max_width)
    if w < 0:
        _check(-w)
    return w


def serialize_block(kind: str, grids, depth: int | None = None) -> tuple[np.ndarray, int]:
    g = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.int64) for x in grids]))
    dim = g.shape[-1]
    nsub = g.shape[0]
    d = ctypes.c_int()
    cap = nsub * 64 * dim * dim // 8
    sym = np.zeros(cap, dtype=np.uint8)
    lib().wbo_serialize_block(0 if kind == "ll" else 1, _ptr(g, ctypes.c_int64), dim, -1 if depth is None else depth,
                              _ptr(sym, ctypes.c_uint8), ctypes.byref(d))
    return sym[: nsub * d.value * dim * dim // 8].copy(), d.value


def encode_block(kind: str, grids) -> bytes:
    g = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.int64) for x in grids]))
    p, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(lib().wbo_encode_block_flat(0 if kind == "ll" else 1, _ptr(g, ctypes.c_int64), g.shape[-1],
                                       ctypes.byref(p), ctypes.byref(n)))
    return _take_bytes(p, n)


def decode_block(data: bytes, dim: int, kind: str, planes_to_keep: int | None = None) -> np.ndarray:
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    nsub = 1 if kind == "ll" else 3
    out = np.zeros((3, dim, dim), dtype=np.int64)
    _check(lib().wbo_decode_block_flat(_ptr(buf, ctypes.c_uint8), buf.size, dim, 0 if kind == "ll" else 1,
                                       -1 if planes_to_keep is None else planes_to_keep, _ptr(out, ctypes.c_int64)))
    return out[:nsub].copy()


def truncate_block(data: bytes, dim: int, kind: str, planes_dropped: int) -> bytes:
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    p, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(lib().wbo_truncate_block(_ptr(buf, ctypes.c_uint8), buf.size, dim, 0 if kind == "ll" else 1,
                                    planes_dropped, ctypes.byref(p), ctypes.byref(n)))
    if not p.value:
        return bytes(data)
    return _take_bytes(p, n)


def decode_tokens(payload: np.ndarray, start_bit: int, end_bit: int, left, right, leaf_symbol, zr_symbol: int,
                  counter_width: int, seg_lengths, out_symbols: np.ndarray, out_seg_starts: np.ndarray):
    """_kernels.decode_tokens (_kernels.py:33-89), same arguments and result."""
    pl = np.ascontiguousarray(payload, dtype=np.uint8)
    l_ = np.ascontiguousarray(left, dtype=np.int32)
    r_ = np.ascontiguousarray(right, dtype=np.int32)
    s_ = np.ascontiguousarray(leaf_symbol, dtype=np.int32)
    sl = np.ascontiguousarray(seg_lengths, dtype=np.int64)
    end = ctypes.c_int64()
    st = lib().wbo_decode_tokens(_ptr(pl, ctypes.c_uint8), start_bit, end_bit, _ptr(l_, ctypes.c_int32),
                                 _ptr(r_, ctypes.c_int32), _ptr(s_, ctypes.c_int32), zr_symbol, counter_width,
                                 _ptr(sl, ctypes.c_int64), sl.size, _ptr(out_symbols, ctypes.c_uint8),
                                 _ptr(out_seg_starts, ctypes.c_int64), ctypes.byref(end))
    return st, end.value


def default_levels(w: int, h: int) -> int:
    return lib().wbo_default_levels(w, h)


def slot_count(w: int, h: int, c: int, levels: int) -> int:
    return int(lib().wbo_slot_count(w, h, c, levels))

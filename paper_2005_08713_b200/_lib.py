"""ctypes binding of libwbpc_b200.so (the C ABI declared in include/wbpc_b200.h).

There is no CPU fallback: importing the package works without a GPU, but every codec call
loads this library and fails loudly (DeviceError) when it is missing or no CUDA device exists.
"""

from __future__ import annotations

import ctypes
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwbpc_b200.so")
_lib = None

STATUS_TO_EXC = {
    1: E.UnsupportedLayoutError,
    2: E.ShapeError,
    3: E.DomainError,
    4: E.LevelRangeError,
    5: E.DepthOverflowError,
    6: E.StreamIndexError,
    7: E.EmptyAlphabetError,
    8: E.CodeLengthError,
    9: E.MalformedTreeError,
    10: E.TruncationError,
    11: E.MalformedPayloadError,
    12: E.BlockParseError,
    13: E.CorruptionError,
    14: E.ContainerParseError,
    15: IndexError,
    100: E.DeviceError,
    101: E.DeviceError,
    103: E.DeviceError,
    104: E.UnsupportedByDeviceError,
}
ST_OUT_CAPACITY = 102

# exported symbols (checked by the CPU test-suite against include/wbpc_b200.h)
EXPORTS = (
    "wbpc_abi_version", "wbpc_last_error", "wbpc_parse_header", "wbpc_slot_count", "wbpc_encode_plan_size",
    "wbpc_encode", "wbpc_decode_plan_size", "wbpc_decode", "wbpc_truncate_plan_size", "wbpc_truncate",
    "wbpc_query_status", "wbpc_decode_tokens", "wbpc_decode_batch", "wbpc_decode_batch_plan_size",
    "wbpc_profile_enable", "wbpc_profile_collect", "wbpc_block_plan_size", "wbpc_encode_blocks",
    "wbpc_decode_blocks", "wbpc_truncate_blocks", "wbpc_decode_region", "wbpc_block_summary", "wbpc_plane_offsets", "wbpc_copy_sized",
    "wbpc_encode_coef_bytes", "wbpc_archive_tile_sizes", "wbpc_archive_index", "wbpc_archive_gather",
    "wbpc_archive_batch_offsets",
)


class Header(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in
                ("width", "height", "channels", "bit_depth", "color_transform", "levels", "block_dim")]


class ImageDesc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_uint32), ("height", ctypes.c_uint32), ("channels", ctypes.c_uint32),
                ("bit_depth", ctypes.c_uint32), ("dtype", ctypes.c_int32), ("layout", ctypes.c_int32),
                ("image_stride_bytes", ctypes.c_uint64)]


DTYPE_U8, DTYPE_U16, DTYPE_I16, DTYPE_I32, DTYPE_U8_DISPLAY = 0, 1, 2, 3, 4
LAYOUT_CHW, LAYOUT_HWC = 0, 1


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise E.DeviceError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp, sz, u32, i32, i64, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.wbpc_abi_version.restype = ctypes.c_int
    L.wbpc_last_error.restype = ctypes.c_char_p
    L.wbpc_parse_header.argtypes = [vp, sz, P(Header)]
    L.wbpc_slot_count.argtypes = [P(Header), P(u64)]
    L.wbpc_encode_plan_size.argtypes = [P(ImageDesc), u32, ctypes.c_int, ctypes.c_int, P(sz), P(sz)]
    L.wbpc_encode_coef_bytes.argtypes = [P(ImageDesc), ctypes.c_int, ctypes.c_int, P(ctypes.c_int)]
    L.wbpc_encode.argtypes = [P(ImageDesc), vp, u32, ctypes.c_int, ctypes.c_int, vp, sz, vp, sz, vp, vp]
    L.wbpc_decode_plan_size.argtypes = [P(Header), ctypes.c_int, P(sz)]
    L.wbpc_decode_batch_plan_size.argtypes = [P(Header), u32, P(sz)]
    L.wbpc_decode.argtypes = [P(Header), vp, sz, ctypes.c_int, ctypes.c_int, vp, i32, vp, ctypes.c_int,
                              ctypes.c_int, vp, sz, vp]
    L.wbpc_decode_batch.argtypes = [P(Header), vp, sz, vp, u32, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int,
                                    ctypes.c_int, vp, sz, vp]
    L.wbpc_truncate_plan_size.argtypes = [P(Header), sz, P(sz), P(sz)]
    L.wbpc_truncate.argtypes = [P(Header), vp, sz, ctypes.c_int, vp, i32, vp, sz, vp, sz, vp, vp]
    L.wbpc_query_status.argtypes = [vp, vp, P(i32), P(u64)]
    L.wbpc_decode_tokens.argtypes = [vp, i64, i64, vp, vp, vp, i32, i32, i32, vp, i32, vp, vp, vp, vp]
    L.wbpc_block_plan_size.argtypes = [ctypes.c_int, u32, P(sz), P(sz)]
    L.wbpc_encode_blocks.argtypes = [ctypes.c_int, u32, vp, vp, vp, sz, vp, sz, vp, vp]
    L.wbpc_decode_blocks.argtypes = [ctypes.c_int, u32, vp, sz, vp, ctypes.c_int, vp, vp, sz, vp]
    L.wbpc_truncate_blocks.argtypes = [ctypes.c_int, u32, vp, sz, vp, ctypes.c_int, vp, sz, vp, sz, vp, vp]
    L.wbpc_decode_region.argtypes = [P(Header), vp, sz, i32, i32, i32, i32, ctypes.c_int, ctypes.c_int, vp,
                                     ctypes.c_int, ctypes.c_int, vp, sz, vp]
    L.wbpc_block_summary.argtypes = [P(Header), vp, sz, vp, vp, vp, sz, vp]
    L.wbpc_plane_offsets.argtypes = [ctypes.c_int, vp, sz, vp, vp, vp, vp, sz, vp]
    L.wbpc_copy_sized.argtypes = [vp, vp, vp, vp]
    L.wbpc_archive_tile_sizes.argtypes = [vp, u32, u32, u32, vp, vp]
    L.wbpc_archive_index.argtypes = [vp, u32, u32, u32, u32, u32, vp, vp, vp, vp]
    L.wbpc_archive_gather.argtypes = [vp, u64, vp, u32, u32, vp, vp, vp]
    L.wbpc_archive_batch_offsets.argtypes = [vp, u32, vp, vp]
    L.wbpc_profile_enable.argtypes = [ctypes.c_int]
    L.wbpc_profile_collect.argtypes = [ctypes.c_char_p, sz, P(ctypes.c_double), P(ctypes.c_int), ctypes.c_int,
                                       P(ctypes.c_int)]
    _lib = L
    return L


def profile_enable(on: bool) -> None:
    load().wbpc_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    """{kernel name: (total ms, launches)} since the last collect (synchronises)."""
    L = load()
    names = ctypes.create_string_buffer(4096)
    ms = (ctypes.c_double * 64)()
    cnt = (ctypes.c_int * 64)()
    n = ctypes.c_int()
    L.wbpc_profile_collect(names, 4096, ms, cnt, 64, ctypes.byref(n))
    keys = names.value.decode().split("\n")
    return {keys[i]: (ms[i], cnt[i]) for i in range(n.value)}


def last_error() -> str:
    return load().wbpc_last_error().decode(errors="replace")


def raise_status(code: int, where: str = "", message: str | None = None) -> None:
    if code == 0:
        return
    exc = STATUS_TO_EXC.get(code, E.DeviceError)
    msg = message if message is not None else last_error()
    raise exc(f"{where}: {msg}" if where else msg)


def check(code: int, where: str = "") -> None:
    raise_status(code, where)

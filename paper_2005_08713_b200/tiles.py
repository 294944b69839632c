"""Tile rendering of the reference's tile service, on the device path.

`_render_tile(reader, ...)` mirrors `_render_tile` (pkg/src/wbpc/service.py:52-100) with the same
signature: the tile (x, y) of `size` pixels at resolution `level` is decoded with
`decode_region` (only the blocks under it), clipped to [0, 2^bit_depth - 1] and, above 8 bits,
rescaled to 8 bits -- fused into the inverse transform's output store
(`WBPC_DTYPE_U8_DISPLAY`) -- and wrapped as a binary PGM / PPM body, or as PNG when the Accept
header asks for image/png (png.py:22-46: 8-bit gray / RGB, filter 0 per scanline, zlib level 9,
host-side), with the same status codes, media types and headers (`X-Sample-Scale`, `ETag`).
The reader keeps one device copy of the container, so serving many tiles of one image uploads
it once.  The HTTP layer itself is out of scope.
"""

from __future__ import annotations

import hashlib
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from .container import (
    BLOCK_DIM,
    ContainerReader,
    _check_region,
    _device,
    decode_region_tensor,
)
from .errors import DomainError, UnsupportedByDeviceError
from .transforms import level_dims


@dataclass
class TileResponse:
    """The fields of the service's starlette Response for one tile."""

    status_code: int
    body: bytes
    media_type: str | None = None
    headers: dict = field(default_factory=dict)


def _png_chunk(tag: bytes, payload: bytes) -> bytes:
    return struct.pack(">I", len(payload)) + tag + payload + struct.pack(">I", zlib.crc32(tag + payload) & 0xFFFFFFFF)


def encode_png(pixels: np.ndarray) -> bytes:
    """(h, w) gray or (h, w, 3) RGB uint8 -> PNG bytes (png.py:22-46 format choices)."""
    px = np.asarray(pixels, dtype=np.uint8)
    if px.ndim == 2:
        ctype, (h, w) = 0, px.shape
    elif px.ndim == 3 and px.shape[2] == 3:
        ctype, (h, w) = 2, px.shape[:2]
    else:
        raise DomainError("expected (h, w) gray or (h, w, 3) RGB")
    rows = np.zeros((h, 1 + w * (3 if ctype == 2 else 1)), dtype=np.uint8)  # filter type 0 per scanline
    rows[:, 1:] = px.reshape(h, rows.shape[1] - 1)
    return (b"\x89PNG\r\n\x1a\n" + _png_chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, ctype, 0, 0, 0))
            + _png_chunk(b"IDAT", zlib.compress(rows.tobytes(), 9)) + _png_chunk(b"IEND", b""))


def _device_container(reader: ContainerReader) -> torch.Tensor:
    buf = getattr(reader, "_dev_buf", None)
    if buf is None or buf.device != _device():
        buf = torch.frombuffer(bytearray(reader.data), dtype=torch.uint8).to(_device())
        reader._dev_buf = buf
    return buf


def _render_tile(reader: ContainerReader, level: int, x: int, y: int, planes_dropped: int, size: int,
                 accept: str) -> TileResponse:
    """Render tile (x, y) of `size` pixels at `level` (service.py:52-100), same signature."""
    header = reader.header
    if not 0 <= level <= header.levels:
        return TileResponse(404, b"level out of range")
    lw, lh = level_dims(header.width, header.height, level)
    x0, y0 = x * size, y * size
    if x < 0 or y < 0 or x0 >= lw or y0 >= lh:
        return TileResponse(404, b"tile outside image")
    w = min(size, lw - x0)
    h = min(size, lh - y0)
    _check_region(header, x0, y0, w, h, level, planes_dropped)  # decode_region's argument errors
    if header.block_dim != BLOCK_DIM:
        raise UnsupportedByDeviceError(f"block_dim {header.block_dim} (this build decodes 128 only)")
    pix = decode_region_tensor(_device_container(reader), x0, y0, w, h, level, planes_dropped, header,
                               out_dtype="display8", layout="hwc")
    if header.color_transform == 1 and header.channels < 3:
        raise IndexError("list index out of range")  # _finish_image on an RCT container
    headers = {}
    maxval = (1 << header.bit_depth) - 1
    if header.bit_depth > 8:
        headers["X-Sample-Scale"] = f"255/{maxval}"
    if header.channels not in (1, 3):
        return TileResponse(400, b"no tile rendering for this layout")
    pixels = pix.cpu().numpy()
    if header.channels == 1:
        if "image/png" in accept:
            body, media = encode_png(pixels[:, :, 0]), "image/png"
        else:
            body, media = b"P5\n%d %d\n255\n" % (w, h) + pixels.tobytes(), "image/x-portable-graymap"
    else:
        if "image/png" in accept:
            body, media = encode_png(pixels), "image/png"
        else:
            body, media = b"P6\n%d %d\n255\n" % (w, h) + pixels.tobytes(), "image/x-portable-pixmap"
    headers["ETag"] = '"' + hashlib.sha256(body).hexdigest() + '"'
    return TileResponse(200, body, media, headers)


def render_tile(data, level: int, x: int, y: int, planes_dropped: int = 0, size: int = 256,
                accept: str = "") -> TileResponse:
    """`_render_tile` on container bytes (or an existing ContainerReader)."""
    reader = data if isinstance(data, ContainerReader) else ContainerReader(data)
    return _render_tile(reader, level, x, y, planes_dropped, size, accept)

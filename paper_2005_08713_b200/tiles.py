"""Tile rendering of the reference's tile service, on the device path.

`render_tile` mirrors `_render_tile` (pkg/src/wbpc/service.py:52-100): the tile (x, y) of
`size` pixels at resolution `level` is decoded with `decode_region` (only the blocks under it),
clipped to [0, 2^bit_depth - 1] and, above 8 bits, rescaled to 8 bits -- fused into the
inverse transform's output store (`WBPC_DTYPE_U8_DISPLAY`) -- and wrapped as a binary PGM
(1 channel) or PPM (3 channels) body with the same status codes, media types and headers
(`X-Sample-Scale`, `ETag`).  The HTTP layer itself and PNG encoding are out of scope (network
serving / file I/O); a request that accepts only PNG raises UnsupportedByDeviceError.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import torch

from .container import (
    BLOCK_DIM,
    ContainerHeader,
    _check_index,
    _device,
    decode_region_tensor,
)
from .errors import UnsupportedByDeviceError
from .transforms import level_dims


@dataclass
class TileResponse:
    """The fields of the service's starlette Response for one tile."""

    status_code: int
    body: bytes
    media_type: str | None = None
    headers: dict = field(default_factory=dict)


def render_tile(data: bytes, level: int, x: int, y: int, planes_dropped: int = 0, size: int = 256,
                accept: str = "") -> TileResponse:
    """Render tile (x, y) of `size` pixels at `level` (service.py:52-100)."""
    data = bytes(data)
    header = ContainerHeader.parse(data)
    _check_index(data, header)  # ContainerReader(data) in the service
    if not 0 <= level <= header.levels:
        return TileResponse(404, b"level out of range")
    lw, lh = level_dims(header.width, header.height, level)
    x0, y0 = x * size, y * size
    if x < 0 or y < 0 or x0 >= lw or y0 >= lh:
        return TileResponse(404, b"tile outside image")
    w = min(size, lw - x0)
    h = min(size, lh - y0)
    if header.block_dim != BLOCK_DIM:
        raise UnsupportedByDeviceError(f"block_dim {header.block_dim} (this build decodes 128 only)")
    buf = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(_device())
    pix = decode_region_tensor(buf, x0, y0, w, h, level, planes_dropped, header, out_dtype="display8",
                               layout="hwc")
    if header.color_transform == 1 and header.channels < 3:
        raise IndexError("list index out of range")  # _finish_image on an RCT container
    headers = {}
    maxval = (1 << header.bit_depth) - 1
    if header.bit_depth > 8:
        headers["X-Sample-Scale"] = f"255/{maxval}"
    if header.channels not in (1, 3):
        return TileResponse(400, b"no tile rendering for this layout")
    if "image/png" in accept:
        raise UnsupportedByDeviceError("PNG tile encoding is out of scope (file I/O); request a PNM tile")
    raw = pix.cpu().numpy().tobytes()
    if header.channels == 1:
        body = b"P5\n%d %d\n255\n" % (w, h) + raw
        media = "image/x-portable-graymap"
    else:
        body = b"P6\n%d %d\n255\n" % (w, h) + raw
        media = "image/x-portable-pixmap"
    headers["ETag"] = '"' + hashlib.sha256(body).hexdigest() + '"'
    return TileResponse(200, body, media, headers)

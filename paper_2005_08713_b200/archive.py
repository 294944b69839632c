"""Tile archive for whole-slide images sharded over GPUs.

A whole slide (BASELINE config 4: 65536^2 RGB) is encoded as independent 4096^2 tile
containers -- the reference's own container format per tile (a single 65536^2 image does not
fit its int64 in-memory design).  Tiles are partitioned contiguously over ranks; each rank
encodes its tiles on its GPU; the only exchange is an all-gather of the per-tile container byte
counts (NCCL over NVLink on the GPU box, gloo in the CPU tests), from which every rank derives
the archive offsets and writes its own byte ranges.

Archive layout (little endian):
    magic "WBPA", u8 version 1, u32 tiles_x, u32 tiles_y,
    (u64 offset, u64 length) per tile in row-major tile order,
    tile containers (each a complete WBPC container).
"""

from __future__ import annotations

import struct

import torch

MAGIC = b"WBPA"
_HDR = struct.Struct("<4sBII")
_ENTRY = struct.Struct("<QQ")


def shard_tiles(n_tiles: int, world: int, rank: int) -> list[int]:
    """Contiguous partition of tile indices over ranks (ceil-sized shards)."""
    per = -(-n_tiles // world)
    return list(range(rank * per, min(n_tiles, (rank + 1) * per)))


def header_bytes(n_tiles: int) -> int:
    return _HDR.size + _ENTRY.size * n_tiles


def tile_offsets(sizes_gathered: torch.Tensor, n_tiles: int | None = None, world: int = 1) -> torch.Tensor:
    """Archive offsets of every tile from the all-gathered, per-rank padded size table.

    sizes_gathered: world * ceil(n_tiles/world) entries, rank-major (as all_gather returns);
    padding entries (ranks with fewer tiles) are dropped.  Runs on the tensor's device.
    """
    sizes = sizes_gathered.to(torch.int64)
    if n_tiles is None:
        n_tiles = sizes.numel()
    per = -(-n_tiles // world)
    keep = [r * per + i for r in range(world) for i in range(per) if r * per + i < n_tiles]
    s = sizes[torch.tensor(keep, device=sizes.device)]
    return header_bytes(n_tiles) + torch.cumsum(s, 0) - s


def pack(containers: list[bytes], tiles_x: int, tiles_y: int) -> bytes:
    n = len(containers)
    assert n == tiles_x * tiles_y
    off = header_bytes(n)
    index = bytearray()
    for c in containers:
        index += _ENTRY.pack(off, len(c))
        off += len(c)
    return _HDR.pack(MAGIC, 1, tiles_x, tiles_y) + bytes(index) + b"".join(containers)


def unpack(data: bytes) -> tuple[int, int, list[bytes]]:
    magic, ver, tx, ty = _HDR.unpack_from(data)
    if magic != MAGIC or ver != 1:
        from .errors import ContainerParseError
        raise ContainerParseError("not a WBPA tile archive")
    out = []
    for i in range(tx * ty):
        o, n = _ENTRY.unpack_from(data, _HDR.size + _ENTRY.size * i)
        out.append(data[o:o + n])
    return tx, ty, out

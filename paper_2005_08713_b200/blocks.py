"""Block-level API of the reference (pkg/src/wbpc/blocks.py:84-304, bitplanes.py:48-81) on the GPU.

``encode_block`` / ``decode_block`` / ``truncate_block`` keep the reference signatures and
exception classes; batched device variants (``encode_blocks`` / ``decode_blocks``) code many
128x128 blocks in one launch sequence.  The kernels are the container kernels in raw-block mode
(C ABI: wbpc_encode_blocks / wbpc_decode_blocks / wbpc_truncate_blocks).  Only 128x128 blocks
(the container's BLOCK_DIM, container.py:54) run on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .container import _WS, _device, _raise_device, _status, _stream_ptr
from .errors import DepthOverflowError, DomainError, ShapeError, UnsupportedByDeviceError

KIND_LL = "ll"
KIND_HP3 = "hp3"
MAX_DEPTH = 63
DIM = 128


@dataclass
class CoefficientBlock:
    """One tile of signed wavelet coefficients (bitplanes.py:48-81)."""

    width: int
    height: int
    kind: str
    depth: int
    coeffs: tuple

    def __post_init__(self) -> None:
        if self.kind not in (KIND_LL, KIND_HP3):
            raise DomainError(f"unknown block kind {self.kind!r}")
        expected = 1 if self.kind == KIND_LL else 3
        if len(self.coeffs) != expected:
            raise ShapeError(f"{self.kind} block needs {expected} grids")
        if self.width % 4 or self.height % 2 or self.width < 4 or self.height < 2:
            raise ShapeError("block dims must be positive multiples of (4, 2)")
        if not 1 <= self.depth <= MAX_DEPTH:
            raise DomainError(f"depth must be 1..{MAX_DEPTH}")
        self.coeffs = tuple(np.asarray(g, dtype=np.int64) for g in self.coeffs)
        for g in self.coeffs:
            if g.shape != (self.height, self.width):
                raise ShapeError(f"grid shape {g.shape} != block dims")

    @property
    def subband_count(self) -> int:
        return len(self.coeffs)

    @property
    def plane_slots(self) -> int:
        return self.depth * self.subband_count

    @classmethod
    def build(cls, kind: str, grids, depth: int | None = None) -> "CoefficientBlock":
        grids = tuple(np.asarray(g, dtype=np.int64) for g in grids)
        if depth is None:
            peak = max(int(np.abs(g).max(initial=0)) for g in grids)
            depth = 1 + peak.bit_length()
        h, w = grids[0].shape
        return cls(width=w, height=h, kind=kind, depth=depth, coeffs=grids)


def _kind_id(kind: str) -> int:
    if kind not in (KIND_LL, KIND_HP3):
        raise DomainError(f"unknown block kind {kind!r}")
    return 0 if kind == KIND_LL else 1


def encode_blocks(kind: str, coeffs: torch.Tensor, depths: torch.Tensor | None = None,
                  out: torch.Tensor | None = None):
    """Device batch: coeffs int32 CUDA tensor (n, nsub, 128, 128) -> (packed bytes, offsets[n+1]).

    `out` (uint8 CUDA tensor) may be a caller buffer of any prior content; every byte of the
    packed blocks is written (no pre-zeroing is needed or assumed).
    """
    k = _kind_id(kind)
    n = coeffs.shape[0]
    planar = coeffs.to(torch.int32).transpose(0, 1).contiguous()  # (nsub, n, 128, 128)
    L = _lib.load()
    ws_n, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(L.wbpc_block_plan_size(k, n, ctypes.byref(ws_n), ctypes.byref(cap)))
    ws = _WS.get(ws_n.value)
    if out is None:
        out = torch.empty(cap.value, dtype=torch.uint8, device=coeffs.device)
    offs = torch.empty(n + 1, dtype=torch.int64, device=coeffs.device)
    dptr = depths.to(torch.int32).contiguous().data_ptr() if depths is not None else None
    _lib.check(L.wbpc_encode_blocks(k, n, planar.data_ptr(), dptr, ws.data_ptr(), ws.numel(), out.data_ptr(),
                                    out.numel(), offs.data_ptr(), _stream_ptr()))
    code, aux = _status(ws)
    if code:
        _raise_device(code, aux, "encode_block")
    return out, offs


def encode_block(block: CoefficientBlock) -> bytes:
    """Serialize, drop all-zero planes, entropy code, emit the block bytes (blocks.py:84-120)."""
    if (block.width, block.height) != (DIM, DIM):
        raise UnsupportedByDeviceError(f"block dims {block.width}x{block.height} (this build codes 128x128)")
    peak = max(int(np.abs(g).max(initial=0)) for g in block.coeffs)
    if peak >= (1 << (block.depth - 1)):  # _smr_planes (bitplanes.py:114-118)
        raise DepthOverflowError(f"coefficient magnitude {peak} needs more than {block.depth - 1} bits")
    if peak >= (1 << 31) - 1 or block.depth > 32:
        raise UnsupportedByDeviceError("coefficients beyond the int32 path")
    dev = _device()
    g = torch.from_numpy(np.stack(block.coeffs).astype(np.int32)).to(dev).unsqueeze(0)
    d = torch.tensor([block.depth], dtype=torch.int32, device=dev)
    out, offs = encode_blocks(block.kind, g, d)
    o = offs.cpu().tolist()
    return out[o[0]:o[1]].cpu().numpy().tobytes()


def _pack(datas: list[bytes], dev):
    offs = np.zeros(len(datas) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(d) for d in datas])
    buf = torch.frombuffer(bytearray(b"".join(datas) or b"\0"), dtype=torch.uint8).to(dev)
    return buf, torch.from_numpy(offs).to(dev), int(offs[-1])


def decode_blocks(kind: str, data: torch.Tensor, offsets: torch.Tensor, planes_to_keep: int | None = None):
    """Device batch: packed block bytes + offsets[n+1] -> int32 (n, nsub, 128, 128) coefficients."""
    k = _kind_id(kind)
    n = offsets.numel() - 1
    nsub = 1 if k == 0 else 3
    L = _lib.load()
    ws_n, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(L.wbpc_block_plan_size(k, n, ctypes.byref(ws_n), ctypes.byref(cap)))
    ws = _WS.get(ws_n.value)
    out = torch.empty((nsub, n, DIM, DIM), dtype=torch.int32, device=data.device)
    keep = -1 if planes_to_keep is None else max(int(planes_to_keep), 0)
    _lib.check(L.wbpc_decode_blocks(k, n, data.data_ptr(), data.numel(), offsets.data_ptr(), keep, out.data_ptr(),
                                    ws.data_ptr(), ws.numel(), _stream_ptr()))
    code, aux = _status(ws)
    if code:
        _raise_device(code, aux, "decode_block")
    return out.transpose(0, 1)


def decode_block(data: bytes, width: int, height: int, kind: str, planes_to_keep: int | None = None) -> CoefficientBlock:
    """Rebuild the coefficient block keeping plane indices < planes_to_keep (blocks.py:195-250)."""
    _kind_id(kind)
    if (width, height) != (DIM, DIM):
        raise UnsupportedByDeviceError(f"block dims {width}x{height} (this build decodes 128x128)")
    dev = _device()
    buf, offs, _ = _pack([bytes(data)], dev)
    g = decode_blocks(kind, buf, offs, planes_to_keep)[0].cpu().numpy().astype(np.int64)
    depth = bytes(data)[0] >> 2  # 6-bit depth field (blocks.py:157); validated by the device parse
    return CoefficientBlock(width=width, height=height, kind=kind, depth=depth, coeffs=tuple(g))


def plane_offsets(data: bytes, width: int, height: int, kind: str) -> list[tuple[tuple[int, int], int]]:
    """((subband, plane), payload bit offset) for every stored plane (blocks.py:253-261)."""
    k = _kind_id(kind)
    if (width, height) != (DIM, DIM):
        raise UnsupportedByDeviceError(f"block dims {width}x{height} (this build parses 128x128)")
    dev = _device()
    buf, _, total = _pack([bytes(data)], dev)
    L = _lib.load()
    ws_n, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(L.wbpc_block_plan_size(k, 1, ctypes.byref(ws_n), ctypes.byref(cap)))
    ws = _WS.get(ws_n.value)
    slots = torch.empty(96, dtype=torch.int32, device=dev)
    offs = torch.empty(96, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(L.wbpc_plane_offsets(k, buf.data_ptr(), total, slots.data_ptr(), offs.data_ptr(), cnt.data_ptr(),
                                    ws.data_ptr(), ws.numel(), _stream_ptr()))
    code, aux = _status(ws)
    if code:
        _raise_device(code, aux, "plane_offsets")
    n = int(cnt.item())
    nsub = 1 if k == 0 else 3
    sl = slots[:n].cpu().tolist()
    of = (offs[:n].cpu().to(torch.int64) & 0xFFFFFFFF).tolist()
    return [((q % nsub, q // nsub), int(o)) for q, o in zip(sl, of)]


def truncate_block(data: bytes, width: int, height: int, kind: str, planes_dropped: int) -> bytes:
    """Cut the payload at the first dropped plane without re-encoding (blocks.py:264-304)."""
    k = _kind_id(kind)
    if planes_dropped < 0:
        raise DomainError("planes_dropped must be >= 0")
    if planes_dropped == 0:
        return bytes(data)
    if (width, height) != (DIM, DIM):
        raise UnsupportedByDeviceError(f"block dims {width}x{height} (this build handles 128x128)")
    dev = _device()
    buf, offs, total = _pack([bytes(data)], dev)
    L = _lib.load()
    ws_n, cap = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(L.wbpc_block_plan_size(k, 1, ctypes.byref(ws_n), ctypes.byref(cap)))
    ws = _WS.get(ws_n.value)
    out = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    oo = torch.empty(2, dtype=torch.int64, device=dev)
    _lib.check(L.wbpc_truncate_blocks(k, 1, buf.data_ptr(), total, offs.data_ptr(), planes_dropped, ws.data_ptr(),
                                      ws.numel(), out.data_ptr(), out.numel(), oo.data_ptr(), _stream_ptr()))
    code, aux = _status(ws)
    if code:
        _raise_device(code, aux, "truncate_block")
    o = oo.cpu().tolist()
    return out[o[0]:o[1]].cpu().numpy().tobytes()

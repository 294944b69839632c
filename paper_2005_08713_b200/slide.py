"""Whole-slide codec: tile-sharded encode/decode with a device-assembled tile archive.

BASELINE configs[3] is a 65536^2 RGB slide encoded as 256 independent 4096^2 tile containers
(each byte-identical to the reference's `encode_image(tile, levels=6, use_rct=True)`,
container.py:167-206; the reference's int64 in-memory design cannot hold the slide as one image).
`SlideCodec` is one rank's share of that job:

* the tiles are partitioned contiguously over ranks (`archive.shard_tiles`);
* each rank encodes its tiles in batches on concurrent streams (`wbpc_encode`), every batch into
  its own region of a device store, offsets staying on the device;
* the per-tile container byte counts are all-gathered (NCCL over NVLink when world > 1 -- the
  path's only collective), `wbpc_archive_index` scans them into the archive header/index and this
  rank's offsets, and `wbpc_archive_gather` moves the rank's containers to their archive offsets;
* decode reads the tiles back from the archive (`wbpc_decode_batch`).

No host round trip happens on the device path.  The host path (`roundtrip_host`) is the same
job from pinned host pixels: H2D + encode per batch, the size exchange, then per batch the D2H of
its containers to their offsets in a host archive (shared by all ranks on a box), the H2D of those
host bytes, decode, and the D2H of the decoded pixels.
"""

from __future__ import annotations

import ctypes
import mmap
import os

import numpy as np
import torch

from . import _lib, archive
from .archive import header_bytes
from .container import COLOR_NONE, COLOR_RCT, ContainerHeader, _DT, _device, _raise_device, _stream_ptr
from .errors import ContainerParseError, DomainError


def _ptr(t: torch.Tensor, elem_offset: int = 0) -> int:
    return t.data_ptr() + elem_offset * t.element_size()


class SlideCodec:
    """One rank's tile shard of a whole-slide encode + archive + decode."""

    def __init__(self, tiles_x: int, tiles_y: int, tile_w: int, tile_h: int, channels: int = 3, bit_depth: int = 8,
                 levels: int = 6, use_rct: bool = True, dtype: torch.dtype = torch.uint8, layout: str = "hwc",
                 world: int = 1, rank: int = 0, group=None, batch: int = 4, streams: int = 4):
        self.dev = _device()
        self.tx, self.ty, self.W, self.H, self.C = tiles_x, tiles_y, tile_w, tile_h, channels
        self.bd, self.L, self.rct = bit_depth, levels, bool(use_rct)
        self.dtype, self.layout = dtype, layout
        self.world, self.rank, self.group = world, rank, group
        self.n_tiles = tiles_x * tiles_y
        self.per = -(-self.n_tiles // world)
        self.first = min(self.n_tiles, rank * self.per)
        self.n_local = max(0, min(self.n_tiles, self.first + self.per) - self.first)
        self.B = max(1, min(batch, self.n_local or 1))
        self.nb = -(-self.n_local // self.B)
        self.S = max(1, min(streams, self.nb))
        elem = torch.empty(0, dtype=dtype).element_size()
        self.tile_bytes = tile_w * tile_h * channels * elem
        lay = _lib.LAYOUT_HWC if layout == "hwc" else _lib.LAYOUT_CHW
        self._lay, self._odt = lay, _DT[dtype]
        self.desc = _lib.ImageDesc(tile_w, tile_h, channels, bit_depth, _DT[dtype], lay, self.tile_bytes)
        self.header = ContainerHeader(tile_w, tile_h, channels, bit_depth, COLOR_RCT if use_rct else COLOR_NONE,
                                      levels)
        self._hc = self.header.to_c()
        L = _lib.load()
        ws_n, cap = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(L.wbpc_encode_plan_size(ctypes.byref(self.desc), self.B, levels, int(self.rct), ctypes.byref(ws_n),
                                           ctypes.byref(cap)))
        self.enc_ws_bytes = ws_n.value
        self.region = (cap.value + 255) // 256 * 256  # store bytes per batch (worst-case container sizes)
        _lib.check(L.wbpc_decode_batch_plan_size(ctypes.byref(self._hc), self.B, ctypes.byref(ws_n)))
        self.dec_ws_bytes = ws_n.value
        cb = ctypes.c_int()
        _lib.check(L.wbpc_encode_coef_bytes(ctypes.byref(self.desc), levels, int(self.rct), ctypes.byref(cb)))
        self.coef_bytes = cb.value
        dev = self.dev
        self.enc_ws = [torch.empty(self.enc_ws_bytes, dtype=torch.uint8, device=dev) for _ in range(self.S)]
        self.dec_ws = [torch.empty(self.dec_ws_bytes, dtype=torch.uint8, device=dev) for _ in range(self.S)]
        self.streams = [torch.cuda.Stream() for _ in range(self.S)]
        self.store = torch.empty(max(1, self.nb) * self.region + 64, dtype=torch.uint8, device=dev)
        self.enc_off = torch.zeros((max(1, self.nb), self.B + 1), dtype=torch.int64, device=dev)
        self.sizes_local = torch.zeros(self.per, dtype=torch.int64, device=dev)
        self.sizes_all = torch.zeros(self.world * self.per, dtype=torch.int64, device=dev)
        self.index = torch.empty(header_bytes(self.n_tiles), dtype=torch.uint8, device=dev)  # archive header+index
        self.local_off = torch.zeros(self.n_local + 1, dtype=torch.int64, device=dev)
        self.base_total = torch.zeros(2, dtype=torch.int64, device=dev)
        # per-batch device status words (encode, decode), captured in stream order after each call
        self.stat = torch.empty((max(1, self.nb), 2, 4), dtype=torch.int64, device=dev)
        self.archive_dev = None  # this rank's archive range on the device (sized after the first encode)
        self._dev_in = None
        self._dev_out = None

    # ----------------------------------------------------------------------------- helpers
    def batch_size(self, k: int) -> int:
        return min(self.B, self.n_local - k * self.B)

    def _fork(self):
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        return cur

    def _join(self, cur):
        for s in self.streams:
            cur.wait_stream(s)

    def _encode_batch(self, k: int, src_ptr: int, s: int) -> None:
        L = _lib.load()
        _lib.check(L.wbpc_encode(ctypes.byref(self.desc), src_ptr, self.batch_size(k), self.L, int(self.rct),
                                 self.enc_ws[s].data_ptr(), self.enc_ws_bytes, _ptr(self.store, k * self.region),
                                 self.region, _ptr(self.enc_off[k]), _stream_ptr()))
        self.stat[k, 0].copy_(self.enc_ws[s][:32].view(torch.int64))

    def _decode_batch(self, k: int, data_ptr: int, data_len: int, off_ptr: int, out_ptr: int, s: int) -> None:
        L = _lib.load()
        _lib.check(L.wbpc_decode_batch(ctypes.byref(self._hc), data_ptr, data_len, off_ptr, self.batch_size(k), 0, 0,
                                       out_ptr, self._odt, self._lay, self.dec_ws[s].data_ptr(), self.dec_ws_bytes,
                                       _stream_ptr()))
        self.stat[k, 1].copy_(self.dec_ws[s][:32].view(torch.int64))

    # ----------------------------------------------------------------------------- device path
    def encode(self, x: torch.Tensor) -> None:
        """Encode this rank's tiles x[(n_local, ...) device tensor] into the store (stream ordered)."""
        if self.n_local and tuple(x.shape[0:1]) != (self.n_local,):
            raise DomainError(f"expected {self.n_local} tiles, got {tuple(x.shape)}")
        cur = self._fork()
        for k in range(self.nb):
            s = k % self.S
            with torch.cuda.stream(self.streams[s]):
                self._encode_batch(k, _ptr(x, k * self.B * (self.tile_bytes // x.element_size())), s)
        self._join(cur)
        _lib.check(_lib.load().wbpc_archive_tile_sizes(self.enc_off.data_ptr(), self.B, self.n_local, self.per,
                                                       self.sizes_local.data_ptr(), _stream_ptr()))

    def exchange(self) -> None:
        """All-gather the per-tile sizes and compute the archive index / this rank's offsets."""
        if self.world > 1:
            import torch.distributed as dist
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(self.sizes_all, self.sizes_local, group=self.group)
            else:  # gloo (CPU tests of the multi-rank path): exchange through host tensors
                got = torch.empty(self.world * self.per, dtype=torch.int64)
                dist.all_gather_into_tensor(got, self.sizes_local.cpu(), group=self.group)
                self.sizes_all.copy_(got)
        else:
            self.sizes_all.copy_(self.sizes_local)
        _lib.check(_lib.load().wbpc_archive_index(self.sizes_all.data_ptr(), self.n_tiles, self.tx, self.ty,
                                                  self.first, self.n_local, self.index.data_ptr(),
                                                  self.local_off.data_ptr(), self.base_total.data_ptr(),
                                                  _stream_ptr()))

    def ensure_archive(self, nbytes: int | None = None) -> None:
        """Allocate the device archive range (synchronises once to read the shard's byte count)."""
        if nbytes is None:
            nbytes = int(self.local_off[-1].item())
        if self.archive_dev is None or self.archive_dev.numel() < nbytes + 64:
            self.archive_dev = torch.empty(nbytes + nbytes // 16 + 4096, dtype=torch.uint8, device=self.dev)

    def assemble(self) -> None:
        """Move this rank's containers to their archive offsets (device archive range)."""
        if self.archive_dev is None:
            raise DomainError("call ensure_archive() after the first encode/exchange")
        _lib.check(_lib.load().wbpc_archive_gather(self.store.data_ptr(), self.region, self.enc_off.data_ptr(),
                                                   self.B, self.n_local, self.archive_dev.data_ptr(),
                                                   self.local_off.data_ptr(), _stream_ptr()))

    def decode(self, out: torch.Tensor) -> torch.Tensor:
        """Decode this rank's tiles from the device archive into out (n_local, ...)."""
        cur = self._fork()
        per_tile = self.tile_bytes // out.element_size()
        for k in range(self.nb):
            s = k % self.S
            with torch.cuda.stream(self.streams[s]):
                self._decode_batch(k, self.archive_dev.data_ptr(), self.archive_dev.numel(),
                                   _ptr(self.local_off, k * self.B), _ptr(out, k * self.B * per_tile), s)
        self._join(cur)
        return out

    def roundtrip_device(self, x: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """The slide round trip with encode and decode interleaved (stream ordered, no host sync).

        Per batch, on its stream: encode into its store region; its tiles' rank-local archive
        offsets from the previous batch's end (`wbpc_archive_batch_offsets`, ordered across
        streams by one event per batch); move its containers into the rank's archive range;
        decode them from there.  Batch k's decode overlaps batch k+1..k+S's encodes, so the
        ALU-bound coder kernels of one batch share the SMs with the latency- and bandwidth-bound
        ones of the others.  Only the archive header/index needs every rank's sizes: the size
        all-gather and `wbpc_archive_index` run once at the end.  The device archive is sized for
        the worst case on the first call.
        """
        L = _lib.load()
        if self.archive_dev is None or self.archive_dev.numel() < self.nb * self.region:
            self.archive_dev = torch.empty(max(1, self.nb) * self.region + 64, dtype=torch.uint8, device=self.dev)
        per_tile = self.tile_bytes // x.element_size()
        self.local_off[:1].zero_()  # batch 0's base (before the fork: every stream waits for it)
        cur = self._fork()
        prev = None
        for k in range(self.nb):
            s = k % self.S
            st = self.streams[s]
            b = self.batch_size(k)
            with torch.cuda.stream(st):
                self._encode_batch(k, _ptr(x, k * self.B * per_tile), s)
                if prev is not None:
                    st.wait_event(prev)
                _lib.check(L.wbpc_archive_batch_offsets(_ptr(self.enc_off[k]), b, _ptr(self.local_off, k * self.B),
                                                        _stream_ptr()))
                prev = torch.cuda.Event()
                prev.record(st)
                _lib.check(L.wbpc_archive_gather(_ptr(self.store, k * self.region), self.region,
                                                 _ptr(self.enc_off[k]), self.B, b, self.archive_dev.data_ptr(),
                                                 _ptr(self.local_off, k * self.B), _stream_ptr()))
                self._decode_batch(k, self.archive_dev.data_ptr(), self.archive_dev.numel(),
                                   _ptr(self.local_off, k * self.B), _ptr(out, k * self.B * per_tile), s)
        self._join(cur)
        _lib.check(L.wbpc_archive_tile_sizes(self.enc_off.data_ptr(), self.B, self.n_local, self.per,
                                             self.sizes_local.data_ptr(), _stream_ptr()))
        self.exchange()
        return out

    def roundtrip_device_phased(self, x: torch.Tensor, out: torch.Tensor, events=None) -> torch.Tensor:
        """encode -> size exchange -> archive assembly -> decode, as separate phases.

        events (optional): 3 CUDA events recorded at start, after assembly, at the end.
        """
        if events:
            events[0].record()
        self.encode(x)
        self.exchange()
        if self.archive_dev is None:
            self.ensure_archive()  # first call only: one sync to size the device archive
        self.assemble()
        if events:
            events[1].record()
        self.decode(out)
        if events:
            events[2].record()
        return out

    def check(self) -> None:
        """Synchronise and raise the first device-reported error of the last encode/decode."""
        torch.cuda.synchronize()
        st = self.stat[: self.nb].cpu().numpy().view(np.uint64)
        for k in range(self.nb):
            for j, what in ((0, "encode"), (1, "decode")):
                key, _, aux, _ = (int(v) for v in st[k, j])
                if key != 0xFFFFFFFFFFFFFFFF:
                    code = key & 0xFF
                    _raise_device(code, aux if code == _lib.ST_OUT_CAPACITY else (key >> 8) & 0xFFFFFFFFFFF,
                                  f"slide {what} (batch {k})")

    def tile_sizes(self) -> list[int]:
        return self.sizes_all[: self.n_tiles].cpu().tolist()

    def archive_header(self) -> bytes:
        return self.index.cpu().numpy().tobytes()

    def local_archive_bytes(self) -> bytes:
        """This rank's contiguous archive range (its tiles' containers) from the device archive."""
        n = int(self.local_off[-1].item())
        return self.archive_dev[:n].cpu().numpy().tobytes()

    # ----------------------------------------------------------------------------- archive files
    def save_archive(self, path: str) -> int:
        """Write the encoded slide to one archive file (after encode / exchange / assemble).

        Every rank writes its own contiguous byte range at its archive offset (`os.pwrite`, no
        rank sees another's bytes); rank 0 also writes the header and index and sizes the file.
        With several ranks, rank 0 must have created the file before the others write (call
        after a barrier, as `bench.py` does for the shared host archive).  Returns the archive size.
        """
        base, total = (int(v) for v in self.base_total.cpu().tolist())
        mine = self.local_archive_bytes()
        if self.rank == 0:
            with open(path, "wb") as f:
                f.truncate(total)
        fd = os.open(path, os.O_WRONLY)
        try:
            if self.rank == 0:
                os.pwrite(fd, self.archive_header(), 0)
            os.pwrite(fd, mine, base)
        finally:
            os.close(fd)
        return total

    def load_archive(self, path: str) -> None:
        """Read this rank's tiles of an archive file into the device archive (then `decode`)."""
        with open(path, "rb") as f:
            head = f.read(archive.header_bytes(self.n_tiles))
            magic, ver, tx, ty = archive._HDR.unpack_from(head)
            if magic != archive.MAGIC or ver != 1 or (tx, ty) != (self.tx, self.ty):
                raise ContainerParseError("not a WBPA tile archive of this slide's tile grid")
            ent = np.frombuffer(head, dtype="<u8", offset=archive._HDR.size).reshape(self.n_tiles, 2)
            offs, lens = ent[:, 0].astype(np.int64), ent[:, 1].astype(np.int64)
            if np.any(offs[1:] != offs[:-1] + lens[:-1]) or offs[0] != len(head):
                raise ContainerParseError("tile index is not contiguous")
            lo = self.first
            hi = self.first + self.n_local
            base, end = int(offs[lo]), int(offs[hi - 1] + lens[hi - 1])
            f.seek(base)
            body = f.read(end - base)
        if len(body) != end - base:
            raise ContainerParseError("archive file is shorter than its index")
        self.ensure_archive(len(body))
        self.archive_dev[: len(body)].copy_(torch.frombuffer(bytearray(body), dtype=torch.uint8))
        rel = np.concatenate([offs[lo:hi] - base, [end - base]]).astype(np.int64)
        self.local_off.copy_(torch.from_numpy(rel))

    # ----------------------------------------------------------------------------- host path
    def roundtrip_host(self, x_host: torch.Tensor, out_host: torch.Tensor, archive_host: torch.Tensor) -> int:
        """Pinned host tiles -> host archive (this rank's range + rank 0's header) -> pinned host tiles.

        Returns the archive's total byte count.  archive_host must be page-locked (pinned or
        cudaHostRegister-ed) and hold the whole archive (ranks share it on one box).
        """
        if self._dev_in is None:
            shape = (self.B,) + tuple(x_host.shape[1:])
            self._dev_in = [torch.empty(shape, dtype=x_host.dtype, device=self.dev) for _ in range(self.S)]
            self._dev_out = [torch.empty(shape, dtype=out_host.dtype, device=self.dev) for _ in range(self.S)]
            self._off_host = torch.zeros((max(1, self.nb), self.B + 1), dtype=torch.int64, pin_memory=True)
        if self.world == 1:
            return self._roundtrip_host_pipelined(x_host, out_host, archive_host)
        cur = self._fork()
        for k in range(self.nb):  # H2D pixels + encode per batch
            s = k % self.S
            b = self.batch_size(k)
            with torch.cuda.stream(self.streams[s]):
                self._dev_in[s][:b].copy_(x_host[k * self.B:k * self.B + b], non_blocking=True)
                self._encode_batch(k, self._dev_in[s].data_ptr(), s)
        self._join(cur)
        _lib.check(_lib.load().wbpc_archive_tile_sizes(self.enc_off.data_ptr(), self.B, self.n_local, self.per,
                                                       self.sizes_local.data_ptr(), _stream_ptr()))
        self.exchange()
        # the one host synchronisation: byte counts for the copies
        lo = self.local_off.cpu().tolist()
        base, total = self.base_total.cpu().tolist()
        if archive_host.numel() < total:
            raise DomainError(f"host archive holds {archive_host.numel()} bytes, the slide needs {total}")
        if self.rank == 0:
            archive_host[: self.index.numel()].copy_(self.index, non_blocking=True)
        cur = self._fork()
        for k in range(self.nb):  # D2H containers -> archive, H2D archive bytes, decode, D2H pixels
            s = k % self.S
            b = self.batch_size(k)
            a0, a1 = base + lo[k * self.B], base + lo[k * self.B + b]
            n = a1 - a0
            reg = self.store[k * self.region:k * self.region + n]
            with torch.cuda.stream(self.streams[s]):
                archive_host[a0:a1].copy_(reg, non_blocking=True)
                reg.copy_(archive_host[a0:a1], non_blocking=True)
                self._decode_batch(k, _ptr(self.store, k * self.region), n, _ptr(self.enc_off[k]),
                                   self._dev_out[s].data_ptr(), s)
                out_host[k * self.B:k * self.B + b].copy_(self._dev_out[s][:b], non_blocking=True)
        self._join(cur)
        return int(total)

    def _roundtrip_host_pipelined(self, x_host, out_host, archive_host) -> int:
        """Single rank: the archive offset of every batch is the header size plus the sizes of the
        batches before it, so each batch's containers go to the host archive as soon as it is
        encoded.  Per batch, on its stream: H2D pixels, encode, D2H offsets (`front`); then, after
        reading that batch's byte count (the only host wait), D2H containers into the archive,
        H2D of those host bytes, decode, D2H pixels (`tail`).  Fronts run `S` batches ahead of the
        tails, so pixel uploads, container round trips and pixel downloads keep both PCIe
        directions busy at once."""
        evs = [None] * self.nb
        hdr = self.index.numel()

        def front(k):
            s = k % self.S
            b = self.batch_size(k)
            with torch.cuda.stream(self.streams[s]):
                self._dev_in[s][:b].copy_(x_host[k * self.B:k * self.B + b], non_blocking=True)
                self._encode_batch(k, self._dev_in[s].data_ptr(), s)
                self._off_host[k].copy_(self.enc_off[k], non_blocking=True)
                evs[k] = torch.cuda.Event()
                evs[k].record(self.streams[s])

        cur = self._fork()
        ahead = min(self.S, self.nb)
        for k in range(ahead):
            front(k)
        pos = hdr
        for k in range(self.nb):
            s = k % self.S
            b = self.batch_size(k)
            evs[k].synchronize()
            n = int(self._off_host[k, b])
            if pos + n > archive_host.numel():
                raise DomainError(f"host archive holds {archive_host.numel()} bytes, the slide needs more")
            reg = self.store[k * self.region:k * self.region + n]
            with torch.cuda.stream(self.streams[s]):
                archive_host[pos:pos + n].copy_(reg, non_blocking=True)
                reg.copy_(archive_host[pos:pos + n], non_blocking=True)
                self._decode_batch(k, _ptr(self.store, k * self.region), n, _ptr(self.enc_off[k]),
                                   self._dev_out[s].data_ptr(), s)
                out_host[k * self.B:k * self.B + b].copy_(self._dev_out[s][:b], non_blocking=True)
            pos += n
            if k + ahead < self.nb:
                front(k + ahead)
        self._join(cur)
        # archive header + index from the per-tile sizes (device scan), to the host
        _lib.check(_lib.load().wbpc_archive_tile_sizes(self.enc_off.data_ptr(), self.B, self.n_local, self.per,
                                                       self.sizes_local.data_ptr(), _stream_ptr()))
        self.exchange()
        archive_host[:hdr].copy_(self.index, non_blocking=True)
        return int(pos)


    def stream_host(self, x_hosts: list, out_hosts: list, archives: list) -> list:
        """Single rank: several slides back to back through the pipelined host path.

        Slide t's pinned tiles x_hosts[t] -> archives[t] (header, index, containers) ->
        out_hosts[t].  Batches keep `S` fronts in flight across slide boundaries, so the next
        slide's uploads and encodes overlap the current slide's last round trips (no pipeline
        drain per slide).  Each batch's per-tile sizes are computed right after its encode;
        slide t's archive index is formed on the stream of slide t+1's first batch, after slide
        t's last encodes and before slide t+1 reuses the size table.  The same tensor may be passed
        for several slides (each slide's bytes are complete before the next overwrites them only in
        stream order: a caller that reads them must sync per slide).  Returns the archive sizes.
        """
        if self.world != 1:
            raise DomainError("stream_host is the single-rank path; use roundtrip_host per slide")
        if self._dev_in is None:
            shape = (self.B,) + tuple(x_hosts[0].shape[1:])
            self._dev_in = [torch.empty(shape, dtype=x_hosts[0].dtype, device=self.dev) for _ in range(self.S)]
            self._dev_out = [torch.empty(shape, dtype=out_hosts[0].dtype, device=self.dev) for _ in range(self.S)]
            self._off_host = torch.zeros((max(1, self.nb), self.B + 1), dtype=torch.int64, pin_memory=True)
        L = _lib.load()
        T = len(x_hosts)
        seq = [(t, k) for t in range(T) for k in range(self.nb)]
        evs = {}
        # every batch's device status words (encode, decode), copied in stream order before the
        # next slide reuses the workspaces; checked once at the end
        stat = torch.empty((T, max(1, self.nb), 2, 4), dtype=torch.int64, pin_memory=True)
        last_ev = [dict() for _ in range(T)]  # slide -> stream -> event of its last front there
        hdr = self.index.numel()

        def index_of(t):  # archive index of slide t from the per-tile sizes of its batches
            _lib.check(L.wbpc_archive_index(self.sizes_local.data_ptr(), self.n_tiles, self.tx, self.ty, 0,
                                            self.n_local, self.index.data_ptr(), self.local_off.data_ptr(),
                                            self.base_total.data_ptr(), _stream_ptr()))
            archives[t][:hdr].copy_(self.index, non_blocking=True)

        def front(t, k):
            s = k % self.S
            b = self.batch_size(k)
            st = self.streams[s]
            with torch.cuda.stream(st):
                if k == 0 and t > 0:
                    for e in last_ev[t - 1].values():
                        st.wait_event(e)
                    index_of(t - 1)
                self._dev_in[s][:b].copy_(x_hosts[t][k * self.B:k * self.B + b], non_blocking=True)
                self._encode_batch(k, self._dev_in[s].data_ptr(), s)
                stat[t, k, 0].copy_(self.enc_ws[s][:32].view(torch.int64), non_blocking=True)
                _lib.check(L.wbpc_archive_tile_sizes(_ptr(self.enc_off[k]), self.B, b, b,
                                                     _ptr(self.sizes_local, k * self.B), _stream_ptr()))
                self._off_host[k].copy_(self.enc_off[k], non_blocking=True)
                e = torch.cuda.Event()
                e.record(st)
                evs[(t, k)] = e
                last_ev[t][s] = e

        cur = self._fork()
        ahead = min(self.S, self.nb)
        for i in range(min(ahead, len(seq))):
            front(*seq[i])
        totals = [0] * T
        pos = hdr
        for i, (t, k) in enumerate(seq):
            if k == 0:
                pos = hdr
            s = k % self.S
            b = self.batch_size(k)
            evs.pop((t, k)).synchronize()
            n = int(self._off_host[k, b])
            arch = archives[t]
            if pos + n > arch.numel():
                raise DomainError(f"host archive holds {arch.numel()} bytes, the slide needs more")
            reg = self.store[k * self.region:k * self.region + n]
            with torch.cuda.stream(self.streams[s]):
                arch[pos:pos + n].copy_(reg, non_blocking=True)
                reg.copy_(arch[pos:pos + n], non_blocking=True)
                self._decode_batch(k, _ptr(self.store, k * self.region), n, _ptr(self.enc_off[k]),
                                   self._dev_out[s].data_ptr(), s)
                stat[t, k, 1].copy_(self.dec_ws[s][:32].view(torch.int64), non_blocking=True)
                out_hosts[t][k * self.B:k * self.B + b].copy_(self._dev_out[s][:b], non_blocking=True)
            pos += n
            totals[t] = pos
            if i + ahead < len(seq):
                front(*seq[i + ahead])
        self._join(cur)
        index_of(T - 1)
        torch.cuda.current_stream().synchronize()
        st = stat.numpy().view(np.uint64)
        for t in range(T):
            for k in range(self.nb):
                for j, what in ((0, "encode"), (1, "decode")):
                    key, _, aux, _ = (int(v) for v in st[t, k, j])
                    if key != 0xFFFFFFFFFFFFFFFF:
                        code = key & 0xFF
                        _raise_device(code, aux if code == _lib.ST_OUT_CAPACITY else (key >> 8) & 0xFFFFFFFFFFF,
                                      f"slide {t} {what} (batch {k})")
        return totals


def shared_host_buffer(path: str, nbytes: int, create: bool) -> tuple[torch.Tensor, object]:
    """A uint8 host tensor backed by a shared-memory file (/dev/shm) and page-locked for DMA.

    Every rank on a box maps the same file, so the ranks' D2H copies land in one archive.
    Returns (tensor, keepalive); call `release_host_buffer(keepalive)` when done.
    """
    if create:
        with open(path, "wb") as f:
            f.truncate(nbytes)
    fd = os.open(path, os.O_RDWR)
    mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
    os.close(fd)
    t = torch.frombuffer(mm, dtype=torch.uint8, count=nbytes)
    rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    if int(rc) != 0:
        raise DomainError(f"cudaHostRegister failed ({rc})")
    return t, (mm, t.data_ptr())


def release_host_buffer(keep) -> None:
    """Unpin a buffer from shared_host_buffer (the mapping goes with its last reference)."""
    torch.cuda.cudart().cudaHostUnregister(keep[1])

"""Encoder output-buffer hygiene and concurrency of the functional API (CUDA path vs the oracle).

* The emit kernel writes into caller buffers of any prior content: blocks whose slots exceed one
  shared-memory window (the multi-window branch) and ordinary containers are encoded into
  buffers pre-filled with 0xFF at unaligned offsets and compared with the oracle byte for byte.
* Functional calls from two threads on two streams round-trip concurrently, bit-exact (per-call
  workspaces; the reference API is pure and thread-safe).
"""

import threading

import numpy as np
import pytest
import torch

import adversarial as A
import inputs

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2005_08713_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_08713_b200 import _lib
    _lib.load()


def test_large_slot_blocks_into_dirty_buffer(oracle_lib):
    cases = [(0, 7, False), (1, 3, False), (2, 12, True), (3, 1, False), (4, 19, True), (5, 9, False)]
    grids, refs = [], []
    for seed, rp, neg in cases:
        g, d, rs = A.large_slot_block(seed, random_plane=rp, negative=neg)
        assert A.slot_payload_bits(oracle_lib, g, rs) > A.EMIT_WINDOW_BITS or neg
        grids.append(g)
        refs.append(oracle_lib.encode_block("hp", list(g)))
    x = torch.from_numpy(np.stack(grids).astype(np.int32)).cuda()
    # repeat with different leading blocks so every block lands at several bit alignments
    for lead in range(4):
        xs = torch.cat([x[lead:], x[:lead]])
        rr = refs[lead:] + refs[:lead]
        out = torch.full((sum(len(r) for r in refs) + 4096,), 0xFF, dtype=torch.uint8, device="cuda")
        buf, offs = P.encode_blocks("hp3", xs, out=out)
        o = offs.cpu().tolist()
        for i, r in enumerate(rr):
            assert buf[o[i]:o[i + 1]].cpu().numpy().tobytes() == r, (lead, i)
    # and the container path: a dirty output buffer gives the oracle's containers
    imgs = [inputs.synth.cfg2_pathology(s, 200, 328) for s in range(3)]
    xb = torch.from_numpy(np.stack(imgs)).cuda()
    dirty = torch.full((1 << 22,), 0xFF, dtype=torch.uint8, device="cuda")
    cont, offs = P.encode_tensor(xb, 8, 3, True, layout="hwc", batched=True, out=dirty)
    for i in range(3):
        ref = oracle_lib.encode_image(inputs.synth.planar(imgs[i]).astype(np.int64), 8, 3, True)
        assert cont[offs[i]:offs[i + 1]].cpu().numpy().tobytes() == ref


def test_large_slot_block_roundtrip():
    g, d, _ = A.large_slot_block(9, random_plane=5)
    blk = P.CoefficientBlock.build("hp3", list(g))
    data = P.encode_block(blk)
    back = P.decode_block(data, 128, 128, "hp3")
    assert back.depth == d and all(np.array_equal(u, v) for u, v in zip(back.coeffs, g))


def test_two_threads_two_streams_roundtrip(oracle_lib):
    imgs = [inputs.synth.planar(inputs.synth.cfg2_pathology(40 + s, 260 + 16 * s, 300)).astype(np.int64)
            for s in range(4)]
    refs = [oracle_lib.encode_image(a, 8, 3, True) for a in imgs]
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for it in range(6):
                    i = (k + it) % len(imgs)
                    x = torch.from_numpy(imgs[i]).to("cuda", torch.uint8)
                    cont, offs = P.encode_tensor(x, 8, 3, True)
                    got = cont[offs[0]:offs[1]].cpu().numpy().tobytes()
                    assert got == refs[i], (k, it)
                    dec = P.decode_tensor(cont[offs[0]:offs[1]], out_dtype="int32")
                    assert np.array_equal(dec.cpu().numpy(), imgs[i]), (k, it)
                    assert P.decode_image(refs[i]).samples.tolist() == imgs[i].tolist()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_sync_false_calls_keep_their_own_status():
    """Two unsynchronised encodes: each returned workspace holds its own call's status."""
    from paper_2005_08713_b200 import _lib
    from paper_2005_08713_b200.container import _status
    a = torch.from_numpy(inputs.synth.planar(inputs.synth.cfg2_pathology(1, 130, 140))).cuda()
    tiny = torch.empty(64, dtype=torch.uint8, device="cuda")  # far below the container size
    _, _, ws_small = P.encode_tensor(a, 8, 2, True, out=tiny, sync=False)
    _, _, ws_ok = P.encode_tensor(a, 8, 2, True, sync=False)
    assert _status(ws_ok)[0] == 0
    assert _status(ws_small)[0] == _lib.ST_OUT_CAPACITY


def test_decode_batch_beyond_4gib(oracle_lib):
    """Containers placed past the 4 GiB mark of one buffer decode (block-relative bit positions)."""
    imgs = [inputs.synth.cfg2_pathology(70 + s, 200, 264) for s in range(2)]
    refs = [oracle_lib.encode_image(inputs.synth.planar(a).astype(np.int64), 8, 3, True) for a in imgs]
    base = (1 << 32) + 12345
    total = base + sum(len(r) for r in refs) + 4096
    buf = torch.empty(total, dtype=torch.uint8, device="cuda")
    offs = [base, base + len(refs[0]), base + len(refs[0]) + len(refs[1])]
    for r, o in zip(refs, offs):
        buf[o:o + len(r)] = torch.frombuffer(bytearray(r), dtype=torch.uint8).cuda()
    dec = P.decode_tensor(buf, P.ContainerHeader(264, 200, 3, 8, 1, 3), out_dtype="uint8", layout="hwc",
                          offsets=torch.tensor(offs, device="cuda"), batch=2)
    assert torch.equal(dec.cpu(), torch.from_numpy(np.stack(imgs)))
    del buf
    torch.cuda.empty_cache()


def _redzoned(n, fill=0x5A, rz=1 << 16):
    buf = torch.full((n + 2 * rz,), fill, dtype=torch.uint8, device="cuda")
    return buf, buf[rz:rz + n], rz


def test_no_writes_outside_buffers(oracle_lib):
    """Bounds check without compute-sanitizer (closed on this pool): every output and workspace
    of encode / decode / truncate / region decode sits between 64 KB red zones that must come
    back untouched."""
    import ctypes
    from paper_2005_08713_b200 import _lib
    from paper_2005_08713_b200.container import _stream_ptr
    L = _lib.load()
    imgs = [inputs.synth.cfg2_pathology(60 + s, 136 + 24 * s, 264) for s in range(2)]
    for img in imgs:
        H, W, _ = img.shape
        x = torch.from_numpy(img).cuda()
        desc = _lib.ImageDesc(W, H, 3, 8, _lib.DTYPE_U8, _lib.LAYOUT_HWC, x.numel())
        ws_n, cap = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(L.wbpc_encode_plan_size(ctypes.byref(desc), 1, 4, 1, ctypes.byref(ws_n), ctypes.byref(cap)))
        wsb, ws, rz = _redzoned(ws_n.value)
        outb, out, _ = _redzoned(cap.value)
        offb, offs, _ = _redzoned(16)
        _lib.check(L.wbpc_encode(ctypes.byref(desc), x.data_ptr(), 1, 4, 1, ws.data_ptr(), ws.numel(), out.data_ptr(),
                                 out.numel(), offs.data_ptr(), _stream_ptr()))
        torch.cuda.synchronize()
        for b in (wsb, outb, offb):
            assert bool((b[:rz] == 0x5A).all()) and bool((b[-rz:] == 0x5A).all())
        n = int(offs.view(torch.int64)[1])
        ref = oracle_lib.encode_image(inputs.synth.planar(img).astype(np.int64), 8, 4, True)
        assert out[:n].cpu().numpy().tobytes() == ref
        # decode (full and region) into red-zoned outputs and workspaces
        hdr = P.ContainerHeader.parse(ref)
        h = hdr.to_c()
        _lib.check(L.wbpc_decode_plan_size(ctypes.byref(h), 0, ctypes.byref(ws_n)))
        wsb, ws, rz = _redzoned(ws_n.value)
        pb, pix, _ = _redzoned(x.numel())
        cont = torch.frombuffer(bytearray(ref), dtype=torch.uint8).cuda()
        _lib.check(L.wbpc_decode(ctypes.byref(h), cont.data_ptr(), cont.numel(), 0, 1, None, 0, pix.data_ptr(),
                                 _lib.DTYPE_U8, _lib.LAYOUT_HWC, ws.data_ptr(), ws.numel(), _stream_ptr()))
        _lib.check(L.wbpc_decode_region(ctypes.byref(h), cont.data_ptr(), cont.numel(), 7, 5, 33, 21, 1, 0,
                                        pix.data_ptr(), _lib.DTYPE_U8, _lib.LAYOUT_HWC, ws.data_ptr(), ws.numel(),
                                        _stream_ptr()))
        torch.cuda.synchronize()
        for b in (wsb, pb):
            assert bool((b[:rz] == 0x5A).all()) and bool((b[-rz:] == 0x5A).all())
        # truncate
        _lib.check(L.wbpc_truncate_plan_size(ctypes.byref(h), cont.numel(), ctypes.byref(ws_n), ctypes.byref(cap)))
        wsb, ws, rz = _redzoned(ws_n.value)
        tb, tout, _ = _redzoned(cap.value)
        lb, tlen, _ = _redzoned(8)
        _lib.check(L.wbpc_truncate(ctypes.byref(h), cont.data_ptr(), cont.numel(), 2, None, 0, ws.data_ptr(),
                                   ws.numel(), tout.data_ptr(), tout.numel(), tlen.data_ptr(), _stream_ptr()))
        torch.cuda.synchronize()
        for b in (wsb, tb, lb):
            assert bool((b[:rz] == 0x5A).all()) and bool((b[-rz:] == 0x5A).all())
        m = int(tlen.view(torch.int64)[0])
        assert tout[:m].cpu().numpy().tobytes() == oracle_lib.truncate_stream(ref, 2)

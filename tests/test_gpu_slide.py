"""Whole-slide path (BASELINE configs[3]) on the device vs the CPU oracle.

* SlideCodec on a small slide: every tile's container equals the oracle's `encode_image` of that
  tile, the device-assembled archive equals `archive.pack` of the oracle's containers, decode
  restores every tile, and the host path writes the same archive bytes.
* Two ranks (two processes on cuda:0, gloo for the size exchange, the CUDA encoder per rank) write
  their shards into one shared host archive; it equals `archive.pack` of the oracle's containers.
* A full 4096^2 cfg4 tile from the GPU generator, L6, RCT: container == the oracle's.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2005_08713_b200")
from paper_2005_08713_b200 import archive, synth  # noqa: E402
from paper_2005_08713_b200.slide import SlideCodec, release_host_buffer, shared_host_buffer  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_08713_b200 import _lib
    _lib.load()


def _tiles(n, size, seed=0):
    return torch.stack([synth.cfg2_pathology_torch(seed + t, size, size, "cuda") for t in range(n)])


def _oracle_archive(oracle_lib, x, tx, ty, L):
    conts = [oracle_lib.encode_image(synth.planar(t.cpu().numpy()).astype(np.int64), 8, L, True) for t in x]
    return conts, archive.pack(conts, tx, ty)


@pytest.mark.parametrize("batch,streams", [(2, 2), (3, 1), (4, 3)])
def test_slide_device_archive_vs_oracle(oracle_lib, batch, streams):
    tx, ty, size, L = 3, 2, 384, 4
    x = _tiles(tx * ty, size, seed=50)
    conts, ref = _oracle_archive(oracle_lib, x, tx, ty, L)
    codec = SlideCodec(tx, ty, size, size, 3, 8, L, True, batch=batch, streams=streams)
    out = torch.empty_like(x)
    codec.encode(x)
    codec.exchange()
    codec.ensure_archive()
    codec.assemble()
    codec.decode(out)
    codec.check()
    assert torch.equal(out, x)
    assert codec.tile_sizes() == [len(c) for c in conts]
    got = codec.archive_header() + codec.local_archive_bytes()
    assert got == ref
    _, _, parts = archive.unpack(got)
    assert parts == conts
    # again through the timed entry point, into dirty buffers
    out.fill_(7)
    codec.archive_dev.fill_(0xFF)
    codec.roundtrip_device(x, out)
    codec.check()
    assert torch.equal(out, x) and codec.archive_header() + codec.local_archive_bytes() == ref
    # host path: pinned tiles -> host archive -> pinned tiles
    xh = x.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    arch = torch.full((len(ref) + 100,), 0xAB, dtype=torch.uint8).pin_memory()
    total = codec.roundtrip_host(xh, oh, arch)
    torch.cuda.synchronize()
    codec.check()
    assert total == len(ref)
    assert arch[:total].numpy().tobytes() == ref
    assert torch.equal(oh, xh)


def _rank_worker(rank, world, port, path, total, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        tx, ty, size, L = 5, 1, 256, 3
        codec = SlideCodec(tx, ty, size, size, 3, 8, L, True, world=world, rank=rank, batch=2, streams=2)
        x = torch.stack([synth.cfg2_pathology_torch(90 + codec.first + i, size, size, "cuda")
                         for i in range(codec.n_local)])
        xh = x.cpu().pin_memory()
        oh = torch.empty_like(xh).pin_memory()
        arch, keep = shared_host_buffer(path, total, create=False)
        n = codec.roundtrip_host(xh, oh, arch)
        torch.cuda.synchronize()
        codec.check()
        ok = bool(torch.equal(oh, xh)) and n == total
        dist.barrier()
        release_host_buffer(keep)
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))


def test_two_ranks_one_shared_archive(oracle_lib, tmp_path):
    import torch.multiprocessing as mp
    tx, size, L = 5, 256, 3
    x = torch.stack([synth.cfg2_pathology_torch(90 + t, size, size, "cuda") for t in range(tx)])
    conts, ref = _oracle_archive(oracle_lib, x, tx, 1, L)
    path = f"/dev/shm/wbpc_test_archive_{os.getpid()}" if os.path.isdir("/dev/shm") else str(tmp_path / "arch")
    with open(path, "wb") as f:
        f.truncate(len(ref))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, path, len(ref), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    with open(path, "rb") as f:
        got = f.read()
    os.unlink(path)
    assert got == ref


def test_archive_file_roundtrip(oracle_lib, tmp_path):
    """save_archive writes the archive.pack layout of the oracle's containers to one file; a
    fresh codec (also as rank 1 of 2: its shard only) reads it back and decodes the tiles."""
    tx, ty, size, L = 2, 3, 320, 3
    x = _tiles(tx * ty, size, seed=70)
    conts, ref = _oracle_archive(oracle_lib, x, tx, ty, L)
    codec = SlideCodec(tx, ty, size, size, 3, 8, L, True, batch=4, streams=2)
    codec.encode(x)
    codec.exchange()
    codec.ensure_archive()
    codec.assemble()
    codec.check()
    path = str(tmp_path / "slide.wbpa")
    assert codec.save_archive(path) == len(ref)
    assert open(path, "rb").read() == ref
    fresh = SlideCodec(tx, ty, size, size, 3, 8, L, True, batch=3, streams=1)
    fresh.load_archive(path)
    out = torch.empty_like(x)
    fresh.decode(out)
    fresh.check()
    assert torch.equal(out, x)
    shard = SlideCodec(tx, ty, size, size, 3, 8, L, True, world=2, rank=1, batch=2, streams=1)
    shard.load_archive(path)
    out1 = torch.empty_like(x[shard.first:shard.first + shard.n_local])
    shard.decode(out1)
    shard.check()
    assert torch.equal(out1, x[shard.first:shard.first + shard.n_local])
    with open(path, "r+b") as f:  # a truncated file is refused
        f.truncate(len(ref) - 100)
    with pytest.raises(P.ContainerParseError):
        SlideCodec(tx, ty, size, size, 3, 8, L, True).load_archive(path)


def test_cfg4_gpu_generated_tile_vs_oracle(oracle_lib):
    """One full cfg4 tile (4096^2 RGB8, L6, RCT) from the GPU generator: bit-exact container,
    lossless decode, and its slide-path container identical to the functional API's."""
    x = synth.cfg4_tile_torch(0, 255, 4096, "cuda")
    ref = oracle_lib.encode_image(synth.planar(x.cpu().numpy()).astype(np.int64), 8, 6, True,
                                  threads=len(os.sched_getaffinity(0)))
    cont, offs = P.encode_tensor(x, 8, 6, True, layout="hwc")
    got = cont[offs[0]:offs[1]].cpu().numpy().tobytes()
    assert got == ref
    dec = P.decode_tensor(cont[offs[0]:offs[1]], out_dtype="uint8", layout="hwc")
    assert torch.equal(dec, x)
    codec = SlideCodec(1, 1, 4096, 4096, 3, 8, 6, True, batch=1, streams=1)
    out = torch.empty_like(x).unsqueeze(0)
    codec.roundtrip_device(x.unsqueeze(0), out)
    codec.check()
    assert torch.equal(out[0], x) and codec.local_archive_bytes() == ref


def test_stream_host_several_slides(oracle_lib):
    """stream_host: three slides back to back (pipelined across slide boundaries), each archive
    equals archive.pack of the oracle's containers and every tile comes back."""
    tx, ty, size, L = 3, 2, 256, 3
    slides = [_tiles(tx * ty, size, seed=200 + 10 * i) for i in range(3)]
    refs = [_oracle_archive(oracle_lib, x, tx, ty, L)[1] for x in slides]
    codec = SlideCodec(tx, ty, size, size, 3, 8, L, True, batch=2, streams=2)
    xh = [x.cpu().pin_memory() for x in slides]
    oh = [torch.empty_like(x).pin_memory() for x in xh]
    arch = [torch.full((len(r) + 64,), 0xCD, dtype=torch.uint8).pin_memory() for r in refs]
    totals = codec.stream_host(xh, oh, arch)
    torch.cuda.synchronize()
    codec.check()
    for i in range(3):
        assert totals[i] == len(refs[i])
        assert arch[i][:totals[i]].numpy().tobytes() == refs[i]
        assert torch.equal(oh[i], xh[i])

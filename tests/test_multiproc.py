"""World-size-2 gloo test of the multi-GPU exchange: per-rank tile containers -> all-gathered
byte counts -> tile-archive offsets (the only collective of the path; NCCL on the GPU box)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def archive_offsets(sizes_all: torch.Tensor) -> torch.Tensor:
    """Exclusive scan of gathered per-tile container sizes -> archive offsets (after a header)."""
    from paper_2005_08713_b200.archive import tile_offsets
    return tile_offsets(sizes_all)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2005_08713_b200 import synth
    from paper_2005_08713_b200.archive import shard_tiles
    n_tiles = 6
    mine = shard_tiles(n_tiles, world, rank)
    conts = []
    for t in mine:
        img = synth.cfg2_pathology(t, 64, 64)
        conts.append(oracle.encode_image(synth.planar(img).astype(np.int64), 8, 2, True))
    local = torch.tensor([len(c) for c in conts] + [0] * (-(-n_tiles // world) - len(conts)), dtype=torch.int64)
    gathered = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(gathered, local)
    sizes = torch.cat(gathered)
    q.put((rank, mine, [len(c) for c in conts], sizes.tolist()))
    dist.destroy_process_group()


def test_gloo_tile_offsets():
    from paper_2005_08713_b200.archive import shard_tiles, tile_offsets
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # every rank sees the same gathered table; tiles partition 0..5 contiguously
    assert res[0][3] == res[1][3]
    assert sorted(res[0][1] + res[1][1]) == list(range(6))
    assert shard_tiles(6, 2, 0) == [0, 1, 2] and shard_tiles(6, 2, 1) == [3, 4, 5]
    per_tile = res[0][2] + res[1][2]
    offs = tile_offsets(torch.tensor(res[0][3]), n_tiles=6, world=2).tolist()
    assert offs[0] > 0 and all(offs[i + 1] - offs[i] == per_tile[i] for i in range(5))

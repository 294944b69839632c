"""Developer statistics: plane bit lengths of the bench workload and the per-lane decode load
under the snake assignment of k_block_planes (LPB lanes per block)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth  # noqa: E402
from paper_2005_08713_b200.blocks import plane_offsets  # noqa: E402
from paper_2005_08713_b200.container import ContainerReader, encode_tensor  # noqa: E402
from paper_2005_08713_b200.errors import CodecError  # noqa: E402

img = torch.from_numpy(synth.cfg2_pathology(1000)).cuda()
buf, offs = encode_tensor(img, bit_depth=8, levels=4, use_rct=True, layout="hwc")
R = ContainerReader(buf[offs[0]:offs[1]].cpu().numpy().tobytes())
lens = []
for i in range(len(R.offsets)):
    blk = R.block_bytes(i)
    try:
        po = plane_offsets(blk, 128, 128, "hp3")
    except CodecError:
        po = plane_offsets(blk, 128, 128, "ll")
    offs = [o for _, o in po] + [8 * len(blk)]
    hdr = offs[0]
    pl = [offs[k + 1] - offs[k] for k in range(len(po))]
    lens.append(pl)
allp = np.concatenate([np.array(p) for p in lens])
print("blocks", len(lens), "planes", allp.size, "mean planes/block", allp.size / len(lens))
print("plane bits: max", allp.max(), "p99", np.percentile(allp, 99), "p90", np.percentile(allp, 90), "median",
      np.median(allp))
for LPB in (16, 32):
    worst = []
    for pl in lens:
        order = np.argsort(-np.array(pl), kind="stable")
        load = np.zeros(LPB)
        for r, j in enumerate(order):
            row, col = divmod(r, LPB)
            lane = LPB - 1 - col if row & 1 else col
            load[lane] += pl[j]
        worst.append(load.max())
    worst = np.array(worst)
    print(f"LPB={LPB}: worst-lane bits per block: max {worst.max()} p90 {np.percentile(worst, 90)} median {np.median(worst)}")
out = os.path.join(ROOT, "gpurun_out", "plane_lengths.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
import json  # noqa: E402
with open(out, "w") as f:
    json.dump(lens, f)

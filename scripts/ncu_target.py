"""ncu target: one profiled round trip after a warm-up (NCU_CFG=cfg4 [default] | cfg2 | cfg1).

cfg4: NCU_TILES (4) cfg4 tiles (4096^2 RGB8, RCT, L6) through SlideCodec with one batch of
NCU_TILES tiles on one stream (the bench's per-batch launch sequence + archive kernels).
cfg2: NCU_IMAGES x 2048^2 RGB8, RCT, L4.  cfg1: one 512^2 gray12, L3.
Run under `ncu --profile-from-start off ...`: only the second round trip is captured.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth  # noqa: E402
from paper_2005_08713_b200.container import Codec  # noqa: E402

cfg = os.environ.get("NCU_CFG", "cfg4")
if cfg == "cfg4":
    from paper_2005_08713_b200.slide import SlideCodec  # noqa: E402
    T = int(os.environ.get("NCU_TILES", "4"))
    x = torch.stack([synth.cfg4_tile_torch(0, t) for t in range(T)])
    out = torch.empty_like(x)
    sc = SlideCodec(T, 1, 4096, 4096, 3, 8, 6, True, batch=T, streams=1)
    sc.roundtrip_device(x, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    sc.roundtrip_device(x, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sc.check()
    assert torch.equal(out, x)
    print("ok")
    sys.exit(0)
if cfg == "cfg1":
    imgs = torch.from_numpy(synth.cfg1_gray12(0).astype("uint16")).cuda().unsqueeze(0)  # (1,1,H,W)
    codec = Codec(512, 512, 1, 12, 3, False, torch.uint16, "chw", batch=1)
else:
    B = int(os.environ.get("NCU_IMAGES", "8"))
    imgs = torch.stack([torch.from_numpy(synth.cfg2_pathology(1000 + i)) for i in range(B)]).cuda()
    codec = Codec(2048, 2048, 3, 8, 4, True, torch.uint8, "hwc", batch=B)
codec.roundtrip_device(imgs)
torch.cuda.synchronize()
torch.cuda.profiler.start()
codec.roundtrip_device(imgs)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
codec.check()
assert torch.equal(codec.pixels_out, imgs)
print("ok")

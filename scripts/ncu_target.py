"""ncu target: one profiled round trip after a warm-up (NCU_CFG=cfg2 [default] | cfg1).

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

cfg = os.environ.get("NCU_CFG", "cfg2")
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

"""One warm encode+decode round trip of a config (for ncu captures)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth
from paper_2005_08713_b200.container import Codec
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
if cfg == "1":
    img, lay, bd, L, rct = synth.cfg1_gray12(0).astype(np.uint16), "chw", 12, 3, False
elif cfg == "3":
    img, lay, bd, L, rct = synth.cfg2_pathology(0, 4096, 4096), "hwc", 8, 5, True
else:
    img, lay, bd, L, rct = synth.cfg2_pathology(0), "hwc", 8, 4, True
x = torch.from_numpy(img).cuda().unsqueeze(0)
H, W, C = img.shape if lay == "hwc" else (img.shape[1], img.shape[2], img.shape[0])
codec = Codec(W, H, C, bd, L, rct, x.dtype, lay)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    codec.roundtrip_device(x)
codec.check()
assert torch.equal(codec.pixels_out, x)
print("ok")

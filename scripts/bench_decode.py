"""Developer timing of the decode kernels on the bench workload (8 x cfg2)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth, _lib
from paper_2005_08713_b200.container import Codec
B = int(os.environ.get("NIMG", "8"))
imgs = torch.stack([torch.from_numpy(synth.cfg2_pathology(1000 + i)) for i in range(B)]).cuda()
codec = Codec(2048, 2048, 3, 8, 4, True, torch.uint8, "hwc", batch=B)
for _ in range(3):
    codec.roundtrip_device(imgs)
codec.check()
assert torch.equal(codec.pixels_out, imgs)
_lib.profile_enable(True)
for _ in range(10):
    codec.roundtrip_device(imgs)
torch.cuda.synchronize()
prof = _lib.profile_collect()
print({k: round(v[0] / 10 * 1e3, 1) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])})

import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth, _lib
from paper_2005_08713_b200.container import Codec
L = _lib.load()
B = 8
imgs = torch.stack([torch.from_numpy(synth.cfg2_pathology(1000 + i)) for i in range(B)]).cuda()
codec = Codec(2048, 2048, 3, 8, 4, True, torch.uint8, "hwc", batch=B)
codec.roundtrip_device(imgs); torch.cuda.synchronize()
codec.encode_device(imgs); torch.cuda.synchronize()
n = 2064
buf = (ctypes.c_ulonglong * (8 * n))()
L.wbpc_adbg_read(buf, 8 * n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
names = ["symbols", "hist+runs", "huff1+cw", "huff2", "slotbits", "meta"]
d = np.diff(a[:, :7], axis=1)
for i, nm in enumerate(names):
    print(f"{nm:10s} mean {d[:, i].mean():9.0f} cyc  p90 {np.percentile(d[:, i], 90):9.0f}")
tot = a[:, 6] - a[:, 0]
print("total per CTA mean", tot.mean(), "max", tot.max(), " kernel span", a[:, 6].max() - a[:, 0].min())

"""Developer timing: per-kernel device times (library CUDA-event marks) for the configs."""
import os, sys, time, json
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2005_08713_b200 as P
from paper_2005_08713_b200 import synth, _lib
from paper_2005_08713_b200.container import Codec

def run(name, img, layout, bd, L, rct, batch=1, iters=10):
    x = torch.from_numpy(img).cuda()
    if batch > 1:
        x = x.unsqueeze(0).repeat(batch, *([1] * img.ndim)).contiguous()
    else:
        x = x.unsqueeze(0)
    if layout == "hwc":
        H, W, C = img.shape
    else:
        C, H, W = img.shape
    codec = Codec(W, H, C, bd, L, rct, x.dtype, layout, batch)
    for _ in range(3):
        codec.roundtrip_device(x)
    codec.check()
    assert torch.equal(codec.pixels_out, x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    enc = []; dec = []
    for _ in range(iters):
        s.record(); codec.encode_device(x); e.record(); torch.cuda.synchronize(); enc.append(s.elapsed_time(e))
        s.record(); codec.decode_device(); e.record(); torch.cuda.synchronize(); dec.append(s.elapsed_time(e))
    _lib.profile_enable(True)
    for _ in range(iters):
        codec.roundtrip_device(x)
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    st = codec.dec_ws[:32].cpu().numpy().view(np.uint64)
    print("   decode fallbacks (cumulative):", int(st[3]))
    _lib.profile_enable(False)
    mp = W * H * batch / 1e6
    te, td = np.median(enc), np.median(dec)
    sizes = codec.container_sizes()
    print(f"== {name}: {mp:.1f} MP  encode {te:.3f} ms ({mp/te*1e3:.0f} MP/s)  decode {td:.3f} ms ({mp/td*1e3:.0f} MP/s)  container {sum(sizes)/1e6:.2f} MB")
    for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:20s} {ms/iters*1e3:9.1f} us/step  ({n//iters} launches/step)")

run("cfg1 gray12 512", synth.cfg1_gray12(0)[0][None].astype(np.uint16), "chw", 12, 3, False)
run("cfg2 rgb 2048", synth.cfg2_pathology(0), "hwc", 8, 4, True)
img3 = synth.cfg2_pathology(0, 4096, 4096)
run("cfg3 rgb 4096", img3, "hwc", 8, 5, True)
run("cfg4 x8 tiles 4096 L6", img3, "hwc", 8, 6, True, batch=8, iters=3)

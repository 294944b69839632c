"""Experiment: 8-image round trip as 1 x batch-8 vs k x batch-(8/k) on k streams (CUDA graphs)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth
from paper_2005_08713_b200.container import Codec
B = 8
imgs = torch.stack([torch.from_numpy(synth.cfg2_pathology(1000 + i)) for i in range(B)]).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

def run(k):
    per = B // k
    codecs = [Codec(2048, 2048, 3, 8, 4, True, torch.uint8, "hwc", batch=per) for _ in range(k)]
    parts = [imgs[i * per:(i + 1) * per].contiguous() for i in range(k)]
    streams = [torch.cuda.Stream() for _ in range(k)]
    for _ in range(2):
        for c, x in zip(codecs, parts):
            c.roundtrip_device(x)
    torch.cuda.synchronize()
    for c, x in zip(codecs, parts):
        c.check(); assert torch.equal(c.pixels_out, x)
    g = torch.cuda.CUDAGraph()
    main = torch.cuda.Stream()
    with torch.cuda.stream(main):
        with torch.cuda.graph(g):
            cur = torch.cuda.current_stream()
            for s in streams:
                s.wait_stream(cur)
            for c, x, s in zip(codecs, parts, streams):
                with torch.cuda.stream(s):
                    c.roundtrip_device(x)
            for s in streams:
                cur.wait_stream(s)
    torch.cuda.synchronize()
    ts = []
    for i in range(30):
        flush.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    for c, x in zip(codecs, parts):
        c.check(); assert torch.equal(c.pixels_out, x)
    print(f"k={k}: {ms:.3f} ms/step  {B * 4.194304 / ms * 1e3:.0f} MP/s")

for k in (1, 2, 4):
    run(k)

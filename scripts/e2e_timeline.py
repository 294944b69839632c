"""Per-stage event timeline of HostPipeline.roundtrip (8 x cfg2) -- developer tool."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import synth, _lib
from paper_2005_08713_b200.container import HostPipeline, _stream_ptr
B, NCH = 8, int(os.environ.get("NCH", "4"))
host = torch.stack([torch.from_numpy(synth.cfg2_pathology(1000 + i)) for i in range(B)]).pin_memory()
pipe = HostPipeline(2048, 2048, 3, 8, 4, True, torch.uint8, "hwc", batch=B, chunk=B // NCH)
for _ in range(3):
    pipe.roundtrip(host)
torch.cuda.synchronize()
L = _lib.load()
ch = pipe.chunk
T0 = torch.cuda.Event(enable_timing=True); T0.record()
marks = {}
def ev(name, s):
    e = torch.cuda.Event(enable_timing=True); e.record(s); marks[name] = e
t_host0 = time.perf_counter()
for k, (c, s) in enumerate(zip(pipe.codecs, pipe.streams)):
    s.wait_event(T0)
    with torch.cuda.stream(s):
        c.dev_in.copy_(host[k * ch:(k + 1) * ch], non_blocking=True); ev(f"{k} h2d_px", s)
        c.encode_device(c.dev_in); ev(f"{k} encode", s)
        L.wbpc_copy_sized(c.host_container.data_ptr(), c.containers.data_ptr(), c.offsets.data_ptr() + 8 * ch, _stream_ptr()); ev(f"{k} d2h_cont", s)
        pipe.off_host[k].copy_(c.offsets, non_blocking=True)
        c.offsets_in.copy_(pipe.off_host[k], non_blocking=True)
        L.wbpc_copy_sized(c.containers_in.data_ptr(), c.host_container.data_ptr(), c.offsets_in.data_ptr() + 8 * ch, _stream_ptr()); ev(f"{k} h2d_cont", s)
        c.decode_device(c.containers_in, c.offsets_in); ev(f"{k} decode", s)
        c.host_pixels.copy_(c.pixels_out, non_blocking=True); ev(f"{k} d2h_px", s)
t_issue = (time.perf_counter() - t_host0) * 1e3
torch.cuda.synchronize()
print("host issue ms %.2f wall ms %.2f" % (t_issue, (time.perf_counter() - t_host0) * 1e3))
for k in range(NCH):
    print(" ".join(f"{n.split()[1]}={T0.elapsed_time(marks[n]):6.2f}" for n in marks if n.startswith(f"{k} ")))

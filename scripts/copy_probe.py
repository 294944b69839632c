import ctypes, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_08713_b200 import _lib
L = _lib.load()
n = 12_500_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
cnt = torch.tensor([n], dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def t(fn, it=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
print("kernel D2H %.1f GB/s" % (n / t(lambda: L.wbpc_copy_sized(h.data_ptr(), d.data_ptr(), cnt.data_ptr(), s)) / 1e6))
print("kernel H2D %.1f GB/s" % (n / t(lambda: L.wbpc_copy_sized(d.data_ptr(), h.data_ptr(), cnt.data_ptr(), s)) / 1e6))
print("memcpy D2H %.1f GB/s" % (n / t(lambda: h.copy_(d, non_blocking=True)) / 1e6))
print("memcpy H2D %.1f GB/s" % (n / t(lambda: d.copy_(h, non_blocking=True)) / 1e6))

import os, sys, struct
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import inputs, oracle
import paper_2005_08713_b200 as P
from paper_2005_08713_b200.container import ContainerHeader, ContainerReader, truncate_tensor
name, a, bd, L, rct = [x for x in inputs.small_inputs() if x[0].startswith("rand_1x13x9")][0]
ref = oracle.encode_image(a, bd, L, rct)
h = ContainerHeader.parse(ref)
buf = torch.frombuffer(bytearray(ref), dtype=torch.uint8).cuda()
out, olen, ws = truncate_tensor(buf, h, 1, sync=False)
torch.cuda.synchronize()
wsb = ws[:4096].cpu().numpy()
print("status", wsb[:32].view(np.uint64))
tm_off = 256
TMS = 216
for blk in range(3):
    t = wsb[tm_off + blk*TMS: tm_off + (blk+1)*TMS]
    new_len, mode, nseg, pad = t[:16].view(np.uint32)
    dst = t[16:56].view(np.uint32); ln = t[56:96].view(np.uint32); src = t[96:176].view(np.uint64); lit = t[176:216].view(np.uint32)
    print(blk, new_len, mode, nseg, dst[:nseg], ln[:nseg], src[:nseg], lit[:nseg])
rd = ContainerReader(ref)
print("offsets", rd.offsets[:4], rd.lengths[:4])
got = out[: int(olen.item())].cpu().numpy().tobytes()
exp = oracle.truncate_stream(ref, 1)
print(exp[:80].hex()); print(got[:80].hex())

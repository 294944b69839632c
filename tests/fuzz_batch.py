"""Randomised consistency run of the large-batch kernels (test infrastructure; not collected by pytest: run by hand on a GPU box).

usage: python tests/fuzz_batch.py [seconds] [seed]
Random equally shaped image batches sized to cross the kernel-selection thresholds (>= 512 and
>= 4096 blocks per call: continuous plane lists, four headers per warp).  Per case: the batched
containers equal the per-image containers (the per-image path is pinned to the oracle by the
parity suite and tests/fuzz_parity.py), image 0's container equals the oracle's, and the
batched decode restores the batch; with corruption, the batched decode reports the same error
class as decoding the damaged image alone.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2005_08713_b200 as P  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
g = torch.Generator(device="cuda")
g.manual_seed(seed)
t0 = time.time()
n = 0
while time.time() - t0 < budget:
    c = int(rng.choice([1, 3]))
    h, w = int(rng.integers(40, 700)), int(rng.integers(40, 900))
    bd = int(rng.choice([8, 8, 10, 12, 16]))
    L = int(rng.integers(0, 6))
    rct = c == 3 and rng.random() < 0.6
    per = oracle.slot_count(w, h, c, L)
    target = int(rng.choice([600, 1500, 4200, 6000]))
    B = max(2, min(400, -(-target // per)))
    dt = torch.uint8 if bd <= 8 else torch.uint16
    if rng.random() < 0.5:
        x = torch.randint(0, 1 << bd, (B, c, h, w), generator=g, device="cuda", dtype=torch.int32).to(dt)
    else:
        yy, xx = torch.meshgrid(torch.arange(h, device="cuda"), torch.arange(w, device="cuda"), indexing="ij")
        base = ((torch.sin(xx / 23.0) * torch.cos(yy / 17.0) + 1) / 2 * ((1 << bd) - 1))
        noise = torch.randint(0, 9, (B, c, h, w), generator=g, device="cuda", dtype=torch.int32)
        x = (base[None, None] + noise).clamp_(0, (1 << bd) - 1).to(torch.int32).to(dt)
    out, offs = P.encode_tensor(x, bd, L, rct, layout="chw", batched=True)
    tag = (n, B, c, h, w, bd, L, rct, per * B)
    for i in sorted(set([0, B - 1, int(rng.integers(0, B))])):
        one, o1 = P.encode_tensor(x[i], bd, L, rct, layout="chw")
        if not torch.equal(one[o1[0]:o1[1]], out[offs[i]:offs[i + 1]]):
            print("BATCH/SINGLE ENCODE MISMATCH", tag, i, flush=True)
            sys.exit(1)
    ref = oracle.encode_image(x[0].cpu().numpy().astype(np.int64), bd, L, rct)
    if out[offs[0]:offs[1]].cpu().numpy().tobytes() != ref:
        print("ORACLE ENCODE MISMATCH", tag, flush=True)
        sys.exit(1)
    hdr = P.ContainerHeader(w, h, c, bd, 1 if rct else 0, L)
    dec = P.decode_tensor(out, hdr, out_dtype="int32", layout="chw", offsets=torch.tensor(offs, device="cuda"), batch=B)
    if not torch.equal(dec.to(dt), x):
        print("BATCH ROUNDTRIP MISMATCH", tag, flush=True)
        sys.exit(1)
    # damage one image's block bytes: same error class (or same pixels) as that image alone
    k = int(rng.integers(0, B))
    lo = offs[k] + 19 + 12 * per
    if offs[k + 1] > lo + 8:
        bad = out.clone()
        pos = int(rng.integers(lo, offs[k + 1]))
        bad[pos] ^= 1 << int(rng.integers(0, 8))

        def cls(fn):
            try:
                return None, fn()
            except Exception as e:  # noqa: BLE001
                return type(e).__name__, None
        eb, db = cls(lambda: P.decode_tensor(bad, hdr, out_dtype="int32", layout="chw",
                                             offsets=torch.tensor(offs, device="cuda"), batch=B))
        es, ds = cls(lambda: P.decode_tensor(bad[offs[k]:offs[k + 1]].clone(), hdr, out_dtype="int32", layout="chw"))
        if eb != es or (eb is None and not torch.equal(db[k], ds)):
            print("CORRUPTION OUTCOME MISMATCH", tag, k, eb, es, flush=True)
            sys.exit(1)
    n += 1
print(f"batch fuzz ok: {n} cases in {time.time() - t0:.0f} s (seed {seed})", flush=True)

"""Randomised differential run of the CUDA path against the CPU oracle (test infrastructure; not collected by pytest: run by hand on a GPU box).

usage: python tests/fuzz_parity.py [seconds] [seed]
Random shapes biased to the sizes the wide-plane DWT kernels take (plane widths >= 512, multiples
and non-multiples of 8 / 16, odd heights), channel counts, bit depths around the packed-lifting
gate, levels, content (noise / smooth / sparse).  Every case: container bytes equal, lossless
round trip equal, one lossy decode and one truncation equal; 8-bit RGB also through the fused
interleaved output.  Prints a summary line; exits 1 on the first mismatch.
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
t0 = time.time()
n = 0
while time.time() - t0 < budget:
    c = int(rng.choice([1, 3, 3, 2, 4]))
    wide = rng.random() < 0.7
    w = int(rng.choice([1024, 1040, 1056, 1088, 1104, 1280, 1536, 2048, 2064, 2080, 2560, 3072, 4096, 4112])) if wide \
        else int(rng.integers(1, 1500))
    if wide and rng.random() < 0.3:
        w += int(rng.integers(-9, 10))
    h = int(rng.integers(1, 700)) if rng.random() < 0.7 else int(rng.integers(700, 1400))
    bd = int(rng.choice([8, 8, 8, 9, 10, 12, 16, 5]))
    L = int(rng.integers(1, 7))
    rct = c == 3 and rng.random() < 0.7
    kind = int(rng.integers(0, 4))
    mx = (1 << bd) - 1
    if kind == 0:
        a = rng.integers(0, mx + 1, (c, h, w))
    elif kind == 1:
        yy, xx = np.mgrid[0:h, 0:w]
        base = (np.sin(xx / rng.uniform(5, 60)) * np.cos(yy / rng.uniform(5, 40)) + 1) / 2 * mx
        a = np.stack([np.clip(base + rng.integers(-4, 5, (h, w)) + 7 * k, 0, mx) for k in range(c)])
    elif kind == 2:
        a = np.full((c, h, w), int(rng.integers(0, mx + 1)))
        m = rng.random((h, w)) < 0.01
        for k in range(c):
            a[k][m] = rng.integers(0, mx + 1, int(m.sum()))
    else:
        yy, xx = np.mgrid[0:h, 0:w]
        a = np.stack([(((xx >> int(rng.integers(0, 4))) ^ (yy >> int(rng.integers(0, 4)))) & 1) * mx for _ in range(c)])
    a = a.astype(np.int64)
    tag = (n, c, h, w, bd, L, rct, kind)
    ref = oracle.encode_image(a, bd, L, rct)
    got = P.encode_image(P.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
    if got != ref:
        print("ENCODE MISMATCH", tag, flush=True)
        sys.exit(1)
    if not np.array_equal(P.decode_image(ref).samples, a):
        print("ROUNDTRIP MISMATCH", tag, flush=True)
        sys.exit(1)
    lev, nd = int(rng.integers(0, L + 1)), int(rng.integers(1, 4))
    o, _ = oracle.decode_image(ref, level=lev, planes_dropped=nd)
    if not np.array_equal(o, P.decode_image(ref, level=lev, planes_dropped=nd).samples):
        print("LOSSY DECODE MISMATCH", tag, lev, nd, flush=True)
        sys.exit(1)
    if P.truncate_stream(ref, nd) != oracle.truncate_stream(ref, nd):
        print("TRUNCATE MISMATCH", tag, nd, flush=True)
        sys.exit(1)
    if c == 3 and bd == 8:
        buf = torch.frombuffer(bytearray(ref), dtype=torch.uint8).cuda()
        hwc = P.decode_tensor(buf, out_dtype="uint8", layout="hwc").cpu().numpy()
        if not np.array_equal(hwc, a.transpose(1, 2, 0).astype(np.uint8)):
            print("HWC DECODE MISMATCH", tag, flush=True)
            sys.exit(1)
    n += 1
print(f"fuzz ok: {n} cases in {time.time() - t0:.0f} s (seed {seed})", flush=True)

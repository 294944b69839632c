"""Developer check: GPU path vs CPU oracle on the small golden inputs (prints mismatches)."""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2005_08713_b200 as P  # noqa: E402

fails = 0
for name, a, bd, L, rct in inputs.small_inputs():
    try:
        ref = oracle.encode_image(a, bd, L, rct)
        img = P.RasterImage.from_planes(list(a), bd)
        t = time.time()
        got = P.encode_image(img, levels=L, use_rct=rct)
        te = time.time() - t
        ok_enc = got == ref
        if not ok_enc:
            fails += 1
            # locate first differing block
            from paper_2005_08713_b200.container import ContainerReader
            ra, rb = ContainerReader(ref), ContainerReader(got)
            for i in range(len(ra.offsets)):
                ba, bb = ra.block_bytes(i), rb.block_bytes(i)
                if ba != bb:
                    print(f"  block {i}: ref len {len(ba)} got {len(bb)}; ref {ba[:24].hex()} got {bb[:24].hex()}")
                    break
        res = [ok_enc]
        for lev in range(L + 1):
            for n in (0, 1, 3):
                d1, _ = oracle.decode_image(ref, level=lev, planes_dropped=n)
                d2 = P.decode_image(ref, level=lev, planes_dropped=n).samples
                ok = d1.shape == d2.shape and np.array_equal(d1, d2)
                res.append(ok)
                if not ok:
                    fails += 1
                    print(f"  decode mismatch level {lev} drop {n}: shapes {d1.shape} {d2.shape}")
        for n in (1, 2, 4):
            t1 = oracle.truncate_stream(ref, n)
            t2 = P.truncate_stream(ref, n)
            res.append(t1 == t2)
            if t1 != t2:
                fails += 1
                print(f"  truncate mismatch n={n}: {len(t1)} vs {len(t2)}")
                from paper_2005_08713_b200.container import ContainerReader
                ra, rb = ContainerReader(t1), ContainerReader(t2)
                for i in range(len(ra.offsets)):
                    ba, bb = ra.block_bytes(i), rb.block_bytes(i)
                    if ba != bb:
                        k = next(j for j in range(min(len(ba), len(bb))) if ba[j] != bb[j])
                        print(f"   block {i} len {len(ba)}/{len(bb)} first diff byte {k}: ref {ba[max(0,k-4):k+12].hex()} got {bb[max(0,k-4):k+12].hex()}")
                        break
        print(name, "OK" if all(res) else "FAIL", f"enc {te*1e3:.1f} ms")
    except Exception:
        fails += 1
        print(name, "EXC")
        traceback.print_exc()
print("FAILS", fails)
sys.exit(1 if fails else 0)

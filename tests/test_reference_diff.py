"""Differential tests: oracle vs the live reference package (build container only).

Skipped when /root/reference is absent (GPU boxes).  Covers random shapes, bit depths,
levels, the lossy paths and the error classes raised on corrupted containers.
"""

import importlib
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def wbpc():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    return importlib.import_module("wbpc")


def _exc_name(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return type(e).__name__
    return None


def test_random_images(oracle_lib, wbpc):
    rng = np.random.default_rng(123)
    for it in range(25):
        c = int(rng.choice([1, 2, 3, 4]))
        h, w = int(rng.integers(1, 150)), int(rng.integers(1, 150))
        bd = int(rng.integers(1, 17))
        L = int(rng.integers(0, 6))
        rct = c == 3 and bool(rng.integers(0, 2))
        if it % 2:
            a = rng.integers(0, 1 << bd, (c, h, w)).astype(np.int64)
        else:
            yy, xx = np.mgrid[0:h, 0:w]
            a = np.stack([(xx * 3 + yy * 5 + k) % (1 << bd) for k in range(c)]).astype(np.int64)
        ref = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
        got = oracle_lib.encode_image(a, bd, L, rct)
        assert got == ref, (c, h, w, bd, L, rct)
        for n in (0, 2):
            lev = int(rng.integers(0, L + 1))
            r = wbpc.decode_image(ref, level=lev, planes_dropped=n).samples
            o, _ = oracle_lib.decode_image(got, level=lev, planes_dropped=n)
            assert np.array_equal(r, o)
        assert wbpc.truncate_stream(ref, 3) == oracle_lib.truncate_stream(got, 3)


def test_encode_errors(oracle_lib, wbpc):
    a = np.zeros((2, 8, 8), dtype=np.int64)
    a[0, 0, 0] = 256
    e1 = _exc_name(lambda: wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), 8)))
    e2 = _exc_name(lambda: oracle_lib.encode_image(a, 8))
    assert e1 == "DomainError" and "DomainError" in str(e2 and oracle_lib.STATUS_NAMES[3])
    b = np.zeros((2, 8, 8), dtype=np.int64)
    assert _exc_name(lambda: wbpc.encode_image(wbpc.RasterImage.from_planes(list(b), 8), use_rct=True)) == \
        "UnsupportedLayoutError"
    with pytest.raises(oracle_lib.OracleError) as ei:
        oracle_lib.encode_image(b, 8, use_rct=True)
    assert ei.value.name == "UnsupportedLayoutError"
    with pytest.raises(oracle_lib.OracleError) as ei:
        oracle_lib.encode_image(b, 8, levels=31)
    assert ei.value.name == "LevelRangeError"


def _oracle_exc(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return getattr(e, "name", type(e).__name__)
    return None


def test_corrupted_containers(oracle_lib, wbpc):
    """Bit flips / truncations / index edits: same exception class (or same output)."""
    rng = np.random.default_rng(7)
    a = rng.integers(0, 256, (3, 70, 90)).astype(np.int64)
    yy, xx = np.mgrid[0:70, 0:90]
    a[1] = (xx + yy) % 256
    data = oracle_lib.encode_image(a, 8, 2, True)
    mism = []
    for it in range(120):
        buf = bytearray(data)
        kind = it % 4
        if kind == 0:  # flip bits in the block payload region
            pos = int(rng.integers(19 + 12 * 30, len(buf)))
            buf[pos] ^= 1 << int(rng.integers(0, 8))
        elif kind == 1:  # truncate
            buf = buf[: int(rng.integers(0, len(buf)))]
        elif kind == 2:  # index entry edit
            e = int(rng.integers(0, 30))
            buf[19 + 12 * e + int(rng.integers(0, 12))] ^= 0xFF
        else:  # header byte edit
            buf[int(rng.integers(0, 19))] ^= 1 << int(rng.integers(0, 8))
        d = bytes(buf)
        for n in (0, 1):
            r = _exc_name(lambda: wbpc.decode_image(d, planes_dropped=n))
            o = _oracle_exc(lambda: oracle_lib.decode_image(d, planes_dropped=n))
            if r != o:
                mism.append((it, kind, n, r, o))
            if r is None and o is None:
                assert np.array_equal(wbpc.decode_image(d, planes_dropped=n).samples,
                                      oracle_lib.decode_image(d, planes_dropped=n)[0])
        r = _exc_name(lambda: wbpc.truncate_stream(d, 2))
        o = _oracle_exc(lambda: oracle_lib.truncate_stream(d, 2))
        if r != o:
            mism.append((it, kind, "trunc", r, o))
    assert not mism, mism[:5]


def test_int16_storage_bound_vs_reference(wbpc):
    """The filter-norm bound that enables int16 encode coefficients (capi.cu make_geom) holds
    on adversarial inputs (noise, random extremes, checkerboards) under the reference's own
    5/3 transform: |low| <= 1.5M + 2, |high| <= 2M + 1 per 1-D pass."""
    from wbpc import transforms as T

    def lo1(m):
        return (3 * m + 1) // 2 + 2

    def hi1(m):
        return 2 * m + 1

    rng = np.random.default_rng(11)
    for trial in range(36):
        bd = int(rng.choice([8, 9, 10]))
        rct = bool(trial % 2)
        C = 3 if rct else 1
        H, W = int(rng.integers(40, 200)), int(rng.integers(40, 200))
        mx = (1 << bd) - 1
        if trial % 3 == 0:
            img = rng.integers(0, mx + 1, (C, H, W))
        elif trial % 3 == 1:
            img = np.where(rng.random((C, H, W)) < 0.5, 0, mx)
        else:
            yy, xx = np.mgrid[0:H, 0:W]
            img = np.stack([((yy + xx + c) % 2) * mx for c in range(C)])
        img = img.astype(np.int64)
        planes = list(T.rct_forward(T.RasterImage.from_planes(list(img), bd))) if rct else list(img)
        for p in planes:
            pyr = T.dwt2d_forward(p, 4)
            m = mx
            for lv in range(4):
                bound_d = max(hi1(lo1(m)), lo1(hi1(m)), hi1(hi1(m)))
                assert max(int(np.abs(d).max()) for d in pyr.details[lv]) <= bound_d
                m = lo1(lo1(m))
            assert int(np.abs(pyr.ll).max()) <= m


def test_long_codes_vs_reference(oracle_lib, wbpc):
    """Blocks with Huffman codes longer than 16 bits: oracle bytes == reference bytes."""
    from wbpc import blocks as rb

    import inputs

    for seed in range(3):
        g = inputs.skewed_ll_block(seed)
        ref = rb.encode_block(rb.CoefficientBlock(width=128, height=128, kind="ll", depth=25, coeffs=(g,)))
        assert oracle_lib.encode_block("ll", [g]) == ref


def test_container_reader_surface_vs_reference(wbpc, golden_small):
    """slots / index / block_bytes of the repo's ContainerReader == the reference's (host side)."""
    import base64
    import paper_2005_08713_b200 as P
    from wbpc import container as rc
    n = 0
    for e in golden_small["images"]:
        if not e["container_b64"]:
            continue
        data = base64.b64decode(e["container_b64"])
        ours, ref = P.ContainerReader(data), rc.ContainerReader(data)
        assert ours.slots == ref.slots
        assert ours.index == ref.index
        assert all(ours.block_bytes(s) == ref.block_bytes(s) for s in ref.slots)
        n += 1
    assert n >= 5
    bad = bytearray(base64.b64decode(golden_small["images"][0]["container_b64"]))
    bad[19] ^= 0xFF  # first index offset
    assert _exc_name(lambda: P.ContainerReader(bytes(bad))) == _exc_name(lambda: rc.ContainerReader(bytes(bad)))


def test_png_writer_vs_reference(wbpc):
    from wbpc import png as rpng
    from paper_2005_08713_b200.tiles import encode_png
    rng = np.random.default_rng(8)
    for shape in ((1, 1), (7, 13), (64, 33, 3), (5, 1, 3), (0, 4)):
        px = rng.integers(0, 256, shape).astype(np.uint8)
        assert encode_png(px) == rpng.encode_png(px), shape
    for bad in (np.zeros((2, 2, 4), np.uint8), np.zeros(5, np.uint8)):
        assert _exc_name(lambda: encode_png(bad)) == _exc_name(lambda: rpng.encode_png(bad))


def test_pnm_vs_reference(wbpc):
    """read_pnm / write_pnm: same rasters, bytes and error classes as the reference."""
    from wbpc import pnm as rp
    from paper_2005_08713_b200 import pnm as op
    rng = np.random.default_rng(21)
    cases = [b"P5\n4 4\n255\n" + bytes(range(16)), b"P6 2 1 255 " + bytes(6), b"P5\n# c\n3 2\n# x\n65535\n" + bytes(12),
             b"P5\n4 4\n255\n" + bytes(10), b"P5\n4 4\n255", b"P7\n1 1\n1\n\0", b"P5\n0 4\n255\n", b"P5\n2 2\n70000\n" + bytes(8),
             b"P5\n2 2\n3\n\x00\x01\x02\x04", b"P5\n2 x\n3\n" + bytes(4), b"P5 1 1 1\r\x01", b"P5\n2 2\n1023\n" + bytes(8)]
    for bd in (1, 7, 8, 12, 16):
        for ch in (1, 3):
            a = rng.integers(0, 1 << bd, (ch, 5, 7))
            cases.append(rp.write_pnm(wbpc.RasterImage.from_planes(list(a), bd)))
    for d in cases:
        e_r = _exc_name(lambda: rp.read_pnm(d))
        e_o = _exc_name(lambda: op.read_pnm(d))
        assert e_r == e_o, (d[:20], e_r, e_o)
        if e_r is None:
            r, o = rp.read_pnm(d), op.read_pnm(d)
            assert (r.width, r.height, r.channels, r.bit_depth) == (o.width, o.height, o.channels, o.bit_depth)
            assert np.array_equal(r.samples, o.samples)
            assert op.write_pnm(o) == rp.write_pnm(r) == d or d.startswith(b"P5\n#") or d.startswith(b"P6 ") \
                or d.startswith(b"P5 ")
    import paper_2005_08713_b200 as P
    a = np.array([[[-3, 5, 300]]])
    for clamp in (False, True):
        e_r = _exc_name(lambda: rp.write_pnm(wbpc.RasterImage(3, 1, 1, 8, a.copy()), clamp=clamp))
        e_o = _exc_name(lambda: op.write_pnm(P.RasterImage(3, 1, 1, 8, a.copy()), clamp=clamp))
        assert e_r == e_o
        if e_r is None:
            assert rp.write_pnm(wbpc.RasterImage(3, 1, 1, 8, a.copy()), clamp=True) == \
                op.write_pnm(P.RasterImage(3, 1, 1, 8, a.copy()), clamp=True)

"""CPU-only: the C-ABI library loads and exports every declared symbol; host-side logic."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "wbpc_b200.h")).read()
    return sorted(set(re.findall(r"\b(wbpc_[a-z_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_2005_08713_b200 import _lib
    L = _lib.load()  # loads without a GPU (no CUDA call at load time)
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) <= set(declared)
    assert L.wbpc_abi_version() == 1


def test_library_is_sm100a():
    """The .so carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2005_08713_b200 import _lib
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_parse_and_errors():
    import paper_2005_08713_b200 as P
    h = P.ContainerHeader(300, 200, 3, 8, 1, 4)
    assert P.ContainerHeader.parse(h.pack()) == h
    with pytest.raises(P.ContainerParseError):
        P.ContainerHeader.parse(b"WBPC")
    with pytest.raises(P.ContainerParseError):
        P.ContainerHeader.parse(b"XBPC" + h.pack()[4:])
    bad = bytearray(h.pack())
    bad[13] = 5  # channels
    with pytest.raises(P.ContainerParseError):
        P.ContainerHeader.parse(bytes(bad))


def test_slot_count_matches_oracle(oracle_lib):
    import paper_2005_08713_b200 as P
    for w, h, c, L in ((512, 512, 1, 3), (2048, 2048, 3, 4), (4096, 4096, 3, 6), (8192, 8192, 4, 5), (1, 1, 1, 0),
                       (300, 17, 2, 6)):
        assert P.slot_count(P.ContainerHeader(w, h, c, 8, 0, L)) == oracle_lib.slot_count(w, h, c, L)
    assert oracle_lib.slot_count(2048, 2048, 3, 4) == 258
    assert oracle_lib.slot_count(4096, 4096, 3, 5) == 1026
    assert oracle_lib.slot_count(8192, 8192, 4, 5) == 5472


def test_index_validation_host(oracle_lib):
    import paper_2005_08713_b200 as P
    from paper_2005_08713_b200.container import _check_index
    a = np.arange(64 * 64).reshape(1, 64, 64) % 256
    data = oracle_lib.encode_image(a, 8, 2)
    h = P.ContainerHeader.parse(data)
    assert _check_index(data, h) == oracle_lib.slot_count(64, 64, 1, 2)
    with pytest.raises(P.ContainerParseError):
        _check_index(data[:25], h)
    bad = bytearray(data)
    bad[19] ^= 0xFF
    with pytest.raises(P.CorruptionError):
        _check_index(bytes(bad), h)


def test_raster_image_and_levels():
    import paper_2005_08713_b200 as P
    img = P.RasterImage.from_planes([np.zeros((3, 5))], 8)
    assert (img.width, img.height, img.channels) == (5, 3, 1)
    with pytest.raises(P.ShapeError):
        P.RasterImage(2, 2, 1, 8, np.zeros((1, 3, 2)))
    with pytest.raises(P.UnsupportedLayoutError):
        P.RasterImage.from_planes([np.zeros((2, 2))] * 5, 8)
    with pytest.raises(P.DomainError):
        P.RasterImage.from_planes([np.zeros((2, 2))], 17)
    with pytest.raises(P.DomainError):
        P.RasterImage.from_planes([np.full((2, 2), 256)], 8).validate_source()
    # default_levels (transforms.py:235-245), test_transforms.py:201-211
    assert P.default_levels(4096, 4096) == 5
    assert P.default_levels(512, 512) == 5
    assert P.default_levels(15, 400) == 0
    assert P.default_levels(16, 16) == 0
    assert P.default_levels(32, 64) == 1
    assert P.level_dims(13, 9, 1) == (7, 5)


def test_error_classes_mirror_reference():
    import paper_2005_08713_b200 as P
    from paper_2005_08713_b200 import _lib
    names = ["UnsupportedLayoutError", "ShapeError", "DomainError", "LevelRangeError", "DepthOverflowError",
             "StreamIndexError", "EmptyAlphabetError", "CodeLengthError", "MalformedTreeError", "TruncationError",
             "MalformedPayloadError", "BlockParseError", "CorruptionError", "ContainerParseError"]
    for i, n in enumerate(names, start=1):
        assert _lib.STATUS_TO_EXC[i] is getattr(P, n)
        assert issubclass(getattr(P, n), P.CodecError)
    assert issubclass(P.StreamIndexError, IndexError)
    with pytest.raises(P.CorruptionError):
        _lib.raise_status(13, message="x")


def test_product_never_imports_oracle():
    """The product package must not route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2005_08713_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "wbo_" not in src and "liboracle" not in src, f


def test_synth_determinism():
    from paper_2005_08713_b200 import synth
    a = synth.cfg1_gray12(3, 128)
    b = synth.cfg1_gray12(3, 128)
    assert a.dtype == np.uint16 and a.shape == (1, 128, 128) and np.array_equal(a, b) and a.max() <= 4095
    c = synth.cfg2_pathology(1, 64, 96)
    assert c.shape == (64, 96, 3) and c.dtype == np.uint8
    assert np.array_equal(c, synth.cfg2_pathology(1, 64, 96))


def test_chunk_count_formula():
    """ceil(L / (2^w - 1)) used by the coder (entropy.py:189) for L <= 2048, w in 2..16."""
    for w in range(2, 17):
        cap = (1 << w) - 1
        L = np.arange(1, 2049)
        assert np.array_equal((L + cap - 1) // cap, -(-L // cap))


def _cascade_rows(n, levels):
    """Dense rows of the linear 5/3 analysis cascade (transforms.py:107-133 without floors):
    per level, (lowpass rows, highpass rows) as matrices over the n input samples."""
    x = np.eye(n)
    out = []
    for _ in range(levels):
        m = x.shape[0]
        if m <= 1:
            out.append((x, np.zeros((0, n))))
            continue
        xe, xo = x[0::2], x[1::2]
        mh = xo.shape[0]
        right = np.concatenate([xe[1:mh], xe[mh - 1:mh]]) if m % 2 == 0 else xe[1:mh + 1]
        hi = xo - (xe[:mh] + right) / 2
        hl = np.concatenate([hi[:1], hi[:-1]] + ([hi[-1:]] if m % 2 else []))
        hr = np.concatenate([hi] + ([hi[-1:]] if m % 2 else []))
        lo = xe + (hl + hr) / 4
        out.append((lo, hi))
        x = lo
    return out


def _dense_coef_bytes(w, h, bd, levels):
    m = (1 << bd) - 1
    if m > 32767:
        return 4
    def norms(n):
        a, b = [1.0], [0.0]
        for lo, hi in _cascade_rows(n, levels):
            a.append(np.abs(lo).sum(1).max())
            b.append(np.abs(hi).sum(1).max() if hi.shape[0] else 0.0)
        return a, b
    aw, bw = norms(w)
    ah, bh = norms(h)
    e = 0.0
    for lv in range(1, levels + 1):
        nrm = max(aw[lv] * ah[lv], aw[lv] * bh[lv], bw[lv] * ah[lv], bw[lv] * bh[lv],
                  aw[lv] * ah[lv - 1], bw[lv] * ah[lv - 1], aw[lv - 1] * ah[lv], aw[lv - 1] * bh[lv])
        if nrm * m * (1 + 1e-9) + 2 * (2 * e + 1) + 1 + 1 > 32767:
            return 4
        e = 1.5 * (1.5 * e + 1) + 1
    return 2


def test_encode_coef_bytes_host():
    """wbpc_encode_coef_bytes (host geometry only, no device): int16 storage exactly when the
    filter-norm bound of the 5/3 lifting keeps every level inside +-2^15, and the plan-size
    argument errors of the encoder."""
    import ctypes

    from paper_2005_08713_b200 import _lib

    L = _lib.load()

    def cb(w, h, c, bd, levels, rct, dt=_lib.DTYPE_U8):
        d = _lib.ImageDesc(w, h, c, bd, dt, _lib.LAYOUT_HWC, w * h * c)
        out = ctypes.c_int()
        rc = L.wbpc_encode_coef_bytes(ctypes.byref(d), levels, int(rct), ctypes.byref(out))
        return rc, out.value

    assert cb(2048, 2048, 3, 8, 4, True) == (0, 2)        # cfg2
    assert cb(4096, 4096, 3, 8, 5, True) == (0, 2)        # cfg3
    assert cb(4096, 4096, 3, 8, 6, True) == (0, 2)        # cfg4 tiles (exact cascade norm bound)
    assert cb(8192, 8192, 4, 16, 5, False, _lib.DTYPE_U16) == (0, 4)  # cfg5: full 16-bit range
    assert cb(8192, 8192, 4, 16, 0, False, _lib.DTYPE_U16) == (0, 4)
    assert cb(512, 512, 1, 12, 3, False, _lib.DTYPE_U16) == (0, 2)    # cfg1
    assert cb(8192, 8192, 3, 8, 9, True) == (0, 2)
    assert cb(65536, 3, 3, 8, 30, True) == (0, 4)   # the floors' error bound grows 2.25x per level
    # the decision against an independent dense evaluation of the same bound
    for (w, h, bd, lv) in [(512, 512, 12, 4), (512, 512, 12, 3), (96, 40, 13, 2), (96, 40, 12, 2), (5, 300, 12, 3),
                           (1, 1, 15, 2), (77, 130, 11, 5), (64, 64, 14, 0), (33, 17, 16, 0)]:
        assert cb(w, h, 1, bd, lv, False, _lib.DTYPE_U16) == (0, _dense_coef_bytes(w, h, bd, lv)), (w, h, bd, lv)
    assert cb(64, 64, 2, 8, 2, True)[0] != 0               # colour transform needs 3 channels
    assert cb(64, 64, 3, 17, 2, False)[0] != 0             # bit depth 1..16


def test_host_conversions_threaded():
    """_host.convert / or_reduce (the drop-in API's sample conversions, split over threads) equal
    numpy's single-thread results, and RasterImage.validate_source keeps the reference's check."""
    import numpy as np
    from paper_2005_08713_b200 import _host
    from paper_2005_08713_b200.errors import DomainError
    from paper_2005_08713_b200.transforms import RasterImage
    rng = np.random.default_rng(4)
    for shape, lo, hi in (((3, 700, 900), 0, 256), ((1, 5, 7), 0, 4096), ((2, 1100, 1300), -40000, 70000)):
        a = rng.integers(lo, hi, shape).astype(np.int64)
        for dt in (np.uint8, np.uint16, np.int32):
            assert np.array_equal(_host.convert(a, dt), a.astype(dt))
        b = a.astype(np.int32)
        assert np.array_equal(_host.convert(b, np.int64), a)
        out = np.empty(shape, np.int64)
        assert _host.convert(b, np.int64, out=out) is out and np.array_equal(out, a)
        assert _host.or_reduce(a) == int(np.bitwise_or.reduce(a, axis=None))
    assert _host.or_reduce(np.empty((0,), np.int64)) == 0
    x = rng.integers(0, 256, (3, 800, 900)).astype(np.int64)
    RasterImage(900, 800, 3, 8, x).validate_source()
    for bad in (-1, 256):
        y = x.copy()
        y[1, 799, 899] = bad
        try:
            RasterImage(900, 800, 3, 8, y).validate_source()
            raise AssertionError("out-of-range sample accepted")
        except DomainError:
            pass

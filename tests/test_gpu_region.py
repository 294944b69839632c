"""decode_region / container_info on the CUDA path vs the reference's fixtures.

decode_region (container.py:338-390) decodes only the blocks whose tiles meet the per-level
boxes; the output equals cropping decode_image, and a corrupt block outside the boxes raises
nothing.  container_info (container.py:420-456) parses every block header on the device.
"""

import json

import numpy as np
import pytest
import torch

from helpers import sha, sha_samples

import inputs

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2005_08713_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_08713_b200 import _lib
    _lib.load()


def _images(golden_region):
    ins = {name: (a, bd, L, rct) for name, a, bd, L, rct in inputs.region_inputs()}
    for e in golden_region["images"]:
        a, bd, L, rct = ins[e["name"]]
        data = P.encode_image(P.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
        assert sha(data) == e["container_sha"], e["name"]
        yield e, a, data


def _outcome(fn):
    try:
        return sha_samples(fn().samples)
    except P.CodecError as ex:
        return type(ex).__name__
    except IndexError:
        return "IndexError"


def _norm(d):
    return json.loads(json.dumps(d))


def test_region_windows(golden_region):
    for e, a, data in _images(golden_region):
        for w in e["windows"]:
            x, y, ww, hh, lev, n = w["args"]
            got = P.decode_region(data, x, y, ww, hh, level=lev, planes_dropped=n).samples
            assert sha_samples(got) == w["sha"], (e["name"], w["args"])


def test_region_errors(golden_region):
    for e, a, data in _images(golden_region):
        for er in e["errors"]:
            x, y, ww, hh, lev, n = er["args"]
            assert _outcome(lambda: P.decode_region(data, x, y, ww, hh, level=lev, planes_dropped=n)) == \
                er["outcome"], (e["name"], er["args"])


def test_region_corruption(golden_region):
    for e, a, data in _images(golden_region):
        for c in e["corrupt"]:
            bad = bytearray(data)
            bad[c["pos"]] ^= c["xor"]
            x, y, ww, hh, lev, n = c["args"]
            got = _outcome(lambda: P.decode_region(bytes(bad), x, y, ww, hh, level=lev, planes_dropped=n))
            assert got == c["region"], (e["name"], c)


def test_container_info(golden_region):
    for e, a, data in _images(golden_region):
        assert _norm(P.container_info(data)) == e["info"], e["name"]
        for c in e["corrupt"]:
            bad = bytearray(data)
            bad[c["pos"]] ^= c["xor"]
            try:
                got = _norm(P.container_info(bytes(bad)))
            except P.CodecError as ex:
                got = type(ex).__name__
            assert got == c["info"], (e["name"], c["pos"])


def test_region_tensor_u8_hwc_matches_crop():
    """Device API with u8 HWC output: odd window offsets exercise the packed-store edges."""
    a = inputs.synth.cfg2_pathology(9, 384, 520)
    t = torch.from_numpy(a).cuda()
    buf, offs = P.encode_tensor(t, 8, 4, use_rct=True, layout="hwc")
    data = buf[offs[0]:offs[1]]
    h = P.ContainerHeader(520, 384, 3, 8, 1, 4)
    full = P.decode_tensor(data, h, out_dtype="uint8", layout="hwc")
    assert torch.equal(full, t)
    rng = np.random.default_rng(5)
    for _ in range(40):
        lev = int(rng.integers(0, 3))
        lw, lh = P.level_dims(520, 384, lev)
        ww, hh = int(rng.integers(1, lw + 1)), int(rng.integers(1, lh + 1))
        x, y = int(rng.integers(0, lw - ww + 1)), int(rng.integers(0, lh - hh + 1))
        ref = P.decode_tensor(data, h, level=lev, out_dtype="int32", layout="hwc")[y:y + hh, x:x + ww]
        for od in ("int32", "int16"):
            got = P.decode_region_tensor(data, x, y, ww, hh, lev, 0, h, out_dtype=od, layout="hwc")
            assert torch.equal(got.to(torch.int32), ref), (x, y, ww, hh, lev, od)
        if lev == 0:
            got = P.decode_region_tensor(data, x, y, ww, hh, 0, 0, h, out_dtype="uint8", layout="hwc")
            assert torch.equal(got, t[y:y + hh, x:x + ww])
        got = P.decode_region_tensor(data, x, y, ww, hh, lev, 1, h, out_dtype="int32", layout="chw")
        ref = P.decode_tensor(data, h, level=lev, planes_dropped=1, out_dtype="int32")[:, y:y + hh, x:x + ww]
        assert torch.equal(got, ref)


def test_region_large_image_matches_crop():
    """A container with more than 512 blocks: region decode through the large-batch kernels (the
    needed-block mask with the continuous plane lists) equals the crop of the full decode."""
    a = inputs.synth.cfg2_pathology(7, 3072, 4096)
    t = torch.from_numpy(a).cuda()
    buf, offs = P.encode_tensor(t, 8, 5, use_rct=True, layout="hwc")
    data = buf[offs[0]:offs[1]]
    h = P.ContainerHeader(4096, 3072, 3, 8, 1, 5)
    assert P.container.slot_count(h) >= 512
    rng = np.random.default_rng(11)
    full = {}
    for _ in range(24):
        lev, nd = int(rng.integers(0, 4)), int(rng.integers(0, 3))
        if (lev, nd) not in full:
            full[(lev, nd)] = P.decode_tensor(data, h, level=lev, planes_dropped=nd, out_dtype="int32", layout="chw")
        f = full[(lev, nd)]
        lh, lw = f.shape[1:]
        ww, hh = int(rng.integers(1, lw + 1)), int(rng.integers(1, lh + 1))
        x, y = int(rng.integers(0, lw - ww + 1)), int(rng.integers(0, lh - hh + 1))
        got = P.decode_region_tensor(data, x, y, ww, hh, lev, nd, h, out_dtype="int32", layout="chw")
        assert torch.equal(got, f[:, y:y + hh, x:x + ww]), (lev, nd, x, y, ww, hh)
    assert torch.equal(P.decode_tensor(data, h, out_dtype="uint8", layout="hwc"), t)

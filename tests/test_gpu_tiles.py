"""Tile rendering (service.py:52-100 PNM branch) on the device vs the reference's responses."""

import pytest
import torch

from helpers import sha

import inputs

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2005_08713_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_08713_b200 import _lib
    _lib.load()


def test_render_tile_vs_reference(golden_tiles):
    ins = {name: (a, bd, L, rct) for name, a, bd, L, rct in inputs.tile_inputs()}
    datas = {}
    for c in golden_tiles["cases"]:
        a, bd, L, rct = ins[c["name"]]
        if c["name"] not in datas:
            datas[c["name"]] = P.encode_image(P.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
            assert sha(datas[c["name"]]) == c["container_sha"]
        level, x, y, pd, size = c["args"]
        r = P.render_tile(datas[c["name"]], level, x, y, pd, size)
        assert r.status_code == c["status"], c
        if r.status_code == 200:
            assert r.media_type == c["media"], c
            assert sha(r.body) == c["body_sha"], c
            assert {k.lower(): v for k, v in r.headers.items()} == c["headers"], c


def test_render_tile_png_is_out_of_scope():
    a = inputs.tile_inputs()[2]
    data = P.encode_image(P.RasterImage.from_planes(list(a[1]), a[2]), levels=a[3])
    with pytest.raises(P.UnsupportedByDeviceError):
        P.render_tile(data, 0, 0, 0, accept="image/png")

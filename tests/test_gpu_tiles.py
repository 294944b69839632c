"""Tile rendering (service.py:52-100, PNM and PNG branches) on the device vs the reference's responses."""

import importlib
import os
import sys

import numpy as np
import pytest
import torch

from helpers import sha

import inputs

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2005_08713_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")  # pip --target install of the unmodified reference


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_08713_b200 import _lib
    _lib.load()


def _containers(golden_tiles):
    ins = {name: (a, bd, L, rct) for name, a, bd, L, rct in inputs.tile_inputs()}
    datas = {}
    for c in golden_tiles["cases"]:
        if c["name"] not in datas:
            a, bd, L, rct = ins[c["name"]]
            datas[c["name"]] = P.encode_image(P.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
            assert sha(datas[c["name"]]) == c["container_sha"]
    return datas


def _check(r, exp, case):
    assert r.status_code == exp["status"], case
    if r.status_code == 200:
        assert r.media_type == exp["media"], case
        assert sha(r.body) == exp["body_sha"], case
        # the fixture keeps the service's own headers (a starlette Response adds content-*)
        got = {k.lower(): v for k, v in r.headers.items() if k.lower() in ("etag", "x-sample-scale")}
        assert got == exp["headers"], case


def test_render_tile_vs_reference(golden_tiles):
    datas = _containers(golden_tiles)
    readers = {k: P.ContainerReader(v) for k, v in datas.items()}
    for c in golden_tiles["cases"]:
        level, x, y, pd, size = c["args"]
        _check(P.render_tile(datas[c["name"]], level, x, y, pd, size), c, c)
        # PNG branch under a browser-style Accept header, through a shared reader
        _check(P.tiles._render_tile(readers[c["name"]], level, x, y, pd, size,
                                    "text/html,image/png;q=0.9,*/*;q=0.8"), c["png"], c)


def test_reference_service_flow_on_repo_reader(golden_tiles):
    """The reference's own service._render_tile, run with this repo's ContainerReader and
    decode_region bound in its namespace, returns the reference's responses byte for byte."""
    if not os.path.isdir(os.path.join(REF_INSTALL, "wbpc")):
        pytest.skip("baseline/_ref (reference install) not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if REF_INSTALL not in sys.path:
        sys.path.append(REF_INSTALL)
    try:
        service = importlib.import_module("wbpc.service")
    except ImportError as e:  # fastapi / numba missing on this host
        pytest.skip(f"reference service not importable: {e}")
    datas = _containers(golden_tiles)
    orig = service.decode_region
    service.decode_region = P.decode_region
    try:
        for c in golden_tiles["cases"]:
            level, x, y, pd, size = c["args"]
            reader = P.ContainerReader(datas[c["name"]])
            _check(service._render_tile(reader, level, x, y, pd, size, ""), c, c)
            _check(service._render_tile(reader, level, x, y, pd, size, "image/png"), c["png"], c)
    finally:
        service.decode_region = orig


def test_container_reader_decode_slot(oracle_lib):
    a = inputs.synth.planar(inputs.synth.cfg2_pathology(5, 300, 260)).astype(np.int64)
    data = oracle_lib.encode_image(a, 8, 2, True)
    rd = P.ContainerReader(data)
    assert len(rd.slots) == len(rd.index) == P.slot_count(rd.header)
    for n in (0, 1, 3):
        blocks = rd.decode_slots(rd.slots, n)
        for slot, blk in zip(rd.slots, blocks):
            bb = rd.block_bytes(slot)
            dim = 128
            keep = None if n == 0 else max((bb[0] >> 2) - n, 0)
            ref = oracle_lib.decode_block(bb, dim, "ll" if slot[0] == "ll" else "hp", keep)
            assert blk.kind == slot[0] and blk.depth == bb[0] >> 2
            assert np.array_equal(np.stack(blk.coeffs), ref), (slot, n)
        one = rd.decode_slot(rd.slots[-1], n)
        assert all(np.array_equal(u, v) for u, v in zip(one.coeffs, blocks[-1].coeffs))

"""Pins the oracle's decode_region (oracle/wbpc_oracle.c decode_core) to the reference.

Fixtures: tests/golden/golden_region.json (make_golden.py --region, from the unmodified
reference's decode_region, container.py:338-390): seeded windows at every level and
planes_dropped, the argument-error classes, and single-byte block corruptions (only blocks
inside the per-level boxes may raise).
"""

import numpy as np
import pytest

from helpers import sha, sha_samples

import inputs


def _images(golden_region):
    ins = {name: (a, bd, L, rct) for name, a, bd, L, rct in inputs.region_inputs()}
    for e in golden_region["images"]:
        yield e, ins[e["name"]]


def _outcome(fn):
    import oracle
    try:
        return sha_samples(fn()[0])
    except oracle.OracleError as ex:
        return ex.name


def test_region_windows(oracle_lib, golden_region):
    for e, (a, bd, L, rct) in _images(golden_region):
        data = oracle_lib.encode_image(a, bd, L, rct)
        assert sha(data) == e["container_sha"], e["name"]
        for w in e["windows"]:
            x, y, ww, hh, lev, n = w["args"]
            d, _ = oracle_lib.decode_region(data, x, y, ww, hh, lev, n)
            assert sha_samples(d) == w["sha"], (e["name"], w["args"])
            # the reference's documented identity: region == crop of decode_image
            full, _ = oracle_lib.decode_image(data, level=lev, planes_dropped=n)
            assert np.array_equal(full[:, y:y + hh, x:x + ww], d)


def test_region_errors_and_corruption(oracle_lib, golden_region):
    for e, (a, bd, L, rct) in _images(golden_region):
        data = oracle_lib.encode_image(a, bd, L, rct)
        for er in e["errors"]:
            x, y, ww, hh, lev, n = er["args"]
            got = _outcome(lambda: oracle_lib.decode_region(data, x, y, ww, hh, lev, n))
            assert got == er["outcome"], (e["name"], er["args"])
        for c in e["corrupt"]:
            bad = bytearray(data)
            bad[c["pos"]] ^= c["xor"]
            x, y, ww, hh, lev, n = c["args"]
            got = _outcome(lambda: oracle_lib.decode_region(bytes(bad), x, y, ww, hh, lev, n))
            assert got == c["region"], (e["name"], c)


def _render_oracle(oracle_lib, data, level, x, y, pd, size, hdr):
    """service._render_tile's PNM branch composed from the oracle's decode_region."""
    import hashlib
    C, W, H, bd, L = hdr
    if not 0 <= level <= L:
        return 404, None, {}, None
    lw, lh = W, H
    for _ in range(level):
        lw, lh = (lw + 1) // 2, (lh + 1) // 2
    x0, y0 = x * size, y * size
    if x < 0 or y < 0 or x0 >= lw or y0 >= lh:
        return 404, None, {}, None
    w, h = min(size, lw - x0), min(size, lh - y0)
    s, _ = oracle_lib.decode_region(data, x0, y0, w, h, level, pd)
    maxval = (1 << bd) - 1
    s = np.clip(s, 0, maxval)
    headers = {}
    if bd > 8:
        s = (s * 255 + maxval // 2) // maxval
        headers["x-sample-scale"] = f"255/{maxval}"
    if C not in (1, 3):
        return 400, None, {}, None
    pix = np.moveaxis(s.astype(np.uint8), 0, 2)
    body = (b"P5\n%d %d\n255\n" % (w, h) + pix[:, :, 0].tobytes()) if C == 1 else \
        (b"P6\n%d %d\n255\n" % (w, h) + pix.tobytes())
    headers["etag"] = '"' + hashlib.sha256(body).hexdigest() + '"'
    return 200, ("image/x-portable-graymap" if C == 1 else "image/x-portable-pixmap"), headers, sha(body)


def test_tile_render_composition(oracle_lib, golden_tiles):
    ins = {name: (a, bd, L, rct) for name, a, bd, L, rct in inputs.tile_inputs()}
    datas = {}
    for c in golden_tiles["cases"]:
        a, bd, L, rct = ins[c["name"]]
        if c["name"] not in datas:
            datas[c["name"]] = oracle_lib.encode_image(a, bd, L, rct)
            assert sha(datas[c["name"]]) == c["container_sha"]
        level, x, y, pd, size = c["args"]
        st, media, headers, body_sha = _render_oracle(oracle_lib, datas[c["name"]], level, x, y, pd, size,
                                                      (a.shape[0], a.shape[2], a.shape[1], bd, L))
        assert st == c["status"], c
        if st == 200:
            assert media == c["media"] and body_sha == c["body_sha"] and headers == c["headers"], c

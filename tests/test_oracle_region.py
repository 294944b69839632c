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

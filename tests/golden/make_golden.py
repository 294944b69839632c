"""Generate the golden fixtures by running the UNMODIFIED reference package.

Run here (the reference is only mounted in the build container):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Writes tests/golden/golden_small.json (known answers + full container bytes of small
images) and, with --big, tests/golden/golden_configs.json (sha256 digests of the
reference's containers / decoded samples / truncated streams for the BASELINE configs,
on the seeded generators of paper_2005_08713_b200/synth.py).  The reference
(`wbpc`) is the oracle of record; oracle/wbpc_oracle.c is checked against these files.
"""

from __future__ import annotations

import base64
import hashlib
import json
import os
import sys
import time

import numpy as np

import wbpc  # the reference, from PYTHONPATH
from wbpc import blocks as ref_blocks
from wbpc import container as ref_container
from wbpc import entropy as ref_entropy

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
import inputs  # noqa: E402
synth = inputs.synth


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def sha_samples(a: np.ndarray) -> str:
    return sha(np.ascontiguousarray(a, dtype="<i8").tobytes())


def b64(b: bytes) -> str:
    return base64.b64encode(b).decode()


def known_answers() -> dict:
    ka = {}
    z = np.zeros((128, 128), dtype=np.int64)
    ka["block_zero_ll"] = ref_blocks.encode_block(wbpc.CoefficientBlock.build("ll", [z])).hex()
    ka["block_zero_hp3"] = ref_blocks.encode_block(wbpc.CoefficientBlock.build("hp3", [z, z, z])).hex()
    ka["block_minus1_ll"] = ref_blocks.encode_block(wbpc.CoefficientBlock.build("ll", [z - 1])).hex()
    ka["optimize_counter_width_5_300_1000_zr3"] = int(ref_entropy.optimize_counter_width([5, 300, 1000], 3))
    hc = ref_entropy.build_huffman({0: 5, 1: 2, 2: 1})
    ka["huffman_0_5_1_2_2_1"] = {
        "lengths": [int(hc.code_lengths[s]) for s in range(3)],
        "values": [int(hc.code_values[s]) for s in range(3)],
        "tree_bits": "".join(str(int(b)) for b in ref_entropy.serialize_tree(hc)),
    }
    # random alphabets: tree bits + code lengths of build_huffman (tie-breaking pins)
    rng = np.random.default_rng(99)
    hs = []
    for i in range(60):
        n = int(rng.integers(1, 257))
        freq = np.zeros(256, dtype=np.int64)
        syms = rng.choice(256, n, replace=False)
        if i % 3 == 0:
            freq[syms] = rng.integers(1, 4, n)  # many ties
        elif i % 3 == 1:
            freq[syms] = rng.integers(1, 100000, n)
        else:
            freq[syms] = (2 ** rng.integers(0, 16, n)).astype(np.int64)
        hc = ref_entropy.build_huffman(freq)
        hs.append({"freq": freq.tolist(), "lengths": hc.code_lengths.astype(int).tolist(),
                   "values": hc.code_values.astype(np.int64).tolist(),
                   "tree_bits": "".join(str(int(b)) for b in ref_entropy.serialize_tree(hc))})
    ka["huffman_random"] = hs
    cws = []
    for i in range(40):
        runs = rng.integers(2, 2049, int(rng.integers(0, 300)))
        zb = int(rng.integers(0, 20))
        cws.append({"runs": runs.tolist(), "zr_bits": zb, "w": int(ref_entropy.optimize_counter_width(runs, zb))})
    ka["counter_width_random"] = cws
    return ka


def block_cases() -> list:
    """encode_block / decode_block / truncate_block on single 128x128 blocks."""
    cases = []
    for i, (kind, grids) in enumerate(inputs.block_grids()):
        blk = ref_blocks.encode_block(wbpc.CoefficientBlock.build(kind, grids))
        trunc = {str(n): sha(ref_blocks.truncate_block(blk, 128, 128, kind, n)) for n in (1, 2, 3, 7)}
        dec = {}
        for keep in (None, 0, 1, 3):
            b = ref_blocks.decode_block(blk, 128, 128, kind, planes_to_keep=keep)
            dec[str(keep)] = sha_samples(np.stack(b.coeffs))
        cases.append({"index": i, "kind": kind, "block_sha": sha(blk), "block_len": len(blk),
                      "block_b64": b64(blk) if len(blk) < 4096 else None, "truncated": trunc, "decoded": dec})
    return cases


def main_small() -> None:
    res = {"reference": "wbpc " + wbpc.__version__, "known_answers": known_answers(), "images": [],
           "blocks": block_cases()}
    for name, a, bd, L, rct in inputs.small_inputs():
        img = wbpc.RasterImage.from_planes(list(a), bd)
        data = wbpc.encode_image(img, levels=L, use_rct=rct)
        entry = {"name": name, "bit_depth": bd, "levels": L, "use_rct": rct, "shape": list(a.shape),
                 "samples_sha": sha_samples(a), "container_sha": sha(data), "container_len": len(data),
                 "container_b64": b64(data) if len(data) <= 8192 else None,
                 "decoded": {}, "truncated": {}}
        for lev in range(0, L + 1):
            for n in (0, 1, 3):
                d = wbpc.decode_image(data, level=lev, planes_dropped=n).samples
                entry["decoded"][f"{lev}/{n}"] = sha_samples(d)
        for n in (1, 2, 4):
            entry["truncated"][str(n)] = sha(wbpc.truncate_stream(data, n))
        res["images"].append(entry)
        print(name, len(data), flush=True)
    with open(os.path.join(HERE, "golden_small.json"), "w") as f:
        json.dump(res, f, indent=1)


def finest_only_truncate(data: bytes, n: int) -> bytes:
    """Reference composition for BASELINE cfg3 wording: truncate_block(., n) on level-1 HP3
    slots only (SURVEY.md §8(d) cfg3 semantics note)."""
    reader = ref_container.ContainerReader(data)
    dim = reader.header.block_dim
    blobs = []
    for slot in reader.slots:
        blob = reader.block_bytes(slot)
        if slot[0] == "hp3" and slot[2] == 1:
            blob = ref_blocks.truncate_block(blob, dim, dim, "hp3", n)
        blobs.append(blob)
    index = bytearray()
    off = ref_container._HEADER.size + ref_container._INDEX_ENTRY.size * len(blobs)
    for b in blobs:
        index += ref_container._INDEX_ENTRY.pack(off, len(b))
        off += len(b)
    return reader.header.pack() + bytes(index) + b"".join(blobs)


def main_big(which: list[int]) -> None:
    path = os.path.join(HERE, "golden_configs.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    res["reference"] = "wbpc " + wbpc.__version__
    if 1 in which:
        a = synth.cfg1_gray12(0).astype(np.int64)
        t = time.time()
        data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), 12), levels=3)
        te = time.time() - t
        e = {"seed": 0, "container_sha": sha(data), "container_len": len(data), "ref_encode_s": te, "decoded": {},
             "truncated": {}}
        for n in (0, 2):
            e["decoded"][f"0/{n}"] = sha_samples(wbpc.decode_image(data, planes_dropped=n).samples)
        e["decoded"]["2/0"] = sha_samples(wbpc.decode_image(data, level=2).samples)
        e["truncated"]["2"] = sha(wbpc.truncate_stream(data, 2))
        res["cfg1"] = e
        print("cfg1", e, flush=True)
    if 2 in which:
        a = synth.planar(synth.cfg2_pathology(0)).astype(np.int64)
        t = time.time()
        data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), 8), levels=4, use_rct=True)
        te = time.time() - t
        t = time.time()
        d = wbpc.decode_image(data).samples
        td = time.time() - t
        e = {"seed": 0, "container_sha": sha(data), "container_len": len(data), "lossless": bool(np.array_equal(d, a)),
             "ref_encode_s": te, "ref_decode_s": td,
             "truncated": {"2": sha(wbpc.truncate_stream(data, 2))},
             "decoded": {"1/0": sha_samples(wbpc.decode_image(data, level=1).samples)}}
        res["cfg2"] = e
        print("cfg2", e, flush=True)
    if 3 in which:
        a = synth.planar(synth.cfg2_pathology(0, 4096, 4096)).astype(np.int64)
        t = time.time()
        data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), 8), levels=5, use_rct=True)
        te = time.time() - t
        e = {"seed": 0, "container_sha": sha(data), "container_len": len(data), "ref_encode_s": te,
             "global": {}, "finest": {}}
        for n in (2, 4):
            t = time.time()
            tr = wbpc.truncate_stream(data, n)
            tt = time.time() - t
            t = time.time()
            d = wbpc.decode_image(data, planes_dropped=n).samples
            td = time.time() - t
            e["global"][str(n)] = {"truncated_sha": sha(tr), "truncated_len": len(tr), "decoded_sha": sha_samples(d),
                                   "psnr": synth.psnr(d, a, 255.0), "ref_truncate_s": tt, "ref_decode_s": td}
            fo = finest_only_truncate(data, n)
            dfo = wbpc.decode_image(fo).samples
            e["finest"][str(n)] = {"truncated_sha": sha(fo), "truncated_len": len(fo), "decoded_sha": sha_samples(dfo),
                                   "psnr": synth.psnr(dfo, a, 255.0)}
        res["cfg3"] = e
        print("cfg3", e, flush=True)
    if 4 in which:
        tiles = {}
        for ti in (0, 255, 77, 160):
            a = synth.planar(synth.cfg4_tile(0, ti)).astype(np.int64)
            t = time.time()
            data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), 8), levels=6, use_rct=True)
            tiles[str(ti)] = {"container_sha": sha(data), "container_len": len(data), "ref_encode_s": time.time() - t}
            print("cfg4 tile", ti, tiles[str(ti)], flush=True)
        res["cfg4"] = {"seed": 0, "tiles": tiles}
    if 5 in which:
        a = synth.cfg5_fluorescence(0).astype(np.int64)
        t = time.time()
        data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), 16), levels=5)
        te = time.time() - t
        t = time.time()
        d = wbpc.decode_image(data).samples
        td = time.time() - t
        res["cfg5"] = {"seed": 0, "container_sha": sha(data), "container_len": len(data), "ref_encode_s": te,
                       "ref_decode_s": td, "lossless": bool(np.array_equal(d, a))}
        print("cfg5", res["cfg5"], flush=True)
    with open(path, "w") as f:
        json.dump(res, f, indent=1)


def main_region() -> None:
    """decode_region windows, container_info and single-byte corruptions (container.py:338-456)."""
    res = {"reference": "wbpc " + wbpc.__version__, "images": []}
    for name, a, bd, L, rct in inputs.region_inputs():
        data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
        C, H, W = a.shape
        e = {"name": name, "container_sha": sha(data), "info": ref_container.container_info(data), "windows": [],
             "errors": [], "corrupt": []}
        for (x, y, w, h, lev, n) in inputs.region_windows(name, W, H, L):
            d = wbpc.decode_region(data, x, y, w, h, level=lev, planes_dropped=n).samples
            e["windows"].append({"args": [x, y, w, h, lev, n], "sha": sha_samples(d)})
        for args in ([0, 0, 1, 1, L + 1, 0], [0, 0, 1, 1, -1, 0], [0, 0, 1, 1, 0, -1], [0, 0, 0, 1, 0, 0],
                     [0, 0, 1, 0, 0, 0], [-1, 0, 1, 1, 0, 0], [0, -1, 1, 1, 0, 0], [W, 0, 1, 1, 0, 0],
                     [0, 0, W + 1, 1, 0, 0], [0, H, 1, 1, 0, 0], [1, 1, W, H, 0, 0]):
            try:
                wbpc.decode_region(data, *args[:4], level=args[4], planes_dropped=args[5])
                e["errors"].append({"args": args, "outcome": "ok"})
            except Exception as ex:  # noqa: BLE001
                e["errors"].append({"args": args, "outcome": type(ex).__name__})
        # single-byte corruption of one block; outcome of decode_region on a seeded window
        reader = ref_container.ContainerReader(data)
        rng = np.random.default_rng(len(name) * 7919)
        wins = inputs.region_windows(name, W, H, L, 24)
        for t in range(24):
            si = int(rng.integers(0, len(reader.slots)))
            off, ln = reader.index[reader.slots[si]]
            pos = off + int(rng.integers(0, ln))
            xor = int(rng.integers(1, 256))
            bad = bytearray(data)
            bad[pos] ^= xor
            x, y, w, h, lev, n = wins[t]
            out = {"pos": pos, "xor": xor, "args": [x, y, w, h, lev, n]}
            try:
                out["region"] = sha_samples(wbpc.decode_region(bytes(bad), x, y, w, h, level=lev,
                                                               planes_dropped=n).samples)
            except Exception as ex:  # noqa: BLE001
                out["region"] = type(ex).__name__
            try:
                out["info"] = ref_container.container_info(bytes(bad))
            except Exception as ex:  # noqa: BLE001
                out["info"] = type(ex).__name__
            e["corrupt"].append(out)
        res["images"].append(e)
        print(name, len(data), flush=True)
    with open(os.path.join(HERE, "golden_region.json"), "w") as f:
        json.dump(res, f, indent=1)


def main_tiles() -> None:
    """The tile service's _render_tile (service.py:52-100), PNM and PNG branches: status, media, headers, body."""
    from wbpc import service as ref_service
    res = {"reference": "wbpc " + wbpc.__version__, "cases": []}
    rng = np.random.default_rng(77)
    for name, a, bd, L, rct in inputs.tile_inputs():
        data = wbpc.encode_image(wbpc.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
        reader = ref_container.ContainerReader(data)
        C, H, W = a.shape
        for t in range(10):
            size = int(rng.choice([32, 64, 100, 256]))
            level = int(rng.integers(0, L + 2)) if t else L + 1
            lw, lh = W, H
            for _ in range(max(0, min(level, L))):
                lw, lh = (lw + 1) // 2, (lh + 1) // 2
            x = int(rng.integers(0, max(1, -(-lw // size)) + (1 if t % 4 == 3 else 0)))
            y = int(rng.integers(0, max(1, -(-lh // size))))
            pd = int(rng.choice([0, 0, 1, 3]))
            r = ref_service._render_tile(reader, level, x, y, pd, size, "")
            case = {"name": name, "container_sha": sha(data), "args": [level, x, y, pd, size],
                    "status": r.status_code, "media": r.media_type,
                    "headers": {k: v for k, v in r.headers.items() if k.lower() in ("etag", "x-sample-scale")},
                    "body_sha": sha(bytes(r.body)), "body_len": len(r.body)}
            # PNG branch (service.py:82-93, png.py:22-46) under a browser-style Accept header
            p = ref_service._render_tile(reader, level, x, y, pd, size, "text/html,image/png;q=0.9,*/*;q=0.8")
            case["png"] = {"status": p.status_code, "media": p.media_type,
                           "headers": {k: v for k, v in p.headers.items() if k.lower() in ("etag", "x-sample-scale")},
                           "body_sha": sha(bytes(p.body)), "body_len": len(p.body)}
            res["cases"].append(case)
        print(name, flush=True)
    with open(os.path.join(HERE, "golden_tiles.json"), "w") as f:
        json.dump(res, f, indent=1)


def main_plane_offsets() -> None:
    """plane_offsets (blocks.py:253-261) of the single-block cases."""
    res = {"reference": "wbpc " + wbpc.__version__, "cases": []}
    for i, (kind, grids) in enumerate(inputs.block_grids()):
        blk = ref_blocks.encode_block(wbpc.CoefficientBlock.build(kind, grids))
        po = ref_blocks.plane_offsets(blk, 128, 128, kind)
        res["cases"].append({"index": i, "kind": kind, "block_sha": sha(blk),
                             "offsets": [[int(s), int(b), int(o)] for (s, b), o in po]})
    with open(os.path.join(HERE, "golden_plane_offsets.json"), "w") as f:
        json.dump(res, f)


if __name__ == "__main__":
    if "--plane-offsets" in sys.argv:
        main_plane_offsets()
    elif "--tiles" in sys.argv:
        main_tiles()
    elif "--region" in sys.argv:
        main_region()
    elif "--big" in sys.argv:
        which = [int(x) for x in sys.argv[sys.argv.index("--big") + 1:]] or [1, 2, 3, 4, 5]
        main_big(which)
    else:
        main_small()

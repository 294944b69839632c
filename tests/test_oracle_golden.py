"""Pins the CPU oracle (oracle/wbpc_oracle.c) to the reference's own outputs.

Every digest / byte string here was produced by the unmodified reference package
(tests/golden/make_golden.py).  Known answers also restate the reference test-suite's pins
(pkg/tests/test_transforms.py, test_bitplanes.py) and SPEC.md examples.
"""

import numpy as np
import pytest

from helpers import b64d, sha, sha_samples

import inputs


def test_known_answer_blocks(oracle_lib, golden_small):
    ka = golden_small["known_answers"]
    z = np.zeros((128, 128), dtype=np.int64)
    assert oracle_lib.encode_block("ll", [z]).hex() == ka["block_zero_ll"] == "0440000000"
    assert oracle_lib.encode_block("hp3", [z, z, z]).hex() == ka["block_zero_hp3"]
    assert oracle_lib.encode_block("ll", [z - 1]).hex() == ka["block_minus1_ll"] == "08401ffc000800000000"


def test_known_answer_counter_width(oracle_lib, golden_small):
    ka = golden_small["known_answers"]
    assert oracle_lib.optimize_counter_width([5, 300, 1000], 3) == ka["optimize_counter_width_5_300_1000_zr3"] == 10
    for case in ka["counter_width_random"]:
        assert oracle_lib.optimize_counter_width(case["runs"], case["zr_bits"]) == case["w"]


def test_known_answer_huffman(oracle_lib, golden_small):
    ka = golden_small["known_answers"]["huffman_0_5_1_2_2_1"]
    h = oracle_lib.huffman([5, 2, 1])
    assert h["code_lengths"][:3].tolist() == ka["lengths"] == [1, 2, 2]
    assert h["code_values"][:3].tolist() == ka["values"]
    assert "".join(map(str, h["tree_bits"])) == ka["tree_bits"]


def test_huffman_random_alphabets(oracle_lib, golden_small):
    """Tie-breaking pins: (frequency, min symbol) merge order, first popped = left."""
    for case in golden_small["known_answers"]["huffman_random"]:
        h = oracle_lib.huffman(case["freq"])
        assert h["code_lengths"].tolist() == case["lengths"]
        assert h["code_values"].astype(np.int64).tolist() == case["values"]
        assert "".join(map(str, h["tree_bits"])) == case["tree_bits"]


def test_lifting_known_values(oracle_lib):
    # test_transforms.py:99-111: [0,1,2,3] -> low [0,2], high [0,1]; constant annihilation
    p = oracle_lib.dwt2d_forward_packed(np.array([[0, 1, 2, 3]]), 1)
    # 1x4 plane, level 1: LH (cw=2, fh=0) empty, HL (fw=2, ch=1) = high, HH empty, LL = low
    assert p.tolist() == [0, 1, 0, 2]
    c = oracle_lib.dwt2d_forward_packed(np.full((8, 8), 37), 1)
    assert (c[:48] == 0).all() and (c[48:] == 37).all()


def test_dwt_round_trip_shapes(oracle_lib):
    rng = np.random.default_rng(5)
    for h, w in ((1, 1), (1, 7), (13, 9), (16, 16), (31, 2)):
        for L in (0, 1, 3, 5):
            x = rng.integers(-70000, 70000, (h, w))
            p = oracle_lib.dwt2d_forward_packed(x, L)
            assert np.array_equal(oracle_lib.dwt2d_inverse_packed(p, w, h, L), x)


def test_block_cases(oracle_lib, golden_small):
    grids = inputs.block_grids()
    for case in golden_small["blocks"]:
        kind, g = grids[case["index"]]
        blk = oracle_lib.encode_block(kind, g)
        assert sha(blk) == case["block_sha"] and len(blk) == case["block_len"]
        for n, digest in case["truncated"].items():
            assert sha(oracle_lib.truncate_block(blk, 128, kind, int(n))) == digest
        for keep, digest in case["decoded"].items():
            k = None if keep == "None" else int(keep)
            assert sha_samples(oracle_lib.decode_block(blk, 128, kind, k)) == digest


@pytest.mark.parametrize("idx", range(24))
def test_small_images(oracle_lib, golden_small, idx):
    allin = inputs.small_inputs()
    if idx >= len(allin):
        pytest.skip("no such input")
    name, a, bd, L, rct = allin[idx]
    entry = next(e for e in golden_small["images"] if e["name"] == name)
    assert sha_samples(a) == entry["samples_sha"]
    data = oracle_lib.encode_image(a, bd, L, rct)
    assert sha(data) == entry["container_sha"]
    if entry["container_b64"]:
        assert data == b64d(entry["container_b64"])
    for key, digest in entry["decoded"].items():
        lev, n = map(int, key.split("/"))
        d, _ = oracle_lib.decode_image(data, level=lev, planes_dropped=n)
        assert sha_samples(d) == digest, key
    for n, digest in entry["truncated"].items():
        assert sha(oracle_lib.truncate_stream(data, int(n))) == digest


def test_cfg1_full(oracle_lib, golden_configs):
    import paper_2005_08713_b200.synth as synth
    g = golden_configs["cfg1"]
    a = synth.cfg1_gray12(0).astype(np.int64)
    data = oracle_lib.encode_image(a, 12, 3, False)
    assert sha(data) == g["container_sha"] and len(data) == g["container_len"]
    for key, digest in g["decoded"].items():
        lev, n = map(int, key.split("/"))
        assert sha_samples(oracle_lib.decode_image(data, level=lev, planes_dropped=n)[0]) == digest
    assert sha(oracle_lib.truncate_stream(data, 2)) == g["truncated"]["2"]


def test_cfg2_full(oracle_lib, golden_configs):
    import paper_2005_08713_b200.synth as synth
    g = golden_configs["cfg2"]
    a = synth.planar(synth.cfg2_pathology(0)).astype(np.int64)
    data = oracle_lib.encode_image(a, 8, 4, True, threads=8)
    assert sha(data) == g["container_sha"]
    d, _ = oracle_lib.decode_image(data, threads=8)
    assert np.array_equal(d, a)
    assert sha(oracle_lib.truncate_stream(data, 2)) == g["truncated"]["2"]
    assert sha_samples(oracle_lib.decode_image(data, level=1, threads=8)[0]) == g["decoded"]["1/0"]


def test_long_codes_exercised(oracle_lib):
    """The skewed blocks really carry codes longer than the device's 16-bit decode table."""
    for seed in range(3):
        g = inputs.skewed_ll_block(seed)
        s, d = oracle_lib.serialize_block("ll", [g])
        assert d == 25
        lengths = oracle_lib.huffman(np.bincount(s, minlength=256))["code_lengths"]
        assert int(lengths.max()) > 16
        back = oracle_lib.decode_block(oracle_lib.encode_block("ll", [g]), 128, "ll")
        assert np.array_equal(back[0], g)

"""Deterministic inputs shared by make_golden.py (run with the reference) and the tests.

Pure numpy + the repo's synthetic generators; no dependency on the reference, so the
tests can rebuild every input from here and compare with the committed digests.
"""

from __future__ import annotations

import importlib.util
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
_spec = importlib.util.spec_from_file_location("_wbpc_synth", os.path.join(REPO, "paper_2005_08713_b200", "synth.py"))
synth = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synth)


def small_inputs():
    """Deterministic small images: (name, samples (C,H,W) int64, bit_depth, levels, use_rct)."""
    rng = np.random.default_rng(20240811)  # the reference conftest seed (conftest.py:52-54)
    out = []
    out.append(("ramp4x4", (np.arange(16).reshape(1, 4, 4) * 17).astype(np.int64), 8, 1, False))
    shapes = [((1, 1, 1), 8, 0, False), ((1, 1, 7), 8, 3, False), ((1, 13, 9), 16, 3, False),
              ((1, 16, 16), 8, 5, False), ((1, 31, 2), 12, 1, False), ((3, 33, 65), 8, 2, True),
              ((3, 130, 257), 8, 3, True), ((4, 64, 64), 16, 5, False), ((2, 129, 1), 16, 4, False),
              ((1, 256, 256), 1, 2, False), ((3, 200, 300), 9, 4, True), ((1, 129, 131), 12, 2, False),
              ((1, 2, 2), 8, 3, False), ((3, 128, 128), 8, 0, True), ((1, 300, 17), 16, 6, False)]
    for (c, h, w), bd, L, rct in shapes:
        a = rng.integers(0, 1 << bd, (c, h, w)).astype(np.int64)
        out.append((f"rand_{c}x{h}x{w}_b{bd}_L{L}{'_rct' if rct else ''}", a, bd, L, rct))
    # smooth content (real zero runs / skewed histograms)
    yy, xx = np.mgrid[0:160, 0:192]
    sm = np.stack([(xx + 2 * yy + 5 * k) * 255 // (192 + 320) for k in range(3)]).astype(np.int64)
    sm = np.clip(sm + rng.integers(-1, 2, sm.shape), 0, 255)
    out.append(("smooth_3x160x192_rct_L3", sm, 8, 3, True))
    out.append(("const_1x64x64_L2", np.full((1, 64, 64), 4095, dtype=np.int64), 12, 2, False))
    out.append(("zeros_1x40x40_L2", np.zeros((1, 40, 40), dtype=np.int64), 8, 2, False))
    c1 = synth.cfg1_gray12(7, 256).astype(np.int64)
    out.append(("cfg1like_256_seed7_L3", c1, 12, 3, False))
    c2 = synth.planar(synth.cfg2_pathology(5, 256, 384)).astype(np.int64)
    out.append(("cfg2like_256x384_seed5_L4", c2, 8, 4, True))
    return out



def region_inputs():
    """Images for the decode_region / container_info fixtures: (name, samples, bd, L, rct)."""
    out = [x for x in small_inputs() if x[0] in ("rand_3x130x257_b8_L3_rct", "rand_1x300x17_b16_L6",
                                                 "smooth_3x160x192_rct_L3", "rand_4x64x64_b16_L5",
                                                 "cfg1like_256_seed7_L3", "cfg2like_256x384_seed5_L4")]
    c2 = synth.planar(synth.cfg2_pathology(3, 600, 776)).astype(np.int64)
    out.append(("cfg2like_600x776_seed3_L4", c2, 8, 4, True))
    c1 = synth.cfg1_gray12(11, 520)[:, :, :392].astype(np.int64)
    out.append(("cfg1like_520x392_seed11_L5", np.ascontiguousarray(c1), 12, 5, False))
    return out


def tile_inputs():
    """Images for the tile-service fixtures: gray 12/16-bit (scaled), RGB8 (RCT), 2 and 4 channels."""
    rng = np.random.default_rng(5150)
    out = [x for x in region_inputs() if x[0] in ("cfg2like_600x776_seed3_L4", "cfg1like_520x392_seed11_L5")]
    out.append(("gray16_300x333_L3", rng.integers(0, 1 << 16, (1, 300, 333)).astype(np.int64), 16, 3, False))
    out.append(("gray6_130x200_L2", rng.integers(0, 1 << 6, (1, 130, 200)).astype(np.int64), 6, 2, False))
    out.append(("two_ch_100x90_L2", rng.integers(0, 256, (2, 100, 90)).astype(np.int64), 8, 2, False))
    out.append(("rgba10_96x160_L3", rng.integers(0, 1024, (4, 96, 160)).astype(np.int64), 10, 3, False))
    return out


def region_windows(name: str, w: int, h: int, L: int, n: int = 14):
    """Seeded (x, y, width, height, level, planes_dropped) windows inside the level dims."""
    rng = np.random.default_rng(sum(map(ord, name)))
    out = []
    for i in range(n):
        lev = int(rng.integers(0, L + 1))
        lw, lh = w, h
        for _ in range(lev):
            lw, lh = (lw + 1) // 2, (lh + 1) // 2
        ww = int(rng.integers(1, lw + 1)) if i % 3 else int(rng.integers(1, min(lw, 9) + 1))
        hh = int(rng.integers(1, lh + 1)) if i % 3 else int(rng.integers(1, min(lh, 9) + 1))
        x = int(rng.integers(0, lw - ww + 1))
        y = int(rng.integers(0, lh - hh + 1))
        out.append((x, y, ww, hh, lev, int(rng.choice([0, 0, 1, 3]))))
    return out


def block_grids():
    """(kind, grids) for the single-block cases: Laplacian coefficients at 6 scales, half zeroed."""
    rng = np.random.default_rng(4242)
    out = []
    for i in range(12):
        kind = "ll" if i % 3 == 0 else "hp3"
        nsub = 1 if kind == "ll" else 3
        scale = [1, 3, 40, 300, 5000, 70000][i % 6]
        grids = []
        for _ in range(nsub):
            g = np.round(rng.laplace(0, scale, (128, 128))).astype(np.int64)
            g[rng.random((128, 128)) < 0.5] = 0
            grids.append(g)
        out.append((kind, grids))
    return out


def _ll_block_from_symbols(sym: np.ndarray) -> np.ndarray:
    """LL magnitudes whose magnitude-plane symbols are sym[plane][area] (bitplanes.py:31 area
    weights; area a = (row a // 32, col a % 32)); non-negative, so the sign plane is all zero."""
    planes = sym.shape[0]
    a = np.arange(2048)
    r, c = a // 32, a % 32
    mag = np.zeros((128, 128), np.int64)
    for b in range(planes):
        for i in range(2):
            for j in range(4):  # area bit 4i + j = coefficient (2r + i, 4c + j)
                mag[2 * r + i, 4 * c + j] |= ((sym[b] >> (4 * i + j)) & 1) << (planes - 1 - b)
    return mag


def deep_table_ll_block(seed: int):
    """LL block whose Huffman tree has ~120 internal nodes at depth 11: 250 symbols seen once
    hang as a balanced subtree under a 4-symbol spine of doubling frequencies (250, 500, 1000,
    rest), so their codes are 11-12 bits and the decoder's second-level subtables run out
    (the first-level entries past the subtable capacity fall back to a tree walk that starts at
    depth 11).  Two magnitude planes, every symbol non-zero (no zero runs)."""
    rng = np.random.default_rng(seed)
    rare = rng.permutation(np.arange(1, 256))[:254]
    vals = np.concatenate([rare[:250], np.full(250, rare[250]), np.full(500, rare[251]),
                           np.full(1000, rare[252]), np.full(4096 - 2000, rare[253])]).astype(np.int64)
    rng.shuffle(vals)
    return _ll_block_from_symbols(vals.reshape(2, 2048))


def skewed_ll_block(seed: int, depth: int = 25, nsym: int = 22):
    """LL block whose magnitude-plane symbols have Fibonacci frequencies (1, 1, 2, 3, 5, ...).

    The Huffman tree of such a block is maximally skewed, so its rarest symbols get codes of
    17-19 bits: longer than the decoder's 16-bit two-level table (the tree-walk path).  Symbols
    are placed at random areas/planes; coefficients are non-negative (all-zero sign plane).
    """
    rng = np.random.default_rng(seed)
    fib = [1, 1]
    while len(fib) < nsym:
        fib.append(fib[-1] + fib[-2])
    slots = (depth - 1) * 2048
    vals = np.concatenate([np.full(f, s + 1, np.int64) for s, f in enumerate(fib)])
    vals = np.concatenate([vals, np.full(slots - vals.size, 255, np.int64)])
    rng.shuffle(vals)
    sym = vals.reshape(depth - 1, 2048)  # [magnitude plane][area]; area a = (row a // 32, col a % 32)
    a = np.arange(2048)
    r, c = a // 32, a % 32
    mag = np.zeros((128, 128), np.int64)
    for b in range(depth - 1):
        for i in range(2):
            for j in range(4):  # area bit 4i + j = coefficient (2r + i, 4c + j) (bitplanes.py:31)
                mag[2 * r + i, 4 * c + j] |= ((sym[b] >> (4 * i + j)) & 1) << (depth - 2 - b)
    return mag

"""Adversarial coefficient blocks that reach rarely used encoder branches.

`large_slot_block` builds an HP3 128x128 block whose bit planes are designed area by area
(4x2 area symbol bit (r&1)*4 + (c&3) = magnitude bit of pixel (r, c), bitplanes.py:31,112-122):
every magnitude plane of every subband holds one constant non-zero symbol, except one plane whose
2048 symbols are drawn from the symbols no constant plane uses.  Those are rare in the block
histogram, get long Huffman codes (entropy.py:194-248), and that one slot's payload exceeds the
emit kernel's single-window capacity (24,576 bits), which takes the multi-window branch.
"""

import numpy as np

DIM = 128
EMIT_WINDOW_BITS = (768 - 2) * 32 - 64  # encode.cu CAPW: slots above this take the windowed path


def _plane_bits(sym_area: np.ndarray) -> np.ndarray:
    """(64, 32) area symbols -> (128, 128) bit plane."""
    r = np.arange(DIM)[:, None]
    c = np.arange(DIM)[None, :]
    s = sym_area[r >> 1, c >> 2].astype(np.int64)
    return (s >> ((r & 1) * 4 + (c & 3))) & 1


def large_slot_block(seed: int = 0, depth: int = 21, random_plane: int = 7, random_sub: int = 1,
                     negative: bool = False):
    """Returns (grids (3,128,128) int64, depth, (64,32) area symbols of the random slot)."""
    rng = np.random.default_rng(seed)
    nsub = 3
    nplanes = depth - 1  # magnitude planes b = 1..depth-1
    consts = rng.permutation(np.arange(1, 256))
    used = consts[: nplanes * nsub]
    unused = np.setdiff1d(np.arange(1, 256), used)
    mags = np.zeros((nsub, DIM, DIM), dtype=np.int64)
    k = 0
    rand_syms = None
    for b in range(1, depth):
        for s in range(nsub):
            if (b, s) == (random_plane, random_sub):
                area = rng.choice(unused, size=(64, 32))
                rand_syms = area
            else:
                area = np.full((64, 32), used[k])
            k += 1
            mags[s] |= _plane_bits(area) << (depth - 1 - b)
    # plane b=1 must hold a set bit somewhere so depth = 1 + bit_length(max) (bitplanes.py:77-79)
    assert int(mags.max()).bit_length() == depth - 1
    grids = -mags if negative else mags
    return grids, depth, rand_syms


def slot_payload_bits(oracle, grids, rand_syms) -> int:
    """Payload bits of the random slot, from the oracle's Huffman code of the block's symbols."""
    sym, depth = oracle.serialize_block("hp", list(grids))
    hist = np.bincount(sym, minlength=256).astype(np.int64)
    hist[0] = 0  # zeros only in unstored (sign) slots here
    code = oracle.huffman(hist)
    return int(code["code_lengths"][rand_syms.ravel()].sum())

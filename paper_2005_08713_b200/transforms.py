"""Host-side image container and geometry helpers (no pixel arithmetic happens here).

Mirrors the reference's public types and helpers (pkg/src/wbpc/transforms.py):
``RasterImage`` (:24-62), ``SubbandPyramid`` (:65-76), ``level_dims`` (:227-232) and
``default_levels`` (:235-245).  The colour transform and the wavelet themselves run on the
GPU inside encode/decode (paper_2005_08713_b200/csrc/dwt.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._host import or_reduce
from .errors import DomainError, ShapeError, UnsupportedLayoutError

MAX_LEVELS = 30


@dataclass
class RasterImage:
    """Integer sample grid, channel planar: samples has shape (channels, h, w) (transforms.py:24-46)."""

    width: int
    height: int
    channels: int
    bit_depth: int
    samples: np.ndarray

    def __post_init__(self) -> None:
        self.samples = np.asarray(self.samples, dtype=np.int64)
        if self.samples.shape != (self.channels, self.height, self.width):
            raise ShapeError(
                f"samples shape {self.samples.shape} != ({self.channels}, {self.height}, {self.width})"
            )
        if not (1 <= self.channels <= 4):
            raise UnsupportedLayoutError(f"channels must be 1..4, got {self.channels}")
        if not (1 <= self.bit_depth <= 16):
            raise DomainError(f"bit depth must be 1..16, got {self.bit_depth}")
        if self.width < 1 or self.height < 1:
            raise DomainError("image dimensions must be >= 1")

    @classmethod
    def from_planes(cls, planes, bit_depth: int) -> "RasterImage":
        stack = np.stack([np.asarray(p, dtype=np.int64) for p in planes])
        c, h, w = stack.shape
        return cls(width=w, height=h, channels=c, bit_depth=bit_depth, samples=stack)

    def plane(self, channel: int) -> np.ndarray:
        return self.samples[channel]

    def validate_source(self) -> None:
        """Encode-input invariant: unsigned samples below 2^bit_depth (transforms.py:57-62)."""
        # one pass: the OR of all samples is in [0, 2^bd) iff every sample is (a negative sample
        # sets the sign bit, a large one a bit at or above bd)
        if self.samples.size and not 0 <= or_reduce(self.samples) < (1 << self.bit_depth):
            raise DomainError(f"samples out of range for bit depth {self.bit_depth}")


@dataclass
class SubbandPyramid:
    """details[k] = (lh, hl, hh) of level k+1 plus the final LL (transforms.py:65-76)."""

    levels: int
    ll: np.ndarray
    details: list


def level_dims(width: int, height: int, level: int) -> tuple[int, int]:
    """Dims of the LL band after `level` splits (iterated ceil halving)."""
    return ((width + (1 << level) - 1) >> level, (height + (1 << level) - 1) >> level)


def default_levels(width: int, height: int) -> int:
    """5 for images larger than 512 px, else the largest L keeping LL >= 16x16 (transforms.py:235-245)."""
    if max(width, height) > 512:
        return 5
    levels = 0
    while levels < MAX_LEVELS:
        w, h = level_dims(width, height, levels + 1)
        if w < 16 or h < 16:
            break
        levels += 1
    return levels

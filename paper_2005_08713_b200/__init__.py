"""B200-native (sm_100a) encode/decode hot path of the arXiv 2005.08713 wavelet bit-plane codec.

Drop-in for the reference package's codec API (pkg/src/wbpc/__init__.py:10-59, hot-path
subset): encode_image / decode_image / truncate_stream / RasterImage / ContainerHeader and the
wbpc.errors classes, plus a device API (encode_tensor / decode_tensor / truncate_tensor) for
callers holding CUDA tensors.  All pixel and bitstream work runs in hand-written CUDA kernels
(csrc/) behind the C ABI of include/wbpc_b200.h; there is no CPU fallback.
"""

from .blocks import (
    KIND_HP3,
    KIND_LL,
    CoefficientBlock,
    decode_block,
    decode_blocks,
    encode_block,
    encode_blocks,
    plane_offsets,
    truncate_block,
)
from .container import (
    BLOCK_DIM,
    Codec,
    CodecGroup,
    ContainerHeader,
    ContainerReader,
    HostPipeline,
    iter_slots,
    container_info,
    decode_image,
    decode_region,
    decode_region_tensor,
    decode_tensor,
    encode_image,
    encode_tensor,
    slot_count,
    truncate_stream,
    truncate_tensor,
)
from .benchmark import BenchReport, BenchRow, run_bench
from .errors import *  # noqa: F401,F403
from .pnm import read_pnm, read_pnm_file, write_pnm, write_pnm_file
from .slide import SlideCodec
from .tiles import TileResponse, encode_png, render_tile
from .transforms import RasterImage, SubbandPyramid, default_levels, level_dims

__version__ = "0.1.0"

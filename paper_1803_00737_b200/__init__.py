"""wavefuse-b200: B200-native (sm_100a) drop-in for the DWT pan-sharpening hot
path of the reference `wavefuse` package (arXiv 1803.00737).

Same public names and signatures as the reference's hot-path subset
(/root/reference/pkg/src/wavefuse/__init__.py:18-51): transforms, DWT fusion,
bilinear resampling and the quality metrics. Compute runs only in the in-tree
sm_100a library `libwavefuse_b200.so` (C ABI: include/wavefuse_b200.h); there
is no CPU fallback.
"""

from .errors import (
    BandCountMismatch,
    ChannelOutOfRange,
    CudaError,
    DimensionMismatch,
    FusionError,
    MalformedHeader,
    MissingTile,
    NotDivisible,
    OddDimension,
    OddLength,
    OddTile,
    TooFewBands,
    TooShort,
    TooSmall,
    Truncated,
    UnsupportedFormat,
    ZeroBandMean,
)
from .fusion import (
    DwtReplace,
    FusionMethod,
    set_exact_default,
    fuse,
    fuse_dwt,
    fuse_quantized,
    fuse_tile_quantized,
    method_from_name,
    quantize,
    resample_bilinear,
)
from .metrics import (PendingReport, QualityReport, d_lambda, d_s, degrade, ergas, fuse_and_qnr,
                      q_index, qnr, qnr_async)
from .pnm import PnmRaster, fuse_pnm, read_pnm, to_plane, write_pnm
from .tiling import (Tile, TileGrid, fuse_tiled, merge, pad_edge, pad_inputs, padded_dims,
                     plan_grid, split)
from .wavelet import (
    FilterBank,
    WaveletKind,
    d4_filters,
    dwt1d_forward,
    dwt1d_inverse,
    dwt2d_forward,
    dwt2d_inverse,
)

__version__ = "0.1.0"

__all__ = [
    "BandCountMismatch",
    "ChannelOutOfRange",
    "CudaError",
    "DimensionMismatch",
    "DwtReplace",
    "FilterBank",
    "FusionError",
    "FusionMethod",
    "MalformedHeader",
    "MissingTile",
    "NotDivisible",
    "OddDimension",
    "OddLength",
    "OddTile",
    "PnmRaster",
    "QualityReport",
    "Tile",
    "TileGrid",
    "TooFewBands",
    "TooShort",
    "TooSmall",
    "Truncated",
    "UnsupportedFormat",
    "WaveletKind",
    "ZeroBandMean",
    "__version__",
    "d4_filters",
    "d_lambda",
    "d_s",
    "degrade",
    "dwt1d_forward",
    "dwt1d_inverse",
    "dwt2d_forward",
    "dwt2d_inverse",
    "ergas",
    "fuse",
    "fuse_and_qnr",
    "fuse_dwt",
    "fuse_pnm",
    "fuse_quantized",
    "fuse_tile_quantized",
    "fuse_tiled",
    "merge",
    "method_from_name",
    "pad_edge",
    "pad_inputs",
    "padded_dims",
    "plan_grid",
    "q_index",
    "qnr",
    "qnr_async",
    "set_exact_default",
    "split",
    "PendingReport",
    "quantize",
    "read_pnm",
    "resample_bilinear",
    "to_plane",
    "write_pnm",
]

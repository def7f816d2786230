"""B200-native HHFFBPA / BPA hot path (arXiv 2506.23568), drop-in for the
reference package ``hhsar``'s reconstruct entry points.

    from paper_2506_23568_b200 import bpa_reconstruct, hhffbpa_reconstruct, FfbpParams

Same signatures, provenance and exceptions as hhsar.bpa_reconstruct
(bpa.py:144) and hhsar.hhffbpa_reconstruct (ffbp.py:415); the compute runs in
hand-written sm_100a CUDA kernels (libhhsar_b200.so, C ABI in
include/hhsar_b200.h) on device-resident complex64 data.  There is no CPU
fallback.
"""

from .bpa import (ImageVolume, backproject, backproject_gather, bpa_reconstruct,
                  check_delay_window, region_grid)
from .errors import (ConfigError, HhsarError, IoFormatError, NativeUnavailableError,
                     NumericDomainError)
from .ffbp import (GRID_PAD, FfbpParams, Subimage, SubimageGrid, build_subimage_grid,
                   default_levels, hhffbpa_reconstruct, hhffbpa_reconstruct_stream,
                   level1_reconstruct, merge_pair)
from .model import (C_LIGHT, DataCube, FrequencyGrid, ImagingRegion, Subarray,
                    SubarrayTree, SyntheticAperture, partition_subarrays, validate_geometry)
from .metrics import (PSNR_SENTINEL_DB, PsfReport, max_intensity_projection, profile_cut,
                      psf_metrics, psnr)
from .rangecomp import RangeProfileSet, range_compress
from .spectrum import SubarrayExtents, default_grid_dims

__version__ = "0.1.0"

__all__ = [
    "C_LIGHT", "ConfigError", "DataCube", "FfbpParams", "FrequencyGrid", "GRID_PAD",
    "HhsarError", "ImageVolume", "ImagingRegion", "IoFormatError", "NativeUnavailableError",
    "NumericDomainError", "PSNR_SENTINEL_DB", "PsfReport", "RangeProfileSet", "Subarray", "SubarrayExtents", "SubarrayTree",
    "Subimage", "SubimageGrid", "SyntheticAperture", "backproject", "backproject_gather",
    "bpa_reconstruct", "build_subimage_grid", "check_delay_window", "default_grid_dims",
    "default_levels", "hhffbpa_reconstruct", "hhffbpa_reconstruct_stream", "level1_reconstruct", "max_intensity_projection",
    "merge_pair", "partition_subarrays", "profile_cut", "psf_metrics", "psnr", "range_compress",
    "region_grid", "validate_geometry",
]

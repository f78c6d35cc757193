"""B200-native depth completion (Ku et al., arXiv 1802.00036) -- drop-in for the
reference package ``depthfill``'s hot path.

Public API (mirrors the reference):
  complete, complete_with_stats, PipelineConfig, BlurMode, FillMode, RunStats,
  STAGE_NAMES, DepthMap, DepthEncoding, KernelShape, Kernel, make_kernel,
  kernel_offsets, EncodingError, DepthRangeError, DegenerateInputError
BASELINE-named entry points:
  fill_in_fast, fill_in_multiscale
Batched device API:
  complete_batch (torch CUDA [B,H,W] float32)
Multi-GPU (frame-sharded, no collective):
  MultiDevicePipeline; ``python -m paper_1802_00036_b200.multi`` under torchrun
Plug-in backend for the reference registry:
  paper_1802_00036_b200.cuda_backend
"""

from .api import DIAMOND_KERNEL_5, fill_in_fast, fill_in_multiscale
from .completion import (STAGE_NAMES, BlurMode, FillMode, MultiscaleConfig, PipelineConfig, RunStats, complete,
                         complete_batch, complete_with_stats)
from .multi import MultiDevicePipeline
from .domain import (INVERSION_OFFSET, VALIDITY_THRESHOLD, DegenerateInputError, DepthEncoding, DepthMap,
                     DepthRangeError, EncodingError, Kernel, KernelShape, ValidityMask, density, kernel_offsets,
                     make_kernel, new_depth_map, validity_mask)

__all__ = [
    "fill_in_fast", "fill_in_multiscale", "DIAMOND_KERNEL_5", "complete", "complete_with_stats",
    "complete_batch", "PipelineConfig", "MultiscaleConfig", "BlurMode", "FillMode", "RunStats", "STAGE_NAMES",
    "DepthMap", "DepthEncoding", "ValidityMask", "KernelShape", "Kernel", "make_kernel", "kernel_offsets",
    "EncodingError", "DepthRangeError", "DegenerateInputError", "VALIDITY_THRESHOLD", "INVERSION_OFFSET",
    "new_depth_map", "validity_mask", "density", "MultiDevicePipeline",
]

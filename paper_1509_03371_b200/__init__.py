"""paper_1509_03371_b200 -- B200-native (sm_100a) SK-net forward labeling, a drop-in for the
hot path of the pixelseg reference (arXiv 1509.03371): conv_sk_forward and friends,
NetRunner::forward and process(), bit-identical to the reference's CPU results.

The compute lives in libgraft_cuda.so (CUDA kernels + C++ host driver behind the C ABI of
include/graft_cuda.h); these modules are the Python mirror of the reference's C++ API.
"""
from .errors import Error, IoError, NumericError, SizeError, SpecError
from .blob import Blob, ColumnBuffer, ConvGeometry, LayerState, Plane
from .netspec import (InitKind, LayerKind, LayerSpec, NetSpec, compute_channels, flop_estimate,
                      load_netspec, output_extent, parse_netspec, parse_netspec_or_throw,
                      propagate_sizes)
from .layers import (conv_sk_forward, gemm, gemm_flops, im2col_sk, maxpool_sk_forward,
                     mergecrop_forward, relu_forward, softmax_forward, upconv_forward)
from .netgraph import NetRunner, NetStates, SolverConfig, init_weights, sgd_step
from .pipeline import (ProcessResult, Processor, band_rows, mirror_pad, normalize_image, process,
                       tile_rows)
from .rng import Rng
from . import malis
from .malis import (AffinityGraph, MalisResult, affinity_backward, affinity_forward, connected_components,
                    malis_gradient, malis_softmax_loss)

__all__ = [
    "Error", "IoError", "NumericError", "SizeError", "SpecError", "Blob", "ColumnBuffer",
    "ConvGeometry", "LayerState", "Plane", "InitKind", "LayerKind", "LayerSpec", "NetSpec",
    "compute_channels", "flop_estimate", "load_netspec", "output_extent", "parse_netspec",
    "parse_netspec_or_throw", "propagate_sizes", "conv_sk_forward", "gemm", "gemm_flops",
    "im2col_sk", "maxpool_sk_forward", "mergecrop_forward", "relu_forward", "softmax_forward",
    "upconv_forward", "NetRunner", "NetStates", "SolverConfig", "init_weights", "sgd_step", "ProcessResult", "Processor",
    "band_rows", "mirror_pad", "normalize_image", "process", "tile_rows", "Rng", "malis",
    "AffinityGraph", "MalisResult", "affinity_backward", "affinity_forward", "connected_components",
    "malis_gradient", "malis_softmax_loss",
]

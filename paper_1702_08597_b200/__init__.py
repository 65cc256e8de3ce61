"""B200-native Winograd layer of arXiv 1702.08597 (forward + backward, sparse CSR / dense W_F).

Hot path: hand-written sm_100a kernels behind the C-ABI in include/wino_cuda.h
(built into libwino_b200.so next to this file).  Python here is the host mirror of
the reference's interfaces:
    WinogradLayer / ForwardCache   -- layer.hpp:19-43, sparse.hpp:78-82 (batched, device-resident)
    compress / reconstruct / PointwiseCsr -- sparse.hpp:19-49
    gen_transforms, lift, conv_winograd, conv_winograd_grad, sparse_conv, density
                                   -- python/bindings.cpp:55-204
    autograd.WinogradConv2d        -- the same layer as a differentiable torch module
    io, infer_bench                -- WGT1 / checkpoints, the infer-bench CSV driver
"""
from ._lib import (CapabilityError, ConsistencyError, CorruptFormatError, CudaError, InvalidArgument,
                   ShapeError, WinoError)
from .api import conv_winograd, conv_winograd_grad, density, gen_transforms, lift, sparse_conv
from .layer import (ForwardCache, PointwiseCsr, WinogradLayer, compress, make_geometry,
                    reconstruct, transforms)

__all__ = [
    "CapabilityError", "ConsistencyError", "CorruptFormatError", "CudaError", "InvalidArgument", "ShapeError",
    "WinoError", "conv_winograd", "conv_winograd_grad", "density", "gen_transforms", "lift",
    "sparse_conv", "ForwardCache", "PointwiseCsr", "WinogradLayer", "compress", "make_geometry",
    "reconstruct", "transforms",
]

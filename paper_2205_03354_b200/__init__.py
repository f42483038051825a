"""B200-native (sm_100a) hot path of the stencil-composition method (arXiv 2205.03354).

Host-side exact composition (`stencil`) + a C-ABI CUDA library
(`libsk_cuda.so`, include/sk_cuda.h) for the data-parallel work: matrix-free
composed apply, fused explicit Cahn-Hilliard stepping, GPU CSR assembly,
SpMV / BLAS-1 and device CG. No CPU fallback: importing the device modules
requires the built library.
"""
from .errors import Errc, StencilkitError  # noqa: F401
from .stencil import (Stencil, StencilSpec, add, bilaplacian, builtin_stencil, compose, laplacian, make,  # noqa: F401
                      outer_product, scale, shift, to_double, weight_sum)

__all__ = [
    "Errc", "StencilkitError", "Stencil", "StencilSpec", "add", "bilaplacian", "builtin_stencil", "compose",
    "laplacian", "make", "outer_product", "scale", "shift", "to_double", "weight_sum",
]

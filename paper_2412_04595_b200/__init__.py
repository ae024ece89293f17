"""B200-native spectral sum-of-Gaussians (SOG) electrostatics for quasi-2D systems
(arXiv 2412.04595): near field + mid-range spectral solver + long-range Fourier-Chebyshev
solver, hand-written sm_100a CUDA behind the C ABI in include/sog.h.

The Python layer only marshals arguments (ctypes); every step of the evaluation runs in
libsog.so.  There is no CPU fallback: importing works without a GPU (plan creation and
describe need none), but evaluation fails loudly without CUDA.
"""
from .sog import DistPlan, Plan, SogError, choose_params, lib_path, load_library, redistribute, slab_owner  # noqa: F401

__all__ = ["DistPlan", "Plan", "SogError", "choose_params", "lib_path", "load_library", "redistribute", "slab_owner"]

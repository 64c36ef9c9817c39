"""B200-native OpTorch data-flow path (arXiv 2105.00619): multi-image
encode / decode and selective batch sampling as sm_100a kernels behind the
C ABI in include/optb_cuda.h.

Submodules mirror the reference's C++ namespaces:
  codec    -> optb::codec   (include/optb/codec.hpp)
  sampler  -> optb::sampler (include/optb/sampler.hpp)
  nn       -> the decode layer of optb::nn (nn.hpp:38-42, nn.cpp:153-192)
  errors   -> include/optb/errors.hpp
Importing the package loads liboptb_cuda.so and fails if it was not built.
"""
from . import _lib  # noqa: F401  (loads the CUDA library or raises)
from . import codec, errors, nn, sampler  # noqa: F401

__all__ = ["codec", "sampler", "nn", "errors"]

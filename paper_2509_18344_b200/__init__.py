"""B200-native SubSpec hot path (arXiv 2509.18344): one lossless tree-speculative decode step.

The method lives in libsubspec.so (CUDA kernels for sm_100a + a C++ engine) behind the C-ABI in
include/subspec.h; `binding.SubSpec` is a thin ctypes wrapper.  See DESIGN.md.
"""
from .build import LIB, build  # noqa: F401


def SubSpec(*a, **kw):
    from .binding import SubSpec as _S
    return _S(*a, **kw)

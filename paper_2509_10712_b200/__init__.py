"""B200-native MinatoLoader preprocessing hot path.

`lfgpu` binds the in-tree CUDA library (liblfgpu.so, include/lfgpu.h);
`loadflow` headers under include/loadflow/ are the reference-shaped C++ API.
"""
from . import lfgpu  # noqa: F401  (raises ImportError if the CUDA library is missing)

__all__ = ["lfgpu"]

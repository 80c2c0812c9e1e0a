"""B200-native FastH (arXiv 2009.13977): blocked Householder products, forward
and backward, the SVD-reparameterised layer and its Sigma-ops, behind the
reference's API (see include/fasth_b200.h for the C ABI and
include/fasth_b200.hpp for the C++ mirror).

The compute is lib/libfasth_b200.so (sm_100a CUDA kernels); importing
``paper_2009_13977_b200.fasth`` loads it and fails loudly if it is absent.
"""
from . import _lib  # noqa: F401

__all__ = ["fasth"]

"""B200-native deep-BSDE training hot path of arXiv:1910.11623.

The product is ``libbsde.so`` (CUDA C++ for sm_100a behind the C-ABI of
``include/bsde.h``); this package is its thin ctypes binding plus the
multilevel host schedule.  Importing it never falls back to a CPU path.
"""
from ._lib import BSDEError, LIB_PATH  # noqa: F401
from .solver import BSDE, nccl_unique_id, step_size  # noqa: F401

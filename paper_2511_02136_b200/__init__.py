"""B200-native batched limit-order-book environment (JaxMARL-HFT hot path).

The product is the CUDA library built from csrc/ (libmlob.so) behind the C ABI
in include/mlob.h; this package is the Python host mirror of the reference's
env API (see env.py).  Importing the package does not load the library; the
first call that needs it does, and fails loudly if it is missing.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]

"""B200-native (sm_100a) CUDASOM hot path (arXiv 1905.09598).

The product is libsom.so (C ABI in include/som.h); ``som`` is its thin
Python binding.  No oracle code is imported here and there is no CPU
fallback.
"""
from . import som
from .som import SOM, SomError

__all__ = ["som", "SOM", "SomError"]

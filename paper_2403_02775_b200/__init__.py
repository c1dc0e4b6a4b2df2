"""B200-native EasyQuant engine (arXiv 2403.02775 hot path).

The product is the CUDA library behind include/ezquant_c.h (and the C++
drop-in include/ezquant/*.hpp). This package exposes it to Python through
ctypes (native.py); it holds no compute of its own and never falls back to
the CPU.
"""
from . import native  # noqa: F401
from .native import (Config, QuantizedWeight, EzqError, InvalidArgument,  # noqa: F401
                     InvariantError, IoError)

__all__ = ["native", "Config", "QuantizedWeight", "EzqError", "InvalidArgument",
           "InvariantError", "IoError"]

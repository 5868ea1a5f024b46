"""B200-native (sm_100a) DOUBLE decode loop — arXiv 2601.05524's retrieval-speculative-parallel
decoding behind the reference's specpar API.  See DESIGN.md.

The compute lives in libdouble_b200.so (CUDA + C++ host orchestrator, C-ABI in include/double_b200.h);
this package is the Python mirror of the reference interface used by tests and bench.py.
"""
from .specpar import *  # noqa: F401,F403
from .specpar import __all__ as _specpar_all
from .models import PRESETS, transformer_config  # noqa: F401
from . import harness  # noqa: F401  (config files -> setup -> methods, harness.cpp)

__all__ = list(_specpar_all) + ["PRESETS", "transformer_config", "harness"]

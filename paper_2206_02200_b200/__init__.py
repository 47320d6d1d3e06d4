"""B200-native GridShift engine (arXiv 2206.02200 hot path).

The product is ``_lib/libgridshift_cuda.so`` (C-ABI in include/gridshift_c.h, C++ API in
include/gridshift/gridshift.hpp).  ``gridshift`` mirrors the reference engine API in Python
over that C-ABI; ``configs`` generates the BASELINE.json synthetic workloads.
"""
from . import gridshift  # noqa: F401
from .gridshift import (ClusterLabeling, Engine, EngineConfig, Error, run)  # noqa: F401

"""B200-native FSBM collision-coalescence hot path (arXiv 2409.07232 / coalbench).

The product is libfsbm_coal.so (sm_100a CUDA kernels behind the C ABI in
include/fsbm_coal.h); ``coalbench`` mirrors the reference's host interface.
"""
from . import _lib
from .coalbench import *  # noqa: F401,F403
from .verify import *  # noqa: F401,F403
from .group import DeviceGroup, GroupDiagnostics, nccl_unique_id  # noqa: F401

__version__ = "0.2.0"

"""B200-native Image-GS hot path (arXiv 2407.01866): renderer + optimizer.

The product is ``libigs_b200.so`` (CUDA for sm_100a behind the C-ABI in
include/igs_b200.h).  ``igs`` is its ctypes binding, mirroring the
reference's igs:: C++ API; ``synth`` generates the reference test-suite's
seeded synthetic inputs; ``fit`` is the host-side encoder loop driving the
device through the ABI.
"""
from .igs import (DEFAULT_K, DEFAULT_LR, OPT_CULL, OPT_DETERMINISTIC, OPT_TILE, OPT_RASTER, OPT_SHARD_ADAM, Context,  # noqa: F401
                  IgsError,
                  LIB_PATH, load_library)

__all__ = ["Context", "IgsError", "load_library", "LIB_PATH", "DEFAULT_K", "DEFAULT_LR", "OPT_CULL", "OPT_RASTER",
           "OPT_DETERMINISTIC", "OPT_TILE", "OPT_SHARD_ADAM"]

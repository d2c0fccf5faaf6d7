"""B200-native SPFOM iteration for the GAM sales-based LP (arXiv 2602.22421).

The product is libspfom.so (include/spfom.h); `spfom` is its ctypes binding.
"""
from .spfom import (  # noqa: F401
    EXPORTED,
    LIB_PATH,
    Params,
    Solver,
    SpfomError,
    load_library,
    nccl_unique_id,
    partition,
)

"""B200-native (sm_100a) MemShare collaborative-filtering KV-block reuse path (arXiv 2507.21433).

The product is ``libmemshare.so`` (CUDA kernels + the C ABI declared in ``include/memshare.h``);
this package holds its ctypes binding (``_lib``), the device-buffer plumbing that enqueues the
four calls (``pipeline``) and the build script (``build``). Importing it requires the built
CUDA library -- there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (fails loudly if libmemshare.so is missing)
from ._lib import (CUR_ALL, CUR_LAST, CUR_RANGE, DIST_FINALIZE, DIST_FULL, DIST_PARTIAL, PAIR_ALIGNED,  # noqa: F401
                   PAIR_CROSS, Dims, KVPool, MemShareError, abi_version)

__all__ = ["_lib", "pipeline"]

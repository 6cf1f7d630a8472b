"""B200-native KV pin pool, memory-manager pressure step and stage mapper for Orla/stageflow.

The product is the C-ABI library ``_lib/libsfkv.so`` (CUDA kernels for sm_100a behind
include/sfkv.h). This package only locates and binds it; there is no Python or CPU compute path,
so a missing library is an import-time error on use, never a silent fallback.
"""
import ctypes as _C
import os as _os

from .abi import Api, Config, Pool, csr  # noqa: F401

PKG_DIR = _os.path.dirname(_os.path.abspath(__file__))
LIB_DIR = _os.path.join(PKG_DIR, "_lib")
# SFKV_LIBRARY: an alternative build of the same ABI (compile-time variants under measurement)
LIB_PATH = _os.environ.get("SFKV_LIBRARY") or _os.path.join(LIB_DIR, "libsfkv.so")
_api = None


def load_library():
    if not _os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    return _C.CDLL(LIB_PATH)


def api() -> Api:
    global _api
    if _api is None:
        _api = Api(load_library())
    return _api

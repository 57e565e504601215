"""tierkv_b200 — B200-native KV-cache data-movement path of LMCache (arXiv 2510.09665).

Host C++ (csrc/*.cpp) mirrors the reference tierkv engine API (Connector,
PagedKVStore, TieredStore, KeyChain) and drives hand-written sm_100a kernels
(csrc/*.cu) through the C-ABI in include/tierkv_b200.h. This Python package
only loads that library (``_lib``) and wraps it (``api``); it never computes a
byte itself and has no CPU fallback.
"""
from ._lib import LIB_PATH, TkvError, check, lib  # noqa: F401


def build(verbose: bool = False) -> str:
    from ._build import build as _b
    return _b(verbose)


def __getattr__(name):
    if name in ("Engine", "chunk_keys", "keychain_next", "plan_tiles", "hash_chains"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)

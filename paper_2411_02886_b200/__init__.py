"""B200-native TokenSelect decode path (arXiv 2411.02886): Selection Cache,
paged Q.K scoring, per-head soft vote, radix top-k and sparse paged
flash-decoding as sm_100a kernels behind the C ABI in include/tokenselect.h.

``paper_2411_02886_b200.selattn`` mirrors the reference's Python module
(proj/python/bindings.cpp). Importing it loads the native library and fails
loudly when it has not been built (there is no CPU implementation).
"""
from __future__ import annotations

import importlib

__all__ = ["selattn", "build"]


def build(force: bool = False) -> str:
    from . import build as _b

    return _b.build(force=force)


def __getattr__(name):
    if name == "selattn":
        return importlib.import_module(".selattn", __name__)
    raise AttributeError(name)

"""hfuse-b200: B200-native horizontal kernel fusion (HFuse, arXiv 2007.01277).

Compiler + sm_100a runtime live in the in-tree ``libhfuse.so`` (C ABI: include/hfuse.h);
``hfuse`` is its Python mirror. See DESIGN.md.

The package itself is lazy: ``pairs`` / ``shard`` / ``crypto`` (workload catalogs, host-side
reduction) import without touching libhfuse.so, so the reference arm of bench.py — which
must run the reference interpreter only — never maps the product library. The first access
to ``hfuse`` or one of its re-exported names loads it (and fails loudly if it is missing).
"""
import importlib

_REEXPORT = ("HFuseError", "Image", "Module", "fuse", "lower", "search")

__all__ = ["hfuse", *_REEXPORT]


def __getattr__(name):
    if name == "hfuse":
        return importlib.import_module(".hfuse", __name__)
    if name in _REEXPORT:
        return getattr(importlib.import_module(".hfuse", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

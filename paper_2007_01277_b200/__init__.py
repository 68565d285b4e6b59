"""hfuse-b200: B200-native horizontal kernel fusion (HFuse, arXiv 2007.01277).

Compiler + sm_100a runtime live in the in-tree ``libhfuse.so`` (C ABI: include/hfuse.h);
``hfuse`` is its Python mirror. See DESIGN.md.
"""
from . import hfuse  # noqa: F401  (fails loudly when libhfuse.so is missing)
from .hfuse import HFuseError, Image, Module, fuse, lower, search  # noqa: F401

__all__ = ["hfuse", "HFuseError", "Image", "Module", "fuse", "lower", "search"]

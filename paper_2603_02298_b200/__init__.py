"""B200-native (sm_100a) hot path underneath the `tla` layout algebra of arXiv 2603.02298:
layout-driven copy, bulk layout evaluation and tiled bf16 GEMM, behind the C ABI of include/tlb.h.

The product is libtlb.so (hand-written CUDA, paper_2603_02298_b200/csrc). This package is the
thin loader / driver; importing it does not load the library until a call needs it, and a missing
library is an error (no CPU fallback).
"""
from . import abi, host, shard  # noqa: F401
from .abi import TlbError, load  # noqa: F401
from .host import L, Layout  # noqa: F401

__all__ = ["abi", "host", "shard", "TlbError", "load", "L", "Layout"]

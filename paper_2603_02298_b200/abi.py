"""ctypes view of include/tlb.h — the C-ABI drop-in boundary of the sm_100a hot path.

Nothing here computes: every call goes into libtlb.so (hand-written CUDA). If the library is
missing the import fails loudly; there is no CPU fallback (the oracle under oracle/ is test
infrastructure and is never imported from this package).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libtlb.so"

TLB_MAX_MODES = 16

(TLB_OK, TLB_ERR_CONTRACT, TLB_ERR_BOUNDS, TLB_ERR_STRUCTURAL, TLB_ERR_SEMIMODULE, TLB_ERR_OVERFLOW, TLB_ERR_CUDA,
 TLB_ERR_UNSUPPORTED, TLB_ERR_INDEX, TLB_ERR_ADMISSIBILITY) = range(10)
STATUS_NAMES = ["ok", "contract_error", "bounds_error", "structural_error", "semimodule_error", "overflow_error",
                "cuda_error", "unsupported", "index_error", "admissibility_error"]
KIND_INT, KIND_BASIS, KIND_XOR = 0, 1, 2
ACC_BUFFER, ACC_COUNTING = 0, 1
LF_ALL_POW2, LF_HAS_NEG, LF_INJECTIVE = 1, 2, 4


class tlb_mode(C.Structure):
    _fields_ = [("extent", C.c_int64), ("stride", C.c_int64), ("kind", C.c_int32), ("axis", C.c_int32)]


class tlb_layout_desc(C.Structure):
    _fields_ = [
        ("n_modes", C.c_int32), ("kind", C.c_int32), ("n_top", C.c_int32), ("flags", C.c_int32),
        ("size", C.c_int64), ("cosize", C.c_int64), ("min_offset", C.c_int64), ("max_offset", C.c_int64),
        ("top_start", C.c_int32 * (TLB_MAX_MODES + 1)),
        ("extent", C.c_int64 * TLB_MAX_MODES), ("stride", C.c_int64 * TLB_MAX_MODES),
        ("magic", C.c_uint64 * TLB_MAX_MODES), ("shift", C.c_uint8 * TLB_MAX_MODES),
        ("log2e", C.c_uint8 * TLB_MAX_MODES),
    ]


class tlb_gemm_tiler(C.Structure):
    _fields_ = [("bm", C.c_int32), ("bn", C.c_int32), ("bk", C.c_int32)]


class tlb_tensor(C.Structure):
    _fields_ = [("layout", C.POINTER(tlb_layout_desc)), ("data", C.c_void_p), ("origin", C.c_int64),
                ("capacity", C.c_int64), ("elem_bytes", C.c_int32), ("accessor", C.c_int32)]


# every symbol include/tlb.h declares: name -> (restype, argtypes)
_P = C.POINTER
SYMBOLS = {
    "tlb_abi_version": (C.c_int, []),
    "tlb_last_error": (C.c_char_p, []),
    "tlb_launch_count": (C.c_uint64, []),
    "tlb_last_plan": (C.c_char_p, []),
    "tlb_config_set": (C.c_int, [C.c_char_p, C.c_char_p]),
    "tlb_layout_lower": (C.c_int, [_P(tlb_mode), C.c_int, _P(tlb_layout_desc)]),
    "tlb_layout_lower_ranked": (C.c_int, [_P(tlb_mode), C.c_int, _P(C.c_int32), C.c_int, _P(tlb_layout_desc)]),
    "tlb_eval_range": (C.c_int, [_P(tlb_layout_desc), C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "tlb_idx2crd_range": (C.c_int, [_P(tlb_layout_desc), C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "tlb_crd2idx_range": (C.c_int, [_P(tlb_layout_desc), C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "tlb_crd2idx_range_checked": (C.c_int, [_P(tlb_layout_desc), C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tlb_rinv_check_range": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), C.c_uint64, C.c_uint64, C.c_void_p,
                                       C.c_void_p]),
    "tlb_compose_check_range": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), _P(tlb_layout_desc), C.c_uint64,
                                          C.c_uint64, C.c_void_p, C.c_void_p]),
    "tlb_compose_check": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), _P(tlb_layout_desc), _P(C.c_uint64), C.c_void_p]),
    "tlb_eval_axes_range": (C.c_int, [_P(tlb_mode), C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "tlb_copy": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), C.c_uint64, C.c_uint64, C.c_void_p]),
    "tlb_copy_plan": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), C.c_uint64, C.c_uint64]),
    "tlb_max_common_vector": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), _P(C.c_int64)]),
    "tlb_copy_set_path": (C.c_int, [C.c_int]),
    "tlb_tensormap_from_divided": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), C.c_int, C.c_int, C.c_void_p,
                                             C.c_void_p]),
    "tlb_tensormap_describe": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), _P(C.c_int32), _P(C.c_uint64),
                                         _P(C.c_uint64), _P(C.c_uint32)]),
    "tlb_tensormap_fetch_tile": (C.c_int, [C.c_void_p, C.c_int, _P(C.c_int32), C.c_uint32, C.c_int, C.c_void_p,
                                           C.c_void_p]),
    "tlb_gemm_bf16": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), C.c_uint32, C.c_uint32, C.c_void_p]),
    "tlb_gemm_bf16_tiled": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), C.c_void_p, C.c_void_p]),
    "tlb_locate_offsets": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), _P(tlb_mode), _P(C.c_int32), C.c_void_p]),
    "tlb_tensormap_cache_stats": (C.c_int, [_P(C.c_uint64), _P(C.c_uint64)]),
    "tlb_workspace_trim": (C.c_int, [C.c_uint64]),
    "tlb_copy_tv": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_layout_desc), C.c_void_p]),
    "tlb_copy_tv_auto": (C.c_int, [_P(tlb_layout_desc), _P(tlb_layout_desc), C.c_int, C.c_int, _P(tlb_mode), _P(C.c_int32), _P(C.c_int32)]),
    "tlb_gemm_tile_count": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), _P(C.c_uint32)]),
    "tlb_gemm_bf16_batched": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int32, C.c_int32, C.c_void_p]),
    "tlb_gemm_f16": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), C.c_uint32, C.c_uint32, C.c_void_p]),
    "tlb_gemm_f16_batched": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), C.c_int64, C.c_int64, C.c_int64,
                                       C.c_int32, C.c_int32, C.c_void_p]),
    "tlb_gemm_i64": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor), C.c_void_p, C.c_void_p]),
    "tlb_gemm_set_path": (C.c_int, [C.c_int]),
    "tlb_gemm_clock_stats": (C.c_int, [_P(C.c_double), _P(C.c_double), _P(C.c_uint32)]),
    "tlb_copy_host": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor)]),
    "tlb_eval_range_host": (C.c_int, [_P(tlb_layout_desc), C.c_uint64, C.c_uint64, C.c_void_p]),
    "tlb_gemm_bf16_host": (C.c_int, [_P(tlb_tensor), _P(tlb_tensor), _P(tlb_tensor)]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libtlb.so (built by paper_2603_02298_b200.build). Raises if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2603_02298_b200.build` "
                               "(the CUDA library is the product; there is no CPU fallback)")
        import os
        # TLB_LIB: a differently built libtlb.so (kernel experiments of tools/, never set by the tests or the bench)
        lib = C.CDLL(os.environ.get("TLB_LIB") or str(LIB_PATH))
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(lib, name)  # AttributeError if the header and the library disagree
            fn.restype = res
            fn.argtypes = args
        if lib.tlb_abi_version() != 1:
            raise RuntimeError("libtlb.so ABI version mismatch")
        _lib = lib
    return _lib


class TlbError(RuntimeError):
    """A non-zero tlb_status. `.status` is the code, `.kind` the reference exception it maps to."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {message}")
        self.status = status
        self.kind = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)


def check(status: int) -> None:
    if status != TLB_OK:
        raise TlbError(status, load().tlb_last_error().decode())

"""TEST INFRASTRUCTURE. ctypes access to the CPU checkers:

  oracle/_build/liboracle.so   plain-C restatement of the reference hot path (oracle/tlb_oracle.c)
  oracle/_ref/libtla_ref.so    the UNMODIFIED reference headers behind C shims (oracle/ref_shim.cpp);
                               present only where it was built from /root/reference (it travels to
                               the GPU box as a prebuilt file)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import this.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

from paper_2603_02298_b200.host import L, Layout

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "_build" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libtla_ref.so"
GOLDEN = ROOT / "tests" / "golden"


class orc_mode(C.Structure):
    _fields_ = [("extent", C.c_int64), ("stride", C.c_int64), ("kind", C.c_int32), ("axis", C.c_int32)]


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        _orc = C.CDLL(str(ORACLE_SO))
        _orc.orc_eval_range.restype = C.c_int
        _orc.orc_copy.restype = C.c_int
        _orc.orc_gemm_i64.restype = C.c_int
        _orc.orc_gemm_bf16.restype = C.c_int
        _orc.orc_gemm_f16.restype = C.c_int
        _orc.orc_gemm_bf16_tn_flat.restype = C.c_int
        _orc.orc_crd2idx_range.restype = C.c_int
    return _orc


def have_ref() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        _ref = C.CDLL(str(REF_SO))
        _ref.ref_last_error.restype = C.c_char_p
    return _ref


def as_layout(x) -> Layout:
    return x if isinstance(x, Layout) else L(x)


def modes_of(lay) -> tuple:
    lay = as_layout(lay)
    arr = (orc_mode * len(lay.modes))()
    for r, (e, k, v, ax) in enumerate(lay.modes):
        arr[r].extent, arr[r].kind, arr[r].stride, arr[r].axis = e, k, v, ax
    return arr, len(lay.modes)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---- the C restatement -------------------------------------------------------------------
def orc_eval_range(lay, i0: int, n: int) -> np.ndarray:
    m, k = modes_of(lay)
    out = np.empty(n, dtype=np.int64)
    st = orc().orc_eval_range(m, k, C.c_int64(i0), C.c_int64(n), _p(out))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out


def orc_eval_axes_range(lay, n_axes: int, i0: int, n: int) -> np.ndarray:
    m, k = modes_of(lay)
    out = np.empty((n, n_axes), dtype=np.int64)
    fn = orc().orc_eval_axes_range
    fn.restype = C.c_int
    st = fn(m, k, n_axes, C.c_int64(i0), C.c_int64(n), _p(out))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out


def orc_idx2crd_range(lay, i0: int, n: int) -> np.ndarray:
    lay = as_layout(lay)
    ext = np.array([e for e, *_ in lay.modes], dtype=np.int64)
    out = np.empty((n, len(ext)), dtype=np.int64)
    orc().orc_idx2crd_range(_p(ext), len(ext), C.c_int64(i0), C.c_int64(n), _p(out))
    return out


def orc_crd2idx_range(lay, crd: np.ndarray) -> np.ndarray:
    lay = as_layout(lay)
    ext = np.array([e for e, *_ in lay.modes], dtype=np.int64)
    crd = np.ascontiguousarray(crd, dtype=np.int64)
    out = np.empty(crd.shape[0], dtype=np.int64)
    st = orc().orc_crd2idx_range(_p(ext), len(ext), _p(crd), C.c_int64(crd.shape[0]), _p(out))
    if st:
        raise RuntimeError(f"oracle status {st}")
    return out


def orc_copy(src_lay, src: np.ndarray | None, dst_lay, dst: np.ndarray, src_origin=0, dst_origin=0, i_begin=0,
             i_end=None) -> int:
    """tla::copy restated; dst is modified in place; returns the status (partial writes stay, as in the reference)."""
    sm, sn = modes_of(src_lay)
    dm, dn = modes_of(dst_lay)
    eb = dst.dtype.itemsize
    if i_end is None:
        i_end = as_layout(src_lay).size
    return orc().orc_copy(sm, sn, _p(src) if src is not None else None, C.c_int64(src_origin),
                          C.c_int64(src.size if src is not None else 0), dm, dn, _p(dst), C.c_int64(dst_origin),
                          C.c_int64(dst.size), eb, C.c_int64(i_begin), C.c_int64(i_end))


def orc_gemm_i64(la, a: np.ndarray, lb, b: np.ndarray, lc, c: np.ndarray) -> int:
    la, lb, lc = as_layout(la), as_layout(lb), as_layout(lc)
    am, an = modes_of(la)
    bm, bn = modes_of(lb)
    cm, cn = modes_of(lc)
    M = 1
    for e, *_ in la.modes[:la.top_leaves[0]]:
        M *= e
    return orc().orc_gemm_i64(am, an, la.top_leaves[0], _p(a), C.c_int64(a.size), bm, bn, lb.top_leaves[0], _p(b),
                              C.c_int64(b.size), cm, cn, lc.top_leaves[0], _p(c), C.c_int64(c.size), C.c_int64(0),
                              C.c_int64(M))


def orc_gemm_bf16(la, a_bits: np.ndarray, lb, b_bits: np.ndarray, lc, c: np.ndarray, want_abs=False, m_begin=0,
                  m_end=None, f16=False):
    """Sequential-k fp32 restatement on bf16 (or, with f16=True, IEEE fp16) bit patterns (uint16).
    Returns (status, abs_sum or None)."""
    la, lb, lc = as_layout(la), as_layout(lb), as_layout(lc)
    am, an = modes_of(la)
    bm, bn = modes_of(lb)
    cm, cn = modes_of(lc)
    M = 1
    for e, *_ in la.modes[:la.top_leaves[0]]:
        M *= e
    ab = np.zeros(c.size, dtype=np.float32) if want_abs else None
    fn = orc().orc_gemm_f16 if f16 else orc().orc_gemm_bf16
    st = fn(am, an, la.top_leaves[0], _p(a_bits), C.c_int64(a_bits.size), bm, bn, lb.top_leaves[0],
                             _p(b_bits), C.c_int64(b_bits.size), cm, cn, lc.top_leaves[0], _p(c), C.c_int64(c.size),
                             _p(ab) if want_abs else None, C.c_int64(m_begin), C.c_int64(M if m_end is None else m_end))
    return st, ab


def orc_gemm_bf16_tn_flat(a_bits, lda, b_bits, ldb, c, ldc, M, N, K, m0, m1, n0, n1) -> None:
    orc().orc_gemm_bf16_tn_flat(_p(a_bits), C.c_int64(lda), _p(b_bits), C.c_int64(ldb), _p(c), C.c_int64(ldc),
                                C.c_int64(M), C.c_int64(N), C.c_int64(K), C.c_int64(m0), C.c_int64(m1), C.c_int64(n0),
                                C.c_int64(n1))


# ---- the unmodified reference ---------------------------------------------------------------
def ref_op(op: str, a: str = "", b: str = "", c: str = ""):
    """Returns (status, text). status 0 ok; otherwise the reference's exception class (ref_shim.cpp)."""
    out = C.create_string_buffer(4096)
    st = ref().ref_op_str(op.encode(), a.encode(), b.encode(), c.encode(), out, C.c_size_t(4096))
    return st, (out.value.decode() if st == 0 else ref().ref_last_error().decode())


def ref_eval_range(text: str, i0: int, n: int, which: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    st = ref().ref_eval_range(text.encode(), C.c_int64(i0), C.c_int64(n), _p(out), which)
    if st:
        raise RuntimeError(f"reference status {st}: {ref().ref_last_error().decode()}")
    return out


def ref_copy(src_text: str, src_cells: np.ndarray | None, dst_text: str, dst_cells: np.ndarray, src_origin=0,
             dst_origin=0) -> int:
    """tla::copy verbatim over int64 cells (dst_cells modified in place)."""
    assert dst_cells.dtype == np.int64
    return ref().ref_copy(src_text.encode(), _p(src_cells) if src_cells is not None else None,
                          C.c_int64(src_cells.size if src_cells is not None else 0), C.c_int64(src_origin),
                          dst_text.encode(), _p(dst_cells), C.c_int64(dst_cells.size), C.c_int64(dst_origin))


def ref_copy_shared(src_text: str, dst_text: str, cells: np.ndarray, src_origin=0, dst_origin=0) -> int:
    """tla::copy verbatim with both tensors viewing ONE storage (cells modified in place)."""
    assert cells.dtype == np.int64
    return ref().ref_copy_shared(src_text.encode(), C.c_int64(src_origin), dst_text.encode(), C.c_int64(dst_origin),
                                 _p(cells), C.c_int64(cells.size))


def ref_eval_axes_range(text: str, n_axes: int, i0: int, n: int) -> np.ndarray:
    out = np.empty((n, n_axes), dtype=np.int64)
    st = ref().ref_eval_axes_range(text.encode(), C.c_int64(i0), C.c_int64(n), n_axes, _p(out))
    if st:
        raise RuntimeError(f"reference status {st}: {ref().ref_last_error().decode()}")
    return out


def ref_copy_bench(src_text: str, dst_text: str, threads: int):
    """(seconds, checksum) of tla::copy on reference-owned storage: verbatim on one core (threads <= 1), or its loop
    body over disjoint i-ranges on `threads` std::threads. Only the copy itself is timed."""
    sec, chk = C.c_double(0), C.c_uint64(0)
    st = ref().ref_copy_bench(src_text.encode(), dst_text.encode(), threads, C.byref(sec), C.byref(chk))
    if st:
        raise RuntimeError(f"reference status {st}: {ref().ref_last_error().decode()}")
    return sec.value, chk.value


def ref_eval_range_mt(text: str, i0: int, n: int, threads: int, which: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    st = ref().ref_eval_range_mt(text.encode(), C.c_int64(i0), C.c_int64(n), _p(out), which, threads)
    if st:
        raise RuntimeError(f"reference status {st}: {ref().ref_last_error().decode()}")
    return out


def ref_gemm(la: str, a: np.ndarray, lb: str, b: np.ndarray, lc: str, c: np.ndarray) -> int:
    return ref().ref_gemm(la.encode(), _p(a), C.c_int64(a.size), lb.encode(), _p(b), C.c_int64(b.size), lc.encode(),
                          _p(c), C.c_int64(c.size))


def golden(name: str):
    return json.loads((GOLDEN / name).read_text())


# ---- small numeric helpers shared by the tests ----------------------------------------------
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def cosize_of(lay) -> int:
    """1 + max offset of an Int-kind layout with non-negative strides (cosize, layout.hpp:277)."""
    lay = as_layout(lay)
    return 1 + sum((e - 1) * v for e, k, v, ax in lay.modes)

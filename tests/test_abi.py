"""CPU: the C-ABI library loads, exports every symbol include/tlb.h declares, and its host-only
entry points (lowering, pre-flight contracts) behave like the reference's checks."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2603_02298_b200 import L, TlbError, abi

ROOT = Path(__file__).resolve().parent.parent


def test_every_declared_symbol_is_exported():
    header = (ROOT / "include" / "tlb.h").read_text()
    declared = set(re.findall(r"\b(tlb_[a-z0-9_]+)\s*\(", header))
    lib = abi.load()
    assert declared, "no declarations found in include/tlb.h"
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} is declared in include/tlb.h but not exported by libtlb.so"
    assert declared == set(abi.SYMBOLS), "abi.py and include/tlb.h disagree on the entry points"


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "tlb.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu %zu\\n",'
                   'sizeof(tlb_layout_desc),sizeof(tlb_tensor),sizeof(tlb_mode),offsetof(tlb_layout_desc,extent),'
                   'offsetof(tlb_layout_desc,log2e));return 0;}\n')
    import subprocess
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [C.sizeof(abi.tlb_layout_desc), C.sizeof(abi.tlb_tensor), C.sizeof(abi.tlb_mode),
            abi.tlb_layout_desc.extent.offset, abi.tlb_layout_desc.log2e.offset]
    assert got == want


def test_header_is_plain_c(tmp_path):
    import subprocess
    src = tmp_path / "c89.c"
    src.write_text('#include "tlb.h"\nint main(void){return TLB_ABI_VERSION - 1;}\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-c", str(src), "-o",
                           str(tmp_path / "c89.o")])


@pytest.mark.parametrize("text,size,cosize,kind,injective", [
    ("(4,8):(1,4)", 32, 32, abi.KIND_INT, True),
    ("(4,8):(20,2)", 32, 75, abi.KIND_INT, True),       # test_layout.cpp:92 cosize golden
    ("((2,2),(4,2)):((1,8),(2,16))", 32, 32, abi.KIND_INT, True),
    ("(8,8):(f1,f9)", 64, -1, abi.KIND_XOR, True),
    ("7:0", 7, 1, abi.KIND_INT, False),
    ("(4,6):(0,1)", 24, 6, abi.KIND_INT, False),
    ("(4,8):(-1,4)", 32, -1, abi.KIND_INT, True),
    ("(4,8):(e0,e1)", 32, -1, abi.KIND_BASIS, False),
    ("(65536,65536):(65536,1)", 2**32, 2**32, abi.KIND_INT, True),
])
def test_lowering(text, size, cosize, kind, injective):
    d = L(text).lower()
    assert d.size == size and d.cosize == cosize and d.kind == kind
    assert bool(d.flags & abi.LF_INJECTIVE) == injective


def test_lowering_errors_map_to_reference_exceptions():
    lib = abi.load()
    d = abi.tlb_layout_desc()
    m = (abi.tlb_mode * 2)()
    m[0].extent, m[0].stride, m[0].kind = 4, 2, abi.KIND_INT
    m[1].extent, m[1].stride, m[1].kind, m[1].axis = 3, 1, abi.KIND_BASIS, 0
    # (4,3):(2,e0) -> semimodule_error (test_layout.cpp:70)
    assert lib.tlb_layout_lower(m, 2, C.byref(d)) == abi.TLB_ERR_SEMIMODULE
    m[1].extent, m[1].stride, m[1].kind = 0, 4, abi.KIND_INT
    # (4,0):(1,4) -> structural_error (test_layout.cpp:71)
    assert lib.tlb_layout_lower(m, 2, C.byref(d)) == abi.TLB_ERR_STRUCTURAL
    assert b"positive" in lib.tlb_last_error()
    big = (abi.tlb_mode * 2)()
    big[0].extent, big[0].stride = 2**40, 1
    big[1].extent, big[1].stride = 2**40, 1
    assert lib.tlb_layout_lower(big, 2, C.byref(d)) == abi.TLB_ERR_OVERFLOW


def test_ranked_lowering_keeps_top_modes():
    d = L("((2,2),8):((1,16),2)").lower(ranked=True)
    assert d.n_top == 2 and list(d.top_start[:3]) == [0, 2, 3]


def test_contracts_are_checked_before_any_device_work():
    """Size mismatch / rank / writability are host-side contract errors, reported even without a GPU."""
    lib = abi.load()
    from paper_2603_02298_b200 import host
    d8, d4 = L("8:1").lower(), L("4:1").lower()
    buf = (C.c_int64 * 8)()
    src = host.make_tensor(d8, C.addressof(buf), 8, 8)
    dst = host.make_tensor(d4, C.addressof(buf), 8, 8)
    # copy requires equal sizes (test_tensor.cpp:113-118)
    assert lib.tlb_copy(C.byref(src), C.byref(dst), 0, 2**64 - 1, None) == abi.TLB_ERR_CONTRACT
    assert b"equal sizes" in lib.tlb_last_error()
    # only buffer accessors are writable (tensor.hpp:93)
    cnt = host.make_tensor(d8, None, 0, 8, counting=True)
    assert lib.tlb_copy(C.byref(src), C.byref(cnt), 0, 2**64 - 1, None) == abi.TLB_ERR_CONTRACT
    # gemm preconditions (test_tensor.cpp:197-203)
    a = host.make_tensor(L("(4,8):(1,4)").lower(ranked=True), C.addressof(buf), 64, 8)
    b = host.make_tensor(L("(6,8):(1,6)").lower(ranked=True), C.addressof(buf), 64, 8)
    c_bad = host.make_tensor(L("(4,5):(1,4)").lower(ranked=True), C.addressof(buf), 64, 8)
    assert lib.tlb_gemm_i64(C.byref(a), C.byref(b), C.byref(c_bad), None, None) == abi.TLB_ERR_CONTRACT
    assert b"extents do not agree" in lib.tlb_last_error()
    # the 2-byte entry points reject other cell sizes, and both check extents before looking for a device
    for fn in (lib.tlb_gemm_bf16, lib.tlb_gemm_f16):
        assert fn(C.byref(a), C.byref(b), C.byref(c_bad), 0, 2**32 - 1, None) == abi.TLB_ERR_CONTRACT
        a2 = host.make_tensor(L("(4,8):(8,1)").lower(ranked=True), C.addressof(buf), 64, 2)
        b2 = host.make_tensor(L("(6,8):(8,1)").lower(ranked=True), C.addressof(buf), 64, 2)
        c8 = host.make_tensor(L("(4,6):(6,1)").lower(ranked=True), C.addressof(buf), 64, 8)
        assert fn(C.byref(a2), C.byref(b2), C.byref(c8), 0, 2**32 - 1, None) == abi.TLB_ERR_CONTRACT
        assert b"element sizes" in lib.tlb_last_error()
    flat = host.make_tensor(L("32:1").lower(ranked=True), C.addressof(buf), 64, 8)
    assert lib.tlb_gemm_i64(C.byref(flat), C.byref(b), C.byref(c_bad), None, None) == abi.TLB_ERR_CONTRACT
    assert b"rank-2" in lib.tlb_last_error()


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    lib = abi.load()
    from paper_2603_02298_b200 import host
    d = L("8:1").lower()
    out = (C.c_int64 * 8)()
    assert lib.tlb_eval_range(C.byref(d), 0, 8, C.addressof(out), None) == abi.TLB_ERR_CUDA
    assert b"no CPU fallback" in lib.tlb_last_error()
    src = host.make_tensor(d, C.addressof(out), 8, 8)
    assert lib.tlb_copy(C.byref(src), C.byref(src), 0, 2**64 - 1, None) == abi.TLB_ERR_CUDA
    assert lib.tlb_copy_host(C.byref(src), C.byref(src)) == abi.TLB_ERR_CUDA
    h16 = (C.c_int16 * 64)()
    hc = (C.c_float * 64)()
    a2 = host.make_tensor(L("(4,8):(8,1)").lower(ranked=True), C.addressof(h16), 64, 2)
    c4 = host.make_tensor(L("(4,4):(4,1)").lower(ranked=True), C.addressof(hc), 64, 4)
    for fn in (lib.tlb_gemm_bf16, lib.tlb_gemm_f16):
        assert fn(C.byref(a2), C.byref(a2), C.byref(c4), 0, 2**32 - 1, None) == abi.TLB_ERR_CUDA
    assert lib.tlb_gemm_bf16_host(C.byref(a2), C.byref(a2), C.byref(c4)) == abi.TLB_ERR_CUDA
    with pytest.raises(TlbError):
        abi.check(lib.tlb_copy_host(C.byref(src), C.byref(src)))


def test_gemm_tile_count_is_host_only():
    """Sharding input: the number of 128x256 tiles of the plan, without a device."""
    import ctypes as C
    from paper_2603_02298_b200 import host
    buf = (C.c_int16 * 16)()
    def t(text, eb):
        return (host.make_tensor(L(text).lower(ranked=True), C.addressof(buf), 1 << 40, eb), None)
    a, b = t("(4096,4096):(4096,1)", 2), t("(4096,4096):(4096,1)", 2)
    assert host.gemm_tile_count(a, b, t("(4096,4096):(1,4096)", 4)) == 512
    assert host.gemm_tile_count(t("(8192,8192):(8192,1)", 2), t("(8192,8192):(8192,1)", 2), t("(8192,8192):(1,8192)", 4)) == 2048
    # ragged: 200 x 300 runs transposed (C m-contiguous): rows = 300 -> 2 blocks, cols = 200 -> 1 block
    assert host.gemm_tile_count(t("(200,136):(136,1)", 2), t("(300,136):(136,1)", 2), t("(200,300):(1,200)", 4)) == 4

"""CPU: host logic of the copy planner (tlb_copy_plan runs the contract checks and the planner without a
device). The plans are what the -m gpu parity tests then execute."""
import ctypes as C

import pytest

from paper_2603_02298_b200 import L, TlbError, abi, host


@pytest.mark.parametrize("s,d,eb,plan", [
    # BASELINE configs C1 and C3 take the swizzle-staged tiled kernel
    ("(8192,8192):(8192,1)", "(8192,8192):(1,8192)", 4, "tiled"),
    ("((8,128),(4,64),4096):((1,2048),(8,32),262144)", "((8,128),(4,64),4096):((128,1),(65536,1024),262144)", 4, "tiled"),
    ("((32,16),(64,4)):((1,32),(512,32768))", "((32,16),(64,4)):((64,8192),(1,2048))", 2, "tiled"),
    ("((32,16),(64,4)):((1,32),(512,32768))", "((32,16),(64,4)):((64,8192),(1,2048))", 8, "tiled"),
    # one mode contiguous on both sides -> vectors along it
    ("4096:1", "4096:1", 4, "vec"),
    ("(64,8,4):(1,256,64)", "(64,8,4):(1,64,512)", 2, "vec"),
    # the Table-1 rows (test_tensor.cpp:93-100)
    ("8:1", "8:1", 8, "vec"), ("(8,2,3):(1,16,32)", "(8,2,3):(1,16,32)", 8, "vec"),
    ("(2,3,2):(42,1,128)", "12:1", 8, "gather"), ("7:0", "7:1", 8, "gather"), ("7:0", "7:0", 8, "last_writer+gather"),
    ("(8,3):(1,8)", "(8,3):(3,1)", 8, "gather"),
    # Xor strides, interleaved runs, ragged rows, aliasing destinations
    ("(8,8):(f1,f9)", "64:1", 8, "gather"),
    # ... but a swizzle that leaves the low bits alone moves whole 16-byte vectors per evaluation, 32 / 64-byte runs when
    # both layouts keep them (Swizzle<3,4,3> on fp32 cells: 16 cells), with 256-bit accesses
    ("(128,8,64):(1,128,1024)", "(128,8,64):(f1,f144,f1024)", 4, "gather_run"),
    ("(128,8,64):(f1,f144,f1024)", "(128,8,64):(1,128,1024)", 2, "gather_run"),
    ("(128,8,64):(f1,f144,f1024)", "(128,8,64):(1,128,1024)", 1, "gather_vec"),
    ("((4,16),(32,4)):((1,512),(4,128))", "((4,16),(32,4)):((2048,1),(16,512))", 4, "tiled_n"),   # 4-cell source runs: narrow staged tiles
    # narrow runs: a whole short mode on one side (a 4M x 24 transpose and back), cell-granular staged tiles
    ("(4194304,24):(24,1)", "(4194304,24):(1,4194304)", 4, "interleave"),     # 24 cells: an interleave size since the last pass
    ("(4194304,20):(20,1)", "(4194304,20):(1,4194304)", 4, "interleave"),
    ("(4194304,27):(27,1)", "(4194304,27):(1,4194304)", 4, "tiled_n"),
    ("(4194304,27):(1,4194304)", "(4194304,27):(27,1)", 4, "tiled_n"),
    ("(4194309,27):(27,1)", "(4194309,27):(1,4194309)", 4, "ragged:tiled_n"),
    ("(4194309,27):(1,4194309)", "(4194309,27):(27,1)", 4, "ragged:tiled_n"),
    ("(4194304,100):(100,1)", "(4194304,100):(1,4194304)", 1, "tiled_n"),
    ("(96,160):(160,1)", "(96,160):(1,96)", 2, "gather"),
    # AoS <-> SoA: register-permuting interleave plan (short mode 2 .. 10, 12, 16, 24 or 32 cells, whole lane pieces, 16-byte alignment)
    ("(4,1048576):(1,4)", "(4,1048576):(1048576,1)", 4, "interleave"),
    ("(224,224,3,16):(3,672,1,150528)", "(224,224,3,16):(1,224,50176,150528)", 1, "interleave"),
    ("(5,1048576):(1,5)", "(5,1048576):(1048576,1)", 4, "interleave"),
    ("(1048576,16):(16,1)", "(1048576,16):(1,1048576)", 4, "interleave"),      # tall-skinny transpose
    ("(27,1048576):(1,27)", "(27,1048576):(1048576,1)", 4, "tiled_n"),         # 27 cells: not an interleave size, narrow staged tiles
    ("(11,1048576):(1,11)", "(11,1048576):(1048576,1)", 8, "tiled_n"),         # 8-byte cells: the common extents only
    ("(4,1048576):(1,4)", "(4,1048576):(1048577,1)", 4, "tiled_n"),            # planar rows not 16-byte aligned: narrow staged tiles
    # ragged extents (rows that are not whole 128-byte pieces / whole tiles): a whole-tile body on the staged plan plus
    # edge strips, from 2^22 elements (smaller copies are one gather launch)
    ("(4000,3000):(3000,1)", "(4000,3000):(1,4000)", 4, "ragged:tiled"),
    ("(4001,3001):(3001,1)", "(4001,3001):(1,4001)", 4, "ragged:tiled_u"),
    ("(300,300,300):(1,300,90000)", "(300,300,300):(90000,300,1)", 4, "ragged:tiled"),
    ("(1000,1000):(1000,1)", "(1000,1000):(1,1000)", 4, "gather"),
    ("(5001,5003):(1,5001)", "(5001,5003):(1,5001)", 1, "ragged:vec"),     # an odd number of contiguous bytes
    ("(33,33):(33,1)", "(33,33):(1,33)", 4, "gather"),
    # no unit stride on the source: the staged plan runs along the smallest-stride mode
    ("(2048,2048):(3,6151)", "(2048,2048):(2048,1)", 2, "tiled_s"),
    ("(2048,2048):(2048,1)", "(2048,2048):(5,10243)", 4, "tiled_s"),
    # stride-0 destination modes: only the slice at their last coordinate survives (last writer wins), an injective copy
    ("(64,64):(1,64)", "(64,64):(1,0)", 4, "last_writer+vec"),
    # genuinely overlapping destination strides: winner election
    ("(32,32,4):(1,32,1024)", "(32,32,4):(1,31,3)", 8, "ordered"),
])
def test_plan_selection(s, d, eb, plan):
    assert host.copy_plan(s, d, eb) == plan


def test_plan_depends_on_alignment_and_range():
    s, d = "(256,128):(128,1)", "(256,128):(1,256)"
    assert host.copy_plan(s, d, 4) == "tiled"
    assert host.copy_plan(s, d, 4, src_align=4) == "tiled_u"           # 16-byte vectors need 16-byte bases: cell-sized accesses
    assert host.copy_plan(s, d, 2, src_align=2) == "tiled_u"           # ... for 1-, 2-, 4- and 8-byte cells
    assert host.copy_plan(s, d, 1, src_align=1) == "tiled_u"           # (1-byte cells: 128-row tiles only)
    assert host.copy_plan("(96,256):(256,1)", "(96,256):(1,96)", 1, src_align=1) == "tiled_n"   # 96 < 128 rows: narrow-run tiles
    assert host.copy_plan(s, d, 4, 0, 256 * 64) == "tiled"             # whole slices of the outermost mode
    assert host.copy_plan(s, d, 4, 5, 777) == "gather"                 # ragged range
    assert host.copy_plan(s, d, 4, 10, 10) == "empty"


def test_plan_contracts():
    with pytest.raises(TlbError) as e:
        host.copy_plan("8:1", "4:1", 8)
    assert e.value.status == abi.TLB_ERR_CONTRACT                      # copy requires equal sizes
    with pytest.raises(TlbError) as e:
        host.copy_plan("(2,2):(e0,e1)", "4:1", 8)
    assert e.value.status == abi.TLB_ERR_SEMIMODULE
    lib = abi.load()
    d = L("4:3").lower()
    buf = (C.c_int64 * 8)()
    src = host.make_tensor(d, C.addressof(buf), 8, 8)                  # 4:3 touches cell 9 of 8
    dst = host.make_tensor(L("4:1").lower(), C.addressof(buf), 8, 8)
    assert lib.tlb_copy_plan(C.byref(src), C.byref(dst), 0, 2**64 - 1) == abi.TLB_ERR_BOUNDS


def test_tensormap_dims_from_divided_layouts():
    """TMA tensor maps are derived from zipped_divide results (algebra.hpp:595): parent flat modes -> globalDim /
    globalStrides (sorted by stride, contiguous leaves merged), tile mode -> boxDim."""
    # zipped_divide((4096,4096):(4096,1), [128,64]) = ((128,64),(32,64)):((4096,1),(524288,64))  (SURVEY.md vocabulary)
    rank, dims, strides, box = host.tensormap_describe("(4096,4096):(4096,1)", "(128,64):(4096,1)")
    assert (rank, dims, strides, box) == (2, [4096, 4096], [1, 4096], [64, 128])
    # config C3 source: modes 0,2,3 merge into one contiguous 2048-element dimension
    rank, dims, strides, box = host.tensormap_describe("((8,128),(4,64),4096):((1,2048),(8,32),262144)",
                                                       "((8,128),4):((1,2048),8)")
    assert (rank, dims, strides, box) == (2, [2048, 128 * 4096], [1, 2048], [32, 128])   # rows of all tiles merge too
    # operands of the GEMM: A (M,K):(K,1) tiled [128,64] -> dims (K, M), box (64, 128)
    assert host.tensormap_describe("(8192,4096):(4096,1)", "(128,64):(4096,1)")[3] == [64, 128]
    with pytest.raises(TlbError) as e:
        host.tensormap_describe("(64,64):(128,2)", "(8,8):(128,2)")          # no stride-1 dimension
    assert e.value.status == abi.TLB_ERR_UNSUPPORTED
    with pytest.raises(TlbError) as e:
        host.tensormap_describe("(8,8):(f1,f9)", "(8,8):(f1,f9)")            # Xor strides
    assert e.value.status == abi.TLB_ERR_SEMIMODULE


def test_cli_plan_and_exit_codes(capsys):
    """python -m paper_2603_02298_b200: exit codes follow the reference CLI (cli.hpp:215-221)."""
    import json
    from paper_2603_02298_b200.__main__ import main
    assert main(["plan", "(8192,8192):(8192,1)", "(8192,8192):(1,8192)", "--elem-bytes", "4"]) == 0
    assert json.loads(capsys.readouterr().out)["plan"] == "tiled"
    assert main(["plan", "8:1", "4:1"]) == 1            # contract_error: sizes differ
    assert main(["plan", "8:1", "(4"]) == 2             # parse error
    assert main(["nonsense"]) == 2                      # usage


def test_max_common_vector_matches_the_reference():
    """tlb_max_common_vector (host only) vs tla::max_common_vector (analysis.hpp:18-28) on the reference's answers for
    Table-1 pairs, gapped / broadcast layouts, config C1 and 60 random stride permutations (tests/golden/mcv.json)."""
    import oracle_util as ou
    from paper_2603_02298_b200 import host
    rows = ou.golden("mcv.json")
    assert len(rows) >= 70
    for row in rows:
        assert host.max_common_vector(row["a"], row["b"]) == row["k"], (row["a"], row["b"])
    assert host.max_common_vector("(8192,8192):(8192,1)", "(8192,8192):(1,8192)") == 1      # C1 has no common vector


def test_vec_plan_width_is_bounded_by_the_common_vector():
    """The vec plan moves min(max_common_vector, 16 bytes) cells per access when the common vector starts the layouts."""
    from paper_2603_02298_b200 import host
    assert host.max_common_vector("(64,32):(1,64)", "(64,32):(1,128)") == 64
    assert host.copy_plan("(64,32):(1,64)", "(64,32):(1,128)", 4) == "vec"
    assert host.max_common_vector("(63,5):(1,63)", "(63,5):(1,64)") == 63


def test_tv_layout_derived_by_raked_product():
    """tlb_copy_tv_auto: V from max_common_vector (analysis.hpp:18-28) capped at 16 bytes, one tile of T vectors =
    raked_product((V):(1), (T):(1)) (algebra.hpp:633: the reference returns (T,V):(V,1)), tiles repeated in the value mode."""
    import oracle_util as ou
    # contiguous on both sides: 16-byte vectors
    assert host.copy_tv_auto("4096:1", "4096:1", 4, 256) == "(256,(4,4)):(4,(1,1024))"
    assert host.copy_tv_auto("4096:1", "4096:1", 2, 128) == "(128,(8,4)):(8,(1,1024))"
    # a transpose has no common vector: scalar values, the tile is T cells
    assert host.max_common_vector("(64,64):(64,1)", "(64,64):(1,64)") == 1
    assert host.copy_tv_auto("(64,64):(64,1)", "(64,64):(1,64)", 4, 256) == "(256,(1,16)):(1,(1,256))"
    # a common run of 8 fp32: capped at 4 per vector
    assert host.max_common_vector("(8,16):(1,8)", "(8,16):(1,16)") == 8
    assert host.copy_tv_auto("(8,16):(1,8)", "(8,16):(1,16)", 4, 32) == "(32,(4,1)):(4,(1,128))"
    if ou.have_ref():
        # the (T, V) tile IS the reference's raked_product of the value and the thread layout
        assert ou.ref_op("raked_product", "4:1", "256:1") == (0, "(256,4):(4,1)")
        assert ou.ref_op("raked_product", "8:1", "128:1") == (0, "(128,8):(8,1)")
    # every coordinate of the tensor is covered exactly once (ragged sizes over-cover: predicated tail)
    tv = host.copy_tv_auto("1000:1", "1000:1", 4, 64)
    idx = ou.orc_eval_range(tv, 0, host.L(tv).size)
    assert sorted(idx.tolist()) == list(range(host.L(tv).size)) and host.L(tv).size >= 1000

"""GPU parity: tla::gemm through the C ABI vs the oracle.

int64 (the reference's own value type): exact.  bf16 -> fp32: exact on the reference's integer fills
(every partial sum < 2^24), and |d| <= 1e-4 * sum_k|a*b| + 1e-6 on random data against the sequential-k
fp32 restatement (the tolerance bounds accumulation-order error only; products are exact in fp32).
"""
import numpy as np
import pytest
import torch

import oracle_util as ou
from gpu_util import dev
from paper_2603_02298_b200 import L, TlbError, abi, host

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-6


def _dims(la, lb):
    La, Lb = L(la), L(lb)
    M = int(np.prod([e for e, *_ in La.modes[:La.top_leaves[0]]]))
    N = int(np.prod([e for e, *_ in Lb.modes[:Lb.top_leaves[0]]]))
    K = int(np.prod([e for e, *_ in La.modes[La.top_leaves[0]:]]))
    return M, N, K


def test_gemm_i64_reference_fixtures():
    for row in ou.golden("gemm.json"):
        a, b, c = dev(np.array(row["a"], dtype=np.int64)), dev(np.array(row["b"], dtype=np.int64)), dev(
            np.array(row["c0"], dtype=np.int64))
        ta, ka = host.tensor_of(row["A"], a, ranked=True)
        tb, kb = host.tensor_of(row["B"], b, ranked=True)
        tc, kc = host.tensor_of(row["C"], c, ranked=True)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        host.gemm_i64((ta, ka), (tb, kb), (tc, kc), st)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        assert c.cpu().numpy().tolist() == row["c"], (row["A"], row["B"], row["C"])


def test_gemm_i64_overflow_is_reported():
    a = dev(np.full(4, 2**62, dtype=np.int64))
    c = dev(np.zeros(4, dtype=np.int64))
    ta, ka = host.tensor_of("(2,2):(1,2)", a, ranked=True)
    tc, kc = host.tensor_of("(2,2):(1,2)", c, ranked=True)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    host.gemm_i64((ta, ka), (ta, ka), (tc, kc), st)
    torch.cuda.synchronize()
    assert int(st.item()) == abi.TLB_ERR_OVERFLOW          # checked_mul (common.hpp:105)


def test_gemm_zero_a_and_preconditions():
    a = dev(np.zeros(16, dtype=np.int64))
    b = dev(np.arange(16, dtype=np.int64))
    c = dev(np.zeros(16, dtype=np.int64))
    t = lambda buf, s: host.tensor_of(s, buf, ranked=True)
    host.gemm_i64(t(a, "(4,4):(1,4)"), t(b, "(4,4):(1,4)"), t(c, "(4,4):(1,4)"))
    torch.cuda.synchronize()
    assert (c.cpu().numpy() == 0).all()                    # test_tensor.cpp:205-214
    s = dev(np.arange(64, dtype=np.int64))
    with pytest.raises(TlbError) as e:                     # test_tensor.cpp:197-203
        host.gemm_i64(t(s, "(4,8):(1,4)"), t(s, "(6,8):(1,6)"), t(s, "(4,5):(1,4)"))
    assert e.value.status == abi.TLB_ERR_CONTRACT


def _bf16_case(la, lb, lc, kat, seed=0, path=0, c_init=True, f16=False, tile_ranges=None):
    M, N, K = _dims(la, lb)
    na, nb, nc = ou.cosize_of(la), ou.cosize_of(lb), ou.cosize_of(lc)
    rng = np.random.default_rng(seed)
    ao = ou.orc_eval_range(la, 0, M * K).reshape(K, M).T
    bo = ou.orc_eval_range(lb, 0, N * K).reshape(K, N).T
    a = np.zeros(na, dtype=np.float32)
    b = np.zeros(nb, dtype=np.float32)
    if kat:
        i, p = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
        a[ao] = (i * 7 + p * 3 + 1) % 11
        j, p = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
        b[bo] = (j * 5 + p * 2 + 2) % 13
        c0 = (np.arange(nc) % 5 - 2).astype(np.float32) if c_init else np.zeros(nc, dtype=np.float32)
    else:
        a[ao] = rng.uniform(-1, 1, (M, K))
        b[bo] = rng.uniform(-1, 1, (N, K))
        c0 = rng.uniform(-1, 1, nc).astype(np.float32) if c_init else np.zeros(nc, dtype=np.float32)
    if f16:
        ab, bb = a.astype(np.float16).view(np.uint16), b.astype(np.float16).view(np.uint16)
    else:
        ab, bb = ou.f32_to_bf16_bits(a), ou.f32_to_bf16_bits(b)
    want = c0.copy()
    st, sabs = ou.orc_gemm_bf16(la, ab, lb, bb, lc, want, want_abs=True, f16=f16)
    assert st == 0
    ta_, tb_, tc_ = dev(ab.view(np.int16)), dev(bb.view(np.int16)), dev(c0)
    ta, ka = host.tensor_of(la, ta_, ranked=True)
    tb, kb = host.tensor_of(lb, tb_, ranked=True)
    tc, kc = host.tensor_of(lc, tc_, ranked=True)
    prev = abi.load().tlb_gemm_set_path(path)
    try:
        fn = host.gemm_f16 if f16 else host.gemm_bf16
        if tile_ranges is None:
            plan = fn((ta, ka), (tb, kb), (tc, kc))
        else:
            for (t0, t1) in tile_ranges:
                plan = fn((ta, ka), (tb, kb), (tc, kc), t0, t1)
    finally:
        abi.load().tlb_gemm_set_path(prev)
    torch.cuda.synchronize()
    got = tc_.cpu().numpy()
    if kat or plan.startswith("simt"):
        assert (got == want).all(), f"{plan}: {int((got != want).sum())} of {got.size} cells differ"
    else:
        err = np.abs(got - want)
        tol = RTOL * sabs + ATOL
        touched = sabs > 0
        assert (err[touched] <= tol[touched]).all(), f"{plan}: max err {err.max()} vs tol {tol[touched].min()}"
        assert (got[~touched] == want[~touched]).all()
    return plan


@pytest.mark.parametrize("fam", [
    ("(4,8):(1,9)", "(6,8):(1,10)", "(4,6):(1,7)"), ("(4,8):(9,1)", "(6,8):(10,1)", "(4,6):(1,7)"),
    ("(6,8):(1,10)", "(4,8):(1,9)", "(6,4):(1,7)"), ("(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)"),
    ("((2,2),8):((1,16),2)", "(6,8):(8,1)", "((2,2),6):((1,3),52)"),
    ("(33,40):(1,33)", "(17,40):(1,17)", "(33,17):(17,1)"),
])
def test_gemm_bf16_layout_families_simt(fam):
    """NT / TN / NTT / BLIS / GETT (test_tensor.cpp:176-189) in bf16: bit-exact vs the sequential restatement."""
    assert _bf16_case(*fam, kat=True).startswith("simt")
    assert _bf16_case(*fam, kat=False, seed=4).startswith("simt")


def _tile_count(la, lb, lc):
    t = lambda s, eb: (host.make_tensor(L(s).lower(ranked=True), 256, 1 << 40, eb), None)
    return host.gemm_tile_count(t(la, 2), t(lb, 2), t(lc, 4))


def test_gemm_simt_fallback_keeps_the_transposed_tile_ids():
    """A fit that runs the problem transposed (m-contiguous C) but whose call falls through to SIMT: a 2-byte C whose
    leading dimension the wide plan's TMA epilogue cannot address, with unequal block counts along m and n. The SIMT
    kernel must index the tile grid the way the tcgen05 fit counted it (columns n >= 256 were skipped). Whole
    range, then an odd partition of the tile ids. (fp32-C problems of this kind now run on the 256 x 256 plan's register
    epilogue: second half.)"""
    shape = ("(200,136):(1,208)", "(300,136):(1,304)", "(200,300):(1,201)")
    assert _c16_case(shape, False).startswith("simt")
    tiles = _tile_count(*shape)
    assert tiles == 4
    assert _c16_case(shape, False, tile_ranges=[(0, 1), (1, 3), (3, tiles)]).startswith("simt")
    big = ("(600,72):(1,608)", "(300,72):(1,304)", "(600,300):(1,601)")
    tiles = _tile_count(*big)
    assert _c16_case(big, True, tile_ranges=[(0, 3), (3, 4), (4, tiles)]).startswith("simt")
    # the same layouts with an fp32 C: MN-major operands on the 256 x 256 plan, any C strides through the register epilogue
    assert _bf16_case(*shape, kat=True) == "umma_2sm_regs"
    assert _bf16_case(*shape, kat=False, seed=3) == "umma_2sm_regs"
    assert _bf16_case(*big, kat=True, tile_ranges=[(0, 4), (4, _tile_count(*big))]).startswith("umma_")


UMMA_SHAPES = [
    ("(128,64):(64,1)", "(256,64):(64,1)", "(128,256):(1,128)"),          # one tile, one k-block
    ("(256,256):(256,1)", "(512,256):(256,1)", "(256,512):(1,256)"),      # 2x2 tiles, TN per PAPER.md:1767
    ("(256,256):(256,1)", "(512,256):(256,1)", "(256,512):(512,1)"),      # N-contiguous C (vector epilogue)
    ("(200,136):(136,1)", "(300,136):(136,1)", "(200,300):(1,200)"),      # ragged M, N, K (TMA zero fill + masks)
    ("(384,512):(520,1)", "(256,512):(528,1)", "(384,256):(1,400)"),      # padded leading dimensions
    ("(1024,1024):(1024,1)", "(1024,1024):(1024,1)", "(1024,1024):(1,1024)"),
    ("(256,128):(128,1)", "(300,128):(128,1)", "(256,300):(1,257)"),      # ldc not a multiple of 4: register epilogue
    ("(256,128):(128,1)", "(256,128):(128,1)", "(256,256):(2,600)"),      # neither mode of C contiguous
]


@pytest.mark.parametrize("cg", [2, 3])
@pytest.mark.parametrize("shape", UMMA_SHAPES)
def test_gemm_bf16_umma_kat_exact(shape, cg):
    plan = _bf16_case(*shape, kat=True, path=cg)
    assert plan.startswith("umma_1sm" if cg == 2 else "umma_2sm")


@pytest.mark.parametrize("cg", [2, 3])
@pytest.mark.parametrize("shape", UMMA_SHAPES[1:5] + UMMA_SHAPES[6:])
def test_gemm_bf16_umma_random_within_tolerance(shape, cg):
    _bf16_case(*shape, kat=False, seed=7, path=cg)


def test_gemm_bf16_auto_plan_is_tensor_core_for_tn():
    assert _bf16_case(*UMMA_SHAPES[1], kat=True).startswith("umma")


def _flat_tn_check(M, N, K, cg, tile_ranges=None, batch=1):
    """Full-size check: KAT fills -> exact; compares sampled 128x256 tiles against the flat restatement."""
    g = torch.Generator(device="cuda")
    i = torch.arange(M, device="cuda").view(M, 1)
    p = torch.arange(K, device="cuda").view(1, K)
    a = ((i * 7 + p * 3 + 1) % 11).to(torch.bfloat16).contiguous()
    j = torch.arange(N, device="cuda").view(N, 1)
    b = ((j * 5 + p * 2 + 2) % 13).to(torch.bfloat16).contiguous()
    c = torch.zeros(N, M, dtype=torch.float32, device="cuda")           # (M,N):(1,M)
    ta, ka = host.tensor_of(f"({M},{K}):({K},1)", a.view(-1).view(torch.int16), ranked=True)
    tb, kb = host.tensor_of(f"({N},{K}):({K},1)", b.view(-1).view(torch.int16), ranked=True)
    tc, kc = host.tensor_of(f"({M},{N}):(1,{M})", c.view(-1), ranked=True)
    prev = abi.load().tlb_gemm_set_path(cg)
    try:
        if tile_ranges is None:
            host.gemm_bf16((ta, ka), (tb, kb), (tc, kc))
        else:
            for (t0, t1) in tile_ranges:
                host.gemm_bf16((ta, ka), (tb, kb), (tc, kc), t0, t1)
    finally:
        abi.load().tlb_gemm_set_path(prev)
    torch.cuda.synchronize()
    # exact integer result via fp64 matmul on the GPU is itself a library call; use it only as a cross-check
    # on the whole matrix, the oracle on sampled tiles is the parity statement.
    an, bn = a.view(torch.int16).cpu().numpy().view(np.uint16), b.view(torch.int16).cpu().numpy().view(np.uint16)
    got = c.cpu().numpy()                                                # [n][m]
    rng = np.random.default_rng(0)
    for _ in range(3):
        m0 = int(rng.integers(0, M // 128)) * 128
        n0 = int(rng.integers(0, N // 256)) * 256
        want = np.zeros((N, M), dtype=np.float32)
        ou.orc_gemm_bf16_tn_flat(an.ravel(), K, bn.ravel(), K, want.ravel(), M, M, N, K, m0, m0 + 16, n0, n0 + 16)
        assert (got[n0:n0 + 16, m0:m0 + 16] == want[n0:n0 + 16, m0:m0 + 16]).all()
    ref = (a.double() @ b.double().t()).t().contiguous()                 # exact: integers below 2^53
    assert torch.equal(c.double(), ref)


@pytest.mark.parametrize("cg", [2, 3])
def test_c2_gemm_4096_full_size_exact(cg):
    """Config C2 at BASELINE size with the reference's integer fills: bit-exact.
    4096^3 is also where the tail wave is split along K (reduce-add of two K-slices per tile)."""
    _flat_tn_check(4096, 4096, 4096, cg)


@pytest.fixture
def force_wide(tlb_config):
    """K-major problems below 48 pair tiles default to the 256 x 256 plan; GEMM_WIDE=1 keeps the small parity shapes
    on the wide kernel."""
    tlb_config("GEMM_WIDE", "1")


WIDE_SHAPES = [
    # (A, B, C) as the kernel runs them: C n-contiguous -> rows = M; 512 x 256 pair tiles need ceil(M/256) even
    ("(512,64):(64,1)", "(256,64):(64,1)", "(512,256):(256,1)"),          # one pair tile, one k-block
    ("(512,1024):(1024,1)", "(512,1024):(1024,1)", "(512,512):(1,512)"),  # m-contiguous C (runs transposed), 16 k-blocks
    ("(1000,200):(200,1)", "(300,200):(200,1)", "(1000,300):(300,1)"),    # ragged M, N, K: TMA zero fill / clipping
    ("(1024,520):(528,1)", "(768,520):(536,1)", "(1024,768):(800,1)"),    # padded leading dimensions
    ("(1024,512):(512,1)", "(1536,512):(512,1)", "(1024,1536):(1,1024)"),  # 12 pair tiles cut into k-ranges per worker
]


@pytest.mark.parametrize("shape", WIDE_SHAPES)
def test_gemm_bf16_wide_plan_kat_exact(shape, force_wide):
    """512 x 256 pair tiles (tlb_gemm_umma_wide.cu): exact on the reference's integer fills, including the stream-K
    cut of the partial wave (partial tiles combine through the reduce-add epilogue)."""
    assert _bf16_case(*shape, kat=True, path=3) == "umma_2sm_wide"


@pytest.mark.parametrize("shape", WIDE_SHAPES[1:])
def test_gemm_bf16_wide_plan_random_within_tolerance(shape, force_wide):
    assert _bf16_case(*shape, kat=False, seed=11, path=3) == "umma_2sm_wide"


MN_MAJOR_SHAPES = [
    # the "N" operands of the paper's layout table: the m / n mode is the contiguous one
    ("(512,256):(1,512)", "(256,256):(1,256)", "(512,256):(1,512)"),      # NT: A, B MN-major, C m-contiguous (runs transposed)
    ("(512,256):(1,512)", "(256,256):(1,256)", "(512,256):(256,1)"),      # NTT: C n-contiguous
    ("(512,256):(256,1)", "(256,256):(1,256)", "(512,256):(256,1)"),      # A K-major, B N-major
    ("(512,256):(1,512)", "(256,256):(256,1)", "(512,256):(256,1)"),      # A M-major, B K-major
    ("(200,136):(1,208)", "(300,136):(1,304)", "(200,300):(1,200)"),      # ragged M, N, K with padded leading dimensions
    ("(640,1000):(1,648)", "(384,1000):(1,392)", "(640,384):(384,1)"),    # odd number of 256-row blocks, K % 64 != 0
]


@pytest.mark.parametrize("shape", MN_MAJOR_SHAPES)
def test_gemm_bf16_mn_major_operands_on_tensor_cores_kat_exact(shape, tlb_config):
    """NT / NTT families on tcgen05: MN-major tiles staged as 64-row chunks, MN-major UMMA descriptors (idesc bits 15/16),
    on every tensor-core plan: the planner's choice (256 x 256 for these short k-loops), one CTA per tile, and the wide plan."""
    assert _bf16_case(*shape, kat=True).startswith("umma_2sm")
    assert _bf16_case(*shape, kat=True, path=2).startswith("umma_1sm")
    tlb_config("GEMM_WIDE", "1")
    assert _bf16_case(*shape, kat=True) == "umma_2sm_wide"


@pytest.mark.parametrize("shape", MN_MAJOR_SHAPES[:2] + MN_MAJOR_SHAPES[4:])
def test_gemm_bf16_mn_major_operands_random_within_tolerance(shape, tlb_config):
    assert _bf16_case(*shape, kat=False, seed=13).startswith("umma_2sm")
    assert _bf16_case(*shape, kat=False, seed=15, f16=True, path=2).startswith("umma_1sm")
    tlb_config("GEMM_WIDE", "1")
    assert _bf16_case(*shape, kat=False, seed=17) == "umma_2sm_wide"


@pytest.mark.parametrize("shape,path,plan", [
    (UMMA_SHAPES[1], 2, "umma_1sm"), (UMMA_SHAPES[2], 3, "umma_2sm"), (UMMA_SHAPES[6], 3, "umma_2sm_regs"),
    (WIDE_SHAPES[1], 0, "umma_2sm_wide"), (WIDE_SHAPES[2], 0, "umma_2sm_wide"), (MN_MAJOR_SHAPES[0], 0, "umma_2sm_wide"),
    (("(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)"), 0, "simt_f16"),
])
def test_gemm_f16_operands(shape, path, plan, tlb_config):
    """tlb_gemm_f16: IEEE fp16 operands on every plan (instruction-descriptor formats 0 instead of 1), exact on the
    reference's integer fills and within the stated tolerance on random data."""
    if plan.endswith("wide"):
        tlb_config("GEMM_WIDE", "1")
    assert _bf16_case(*shape, kat=True, path=path, f16=True) == plan
    assert _bf16_case(*shape, kat=False, seed=17, path=path, f16=True) == plan


@pytest.mark.parametrize("f16", [False, True])
@pytest.mark.parametrize("shape", [
    ("(512,256):(256,1)", "(256,256):(256,1)", "(512,256):(256,1)"),      # n-contiguous C in the operands' type
    ("(512,256):(256,1)", "(256,256):(256,1)", "(512,256):(1,512)"),      # m-contiguous C (runs transposed)
    ("(1000,200):(200,1)", "(300,200):(200,1)", "(1000,300):(304,1)"),    # ragged, padded C rows
    ("(512,256):(1,512)", "(256,256):(1,256)", "(512,256):(256,1)"),      # MN-major operands
    ("(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)"),                     # SIMT plan
])
def test_gemm_c_in_the_operand_type(shape, f16):
    """C with the operands' 2-byte type (the reference's tensors share one value type): fp32 accumulation in TMEM, one
    rounding to bf16 / fp16, added to C in that type (L2 reduction on the wide plan, in registers on the SIMT plan).
    Tolerance: one unit in the last place of the result type on |C| + sum |a b| (2^-7 bf16, 2^-10 fp16)."""
    plan = _c16_case(shape, f16)
    if shape[0].startswith("(4,8)"):
        assert plan == ("simt_f16" if f16 else "simt_bf16")
        return
    assert plan.startswith("umma_2sm") and not plan.endswith("regs")     # the planner's choice: 256 x 256 for short k-loops
    prev = abi.load().tlb_gemm_set_path(2)
    try:
        assert _c16_case(shape, f16).startswith("umma_1sm")              # one CTA per tile
    finally:
        abi.load().tlb_gemm_set_path(prev)
    host.config("GEMM_WIDE", "1")
    try:
        assert _c16_case(shape, f16) == "umma_2sm_wide"                  # and the 512 x 256 plan
    finally:
        host.config("GEMM_WIDE", None)


def _c16_case(shape, f16, tile_ranges=None):
    la, lb, lc = shape
    M, N, K = _dims(la, lb)
    rng = np.random.default_rng(31)
    na, nb, nc = ou.cosize_of(la), ou.cosize_of(lb), ou.cosize_of(lc)
    ao = ou.orc_eval_range(la, 0, M * K).reshape(K, M).T
    bo = ou.orc_eval_range(lb, 0, N * K).reshape(K, N).T
    a, b = np.zeros(na, dtype=np.float32), np.zeros(nb, dtype=np.float32)
    a[ao] = rng.uniform(-1, 1, (M, K))
    b[bo] = rng.uniform(-1, 1, (N, K))
    c0 = rng.uniform(-1, 1, nc).astype(np.float32)
    if f16:
        conv = lambda x: x.astype(np.float16).view(np.uint16)
        back = lambda u: u.view(np.float16).astype(np.float32)
        ulp = 2.0 ** -10
    else:
        conv = ou.f32_to_bf16_bits
        back = lambda u: (u.astype(np.uint32) << 16).view(np.float32)
        ulp = 2.0 ** -7
    ab, bb, cb = conv(a), conv(b), conv(c0)
    want = back(cb).copy()                                               # fp32 restatement starting from the rounded C
    st, sabs = ou.orc_gemm_bf16(la, ab, lb, bb, lc, want, want_abs=True, f16=f16)
    assert st == 0
    ta_, tb_, tc_ = dev(ab.view(np.int16)), dev(bb.view(np.int16)), dev(cb.view(np.int16))
    ta, ka = host.tensor_of(la, ta_, ranked=True)
    tb, kb = host.tensor_of(lb, tb_, ranked=True)
    tc, kc = host.tensor_of(lc, tc_, ranked=True)
    fn = host.gemm_f16 if f16 else host.gemm_bf16
    if tile_ranges is None:
        plan = fn((ta, ka), (tb, kb), (tc, kc))
    else:
        for (t0, t1) in tile_ranges:
            plan = fn((ta, ka), (tb, kb), (tc, kc), t0, t1)
    torch.cuda.synchronize()
    got = back(tc_.cpu().numpy().view(np.uint16))
    scale = np.abs(back(cb)) + sabs
    touched = sabs > 0
    assert (np.abs(got - want)[touched] <= 2 * ulp * scale[touched] + 1e-6).all()
    assert (got[~touched] == back(cb)[~touched]).all()                   # cells the layout does not address stay untouched
    return plan


def test_gemm_wide_plan_whole_tiles_then_k_ranges():
    """128 pair tiles on 74 CTA pairs: 54 tiles are cut into one k-range per pair and run first, 74 whole tiles follow."""
    _flat_tn_check(4096, 4096, 1024, 3)


def test_gemm_wide_plan_tile_ranges_partition_the_output(force_wide):
    """Sharding on groups of 4 tile ids (512 x 256 pair tiles, shard.gemm_tile_range): every shard runs the wide plan and
    disjoint ranges compose to the full product."""
    tiles = (1024 // 256) * (2048 // 256) * 2
    cuts = [0, 16, 20, 48, tiles]
    _flat_tn_check(1024, 2048, 512, 3, tile_ranges=list(zip(cuts[:-1], cuts[1:])))
    assert abi.load().tlb_last_plan().decode() == "umma_2sm_wide"


def test_gemm_wide_plan_takes_large_problems_with_an_odd_number_of_row_blocks(force_wide):
    """ceil(M/256) odd: the full range of a problem still runs 512 x 256 pair tiles (the last one is clipped by the
    TMA bounds); 3 x 16 = 48 pair tiles. (Forced: with K = 64 the planner would keep the 256 x 256 plan.)"""
    assert _bf16_case("(1280,64):(64,1)", "(4096,64):(64,1)", "(1280,4096):(4096,1)", kat=True) == "umma_2sm_wide"


def test_gemm_plan_selection_by_k_and_size():
    """The planner's crossover (measured, tlb_gemm_umma_wide.cu): the 512 x 256 plan needs at least 48 pair tiles AND 64
    k-blocks (K >= 4096); shorter k-loops keep the 256 x 256 plan, whose flush overlaps the next tile. Host-side decision,
    checked through tlb_last_plan on zero-filled operands (nothing to compare: the parity tests cover both kernels)."""
    def plan(M, N, K):
        a = torch.zeros(M * K, dtype=torch.bfloat16, device="cuda")
        b = torch.zeros(N * K, dtype=torch.bfloat16, device="cuda")
        c = torch.zeros(M * N, dtype=torch.float32, device="cuda")
        return host.gemm_bf16(host.tensor_of(f"({M},{K}):({K},1)", a.view(torch.int16), ranked=True),
                              host.tensor_of(f"({N},{K}):({K},1)", b.view(torch.int16), ranked=True),
                              host.tensor_of(f"({M},{N}):({N},1)", c, ranked=True))
    assert plan(4096, 4096, 4096) == "umma_2sm_wide"
    assert plan(4096, 4096, 2048) == "umma_2sm"
    assert plan(2048, 2048, 8192) == "umma_2sm"          # 32 pair tiles
    assert plan(3072, 4096, 4096) == "umma_2sm_wide"     # 96 pair tiles


def test_gemm_wide_plan_falls_back_when_it_does_not_apply(tlb_config):
    # ceil(M/256) odd: no m-adjacent block pairs -> 256 x 256 plan
    assert _bf16_case("(768,128):(128,1)", "(256,128):(128,1)", "(768,256):(256,1)", kat=True, path=3) == "umma_2sm"
    assert _bf16_case(*WIDE_SHAPES[1], kat=True, path=3) == "umma_2sm"          # 2 pair tiles: too small for the wide plan
    tlb_config("GEMM_WIDE", "0")
    assert _bf16_case("(2048,64):(64,1)", "(4096,64):(64,1)", "(2048,4096):(4096,1)", kat=True, path=3) == "umma_2sm"


def test_gemm_wide_plan_without_k_split_is_reproducible(tlb_config):
    """TLB_GEMM_SPLIT_TAIL=0: every tile is summed by one CTA pair in k order, so two runs agree bit for bit (with the
    k-range cut of the partial wave the partial sums meet in L2 in arrival order)."""
    tlb_config("GEMM_SPLIT_TAIL", "0")
    tlb_config("GEMM_WIDE", "1")
    assert _bf16_case(*WIDE_SHAPES[4], kat=False, seed=5, path=3) == "umma_2sm_wide"
    M, N, K = 2048, 2304, 512                                            # 36 pair tiles on 74 CTA pairs
    g = torch.Generator(device="cuda").manual_seed(9)
    a = (torch.rand(M * K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(N * K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    outs = []
    for _ in range(2):
        c = torch.zeros(M * N, dtype=torch.float32, device="cuda")
        ta = host.tensor_of(f"({M},{K}):({K},1)", a.view(torch.int16), ranked=True)
        tb = host.tensor_of(f"({N},{K}):({K},1)", b.view(torch.int16), ranked=True)
        tc = host.tensor_of(f"({M},{N}):({N},1)", c, ranked=True)
        assert host.gemm_bf16(ta, tb, tc) == "umma_2sm_wide"
        torch.cuda.synchronize()
        outs.append(c)
    assert torch.equal(outs[0], outs[1])
    ref = a.view(M, K).float() @ b.view(N, K).float().t()
    assert torch.allclose(outs[0].view(M, N), ref, rtol=1e-3, atol=1e-2)


def test_gemm_register_epilogue_matches_tma_epilogue(tlb_config):
    tlb_config("GEMM_EPILOGUE", "regs")
    assert _bf16_case(*UMMA_SHAPES[1], kat=True, path=2) == "umma_1sm_regs"
    assert _bf16_case(*UMMA_SHAPES[2], kat=False, seed=3, path=3) == "umma_2sm_regs"
    _flat_tn_check(4096, 4096, 1024, 2)


@pytest.mark.parametrize("cg", [2, 3])
def test_gemm_tile_ranges_partition_the_output(cg):
    """Sharding by tile-coordinate ranges: disjoint ranges compose to the full product."""
    tiles = (1024 // 256) * (2048 // 256) * 2
    cuts = [0, 6, 20, tiles - 2, tiles]
    _flat_tn_check(1024, 2048, 512, cg, tile_ranges=list(zip(cuts[:-1], cuts[1:])))


@pytest.mark.parametrize("cg", [2, 3])
def test_gemm_batched_matches_per_batch(cg):
    M, N, K, B = 256, 512, 192, 3
    rng = np.random.default_rng(2)
    a = ou.f32_to_bf16_bits(rng.uniform(-1, 1, (B, M, K)).astype(np.float32))
    b = ou.f32_to_bf16_bits(rng.uniform(-1, 1, (B, N, K)).astype(np.float32))
    c0 = rng.uniform(-1, 1, (B, N, M)).astype(np.float32)
    ta_, tb_, tc_ = dev(a.view(np.int16)), dev(b.view(np.int16)), dev(c0)
    la, lb, lc = f"({M},{K}):({K},1)", f"({N},{K}):({K},1)", f"({M},{N}):(1,{M})"
    ta = host.make_tensor(L(la).lower(ranked=True), ta_.data_ptr(), ta_.numel(), 2)
    tb = host.make_tensor(L(lb).lower(ranked=True), tb_.data_ptr(), tb_.numel(), 2)
    tc = host.make_tensor(L(lc).lower(ranked=True), tc_.data_ptr(), tc_.numel(), 4)
    prev = abi.load().tlb_gemm_set_path(cg)
    try:
        host.gemm_bf16_batched((ta, None), (tb, None), (tc, None), M * K, N * K, M * N, 1, 3)   # batches 1..2 only
    finally:
        abi.load().tlb_gemm_set_path(prev)
    torch.cuda.synchronize()
    got = tc_.cpu().numpy()
    assert (got[0] == c0[0]).all()                                       # batch 0 untouched
    for bi in (1, 2):
        want = c0[bi].copy().ravel()
        st, sabs = ou.orc_gemm_bf16(la, a[bi].ravel(), lb, b[bi].ravel(), lc, want, want_abs=True)
        assert st == 0
        assert (np.abs(got[bi].ravel() - want) <= RTOL * sabs + ATOL).all()


def test_gemm_batched_with_c_in_the_operand_type():
    """Batches 1..2 of a 3-batch problem with bf16 C: batch strides and a batch range on the 2-byte reduction epilogue."""
    M, N, K, B = 256, 512, 192, 3
    rng = np.random.default_rng(4)
    a = ou.f32_to_bf16_bits(rng.uniform(-1, 1, (B, M, K)).astype(np.float32))
    b = ou.f32_to_bf16_bits(rng.uniform(-1, 1, (B, N, K)).astype(np.float32))
    c0 = ou.f32_to_bf16_bits(rng.uniform(-1, 1, (B, N, M)).astype(np.float32))
    back = lambda u: (u.astype(np.uint32) << 16).view(np.float32)
    ta_, tb_, tc_ = dev(a.view(np.int16)), dev(b.view(np.int16)), dev(c0.view(np.int16))
    la, lb, lc = f"({M},{K}):({K},1)", f"({N},{K}):({K},1)", f"({M},{N}):(1,{M})"
    ta = host.make_tensor(L(la).lower(ranked=True), ta_.data_ptr(), ta_.numel(), 2)
    tb = host.make_tensor(L(lb).lower(ranked=True), tb_.data_ptr(), tb_.numel(), 2)
    tc = host.make_tensor(L(lc).lower(ranked=True), tc_.data_ptr(), tc_.numel(), 2)
    assert host.gemm_bf16_batched((ta, None), (tb, None), (tc, None), M * K, N * K, M * N, 1, 3).startswith("umma_2sm")
    torch.cuda.synchronize()
    got = back(tc_.cpu().numpy().view(np.uint16))
    assert (got[0] == back(c0[0])).all()                                 # batch 0 untouched
    for bi in (1, 2):
        want = back(c0[bi]).copy().ravel()
        st, sabs = ou.orc_gemm_bf16(la, a[bi].ravel(), lb, b[bi].ravel(), lc, want, want_abs=True)
        assert st == 0
        assert (np.abs(got[bi].ravel() - want) <= 2 * 2.0 ** -7 * (np.abs(back(c0[bi]).ravel()) + sabs) + 1e-6).all()


def test_gemm_host_entry_point():
    M, N, K = 256, 256, 128
    i, p = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
    a = ou.f32_to_bf16_bits(((i * 7 + p * 3 + 1) % 11).astype(np.float32))
    j, p = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    b = ou.f32_to_bf16_bits(((j * 5 + p * 2 + 2) % 13).astype(np.float32))
    c = np.ones(M * N, dtype=np.float32)
    la, lb, lc = f"({M},{K}):({K},1)", f"({N},{K}):({K},1)", f"({M},{N}):(1,{M})"
    want = c.copy()
    st, _ = ou.orc_gemm_bf16(la, a.ravel(), lb, b.ravel(), lc, want)
    ha, hb, hc = torch.from_numpy(a.view(np.int16).ravel().copy()), torch.from_numpy(b.view(np.int16).ravel().copy()), torch.from_numpy(c)
    ta, ka = host.tensor_of(la, ha, ranked=True)
    tb, kb = host.tensor_of(lb, hb, ranked=True)
    tc, kc = host.tensor_of(lc, hc, ranked=True)
    host.gemm_bf16_host((ta, ka), (tb, kb), (tc, kc))
    assert (hc.numpy() == want).all()


@pytest.mark.parametrize("lc_kind", ["m_contiguous", "n_contiguous"])
def test_gemm_host_entry_point_pipelined_panels(lc_kind, tlb_config):
    """tlb_gemm_bf16_host on a problem with several 512-row panels (ragged last panel, padded leading dimensions): the
    upload / compute / download pipeline must produce exactly what the one-shot path does, and the oracle's cells."""
    tlb_config("HOST_PANEL", "512")
    M, N, K = 1300, 1400, 72
    lda, ldb = 80, 88
    rng = np.random.default_rng(21)
    i, p = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
    j, p2 = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    a = np.zeros(M * lda, dtype=np.float32)
    b = np.zeros(N * ldb, dtype=np.float32)
    a[(i * lda + p).ravel()] = ((i * 7 + p * 3 + 1) % 11).ravel()
    b[(j * ldb + p2).ravel()] = ((j * 5 + p2 * 2 + 2) % 13).ravel()
    ab, bb = ou.f32_to_bf16_bits(a), ou.f32_to_bf16_bits(b)
    la, lb = f"({M},{K}):({lda},1)", f"({N},{K}):({ldb},1)"
    lc = f"({M},{N}):(1,{M + 4})" if lc_kind == "m_contiguous" else f"({M},{N}):({N + 4},1)"
    nc = ou.cosize_of(lc)
    c0 = (np.arange(nc) % 7 - 3).astype(np.float32)
    want = c0.copy()
    st, _ = ou.orc_gemm_bf16(la, ab, lb, bb, lc, want)
    assert st == 0
    outs = []
    for pipe in ("1", "0"):
        tlb_config("HOST_PIPELINE", pipe)
        ha, hb, hc = (torch.from_numpy(x.copy()) for x in (ab.view(np.int16), bb.view(np.int16), c0))
        ta, ka = host.tensor_of(la, ha, ranked=True)
        tb, kb = host.tensor_of(lb, hb, ranked=True)
        tc, kc = host.tensor_of(lc, hc, ranked=True)
        host.gemm_bf16_host((ta, ka), (tb, kb), (tc, kc))
        outs.append(hc.numpy().copy())
    assert (outs[0] == want).all() and (outs[1] == want).all()


def test_c4_batched_8192_two_batches_exact():
    """Config C4 shape (8192^3 per batch, batch strides, TN with m-contiguous C) on 2 of the 64 batches with the
    reference's integer fills: K = 8192 keeps every partial sum below 2^24 (10 * 12 * 8192 = 983040), so the result
    must be exact. Checked against the flat restatement on sampled tiles and against an exact fp64 product."""
    M = N = K = 8192
    B = 2
    i = torch.arange(M, device="cuda").view(M, 1)
    p = torch.arange(K, device="cuda").view(1, K)
    a1 = ((i * 7 + p * 3 + 1) % 11).to(torch.bfloat16)
    b1 = ((i * 5 + p * 2 + 2) % 13).to(torch.bfloat16)
    a = torch.stack([a1, a1.flip(0)]).contiguous()
    b = torch.stack([b1, b1.flip(0)]).contiguous()
    c = torch.ones(B, N, M, dtype=torch.float32, device="cuda")
    ta = host.make_tensor(L(f"({M},{K}):({K},1)").lower(ranked=True), a.data_ptr(), a.numel(), 2)
    tb = host.make_tensor(L(f"({N},{K}):({K},1)").lower(ranked=True), b.data_ptr(), b.numel(), 2)
    tc = host.make_tensor(L(f"({M},{N}):(1,{M})").lower(ranked=True), c.data_ptr(), c.numel(), 4)
    plan = host.gemm_bf16_batched((ta, None), (tb, None), (tc, None), M * K, N * K, M * N, 0, B)
    torch.cuda.synchronize()
    assert plan == "umma_2sm_wide"
    for bi in range(B):
        ref = (a[bi].double() @ b[bi].double().t()).t() + 1.0
        assert torch.equal(c[bi].double(), ref)
    an = a[1].view(torch.int16).cpu().numpy().view(np.uint16)
    bn = b[1].view(torch.int16).cpu().numpy().view(np.uint16)
    want = np.ones((N, M), dtype=np.float32)
    ou.orc_gemm_bf16_tn_flat(an.ravel(), K, bn.ravel(), K, want.ravel(), M, M, N, K, 4096, 4104, 8000, 8008)
    assert (c[1].cpu().numpy()[8000:8008, 4096:4104] == want[8000:8008, 4096:4104]).all()


# ---- layout-driven tiling (north_star: "tiled GEMM partitioned by local_tile / local_partition / TiledMMA") ----------------
TILERS = [(128, 128, 64), (128, 256, 64), (256, 128, 64), (256, 256, 64), (512, 256, 64)]
TILER_PLANS = {(128, 128): "umma_1sm_n128", (128, 256): "umma_1sm", (256, 128): "umma_2sm_n128", (256, 256): "umma_2sm",
               (512, 256): "umma_2sm_wide"}


def _tiled_case(la, lb, lc, tiler, kat=True, seed=0):
    M, N, K = _dims(la, lb)
    na, nb, nc = ou.cosize_of(la), ou.cosize_of(lb), ou.cosize_of(lc)
    rng = np.random.default_rng(seed)
    ao = ou.orc_eval_range(la, 0, M * K).reshape(K, M).T
    bo = ou.orc_eval_range(lb, 0, N * K).reshape(K, N).T
    a, b = np.zeros(na, dtype=np.float32), np.zeros(nb, dtype=np.float32)
    if kat:
        i, p = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
        a[ao] = (i * 7 + p * 3 + 1) % 11
        j, p = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
        b[bo] = (j * 5 + p * 2 + 2) % 13
        c0 = (np.arange(nc) % 5 - 2).astype(np.float32)
    else:
        a[ao] = rng.uniform(-1, 1, (M, K))
        b[bo] = rng.uniform(-1, 1, (N, K))
        c0 = rng.uniform(-1, 1, nc).astype(np.float32)
    ab, bb = ou.f32_to_bf16_bits(a), ou.f32_to_bf16_bits(b)
    want = c0.copy()
    st, sabs = ou.orc_gemm_bf16(la, ab, lb, bb, lc, want, want_abs=True)
    assert st == 0
    ta_, tb_, tc_ = dev(ab.view(np.int16)), dev(bb.view(np.int16)), dev(c0)
    ta, tb, tc = (host.tensor_of(t, buf, ranked=True) for t, buf in ((la, ta_), (lb, tb_), (lc, tc_)))
    plan = host.gemm_bf16_tiled(ta, tb, tc, tiler)
    torch.cuda.synchronize()
    got = tc_.cpu().numpy()
    if kat:
        assert (got == want).all(), f"{plan} tiler {tiler}: {int((got != want).sum())} of {got.size} cells differ"
    else:
        touched = sabs > 0
        assert (np.abs(got - want)[touched] <= (RTOL * sabs + ATOL)[touched]).all()
        assert (got[~touched] == want[~touched]).all()
    return plan


@pytest.mark.parametrize("tiler", TILERS)
@pytest.mark.parametrize("shape", [
    ("(512,256):(256,1)", "(768,256):(256,1)", "(512,768):(768,1)"),      # n-contiguous C: the tiler applies as given
    ("(1000,200):(200,1)", "(300,200):(200,1)", "(1000,300):(300,1)"),    # ragged M, N, K
    ("(1024,520):(528,1)", "(768,520):(536,1)", "(1024,768):(800,1)"),    # padded leading dimensions
])
def test_gemm_partitioned_by_a_caller_chosen_tiler(shape, tiler):
    """tlb_gemm_bf16_tiled: the CTA tile, the k-block boxes and the UMMA atom all follow from the tiler [bm, bn, bk]
    (zipped_divide tile modes -> tensor maps; 128 x N x 16 or 256 x N x 16 atoms): every tiler gives the exact result."""
    assert _tiled_case(*shape, tiler, kat=True) == TILER_PLANS[tiler[:2]]
    _tiled_case(*shape, tiler, kat=False, seed=23)


@pytest.mark.parametrize("tiler", TILERS)
def test_gemm_tiler_on_the_papers_tn_layout(tiler):
    """TN: C is m-contiguous, the plan runs C^T, so the caller's [bm, bn] becomes [bn, bm] rows x columns."""
    shape = ("(768,256):(256,1)", "(512,256):(256,1)", "(768,512):(1,768)")
    user = (tiler[1], tiler[0], 64)                                     # chosen so that the plan's tile is `tiler`
    assert _tiled_case(*shape, user, kat=True) == TILER_PLANS[tiler[:2]]


def test_gemm_tiler_contracts():
    shape = ("(512,256):(256,1)", "(768,256):(256,1)", "(512,768):(768,1)")
    for bad in [(64, 128, 64), (128, 64, 64), (128, 128, 32), (512, 128, 64), (192, 256, 64)]:
        with pytest.raises(TlbError) as e:
            _tiled_case(*shape, bad)
        assert e.value.status == abi.TLB_ERR_UNSUPPORTED
    with pytest.raises(TlbError) as e:                                  # BLIS strides: SIMT plan, no tiler
        _tiled_case("(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)", (128, 128, 64))
    assert e.value.status == abi.TLB_ERR_UNSUPPORTED


def test_gemm_tensor_maps_come_from_the_divided_layouts_and_are_cached():
    """The tensor maps of a GEMM call are derived from zipped_divide tile modes (tlb_tensormap_describe shows the same
    dimensions) and encoded once: a second call on the same buffers is served from the mutex-guarded cache."""
    rank, dims, strides, box = host.tensormap_describe("(4096,4096):(4096,1)", "(256,64):(4096,1)")
    assert (rank, dims, strides, box) == (2, [4096, 4096], [1, 4096], [64, 256])      # A k-blocks of the wide plan
    M = 1024
    a = torch.zeros(M * M, dtype=torch.int16, device="cuda")
    c = torch.zeros(M * M, dtype=torch.float32, device="cuda")
    ta = host.tensor_of(f"({M},{M}):({M},1)", a, ranked=True)
    tc = host.tensor_of(f"({M},{M}):({M},1)", c, ranked=True)
    host.gemm_bf16(ta, ta, tc)
    h0, m0 = host.tensormap_cache_stats()
    for _ in range(5):
        host.gemm_bf16(ta, ta, tc)
    torch.cuda.synchronize()
    h1, m1 = host.tensormap_cache_stats()
    assert m1 == m0 and h1 - h0 >= 10                                    # 5 calls x (A = B map, C map), no new encode


def test_locate_offsets_matches_the_reference():
    """tlb_locate_offsets vs tla::locate_offsets (analysis.hpp:40-56): the reference's own goldens (test_analysis.cpp:84-108),
    the tcgen05.ld 32x32b partition of TMEM accumulators, and inadmissible offsets."""
    for row in ou.golden("locate.json"):
        if row["status"] != 0:
            with pytest.raises(TlbError) as e:
                host.locate_offsets(row["A"], row["T"])
            assert e.value.status == abi.TLB_ERR_ADMISSIBILITY, (row["A"], row["T"])
            continue
        modes = host.locate_offsets(row["A"], row["T"])
        n = len(row["R_values"])
        text = (f"{modes[0][0]}:{modes[0][1]}" if len(modes) == 1 else
                "(" + ",".join(str(e) for e, _ in modes) + "):(" + ",".join(str(s) for _, s in modes) + ")")
        assert ou.orc_eval_range(text, 0, n).tolist() == row["R_values"], (row["A"], row["T"], text)
    # the partition the kernels use: 32 lanes x 32 columns per tcgen05.ld.32x32b.x32 of a (128, N):(65536, 1) accumulator
    assert host.locate_offsets("(128,512):(65536,1)", "(32,32):(1,65536)") == [(32, 128), (32, 1)]


# ---- folded (GETT) and strided (BLIS) operand families at scale (test_tensor.cpp:187-189) ---------------
GETT_SHAPES = [
    # A[(m0,m1),(k0,k1)] K-major with folded rows AND folded k, B[n,(k0,k1)], plain C: rank-5 / rank-4 operand maps
    ("((128,8),(64,8)):((64,65536),(1,8192))", "(512,(64,8)):(64,(1,32768))", "(1024,512):(512,1)"),
    # the same contraction with the paper's TN output
    ("((128,8),(64,8)):((64,65536),(1,8192))", "(512,(64,8)):(64,(1,32768))", "(1024,512):(1,1024)"),
    # A[(m0,m1),k] m0-contiguous (MN-major, folded m), C[(m0,m1),n] folded the same way: the epilogue's reduce-add map is rank 4
    ("((64,16),512):((1,32768),64)", "(768,512):(512,1)", "((64,16),768):((1,49152),64)"),
    # folded n on B and on C's columns, ragged K
    ("(512,200):(200,1)", "((64,8),200):((200,16000),1)", "(512,(64,8)):(1024,(1,128))"),
]


@pytest.mark.parametrize("shape", GETT_SHAPES)
def test_gemm_gett_folded_modes_on_tensor_cores(shape):
    """GETT: modes folded into several leaves. Each leaf is a TMA dimension of a rank-4/5 tensor map derived from the
    divided layout; the producer decomposes a tile's 1-D coordinate into per-leaf coordinates. Exact on the reference's
    integer fills, within tolerance on random data."""
    assert _bf16_case(*shape, kat=True).startswith("umma_2sm")
    assert _bf16_case(*shape, kat=False, seed=29).startswith("umma_2sm")


def test_gemm_gett_folded_modes_on_every_tensor_core_plan(tlb_config):
    shape = GETT_SHAPES[0]
    assert _bf16_case(*shape, kat=True, path=2) == "umma_1sm"
    assert _bf16_case(*shape, kat=True, path=3) == "umma_2sm"
    tlb_config("GEMM_WIDE", "1")
    assert _bf16_case(*shape, kat=True, path=3) == "umma_2sm_wide"
    assert _tiled_case(*shape, (128, 128, 64)) == "umma_1sm_n128"


@pytest.mark.parametrize("shape", [
    ("(512,256):(3,1549)", "(384,256):(2,771)", "(512,384):(5,2563)"),                       # BLIS: no unit stride anywhere
    ("((2,256),256):((1,512),2)", "(384,256):(256,1)", "((2,256),384):((1,2),512)"),           # the reference's GETT row scaled: k stride 2
    ("(300,200):(f1,f512)", "(100,200):(200,1)", "(300,100):(1,300)"),                       # Xor-strided operand
    ("(333,77):(77,1)", "(129,77):(1,129)", "(333,129):(129,1)"),                            # odd extents, unaligned leading dimensions
])
def test_gemm_simt_tiled_plan_is_exact_on_strided_families(shape):
    """Layouts TMA cannot address (no unit-stride leaf, strides that are not multiples of 16 bytes, Xor strides) run on the
    tiled SIMT plan: offset tables per tile, fp32 staging in shared memory, k ascending per output -> bit-exact."""
    assert _bf16_case(*shape, kat=True).startswith("simt")
    assert _bf16_case(*shape, kat=False, seed=31).startswith("simt")
    assert _bf16_case(*shape, kat=False, seed=37, f16=True).startswith("simt")


PACKED_SHAPES = [
    ("(512,256):(3,1549)", "(384,256):(2,771)", "(512,384):(5,2563)"),                       # BLIS: no unit stride anywhere
    ("((2,256),256):((1,512),2)", "(384,256):(256,1)", "((2,256),384):((1,2),512)"),           # GETT row with k stride 2
    ("(300,200):(f1,f512)", "(100,200):(200,1)", "(300,100):(1,300)"),                       # Xor-strided operand
    ("(333,77):(77,1)", "(129,77):(1,129)", "(333,129):(129,1)"),                            # unaligned leading dimensions
    ("(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)"),                                        # test_tensor.cpp:187 verbatim
]


@pytest.mark.parametrize("shape", PACKED_SHAPES)
def test_gemm_packed_plan_runs_unaddressable_layouts_on_tensor_cores(shape, tlb_config):
    """Layouts no tensor map can address take the packed plan once the problem is large enough: tlb_copy packs A, B
    (K-major) and C (n-contiguous), the tcgen05 plan runs on the packed tensors, tlb_copy scatters C back. Forced here
    on small shapes (GEMM_PACK_MIN = 0) so the oracle stays cheap: exact on the reference's integer fills, within the
    GEMM tolerance on random data, C += semantics kept (c_init)."""
    tlb_config("GEMM_PACK_MIN", "0")
    assert _bf16_case(*shape, kat=True).startswith("packed+umma")
    assert _bf16_case(*shape, kat=False, seed=41).startswith("packed+umma")
    assert _bf16_case(*shape, kat=False, seed=43, f16=True).startswith("packed+umma")
    tlb_config("GEMM_PACK", "0")
    assert _bf16_case(*shape, kat=True).startswith("simt")


def test_gemm_packed_plan_default_threshold_and_size():
    """Default knobs: a 1024 x 768 x 512 BLIS-strided problem (2^28.6 MACs) is packed; partial tile ranges and the
    forced SIMT path are not. C cells outside the layout's image stay untouched (cosize > size)."""
    shape = ("(1024,512):(3,3079)", "(768,512):(2,1543)", "(1024,768):(5,5123)")
    assert _bf16_case(*shape, kat=True) == "packed+umma_2sm_wide" or _bf16_case(*shape, kat=True).startswith("packed+umma")
    assert _bf16_case(*shape, kat=True, path=1).startswith("simt")
    tiles = _tile_count(*shape)
    assert _bf16_case(*shape, kat=True, tile_ranges=[(0, 2), (2, tiles)]).startswith("simt")


def _im2col(n, h, w, c, r, s, kout):
    """NHWC activations, stride 1, no padding: A = ((Q,P,N),(C,S,R)) over the input buffer, B = filters (Kout, C S R),
    C = NHWC output. A is non-injective (windows overlap): it is only read."""
    p, q = h - r + 1, w - s + 1
    la = f"(({q},{p},{n}),({c},{s},{r})):(({c},{w * c},{h * w * c}),(1,{c},{w * c}))"
    lb = f"({kout},{c * s * r}):({c * s * r},1)"
    lc = f"({q * p * n},{kout}):({kout},1)"
    return la, lb, lc


@pytest.mark.parametrize("dims", [(2, 18, 18, 64, 3, 3, 128), (1, 34, 34, 64, 3, 3, 256), (4, 10, 18, 64, 3, 3, 64)])
def test_gemm_conv_im2col_layout_on_tensor_cores(dims):
    """CONV row of the paper's GEMM table: fprop as C(m, kout) += A(m, k) B(kout, k) with A the im2col
    LAYOUT of the input (five leaves -> a rank-5 tensor map without a batch dimension), no im2col buffer is materialised.
    Exact on the reference's integer fills against the oracle's evaluation of the same layouts."""
    shape = _im2col(*dims)
    assert _bf16_case(*shape, kat=True).startswith("umma_")
    assert _bf16_case(*shape, kat=False, seed=47).startswith("umma_")


def test_gemm_wide_plan_chunked_launches_are_exact(tlb_config):
    """Long tile ranges are cut into several launches of a few waves each (the workers of a persistent launch drift apart
    and stop sharing operand panels in L2: DESIGN.md 3.3). Forced here with one wave per launch on a 5-batch problem whose
    launch boundaries fall inside batches: same exact result as one launch, more launches counted."""
    M, N, K, B = 2048, 2048, 256, 5
    i = torch.arange(M, device="cuda").view(M, 1)
    p = torch.arange(K, device="cuda").view(1, K)
    a1 = ((i * 7 + p * 3 + 1) % 11).to(torch.bfloat16)
    b1 = ((i * 5 + p * 2 + 2) % 13).to(torch.bfloat16)
    a = torch.stack([a1.roll(bi, 0) for bi in range(B)]).contiguous()
    b = torch.stack([b1.roll(-bi, 0) for bi in range(B)]).contiguous()
    ta = host.make_tensor(L(f"({M},{K}):({K},1)").lower(ranked=True), a.data_ptr(), a.numel(), 2)
    tb = host.make_tensor(L(f"({N},{K}):({K},1)").lower(ranked=True), b.data_ptr(), b.numel(), 2)
    lib = abi.load()
    tlb_config("GEMM_WIDE", "1")
    results, launches = [], []
    for waves in ("0", "1"):
        tlb_config("GEMM_CHUNK_WAVES", waves)
        c = torch.ones(B, N, M, dtype=torch.float32, device="cuda")
        tc = host.make_tensor(L(f"({M},{N}):(1,{M})").lower(ranked=True), c.data_ptr(), c.numel(), 4)
        n0 = lib.tlb_launch_count()
        assert host.gemm_bf16_batched((ta, None), (tb, None), (tc, None), M * K, N * K, M * N, 0, B) == "umma_2sm_wide"
        torch.cuda.synchronize()
        launches.append(int(lib.tlb_launch_count() - n0))
        results.append(c)
    assert launches[0] == 1 and launches[1] >= 2
    for bi in range(B):
        ref = (a[bi].double() @ b[bi].double().t()).t() + 1.0
        assert torch.equal(results[0][bi].double(), ref)
        assert torch.equal(results[1][bi].double(), ref)


@pytest.mark.parametrize("dims", [(512, 1024, 128), (1000, 1024, 200), (768, 512, 72)])
def test_gemm_wide_multicast_plan_matches_the_oracle(dims, tlb_config):
    """Clusters of 4: two CTA pairs on n-adjacent pair tiles share the A rows, every CTA loads a quarter and multicasts it
    to its counterpart (cta_group::2 + multicast TMA; stage release needs both pairs). Exact on the integer fills against
    the oracle, incl. a ragged M and a K that is not a multiple of 64; random data within the GEMM tolerance."""
    M, N, K = dims
    tlb_config("GEMM_WIDE", "1")
    tlb_config("GEMM_MCAST", "1")
    la, lb, lc = f"({M},{K}):({K},1)", f"({N},{K}):({K},1)", f"({M},{N}):({N},1)"
    assert _bf16_case(la, lb, lc, kat=True) == "umma_2sm_wide_mc"
    assert _bf16_case(la, lb, lc, kat=False, seed=53) == "umma_2sm_wide_mc"
    # m-contiguous C (the paper's TN row) runs transposed: the columns of the plan are then m
    assert _bf16_case(la, lb, f"({M},{N}):(1,{M})", kat=True) == ("umma_2sm_wide_mc" if ((M + 255) // 256) % 2 == 0 else "umma_2sm_wide")


def test_gemm_wide_multicast_plan_stream_k_exact(tlb_config):
    """64 cluster tiles on the 33 co-resident clusters of 4: the partial wave is cut into k-ranges that BOTH pairs of a
    cluster walk in lockstep. Exact against an fp64 product of the integer fills."""
    M = N = 4096
    K = 1024
    i = torch.arange(M, device="cuda").view(M, 1)
    p = torch.arange(K, device="cuda").view(1, K)
    a = ((i * 7 + p * 3 + 1) % 11).to(torch.bfloat16).contiguous()
    b = ((i * 5 + p * 2 + 2) % 13).to(torch.bfloat16).contiguous()
    ref = a.double() @ b.double().t() + 1.0
    ta = host.make_tensor(L(f"({M},{K}):({K},1)").lower(ranked=True), a.data_ptr(), a.numel(), 2)
    tb = host.make_tensor(L(f"({N},{K}):({K},1)").lower(ranked=True), b.data_ptr(), b.numel(), 2)
    tlb_config("GEMM_MCAST", "1")
    tlb_config("GEMM_WIDE", "1")
    c = torch.ones(M, N, dtype=torch.float32, device="cuda")
    tc = host.make_tensor(L(f"({M},{N}):({N},1)").lower(ranked=True), c.data_ptr(), c.numel(), 4)
    assert host.gemm_bf16((ta, None), (tb, None), (tc, None)) == "umma_2sm_wide_mc"
    torch.cuda.synchronize()
    assert torch.equal(c.double(), ref)


def test_c4_full_size_64_batches_by_linearity():
    """Config C4 at BASELINE's full size: 64 x (8192 x 8192 x 8192), batch strides, TN with m-contiguous C, one call (cut into
    one launch per batch by the library). The oracle cannot run 7e13 MACs, so the check is a size-independent property of
    the exact integer fills (every partial sum < 2^24, fp32 accumulation exact in any order): for every batch,
    row sums and column sums of C - C0 equal the matrix-vector products with the operands' column sums (linearity),
    computed exactly in fp64 / int64. A wrong, missing or doubled tile changes at least one row sum and one column sum."""
    M = N = K = 8192
    B = 64
    i = torch.arange(M, device="cuda").view(M, 1)
    p = torch.arange(K, device="cuda").view(1, K)
    a = torch.empty(B, M, K, dtype=torch.bfloat16, device="cuda")
    b = torch.empty(B, N, K, dtype=torch.bfloat16, device="cuda")
    for bi in range(B):
        a[bi] = ((i * 7 + p * 3 + 1 + bi) % 11).to(torch.bfloat16)
        b[bi] = ((i * 5 + p * 2 + 2 + 3 * bi) % 13).to(torch.bfloat16)
    c = torch.ones(B, N, M, dtype=torch.float32, device="cuda")           # C(m, n) at m + M n: stored as [n][m]
    ta = host.make_tensor(L(f"({M},{K}):({K},1)").lower(ranked=True), a.data_ptr(), a.numel(), 2)
    tb = host.make_tensor(L(f"({N},{K}):({K},1)").lower(ranked=True), b.data_ptr(), b.numel(), 2)
    tc = host.make_tensor(L(f"({M},{N}):(1,{M})").lower(ranked=True), c.data_ptr(), c.numel(), 4)
    lib = abi.load()
    n0 = lib.tlb_launch_count()
    assert host.gemm_bf16_batched((ta, None), (tb, None), (tc, None), M * K, N * K, M * N, 0, B) == "umma_2sm_wide"
    torch.cuda.synchronize()
    assert lib.tlb_launch_count() - n0 == B                                 # one launch per batch (GEMM_CHUNK_WAVES)
    for bi in range(B):
        ad, bd = a[bi].double(), b[bi].double()
        cd = c[bi].double() - 1.0                                           # [n][m]
        # sum over n of C(m, n) = sum_k A(m, k) * colsum_B(k); sum over m of C(m, n) = sum_k B(n, k) * colsum_A(k)
        assert torch.equal(cd.sum(dim=0), ad @ bd.sum(dim=0)), f"batch {bi}: row sums"
        assert torch.equal(cd.sum(dim=1), bd @ ad.sum(dim=0)), f"batch {bi}: column sums"
    # and one sampled tile of the last batch against the flat restatement
    an = a[B - 1].view(torch.int16).cpu().numpy().view(np.uint16)
    bn = b[B - 1].view(torch.int16).cpu().numpy().view(np.uint16)
    want = np.ones((N, M), dtype=np.float32)
    ou.orc_gemm_bf16_tn_flat(an.ravel(), K, bn.ravel(), K, want.ravel(), M, M, N, K, 512, 520, 7680, 7688)
    assert (c[B - 1].cpu().numpy()[7680:7688, 512:520] == want[7680:7688, 512:520]).all()


def _fuzz_gemm_case(rng):
    """One random GEMM problem over the layout families of test_tensor.cpp:176-195: K- or MN-major operands with padded
    (aligned or unaligned) leading dimensions, optionally a mode folded into two leaves (GETT) or strided (BLIS), C m- or
    n-contiguous."""
    M, N, K = int(rng.integers(1, 18)) * 64, int(rng.integers(1, 14)) * 64, int(rng.integers(1, 40)) * 16
    if rng.random() < 0.3:
        M, N, K = M - int(rng.integers(0, 60)), N - int(rng.integers(0, 60)), K - int(rng.integers(0, 15))

    def operand(rows, k):
        kind = rng.choice(["k_major", "mn_major", "folded", "strided"], p=[0.4, 0.3, 0.2, 0.1])
        pad = int(rng.choice([0, 8, 24, 3]))
        if kind == "k_major":
            return f"({rows},{k}):({k + pad},1)"
        if kind == "mn_major":
            return f"({rows},{k}):(1,{rows + pad})"
        if kind == "folded" and rows % 128 == 0 and k % 64 == 0:
            r0, k0 = 64, 32                                  # rows = (r0, rows / r0), k = (k0, k / k0): four leaves
            return f"(({r0},{rows // r0}),({k0},{k // k0})):(({k0},{k0 * r0 * (k // k0)}),(1,{k0 * r0}))"
        if kind == "strided":
            return f"({rows},{k}):(3,{3 * rows + 5})"
        return f"({rows},{k}):({k + pad},1)"

    la, lb = operand(M, K), operand(N, K)
    pad = int(rng.choice([0, 4, 12, 1]))
    lc = f"({M},{N}):({N + pad},1)" if rng.random() < 0.5 else f"({M},{N}):(1,{M + pad})"
    return la, lb, lc


_FUZZ_PLANS = set()


@pytest.mark.parametrize("seed", range(20))
def test_gemm_fuzz_layout_families_against_the_oracle(seed, tlb_config):
    """Differential fuzz through every GEMM plan the planner may pick (tcgen05 1-CTA / 2-CTA / wide, register and TMA
    epilogues, rank-4/5 tensor maps, packed, SIMT): 8 random problems per seed against the sequential-k restatement,
    bf16 and fp16, exact where the plan keeps the reference's order, within the stated tolerance elsewhere."""
    rng = np.random.default_rng(1000 + seed)
    if seed % 2:
        tlb_config("GEMM_WIDE", "1")   # odd seeds: the wide plan wherever it applies (the planner keeps it for K >= 4096)
    plans = set()
    for _ in range(8):
        la, lb, lc = _fuzz_gemm_case(rng)
        plans.add(_bf16_case(la, lb, lc, kat=bool(rng.random() < 0.3), seed=int(rng.integers(1 << 30)), f16=bool(rng.random() < 0.3)))
    _FUZZ_PLANS.update(plans)
    if seed == 19:   # the fuzz must actually reach the tensor-core plans, the packed plan and the SIMT plan
        kinds = {p.split("+")[0].replace("_regs", "") for p in _FUZZ_PLANS}
        assert {"umma_2sm", "umma_2sm_wide", "packed"} <= kinds and any(k.startswith("simt") for k in kinds), _FUZZ_PLANS


@pytest.mark.parametrize("shape", [
    ("(1,64):(64,1)", "(256,64):(64,1)", "(1,256):(256,1)"),        # one row of C
    ("(256,64):(64,1)", "(1,64):(64,1)", "(256,1):(1,256)"),        # one column of C
    ("(128,1):(1,128)", "(128,1):(1,128)", "(128,128):(128,1)"),    # K = 1: an outer product
    ("(1,1):(1,1)", "(1,1):(1,1)", "(1,1):(1,1)"),                  # a single multiply-add
    ("(8,8):(8,1)", "(8,8):(8,1)", "(8,8):(8,1)"),                  # far below one tile
    ("((1,130),(1,72)):((5,72),(7,1))", "(65,72):(72,1)", "(130,(65,1)):(65,(1,9))"),   # extent-1 leaves inside the modes
    ("(257,72):(72,1)", "(513,72):(72,1)", "(257,513):(520,1)"),    # one row / column past a tile boundary
])
def test_gemm_degenerate_and_ragged_extents(shape):
    """Degenerate extents (single rows / columns, K = 1, extent-1 leaves) and shapes one past a tile boundary, on whatever
    plan the planner picks, in both value types: exact on the integer fills, within tolerance on random data."""
    _bf16_case(*shape, kat=True)
    _bf16_case(*shape, kat=False, seed=61)
    _bf16_case(*shape, kat=False, seed=67, f16=True)
    _bf16_case(*shape, kat=True, path=1)                             # and on the SIMT plan


@pytest.mark.parametrize("f16", [False, True])
def test_gemm_packed_plan_with_c_in_the_operand_type(f16, tlb_config):
    """The packed plan with a 2-byte C: C is gathered into an n-contiguous 2-byte tile buffer, the tcgen05 plan adds into it
    in that type (one rounding), and the copy scatters it back through C's strided layout."""
    tlb_config("GEMM_PACK_MIN", "0")
    assert _c16_case(("(512,256):(3,1549)", "(384,256):(2,771)", "(512,384):(5,2563)"), f16).startswith("packed+umma")
    assert _c16_case(("(300,200):(f1,f512)", "(100,200):(200,1)", "(300,100):(1,301)"), f16).startswith("packed+umma")

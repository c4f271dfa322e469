"""GPU parity: bulk layout evaluation (config C5) through the C ABI vs the oracle — bit-exact int64."""
import numpy as np
import pytest
import torch

import oracle_util as ou
from gpu_util import dev
from paper_2603_02298_b200 import L, TlbError, abi, host

pytestmark = pytest.mark.gpu


def _eval(text, i0, n):
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    host.eval_range(text, i0, n, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def test_eval_matches_reference_fixtures():
    for row in ou.golden("eval.json"):
        want = np.array(row["values"], dtype=np.int64)
        got = _eval(row["layout"], 0, len(want))
        assert (got == want).all(), row["layout"]


def test_eval_known_answers_from_reference_tests():
    assert _eval("((2,2),(4,2)):((1,8),(2,16))", 22, 1)[0] == 26      # test_layout.cpp:76
    assert _eval("(4,8):(-1,4)", 3, 1)[0] == -3                      # test_layout.cpp:184
    assert _eval("(8,8):(f1,f9)", 9, 1)[0] == 8                      # test_layout.cpp:96
    x = np.arange(4096, dtype=np.int64)
    assert (_eval("(128,8,4):(f1,f144,f1024)", 0, 4096) == (x ^ ((x >> 3) & 0x70))).all()  # Swizzle<3,4,3>


@pytest.mark.parametrize("text", [
    "(3,5,7):(35,7,1)", "(6,(5,3)):(1,(18,6))", "((3,5),2):((7,0),100)", "(5,6):(f3,f40)", "(1000,999):(999,1)",
    "((128,64),(512,1024)):((65536,1),(8388608,64))", "(64,1024,128,512):(128,4194304,1,8192)", "(7,11,13,17):(1,7,77,1001)",
])
@pytest.mark.parametrize("odd", [False, True])
def test_eval_random_windows_vs_oracle(text, odd):
    size = L(text).size
    rng = np.random.default_rng(1)
    for i0 in [0, int(rng.integers(0, max(size - 5000, 1)))]:
        n = min(4097 if odd else 4096, size - i0)
        out = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        view = out[1:] if odd else out[:n]                      # odd: misaligned output (scalar store path)
        host.eval_range(text, i0, n, view)
        torch.cuda.synchronize()
        assert (view.cpu().numpy()[:n] == ou.orc_eval_range(text, i0, n)).all()


def test_c5_index_maps_sampled_at_full_size():
    """2^32-element divided layout: windows spread over the whole domain + the reference's sampled anchors."""
    ops = ou.golden("ops.json")
    Lt, Rt = ops["C5_L"], ops["C5_R"]
    for i0 in [0, 2**31 - 2048, 2**32 - 4096, 123456789, 3 * 2**30 + 77]:
        assert (_eval(Lt, i0, 4096) == ou.orc_eval_range(Lt, i0, 4096)).all()
        assert (_eval(Rt, i0, 4096) == ou.orc_eval_range(Rt, i0, 4096)).all()
    idx = ops["C5_samples_i"]
    for i, lv, rv in list(zip(idx, ops["C5_L_values"], ops["C5_R_values"]))[::64]:
        assert _eval(Lt, i, 1)[0] == lv and _eval(Rt, i, 1)[0] == rv


@pytest.mark.parametrize("i0", [0, 15 * 2**28, 2**32 - 2**21, 5 * 2**28 + 96])
def test_c5_windows_through_the_kernel_the_bench_times(i0):
    """bench.py materialises C5 in 2^28-element chunks, which selects eval_warp_kernel<32> (groups of 32 indices, one peel
    per lane, bases by shuffle). The 4096-element windows above select G = 8, so this runs 2^21-element windows through
    the G = 32 warp kernel (asserted through tlb_last_plan) at the first chunk, the last chunk, the end of the domain and
    a start that is 32- but not 128-aligned, against the oracle on every element. The output is 32-byte aligned as in
    the bench."""
    ops = ou.golden("ops.json")
    n = 2**21
    for text in (ops["C5_L"], ops["C5_R"]):
        got = _eval(text, i0, n)
        assert abi.load().tlb_last_plan().decode() == "eval_warp32"
        assert (got == ou.orc_eval_range(text, i0, n)).all()


def test_c5_non_group_aligned_start_falls_back_and_stays_exact():
    ops = ou.golden("ops.json")
    n = 2**20 + 5
    got = _eval(ops["C5_L"], 7 * 2**28 + 3, n)                # i0 % 2 != 0: no group size applies, the odometer kernel
    assert abi.load().tlb_last_plan().decode() == "eval_odo"
    assert (got == ou.orc_eval_range(ops["C5_L"], 7 * 2**28 + 3, n)).all()
    got = _eval(ops["C5_L"], 7 * 2**28 + 16, n)               # i0 % 16 == 0: G = 16 warp kernel + group + scalar tails
    assert abi.load().tlb_last_plan().decode() == "eval_warp16"
    assert (got == ou.orc_eval_range(ops["C5_L"], 7 * 2**28 + 16, n)).all()


@pytest.mark.parametrize("text", [
    "(3,1048576,64):(1,3,3145728)",            # leading leaf of 3 cells
    "(5,7,11,13,1000):(1,5,35,385,5005)",      # small odd leaves: leaf 1 wraps every 35 indices
    "(3,2,1000,1000):(2000000,7,1,1000)",      # e0 * e1 = 6 < the 8 indices of a thread: several re-peels per thread
    "(6,100000):(100000,1)",                   # two leaves: leaf 1 is the last leaf, unbounded
    "(7,9,100):(-1,-7,63)",                    # negative strides
    "(1,3,1,50,4000):(9,1,9,3,150)",           # extent-1 leaves in front
])
def test_eval_odometer_for_leading_leaves_no_group_size_divides(text):
    """Layouts whose leading leaf is not a multiple of 2 (or whose range starts at an odd index) are walked 8 indices per
    thread by an odometer over leaves 0 and 1 (round 2: the per-index peel before, 2 TB/s against 7 TB/s). Every value
    against the oracle, ranges that start anywhere, the extended domain, and the per-index kernel as a cross-check."""
    size = L(text).size
    for i0, n in ((0, min(size, 300000)), (1, 4099), (12345, 65536 + 3), (max(0, size - 1000), 1000 + 77)):
        got = _eval(text, i0, n)
        assert (got == ou.orc_eval_range(text, i0, n)).all(), (text, i0, n, abi.load().tlb_last_plan().decode())
    _eval(text, 1, 4099)                       # an odd start rules out every group size
    assert abi.load().tlb_last_plan().decode() == "eval_odo"
    host.config("EVAL_ODOMETER", "0")
    try:
        got = _eval(text, 1, 4099)
        assert abi.load().tlb_last_plan().decode() == "eval_scalar"
        assert (got == ou.orc_eval_range(text, 1, 4099)).all()
    finally:
        host.config("EVAL_ODOMETER", None)


def test_c5_right_inverse_identity_on_device():
    """L(R(k)) == k for all k of a 2^26 slice at both ends of the 2^32 domain (property at full size)."""
    ops = ou.golden("ops.json")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for k0 in [0, 2**32 - 2**26]:
        host.rinv_check_range(ops["C5_L"], ops["C5_R"], k0, 2**26, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    # and a wrong inverse is detected
    host.rinv_check_range(ops["C5_L"], "(64,1024,128,512):(129,4194304,1,8192)", 0, 2**20, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) > 0


def test_compose_check_on_device():
    # compose((8192,8192):(1,8192), rinv((8192,8192):(8192,1))) = (8192,8192):(8192,1)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    host.compose_check_range("(8192,8192):(1,8192)", "(8192,8192):(8192,1)", "(8192,8192):(8192,1)", 0, 2**26, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    host.compose_check_range("(8192,8192):(1,8192)", "(8192,8192):(8192,1)", "(8192,8192):(8192,2)", 0, 2**20, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) > 0


def test_locate_offsets_verification_on_device():
    """locate_offsets (analysis.hpp:40-56) = compose(left_inverse(A), T) on the host, then the O(size(T)) loop
    A(R(i)) == T(i) that decides admissibility. That loop is tlb_compose_check_range(A, R, T); goldens are the
    reference's own (test_analysis.cpp:84-108): the TMEM-style lane-major accumulator row is admissible, the offset
    that falls into the stride gap of (4,8):(1,5) is not."""
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    # (128,512):(16384,1) located by (1,128):(1,16384) is R = (1,128):(0,1)
    host.compose_check_range("(128,512):(16384,1)", "(1,128):(0,1)", "(1,128):(1,16384)", 0, 128, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    # (4,8):(1,4) located by 5:7: R from the reference evaluates back to 7 i
    host.compose_check_range("(4,8):(1,4)", "5:7", "5:7", 0, 5, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    # (4,8):(1,5) against 2:4: compose(left_inverse(A), T) = 2:4, and A(4) = 5 != 4 -> admissibility_error upstream
    host.compose_check_range("(4,8):(1,5)", "2:4", "2:4", 0, 2, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 1


def test_idx2crd_and_crd2idx_roundtrip():
    text = "((3,2),((2,3),2)):((4,1),((2,15),100))"
    n = L(text).size
    crd = torch.empty(n, 5, dtype=torch.int64, device="cuda")
    host.idx2crd_range(text, 0, n, crd)
    torch.cuda.synchronize()
    assert (crd.cpu().numpy() == ou.orc_idx2crd_range(text, 0, n)).all()
    idx = torch.empty(n, dtype=torch.int64, device="cuda")
    host.crd2idx_range(text, crd, n, idx)
    torch.cuda.synchronize()
    assert (idx.cpu().numpy() == np.arange(n)).all()
    # large shape, window far from zero
    big = "((128,64),(512,1024)):((65536,1),(8388608,64))"
    crd = torch.empty(4096, 4, dtype=torch.int64, device="cuda")
    host.idx2crd_range(big, 2**32 - 4096, 4096, crd)
    host.crd2idx_range(big, crd, 4096, idx := torch.empty(4096, dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    assert (crd.cpu().numpy() == ou.orc_idx2crd_range(big, 2**32 - 4096, 4096)).all()
    assert (idx.cpu().numpy() == np.arange(2**32 - 4096, 2**32)).all()


def test_eval_axes_matches_reference_fixtures_and_oracle():
    """tlb_eval_axes_range (layout_eval_axes, layout.hpp:103) over whole domains: the reference's fixtures (incl.
    coordinate_identity((8,8)) = (8,8):(e0,e1), Table 2: L(c) = c) and the oracle on every index of larger windows."""
    for row in ou.golden("axes.json"):
        na = row["n_axes"]
        for w in row["windows"]:
            want = np.array(w["values"], dtype=np.int64).reshape(-1, na)
            out = torch.empty(want.shape[0], na, dtype=torch.int64, device="cuda")
            host.eval_axes_range(row["layout"], na, w["i0"], want.shape[0], out)
            torch.cuda.synchronize()
            assert (out.cpu().numpy() == want).all(), row["layout"]
    # TMA coordinates of a tiled identity: zipped_divide(coordinate_identity((4096,8192)), [128,64]) evaluated over 2^20
    # indices from a start far from zero; coordinate (tile, in-tile) -> (row, column) of the tile's elements
    t = "((128,64),(32,128)):((e0,e1),(128*e0,64*e1))"
    i0, n = 17 * 2**20 + 13, 2**20
    out = torch.empty(n, 2, dtype=torch.int64, device="cuda")
    host.eval_axes_range(t, 2, i0, n, out)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == ou.orc_eval_axes_range(t, 2, i0, n)).all()
    for t, na in [("(3,5,7):(e2,e0,e1)", 3), ("(2,3,2,5):(e0,2*e1,e2,7*e3)", 4), ("(2,2,2,2,2):(e0,e1,e2,e3,e4)", 5), ("(6,4):(e0,e0)", 1)]:
        n = L(t).size + 3
        out = torch.empty(n + 1, na, dtype=torch.int64, device="cuda")
        for view in (out[:n], out[1:]):                        # aligned and misaligned outputs (vector / scalar stores)
            host.eval_axes_range(t, na, 0, n, view)
            torch.cuda.synchronize()
            assert (view.cpu().numpy() == ou.orc_eval_axes_range(t, na, 0, n)).all(), t


def test_eval_axes_overflow_is_proven_before_launch():
    out = torch.empty(8, 2, dtype=torch.int64, device="cuda")
    with pytest.raises(TlbError) as e:                         # checked_mul in eval_leaf (stride.hpp:152) would wrap
        host.eval_axes_range("(4,8):(4611686018427387904*e0,e1)", 2, 0, 8, out)
    assert e.value.status == abi.TLB_ERR_OVERFLOW


def test_crd2idx_checked_arithmetic():
    """tla::crd2idx accepts any coordinate values and throws overflow_error on a checked_mul / checked_add wrap
    (int_tuple.hpp:154): out-of-range and negative coordinates produce the reference's (oracle's) value, a wrap is
    reported through the status word and leaves the output cell untouched."""
    text = "(4,8,16):(1,4,32)"
    crd = np.array([[1, 2, 3], [7, 9, 20], [-1, 3, 2], [3, -8, 1], [0, 0, 2**40]], dtype=np.int64)
    got = torch.full((5,), -7, dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    host.crd2idx_range(text, dev(crd), 5, got, status_buf=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert (got.cpu().numpy() == ou.orc_crd2idx_range(text, crd)).all()
    bad = np.array([[1, 2, 3], [0, 0, 2**62], [2, 2, 2]], dtype=np.int64)     # 2^62 * 32 wraps
    got = torch.full((3,), -7, dtype=torch.int64, device="cuda")
    host.crd2idx_range(text, dev(bad), 3, got, status_buf=st)
    torch.cuda.synchronize()
    assert int(st.item()) == abi.TLB_ERR_OVERFLOW
    assert got.cpu().numpy().tolist() == [1 + 2 * 4 + 3 * 32, -7, 2 + 2 * 4 + 2 * 32]
    with pytest.raises(RuntimeError):
        ou.orc_crd2idx_range(text, bad)                        # the oracle (and the reference) raise on the same input


def test_eval_axes_coordinate_layout():
    # (4,(4,2)):(e1,(e0,6*e1)) at (1,(2,1)) -> axes (2, 7)   (test_layout.cpp:84-89)
    text = "(4,(4,2)):(e1,(e0,6*e1))"
    out = torch.empty(32, 2, dtype=torch.int64, device="cuda")
    host.eval_axes_range(text, 2, 0, 32, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    i = 1 + 4 * (2 + 4 * 1)
    assert list(got[i]) == [2, 7]


def test_eval_error_contracts():
    out = torch.empty(8, dtype=torch.int64, device="cuda")
    with pytest.raises(TlbError) as e:
        host.eval_range("(4,8):(e0,e1)", 0, 8, out)
    assert e.value.status == abi.TLB_ERR_SEMIMODULE
    with pytest.raises(TlbError) as e:
        host.eval_range("(4,8):(4611686018427387904,1)", 0, 8, out)     # checked_mul would overflow
    assert e.value.status == abi.TLB_ERR_OVERFLOW

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

"""TEST INFRASTRUCTURE: device-side helpers for the -m gpu parity tests."""
import numpy as np
import torch

import oracle_util as ou
from paper_2603_02298_b200 import L, host

NP2T = {np.dtype("uint8"): torch.uint8, np.dtype("int16"): torch.int16, np.dtype("int32"): torch.int32,
        np.dtype("int64"): torch.int64, np.dtype("float32"): torch.float32}


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cells(n: int, eb: int, seed: int = 0, fill=None) -> np.ndarray:
    """n opaque cells of eb bytes as a numpy array of a signed integer dtype (16-byte cells: int64 pairs)."""
    dt = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64, 16: np.int64}[eb]
    m = n * (2 if eb == 16 else 1)
    if fill is not None:
        return np.full(m, fill, dtype=dt)
    rng = np.random.default_rng(seed)
    info = np.iinfo(dt)
    return rng.integers(info.min, info.max, m, dtype=dt, endpoint=True)


def run_copy_case(s: str, d: str, eb: int = 8, src_origin=0, dst_origin=0, path=0, slack=0, seed=0, i_begin=0, i_end=2**64 - 1):
    """GPU tlb_copy vs the C restatement on the same seeded cells; returns the plan name."""
    from paper_2603_02298_b200 import abi
    ns, nd = ou.cosize_of(s) + src_origin + slack, ou.cosize_of(d) + dst_origin + slack
    src = cells(ns, eb, seed)
    dst0 = cells(nd, eb, fill=-1 if eb != 1 else 255)
    want = dst0.copy()
    if eb == 16:
        sv, wv = src.view([("a", np.int64), ("b", np.int64)]), want.view([("a", np.int64), ("b", np.int64)])
        st = ou.orc_copy(s, sv, d, wv, src_origin, dst_origin, i_begin=i_begin, i_end=min(i_end, L(s).size))
    else:
        st = ou.orc_copy(s, src, d, want, src_origin, dst_origin, i_begin=i_begin, i_end=min(i_end, L(s).size))
    assert st == 0
    tsrc, tdst = dev(src), dev(dst0)
    ls, ld = L(s), L(d)
    ds, dd = ls.lower(), ld.lower()
    a = host.make_tensor(ds, tsrc.data_ptr(), ns, eb, src_origin)
    b = host.make_tensor(dd, tdst.data_ptr(), nd, eb, dst_origin)
    prev = abi.load().tlb_copy_set_path(path)
    try:
        plan = host.copy((a, None), (b, None), i_begin, i_end)
    finally:
        abi.load().tlb_copy_set_path(prev)
    torch.cuda.synchronize()
    got = tdst.cpu().numpy()
    assert (got == want).all(), f"copy {s} -> {d} eb={eb} plan={plan}: {int((got != want).sum())} cells differ"
    return plan

"""TEST INFRASTRUCTURE. Regenerates tests/golden/*.json by running the UNMODIFIED reference
(oracle/_ref/libtla_ref.so, built from /root/reference by oracle/Makefile) in this container.
The GPU box has no /root/reference; the committed fixtures are what its tests compare against.

    make -C oracle ref && python oracle/gen_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle_util as ou  # noqa: E402

OUT = ROOT / "tests" / "golden"

EVAL_LAYOUTS = [
    # proj/tests/test_layout.cpp:74-99, test_tensor.cpp:28-32,225-229, acceptance.cpp:33-46
    "((2,2),(4,2)):((1,8),(2,16))", "(4,8):(8,1)", "(4,8):(1,4)", "((3,2),((2,3),2)):((4,1),((2,15),100))",
    "(8,8):(f1,f9)", "(4,8):(-1,4)", "(128,8,4):(f1,f144,f1024)", "(128,8):(f1,f144)",
    # the Table-1 copy layouts (test_tensor.cpp:93-100)
    "8:1", "(8,2,3):(1,16,32)", "(2,3,2):(42,1,128)", "12:1", "7:0", "7:1", "(8,3):(1,8)", "(8,3):(3,1)",
    "(8,(3,5)):(1,(57,8))", "(8,15):(1,8)",
    # gemm families (test_tensor.cpp:176-189)
    "(4,8):(1,9)", "(6,8):(1,10)", "(4,6):(1,7)", "(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)",
    "((2,2),8):((1,16),2)", "((2,2),6):((1,3),52)",
    # non power-of-two / mixed radices / zero strides
    "(3,5,7):(35,7,1)", "(6,(5,3)):(1,(18,6))", "(3,4):(0,1)", "((3,5),2):((7,0),100)", "(5,6):(f3,f40)",
]

COPY_PAIRS = [
    # Table 1 (proj/tests/test_tensor.cpp:93-100, acceptance.cpp:282-285)
    ["8:1", "8:1"], ["(8,2,3):(1,16,32)", "(8,2,3):(1,16,32)"], ["(2,3,2):(42,1,128)", "12:1"],
    ["12:1", "(2,3,2):(42,1,128)"], ["7:0", "7:1"], ["7:0", "7:0"], ["(8,3):(1,8)", "(8,3):(3,1)"],
    ["(8,(3,5)):(1,(57,8))", "(8,15):(1,8)"],
    # beyond Table 1: transposes that hit the tiled plan, swizzles, non-injective destinations, mixed radices
    ["(64,64):(64,1)", "(64,64):(1,64)"], ["(32,128):(1,32)", "(32,128):(128,1)"],
    ["((8,16),(4,8)):((1,256),(8,32))", "((8,16),(4,8)):((16,1),(1024,128))"],
    ["(8,8):(f1,f9)", "64:1"], ["64:1", "(8,8):(f1,f9)"], ["(128,8):(f1,f144)", "(128,8):(8,1)"],
    ["12:1", "(4,3):(1,2)"], ["(4,6):(1,4)", "(4,6):(0,1)"], ["(6,4):(4,1)", "(4,6):(1,4)"],
    ["(3,5,7):(35,7,1)", "(3,5,7):(1,3,15)"], ["(16,3):(3,1)", "(16,3):(1,16)"],
]

GEMM_FAMILIES = [
    # proj/tests/test_tensor.cpp:176-189 (NT, TN, NTT, BLIS, GETT)
    ["(4,8):(1,9)", "(6,8):(1,10)", "(4,6):(1,7)"],
    ["(4,8):(9,1)", "(6,8):(10,1)", "(4,6):(1,7)"],
    ["(6,8):(1,10)", "(4,8):(1,9)", "(6,4):(1,7)"],
    ["(4,8):(3,13)", "(6,8):(2,17)", "(4,6):(5,23)"],
    ["((2,2),8):((1,16),2)", "(6,8):(8,1)", "((2,2),6):((1,3),52)"],
    # larger TN / NT instances and an Xor-strided operand
    ["(40,24):(24,1)", "(56,24):(24,1)", "(40,56):(1,40)"],
    ["(40,24):(24,1)", "(56,24):(24,1)", "(40,56):(56,1)"],
    ["(8,8):(f1,f9)", "(6,8):(8,1)", "(8,6):(1,8)"],
]


AXES_LAYOUTS = [
    # coordinate_identity goldens (proj/tests/test_layout.cpp:158-160), Table 2's (8,8):(e0,e1), the per-axis
    # coordinates of test_layout.cpp:99 and TMA-style coordinate tensors of a divided identity
    ["(4,8):(e0,e1)", 2], ["7:e0", 1], ["(4,(3,2)):(e0,(e1,3*e1))", 2], ["(8,8):(e0,e1)", 2],
    ["((4,2),(8,4)):((e0,4*e0),(e1,8*e1))", 2], ["((128,64),(4,8)):((e0,e1),(128*e0,64*e1))", 2],
    ["(3,5,7):(e2,e0,e1)", 3], ["(4,6):(0,e1)", 2], ["(2,3,2,5):(e0,2*e1,e2,7*e3)", 4], ["(6,4):(e0,e0)", 1],
    ["(2,2,2,2,2):(e0,e1,e2,e3,e4)", 5],
]

ALIAS_CASES = [
    # [src layout, src origin, dst layout, dst origin, storage cells]: both tensors view ONE storage (tensor.hpp:29)
    ["16:1", 0, "16:1", 1, 20],          # shift right by one: every cell becomes cell 0 (read-after-write chain)
    ["16:1", 1, "16:1", 0, 20],          # shift left by one: a plain move (reads stay ahead of the writes)
    ["16:1", 0, "16:1", 0, 16],          # in place
    ["(4,4):(4,1)", 0, "(4,4):(1,4)", 0, 16],   # in-place transpose under the serial order
    ["(8,2):(1,8)", 0, "(8,2):(2,1)", 3, 24],
    ["12:1", 0, "12:2", 1, 30],
    ["(4,6):(1,4)", 2, "(4,6):(6,1)", 0, 30],
    ["(4,6):(1,4)", 0, "(4,6):(0,1)", 2, 30],   # non-injective destination AND overlap
    ["7:0", 3, "7:1", 0, 8],
    ["(8,8):(f1,f9)", 0, "64:1", 8, 80],
]


LOCATE_CASES = [
    # proj/tests/test_analysis.cpp:84-108 first, then TMEM-style tiles with the hardware lane stride (65536) and the paper's (16384)
    ["(128,512):(16384,1)", "(1,128):(1,16384)"], ["(4,8):(1,4)", "5:7"], ["(4,8):(2,8)", "3:3"], ["(4,8):(1,5)", "2:4"],
    ["(128,512):(65536,1)", "(32,32):(1,65536)"], ["(128,256):(65536,1)", "(32,32):(1,65536)"], ["(128,128):(65536,1)", "(32,32):(1,65536)"],
    ["(128,512):(16384,1)", "(2,128):(1,16384)"], ["(128,512):(16384,1)", "(8,(16,4)):(1,(16384,524288))"],
    ["(8,16):(16,1)", "(4,2):(1,32)"], ["(8,16):(16,1)", "(4,4):(2,16)"], ["(6,10):(10,1)", "(3,2):(2,10)"], ["(8,16):(32,1)", "3:16"],
]


def cosize(text):
    st, r = ou.ref_op("cosize", text)
    if st == 0:
        return int(r)
    # Xor / negative-stride layouts: span of the image
    v = ou.ref_eval_range(text, 0, int(ou.ref_op("size", text)[1]))
    return int(v.max() - min(int(v.min()), 0)) + 1


def main():
    assert ou.have_ref(), "build oracle/_ref first: make -C oracle ref"
    OUT.mkdir(parents=True, exist_ok=True)

    ev = []
    for t in EVAL_LAYOUTS:
        n = int(ou.ref_op("size", t)[1])
        vals = ou.ref_eval_range(t, 0, n + 5, 0)           # 5 extended-domain points past the size
        vals2 = ou.ref_eval_range(t, 0, n + 5, 1)          # oracle::oracle_eval_int agrees
        assert (vals == vals2).all(), t
        ev.append({"layout": t, "size": n, "values": vals.tolist()})
    (OUT / "eval.json").write_text(json.dumps(ev))

    cp = []
    for s, d in COPY_PAIRS:
        n_s, n_d = cosize(s), cosize(d)
        src = np.arange(n_s, dtype=np.int64) * 3 + 1       # acceptance.cpp:289 fill
        dst = np.full(n_d, -1, dtype=np.int64)             # test_tensor.cpp:104 pre-fill
        st = ou.ref_copy(s, src, d, dst)
        cp.append({"src": s, "dst": d, "src_len": n_s, "dst_len": n_d, "status": st, "dst_cells": dst.tolist()})
    # counting source, origins, and the error contracts
    dst = np.full(32, -1, dtype=np.int64)
    st = ou.ref_copy("(4,8):(1,4)", None, "(4,8):(8,1)", dst, src_origin=5)
    cp.append({"src": "(4,8):(1,4)", "dst": "(4,8):(8,1)", "counting_base": 5, "dst_len": 32, "status": st,
               "dst_cells": dst.tolist()})
    dst = np.full(8, -1, dtype=np.int64)
    st = ou.ref_copy("8:1", np.arange(8, dtype=np.int64), "4:1", dst)
    cp.append({"src": "8:1", "dst": "4:1", "src_len": 8, "dst_len": 8, "status": st, "error": "size mismatch"})
    dst = np.full(8, -1, dtype=np.int64)
    st = ou.ref_copy("4:3", np.arange(8, dtype=np.int64), "4:1", dst)
    cp.append({"src": "4:3", "dst": "4:1", "src_len": 8, "dst_len": 8, "status": st, "error": "source out of bounds"})
    (OUT / "copy.json").write_text(json.dumps(cp))

    gm = []
    for la, lb, lc in GEMM_FAMILIES:
        La, Lb, Lc = ou.as_layout(la), ou.as_layout(lb), ou.as_layout(lc)
        na, nb, nc = cosize(la), cosize(lb), cosize(lc)
        M = int(np.prod([e for e, *_ in La.modes[:La.top_leaves[0]]]))
        N = int(np.prod([e for e, *_ in Lb.modes[:Lb.top_leaves[0]]]))
        K = int(np.prod([e for e, *_ in La.modes[La.top_leaves[0]:]]))
        a = np.zeros(na, dtype=np.int64)
        b = np.zeros(nb, dtype=np.int64)
        c = np.zeros(nc, dtype=np.int64)
        # the reference's own fills (test_tensor.cpp:155,161), stored through the layouts
        for i in range(M):
            for p in range(K):
                st, off = ou.ref_op("eval_coord", la, f"({i},{p})")
                a[int(off.lstrip("f"))] = (i * 7 + p * 3 + 1) % 11
        for j in range(N):
            for p in range(K):
                st, off = ou.ref_op("eval_coord", lb, f"({j},{p})")
                b[int(off.lstrip("f"))] = (j * 5 + p * 2 + 2) % 13
        c0 = (np.arange(nc, dtype=np.int64) % 5) - 2        # C += ...: a non-zero starting accumulator
        c[:] = c0
        st = ou.ref_gemm(la, a, lb, b, lc, c)
        gm.append({"A": la, "B": lb, "C": lc, "M": M, "N": N, "K": K, "a": a.tolist(), "b": b.tolist(),
                   "c0": c0.tolist(), "c": c.tolist(), "status": st})
    (OUT / "gemm.json").write_text(json.dumps(gm))

    # config C5 and C3 layouts as the reference derives them
    ops = {}
    st, ops["C5_L"] = ou.ref_op("zipped_divide", "(65536,65536):(65536,1)", "[128,64]")
    st, ops["C5_R"] = ou.ref_op("right_inverse", ops["C5_L"])
    st, ops["C3_src_rinv"] = ou.ref_op("right_inverse", "((8,128),(4,64),4096):((1,2048),(8,32),262144)")
    st, ops["C3_dst_rinv"] = ou.ref_op("right_inverse", "((8,128),(4,64),4096):((128,1),(65536,1024),262144)")
    st, ops["C1_mcv"] = ou.ref_op("max_common_vector", "(64,64):(64,1)", "(64,64):(1,64)")
    st, ops["local_tile_3_5"] = ou.ref_op("slice", ou.ref_op("zipped_divide", "(4096,4096):(4096,1)", "[128,64]")[1],
                                          "(_,(3,5))", "0")
    # sampled values of the 2^32-element maps (bit-exact anchors at full size)
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([rng.integers(0, 2**32, 4096), [0, 1, 2**32 - 1, 2**31, 8191, 8192]]))
    ops["C5_samples_i"] = idx.tolist()
    ops["C5_L_values"] = [int(ou.ref_eval_range(ops["C5_L"], int(i), 1)[0]) for i in idx]
    ops["C5_R_values"] = [int(ou.ref_eval_range(ops["C5_R"], int(i), 1)[0]) for i in idx]
    (OUT / "ops.json").write_text(json.dumps(ops, indent=1))
    ax = []
    for t, na in AXES_LAYOUTS:
        n = int(ou.ref_op("size", t)[1])
        # whole domain + 3 extended-domain points when small, else a head window and a tail window
        wins = [(0, n + 3)] if n <= 2048 else [(0, 1024), (n - 1024, 1027)]
        ax.append({"layout": t, "n_axes": na, "size": n,
                   "windows": [{"i0": i0, "values": ou.ref_eval_axes_range(t, na, i0, cnt).tolist()} for i0, cnt in wins]})
    st, ci = ou.ref_op("coordinate_identity", "(8,8)")
    assert st == 0 and ci == "(8,8):(e0,e1)", ci
    (OUT / "axes.json").write_text(json.dumps(ax))

    al = []
    for s, so, d, do, cells in ALIAS_CASES:
        buf = np.arange(cells, dtype=np.int64) * 3 + 1
        st = ou.ref_copy_shared(s, d, buf, so, do)
        al.append({"src": s, "src_origin": so, "dst": d, "dst_origin": do, "cells": cells, "status": st,
                   "result": buf.tolist()})
    (OUT / "alias.json").write_text(json.dumps(al))
    # max_common_vector (analysis.hpp:18-28): Table-1 pairs, gaps, broadcasts and 60 random stride permutations of (2,4,3,8)
    mc = [["8:1", "8:1"], ["(8,2,3):(1,16,32)", "(8,2,3):(1,16,32)"], ["(2,3,2):(42,1,128)", "12:1"], ["12:1", "(2,3,2):(42,1,128)"],
          ["(8,3):(1,8)", "(8,3):(3,1)"], ["(8,(3,5)):(1,(57,8))", "(8,15):(1,8)"], ["(64,64):(64,1)", "(64,64):(1,64)"],
          ["(4,8):(8,1)", "(4,8):(8,1)"], ["(4,8):(1,4)", "32:1"], ["(4,8):(1,8)", "(4,8):(1,8)"], ["(4,8):(1,8)", "(4,8):(1,4)"],
          ["7:0", "7:1"], ["(4,6):(1,4)", "(4,6):(0,1)"], ["(8192,8192):(8192,1)", "(8192,8192):(1,8192)"]]
    rng2 = np.random.default_rng(0)
    shp = [2, 4, 3, 8]
    for _ in range(60):
        def build(perm):
            st_, run = [0] * 4, 1
            for i in perm:
                st_[i] = run
                run *= shp[i]
            return "(" + ",".join(map(str, shp)) + "):(" + ",".join(map(str, st_)) + ")"
        mc.append([build(rng2.permutation(4)), build(rng2.permutation(4))])
    (OUT / "mcv.json").write_text(json.dumps([{"a": a, "b": b, "k": int(ou.ref_op("max_common_vector", a, b)[1])} for a, b in mc]))

    lo = []
    for a, t in LOCATE_CASES:
        st, r = ou.ref_op("locate_offsets", a, t)
        row = {"A": a, "T": t, "status": st}
        if st == 0:
            row["R"] = r
            row["R_values"] = ou.ref_eval_range(r, 0, int(ou.ref_op("size", t)[1])).tolist()
        lo.append(row)
    (OUT / "locate.json").write_text(json.dumps(lo))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

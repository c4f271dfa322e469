"""GPU parity: tla::copy through the C ABI vs the oracle — bit-exact on every cell, including the
cells the copy must NOT touch (destinations are pre-filled with -1, test_tensor.cpp:104)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle_util as ou
from gpu_util import cells, dev, run_copy_case
from paper_2603_02298_b200 import L, TlbError, abi, host

pytestmark = pytest.mark.gpu


def test_copy_reference_fixtures():
    """Every row of tests/golden/copy.json (Table 1 + extras), int64 cells exactly as the reference ran them."""
    for row in ou.golden("copy.json"):
        if "error" in row:
            continue
        nd = row["dst_len"]
        tdst = dev(np.full(nd, -1, dtype=np.int64))
        dd = L(row["dst"]).lower()
        dst = host.make_tensor(dd, tdst.data_ptr(), nd, 8)
        ds = L(row["src"]).lower()
        if "counting_base" in row:
            src = host.make_tensor(ds, None, 0, 8, row["counting_base"], counting=True)
            keep = None
        else:
            keep = dev(np.arange(row["src_len"], dtype=np.int64) * 3 + 1)
            src = host.make_tensor(ds, keep.data_ptr(), row["src_len"], 8)
        host.copy((src, None), (dst, None))
        torch.cuda.synchronize()
        assert tdst.cpu().numpy().tolist() == row["dst_cells"], (row["src"], row["dst"])


TABLE1 = [("8:1", "8:1"), ("(8,2,3):(1,16,32)", "(8,2,3):(1,16,32)"), ("(2,3,2):(42,1,128)", "12:1"),
          ("12:1", "(2,3,2):(42,1,128)"), ("7:0", "7:1"), ("7:0", "7:0"), ("(8,3):(1,8)", "(8,3):(3,1)"),
          ("(8,(3,5)):(1,(57,8))", "(8,15):(1,8)")]


@pytest.mark.parametrize("eb", [1, 2, 4, 8, 16])
def test_copy_table1_all_element_sizes(eb):
    for s, d in TABLE1:
        run_copy_case(s, d, eb)


@pytest.mark.parametrize("s,d", [
    ("(256,128):(128,1)", "(256,128):(1,256)"),                           # 256-row tiles
    ("(128,384):(1,128)", "(128,384):(384,1)"),                           # 128-row tiles, three 128-byte column blocks
    ("((8,128),(4,64),4):((1,2048),(8,32),262144)", "((8,128),(4,64),4):((128,1),(65536,1024),262144)"),  # C3, 4 tiles
    ("(512,128,3):(128,1,65536)", "(512,128,3):(1,512,65536)"),           # batched transpose
])
def test_copy_tiled_plan_one_byte_cells(s, d):
    """1-byte cells (fp8-sized): 16 x 16 byte blocks per lane, rotated row reads + barrel rotation, full-line stores."""
    assert run_copy_case(s, d, 1) == "tiled"
    assert run_copy_case("(96,160):(160,1)", "(96,160):(1,96)", 1) == "tiled_n"  # no 128-row B run: the 96-cell destination run whole, narrow-run tiles


@pytest.mark.parametrize("eb", [1, 2, 4, 8])
@pytest.mark.parametrize("s,d,so,do", [
    ("(256,128):(129,1)", "(256,128):(1,256)", 0, 0),                     # padded source rows: not a multiple of 16 bytes
    ("(256,128):(128,1)", "(256,128):(1,257)", 0, 0),                     # padded destination columns
    ("(256,128):(128,1)", "(256,128):(1,256)", 1, 3),                     # odd origins on both sides
    ("(96,160):(161,1)", "(96,160):(1,97)", 0, 1),                        # 32-row tiles
])
def test_copy_tiled_plan_unaligned(s, d, so, do, eb):
    """Leading dimensions / origins that break 16-byte alignment keep the staged plan with cell-sized global accesses."""
    plan = run_copy_case(s, d, eb, src_origin=so, dst_origin=do)
    if s.startswith("(96,160)") and eb == 2:
        assert plan == "gather"            # 160 two-byte cells are not a whole number of 128-byte rows
    elif s.startswith("(96,160)") and eb == 1:
        assert plan == "tiled_n"           # 96 rows < the 128 a 1-byte tile needs: the destination run whole, narrow-run tiles
    else:
        assert plan == "tiled_u"


@pytest.mark.parametrize("eb", [2, 4, 8, 16])
@pytest.mark.parametrize("s,d", [
    ("(256,128):(128,1)", "(256,128):(1,256)"),                           # C1 shape in small
    ("(128,256):(1,128)", "(128,256):(256,1)"),
    ("(96,160):(160,1)", "(96,160):(1,96)"),                              # Lb = 32 tiles
    ("((8,128),(4,64),4):((1,2048),(8,32),262144)", "((8,128),(4,64),4):((128,1),(65536,1024),262144)"),  # C3, 4 tiles
    ("(64,64,8):(512,1,64)", "(64,64,8):(1,512,64)"),                     # batched transpose, padded rows
    ("((32,16),(64,4)):((1,32),(512,32768))", "((32,16),(64,4)):((64,8192),(1,2048))"),   # 4-mode permutation
])
def test_copy_tiled_plan(s, d, eb):
    plan = run_copy_case(s, d, eb)
    if s.startswith("(96,160)") and eb == 2:
        assert plan == "gather"            # 160 two-byte cells are not a whole number of 128-byte rows
    else:
        assert plan == "tiled", plan


@pytest.mark.parametrize("eb", [2, 4, 8])
@pytest.mark.parametrize("s,d", [
    ("(256,128):(128,1)", "(256,128):(1,256)"),
    ("(128,256):(1,128)", "(128,256):(256,1)"),
    ("(96,160):(160,1)", "(96,160):(1,96)"),
    ("((8,128),(4,64),20):((1,2048),(8,32),262144)", "((8,128),(4,64),20):((128,1),(65536,1024),262144)"),  # 20 tiles: ragged last CTA
    ("(64,64,8):(512,1,64)", "(64,64,8):(1,512,64)"),
    ("((32,16),(64,4)):((1,32),(512,32768))", "((32,16),(64,4)):((64,8192),(1,2048))"),
])
def test_copy_tiled_tma_plan(s, d, eb):
    """The TMA-fed variant (tensor map derived from the source layout, hardware 128-byte swizzle) is bit-identical."""
    if s.startswith("(96,160)") and eb == 2:
        pytest.skip("160 two-byte cells are not a whole number of 128-byte rows")
    assert run_copy_case(s, d, eb, path=3) == "tiled_tma"


@pytest.mark.parametrize("s,d", [
    ("(256,128,4):(128,1,-32768)", "(256,128,4):(1,256,32768)"),          # reversed batch mode on the source
    ("(256,128):(-128,1)", "(256,128):(1,256)"),                          # reversed rows: the B run's source stride is negative
    ("(256,128):(128,1)", "(256,128):(1,-256)"),                          # reversed columns on the destination
])
def test_copy_tiled_plan_with_reversed_modes(s, d):
    """Negative strides (test_layout.cpp:183-186 evaluates them) stay on the tiled plan when they are not along the two
    contiguous runs; origins put the most negative offset at cell 0."""
    ds, dd = L(s).lower(), L(d).lower()
    so, do = max(0, -ds.min_offset), max(0, -dd.min_offset)
    ns, nd = ds.max_offset + so + 1, dd.max_offset + do + 1
    src, want = cells(ns, 4, 5), cells(nd, 4, fill=-1)
    assert ou.orc_copy(s, src, d, want, so, do) == 0
    tsrc, tdst = dev(src), dev(cells(nd, 4, fill=-1))
    a = host.make_tensor(ds, tsrc.data_ptr(), ns, 4, so)
    b = host.make_tensor(dd, tdst.data_ptr(), nd, 4, do)
    assert host.copy((a, None), (b, None)) == "tiled"
    torch.cuda.synchronize()
    assert (tdst.cpu().numpy() == want).all()


def test_copy_interleaved_runs_take_narrow_tiles():
    """The destination-contiguous run continues inside the source-contiguous run: no clean 128-byte A x B tile; since round 2
    the 4-cell source run is staged whole on the narrow-run kernel (the gather before)."""
    assert run_copy_case("((4,16),(32,4)):((1,512),(4,128))", "((4,16),(32,4)):((2048,1),(16,512))", 4) == "tiled_n"
    host.config("COPY_CELL_TILES", "0")
    try:
        assert run_copy_case("((4,16),(32,4)):((1,512),(4,128))", "((4,16),(32,4)):((2048,1),(16,512))", 4, seed=1) == "gather"
    finally:
        host.config("COPY_CELL_TILES", None)


@pytest.mark.parametrize("s,d,plan", [
    ("4096:1", "4096:1", "vec"),
    ("(64,32):(1,64)", "(64,32):(1,128)", "vec"),                         # row gather with padding
    ("(64,8,4):(1,256,64)", "(64,8,4):(1,64,512)", "vec"),                # mode permutation, contiguous rows
    ("(63,5):(1,63)", "(63,5):(1,64)", "gather"),                         # nothing to vectorise along 63 with 8-byte... still ok
])
def test_copy_vec_plan(s, d, plan):
    for eb in (2, 4, 8, 16):
        got = run_copy_case(s, d, eb)
        if plan == "vec":
            assert got == "vec", (got, eb)


def test_copy_forced_gather_equals_tiled():
    s, d = "(256,128):(128,1)", "(256,128):(1,256)"
    assert run_copy_case(s, d, 4, path=1) == "gather"
    assert run_copy_case(s, d, 4, path=2) == "tiled"


def test_copy_misaligned_origins_fall_back_and_stay_exact():
    assert run_copy_case("(256,128):(128,1)", "(256,128):(1,256)", 4, src_origin=1, dst_origin=3) == "tiled_u"
    assert run_copy_case("(256,128):(128,1)", "(256,128):(1,256)", 2, src_origin=1, dst_origin=3) == "tiled_u"
    assert run_copy_case("(256,128):(128,1)", "(256,128):(1,256)", 1, src_origin=1, dst_origin=3) == "tiled_u"   # 1-byte cells: the cell-granular staged kernel (round 2)
    assert run_copy_case("4096:1", "4096:1", 2, src_origin=1, dst_origin=1) in ("vec", "gather")


def test_copy_random_layout_pairs_vs_oracle():
    rng = np.random.default_rng(3)
    from test_oracle_pinned import _random_layout
    done = 0
    while done < 120:
        s, d = _random_layout(rng), _random_layout(rng)
        if L(s).size != L(d).size:
            d = "%d:%d" % (L(s).size, int(rng.integers(0, 3)))
        run_copy_case(s, d, int(rng.choice([1, 2, 4, 8, 16])), seed=done)
        done += 1


def _structured_pair(rng):
    """A (source, destination) pair over one shape of 3-5 power-of-two modes: each side assigns compact strides in its own
    random mode order (permutes / transposes), optionally scaled (no unit stride), padded, with a reversed mode, a
    broadcast (stride-0) destination mode, or a swizzled (Xor) destination. Returns (src, dst, src_origin, dst_origin, slack)."""
    if rng.random() < 0.15:
        r = int(rng.choice([2, 8, 32]))
        order = rng.permutation(3)
        ext = [128, 8, r]
        st = [0, 0, 0]
        acc = 1
        for m in order:
            st[m] = acc
            acc *= ext[m]
        return f"(128,8,{r}):({st[0]},{st[1]},{st[2]})", f"(128,8,{r}):(f1,f144,f1024)", 0, 0, 0
    nm = int(rng.integers(2, 5))
    ext = [int(rng.choice([4, 16, 32, 64, 128, 256])) for _ in range(nm)]
    while np.prod(ext) > (1 << 18):
        ext[int(np.argmax(ext))] //= 2
    def side(scale_choices, allow_zero):
        order = rng.permutation(nm)
        scale = int(rng.choice(scale_choices))
        st = [0] * nm
        acc = scale
        for k, m in enumerate(order):
            st[m] = acc
            acc *= ext[m]
            if k == nm - 2 and rng.random() < 0.3:
                acc += int(rng.choice([1, 4, 8])) * scale          # padded outermost mode
        origin = 0
        if rng.random() < 0.12:                                    # one reversed mode
            m = int(rng.integers(nm))
            origin = (ext[m] - 1) * st[m]
            st[m] = -st[m]
        if allow_zero and rng.random() < 0.15:
            st[int(rng.integers(nm))] = 0
        return st, origin
    ss, so = side([1, 1, 1, 2, 3], False)
    ds, do = side([1, 1, 1, 1, 5], True)
    shape = ",".join(str(e) for e in ext)
    mk = lambda st: f"({shape}):({','.join(str(x) for x in st)})"
    return mk(ss), mk(ds), so, do, max(so, do)


def test_copy_structured_fuzz_reaches_every_plan():
    """Differential fuzz over permutes / transposes / strided / padded / reversed / broadcast / swizzled layout pairs large
    enough for the staged plans, all cell sizes, against the oracle; the run must reach every family of plans."""
    rng = np.random.default_rng(11)
    plans = set()
    for case in range(220):
        s, d, so, do, slack = _structured_pair(rng)
        plans.add(run_copy_case(s, d, int(rng.choice([1, 2, 4, 8, 16])), src_origin=so, dst_origin=do, slack=slack, seed=case))
    kinds = {p.split("+")[0] for p in plans}
    assert {"vec", "tiled", "gather", "last_writer"} <= kinds and kinds & {"tiled_u", "tiled_s"} and kinds & {"gather_vec", "gather_run"}, plans


@pytest.mark.parametrize("eb", [2, 4, 8, 16])
def test_copy_ragged_extents_take_the_staged_plan(eb):
    """Extents that are not whole tiles (a 403 x 301 transpose, a ragged hierarchical permute, padded rows, origins, a
    sub-range of whole outer slices): the call is cut into a whole-tile body on the staged plan and edge strips; every cell
    of the destination, pre-fill included, equals tla::copy's (tensor.hpp:195-199). The cut starts at 2^22 elements by
    default (smaller copies are one gather launch); the small cases lower that bound through the knob."""
    assert run_copy_case("(2403,1801):(1801,1)", "(2403,1801):(1,2403)", eb).startswith("ragged:tiled")     # default threshold
    assert run_copy_case("(403,301):(301,1)", "(403,301):(1,403)", eb, seed=7) == "gather"
    host.config("COPY_RAGGED", "14")
    try:
        assert run_copy_case("(403,301):(301,1)", "(403,301):(1,403)", eb).startswith("ragged:tiled")
        assert run_copy_case("(403,301):(1,403)", "(403,301):(301,1)", eb, seed=1).startswith("ragged:tiled")
        assert run_copy_case("(520,300):(304,1)", "(520,300):(1,528)", eb, slack=40, seed=2).startswith("ragged:tiled")   # padded leading dimensions
        assert run_copy_case("(70,50,40):(1,70,3500)", "(70,50,40):(2000,40,1)", eb, seed=3).startswith("ragged:")        # rank-3 reversal
        assert run_copy_case("(403,301):(301,1)", "(403,301):(1,403)", eb, src_origin=3, dst_origin=5, seed=4).startswith("ragged:")
        if eb == 4:
            # a sub-range of whole outer slices of a ragged rank-3 permute
            s, d = "(300,70,8):(70,1,21000)", "(300,70,8):(1,300,21000)"
            assert run_copy_case(s, d, eb, i_begin=2 * 21000, i_end=7 * 21000, seed=5).startswith("ragged:")
        if eb < 16:
            # one contiguous mode that is not a whole number of 16-byte vectors: whole vectors on the vec plan, the rest gathered
            n_odd = 16 // eb * 1237 + 1
            assert run_copy_case(f"({n_odd},29):(1,{n_odd})", f"({n_odd},29):(1,{n_odd})", eb, seed=8) == "ragged:vec"
            # a run that starts off a 16-byte boundary by the same amount on both sides (a[1:] -> b[1 + 16 / eb:]): head cells too
            v = 16 // eb
            assert run_copy_case("40001:1", "40001:1", eb, src_origin=1, dst_origin=1 + v, seed=9) == "ragged:vec"
            assert run_copy_case(f"({v * 640},33):(1,{v * 640})", f"({v * 640},33):(1,{v * 800})", eb, src_origin=v - 1, dst_origin=2 * v - 1, seed=10) == "ragged:vec"
            # different misalignments: no common vector boundary, cell by cell
            assert run_copy_case("40001:1", "40001:1", eb, src_origin=1, dst_origin=2, seed=11) in ("vec", "gather")
        host.config("COPY_RAGGED", "0")
        assert run_copy_case("(2403,1801):(1801,1)", "(2403,1801):(1,2403)", eb, seed=6) == "gather"
    finally:
        host.config("COPY_RAGGED", None)


_IL_COMMON = [2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 16, 24, 32]
_IL_ALL = list(range(2, 27)) + [28, 30, 32]


@pytest.mark.parametrize("eb,ec", [(eb, ec) for eb in (1, 2, 4, 8) for ec in (_IL_ALL if eb in (2, 4) else _IL_COMMON)])
def test_copy_interleave_plan(eb, ec):
    """AoS <-> SoA and tall-skinny transposes (a short mode of 2 .. 26, 28, 30 or 32 cells for 2- and 4-byte cells, the common extents for 1- and 8-byte cells, against a long one): the register-permuting interleave plan, both
    directions, with outer modes, padded planar rows, origins that break the 32-byte alignment of the 256-bit accesses,
    a sub-range of whole outer slices, and a j extent that is not a whole number of lane pieces (gather)."""
    nj = 16 // eb * (2 if ec % 2 else 1)          # j per lane
    J = nj * 37
    aos, soa = f"({ec},{J}):(1,{ec})", f"({ec},{J}):({J},1)"
    assert run_copy_case(aos, soa, eb) == "interleave"
    assert run_copy_case(soa, aos, eb, seed=1) == "interleave"
    # three outer images, planar rows padded by 2 lane pieces, interleaved images padded too
    pj = J + 2 * nj
    aos3, soa3 = f"({ec},{J},3):(1,{ec},{ec * pj})", f"({ec},{J},3):({pj},1,{ec * pj})"
    assert run_copy_case(aos3, soa3, eb, seed=2) == "interleave"
    assert run_copy_case(soa3, aos3, eb, seed=3) == "interleave"
    # origins of 16 bytes: 128-bit accesses only
    assert run_copy_case(aos, soa, eb, src_origin=16 // eb, dst_origin=16 // eb, seed=4) == "interleave"
    assert run_copy_case(soa3, aos3, eb, src_origin=16 // eb, dst_origin=48 // eb, seed=5) == "interleave"
    # whole outer slices 1 .. 2 of the three images
    n1 = ec * J
    assert run_copy_case(aos3, soa3, eb, i_begin=n1, i_end=3 * n1, seed=6) == "interleave"
    # not a whole number of lane pieces / an unaligned origin: the narrow-run staged tiles when the long mode has whole
    # 32-cell pieces, else the gather plans
    assert run_copy_case(f"({ec},{J + 1}):(1,{ec})", f"({ec},{J + 1}):({J + 1},1)", eb, seed=7) in ("gather", "gather_vec", "tiled_n")
    assert run_copy_case(aos, soa, eb, src_origin=1, seed=8) in ("gather", "tiled_n")
    host.config("COPY_INTERLEAVE", "0")
    try:
        assert run_copy_case(aos, soa, eb, seed=9) in ("gather", "gather_vec", "tiled_n")
    finally:
        host.config("COPY_INTERLEAVE", None)
    # a long mode that is not a whole number of lane pieces (planar rows still 16-byte aligned): whole pieces + the last j
    host.config("COPY_RAGGED", "4")
    try:
        jr, pr = J + 1, J + nj
        assert run_copy_case(f"({ec},{jr}):(1,{ec})", f"({ec},{jr}):({pr},1)", eb, seed=10) == "ragged:interleave"
        assert run_copy_case(f"({ec},{jr}):({pr},1)", f"({ec},{jr}):(1,{ec})", eb, seed=11) == "ragged:interleave"
    finally:
        host.config("COPY_RAGGED", None)


@pytest.mark.parametrize("eb", [1, 2, 4, 8])
def test_copy_narrow_runs_take_the_cell_granular_tiles(eb):
    """A whole short mode as the source-contiguous run (fewer cells than a 128-byte row) or as the destination-contiguous
    run (fewer than 32 cells): run-time tile extents on the cell-granular staged kernel, both directions, outer modes,
    origins, hierarchical short runs; extents of the long mode that are not whole tiles through the ragged cut."""
    for k, nn in enumerate((5, 27, 29, 31)):
        if nn * eb >= 128:
            continue
        fwd = run_copy_case(f"(512,{nn}):({nn},1)", f"(512,{nn}):(1,512)", eb, seed=k)
        bwd = run_copy_case(f"(512,{nn}):(1,512)", f"(512,{nn}):({nn},1)", eb, seed=10 + k)
        assert fwd in ("tiled_n", "interleave") and bwd in ("tiled_n", "interleave"), (nn, fwd, bwd)
    nn = 27 if eb < 8 else 11     # a short mode below one 128-byte row that is not an interleave size for this cell size
    assert run_copy_case(f"({nn},256,3):(1,{nn},7000)", f"({nn},256,3):(300,1,8100)", eb, src_origin=1, dst_origin=2, seed=20) == "tiled_n"
    assert run_copy_case(f"({nn},256,3):(300,1,8100)", f"({nn},256,3):(1,{nn},7000)", eb, src_origin=3, dst_origin=1, seed=21) == "tiled_n"
    if eb == 4:
        assert run_copy_case("((4,16),(32,4)):((1,512),(4,128))", "((4,16),(32,4)):((2048,1),(16,512))", eb, seed=22) == "tiled_n"
    host.config("COPY_RAGGED", "4")
    try:
        want = "ragged:tiled_n" if 27 * eb < 128 else "ragged:tiled_u"   # 27 eight-byte cells are more than a 128-byte row
        assert run_copy_case("(421,27):(27,1)", "(421,27):(1,421)", eb, seed=23) == want
        assert run_copy_case("(421,27):(1,421)", "(421,27):(27,1)", eb, seed=24) == "ragged:tiled_n"
    finally:
        host.config("COPY_RAGGED", None)
    host.config("COPY_CELL_TILES", "0")
    try:
        assert run_copy_case("(512,27):(27,1)", "(512,27):(1,512)", eb, seed=25).startswith("gather")
    finally:
        host.config("COPY_CELL_TILES", None)


@pytest.mark.parametrize("eb", [2, 4, 8])
@pytest.mark.parametrize("rows", [96, 160, 192, 224])
def test_copy_tiles_of_96_to_224_rows(eb, rows):
    """A destination-contiguous run of 96 / 160 / 192 / 224 cells is one staged tile (384 .. 1792-byte destination segments)
    instead of 32-row tiles: both directions, an outer mode, several tiles per CTA for the 96-row tiles; the power-of-two
    tiles under COPY_ODD_TILES=0 give the same cells."""
    cols = 128
    s, d = f"({rows},{cols},3):({cols},1,{rows * cols})", f"({rows},{cols},3):(1,{rows},{rows * cols})"
    assert run_copy_case(s, d, eb) == "tiled"
    run_copy_case(d, s, eb, seed=1)            # the opposite direction (its source run is `rows` cells: staged only when that is whole 128-byte rows)
    big_s, big_d = f"({rows},16384):(16384,1)", f"({rows},16384):(1,{rows})"       # enough tiles for several per CTA
    assert run_copy_case(big_s, big_d, eb, seed=2) == "tiled"
    host.config("COPY_ODD_TILES", "0")
    try:
        assert run_copy_case(s, d, eb, seed=3) == "tiled"
    finally:
        host.config("COPY_ODD_TILES", None)


def test_copy_round2_plans_differential_fuzz():
    """Random permutes of 2 - 4 modes with random extents (whole tiles or not), paddings and origins, every cell size, with the
    ragged cut enabled from 16 elements: the run must reach the ragged / interleave / narrow / cell-granular plans, and every
    cell of every destination (pre-fill included) must equal tla::copy's."""
    rng = np.random.default_rng(2026)
    plans = set()
    host.config("COPY_RAGGED", "4")
    try:
        for case in range(260):
            rank = int(rng.integers(2, 5))
            if rank == 2:
                ext = [int(rng.choice([3, 4, 5, 9, 16, 24, 33, 64, 100, 129, 200, 257, 300])) for _ in range(2)]
            else:
                ext = [int(rng.choice([2, 3, 4, 5, 7, 8, 12, 16, 31, 32, 40, 65])) for _ in range(rank)]
            pad_s, pad_d = int(rng.choice([0, 0, 1, 4, 8])), int(rng.choice([0, 0, 1, 4, 8]))
            def compact(order, pad):
                strides, run = [0] * rank, 1
                for k, m in enumerate(order):
                    strides[m] = run
                    run *= ext[m]
                    if k == 0:
                        run += pad        # padded leading dimension
                return strides
            so = list(rng.permutation(rank))
            do = list(rng.permutation(rank))
            ss, ds = compact(so, pad_s), compact(do, pad_d)
            s = "(" + ",".join(map(str, ext)) + "):(" + ",".join(map(str, ss)) + ")"
            d = "(" + ",".join(map(str, ext)) + "):(" + ",".join(map(str, ds)) + ")"
            eb = int(rng.choice([1, 2, 4, 8, 16]))
            o_s, o_d = (int(rng.choice([0, 0, 1, 4, 16])) for _ in range(2))
            plans.add(run_copy_case(s, d, eb, src_origin=o_s, dst_origin=o_d, seed=case))
    finally:
        host.config("COPY_RAGGED", None)
    kinds = {p.split(":")[0] for p in plans} | {p.split(":")[-1] for p in plans}
    assert {"ragged", "interleave", "tiled_n", "tiled_u", "tiled", "vec"} <= kinds, plans


def test_copy_xor_layouts():
    run_copy_case("(8,8):(f1,f9)", "64:1", 8)
    run_copy_case("64:1", "(8,8):(f1,f9)", 4)
    # staging layout of config C3: Swizzle<3,4,3> per 1 KiB == (128,8):(f1,f144)
    run_copy_case("(128,8):(f1,f144)", "(128,8):(8,1)", 1)
    # Xor offsets act on the absolute position, origin included (tensor.hpp:57)
    ns = 64 + 64
    src, want = cells(ns, 8, 1), cells(ns, 8, fill=-1)
    assert ou.orc_copy("(8,8):(f1,f9)", src, "64:1", want, src_origin=64, dst_origin=5) == 0
    tsrc, tdst = dev(src), dev(cells(ns, 8, fill=-1))
    a = host.make_tensor(L("(8,8):(f1,f9)").lower(), tsrc.data_ptr(), ns, 8, 64)
    b = host.make_tensor(L("64:1").lower(), tdst.data_ptr(), ns, 8, 5)
    host.copy((a, None), (b, None))
    torch.cuda.synchronize()
    assert (tdst.cpu().numpy() == want).all()


@pytest.mark.parametrize("eb,plan", [(1, "gather_vec"), (2, "gather_run"), (4, "gather_run"), (8, "gather_run"), (16, "gather_run")])
def test_copy_xor_layouts_vectorised(eb, plan):
    """Swizzled (Xor) layouts keep the low coordinate bits contiguous (leaf 0 is f1, the other masks start at bit 4): the
    gather evaluates both layouts once per 16-byte vector (max_common_vector, analysis.hpp:18-28, extended to Xor leaves),
    or once per 32 / 64-byte run moved with 256-bit accesses when both layouts keep that much contiguous ("gather_run").
    Both directions, an Xor layout on both sides, origins (Xor acts on the absolute position, tensor.hpp:57) and a range
    that is not a whole number of vectors (falls back to one cell per thread)."""
    sw, flat = "(128,8,32):(f1,f144,f1024)", "(128,8,32):(1,128,1024)"
    assert run_copy_case(flat, sw, eb) == plan
    assert run_copy_case(sw, flat, eb, seed=1) == plan
    assert run_copy_case(sw, "(128,8,32):(f1,f160,f1024)", eb, seed=2) == plan   # two different swizzles
    assert run_copy_case(flat, sw, eb, src_origin=16, dst_origin=32768, seed=3) == plan
    assert run_copy_case(flat, sw, eb, src_origin=1, dst_origin=32768, seed=4) in ("gather", "gather_vec")   # unaligned source
    host.config("COPY_GATHER_RUN", "0")
    try:
        assert run_copy_case(flat, sw, eb, seed=5) == ("gather" if eb == 16 else "gather_vec")
    finally:
        host.config("COPY_GATHER_RUN", None)


@pytest.mark.parametrize("eb", [2, 4, 8])
def test_copy_strided_runs_take_the_staged_plan(eb):
    """No unit stride on one side (BLIS-style general strides): the staged plan runs along the smallest-stride mode with
    cell-sized strided accesses ("tiled_s"). Packing a strided matrix into rows, scattering rows into a strided matrix,
    strided on both sides, a reversed outer mode, and the cases that must stay on the gather (same mode fastest on both
    sides, strides too far apart)."""
    assert run_copy_case("(256,128):(3,779)", "(256,128):(128,1)", eb) == "tiled_s"            # pack: m stride 3 -> rows
    assert run_copy_case("(256,128):(128,1)", "(256,128):(5,1291)", eb, seed=1) == "tiled_s"   # scatter: rows -> m stride 5
    assert run_copy_case("(256,256):(3,779)", "(256,256):(1543,2)", eb, seed=2) == "tiled_s"   # strided on both sides
    assert run_copy_case("(256,128):(3,-779)", "(256,128):(128,1)", eb, src_origin=779 * 127, slack=779 * 127, seed=3) == "tiled_s"
    assert run_copy_case("(256,128):(3,779)", "(256,128):(2,515)", eb, seed=4) in ("gather", "gather_vec")  # same fastest mode
    assert run_copy_case("(64,64):(100,6400)", "(64,64):(64,1)", eb, seed=5) in ("gather", "gather_vec")    # stride 100: no gain


def test_copy_non_injective_destination_last_writer_wins():
    """7:0 -> 7:0 makes dst[0] = src(6) (test_tensor.cpp:98); larger aliasing cases vs the oracle."""
    # stride-0 (broadcast) destination modes: the copy equals the injective copy of the slice at their last coordinate
    assert run_copy_case("7:1", "7:0", 8) == "last_writer+gather"
    assert run_copy_case("(64,64):(1,64)", "(64,64):(1,0)", 4) == "last_writer+vec"
    assert run_copy_case("(64,64):(64,1)", "(64,64):(0,1)", 4).startswith("last_writer+")
    assert run_copy_case("(256,128,3):(128,1,32768)", "(256,128,3):(1,256,0)", 4) == "last_writer+tiled"   # a transpose under a broadcast
    assert run_copy_case("(6,35):(1,6)", "((2,3),(5,7)):((0,2),(6,0))", 8).startswith("last_writer+")       # broadcast leaves inside both modes
    assert run_copy_case("(64,64):(1,64)", "(64,64):(1,0)", 4, path=1) == "ordered"                          # forced fallback keeps the election
    # genuinely overlapping strides: winner election (atomicMax of i per cell, then only the winners store)
    assert run_copy_case("(32,32,4):(1,32,1024)", "(32,32,4):(1,31,3)", 8) == "ordered"
    assert run_copy_case("(16,16,4):(1,16,256)", "(16,16,4):(1,15,0)", 4) == "ordered"                       # broadcast AND overlap
    # the winner arrays came from the library's own stream-ordered pool: give its cached blocks back, then use it again
    assert abi.load().tlb_workspace_trim(0) == 0
    assert run_copy_case("(32,32,4):(1,32,1024)", "(32,32,4):(1,31,3)", 4, seed=9) == "ordered"


def _alias_case(s, d, so, do, cells_n, eb=8, seed=0):
    """Both tensors view ONE device buffer; compare with the restatement run in place on the same cells."""
    buf = cells(cells_n, eb, seed)
    want = buf.copy()
    if eb == 16:
        wv = want.view([("a", np.int64), ("b", np.int64)])
        assert ou.orc_copy(s, wv, d, wv, so, do) == 0
    else:
        assert ou.orc_copy(s, want, d, want, so, do) == 0
    t = dev(buf)
    a = host.make_tensor(L(s).lower(), t.data_ptr(), cells_n, eb, so)
    b = host.make_tensor(L(d).lower(), t.data_ptr(), cells_n, eb, do)
    plan = host.copy((a, None), (b, None))
    torch.cuda.synchronize()
    got = t.cpu().numpy()
    assert (got == want).all(), f"aliased copy {s}@{so} -> {d}@{do} plan={plan}: {int((got != want).sum())} cells differ"
    return plan


def test_copy_aliased_views_of_one_buffer_keep_the_serial_order():
    """Source and destination ranges overlap inside one buffer (the reference's views share storage, tensor.hpp:29):
    the result is the serial ascending-i one. Reference fixtures first (tests/golden/alias.json), then larger cases."""
    for row in ou.golden("alias.json"):
        t = dev(np.arange(row["cells"], dtype=np.int64) * 3 + 1)
        a = host.make_tensor(L(row["src"]).lower(), t.data_ptr(), row["cells"], 8, row["src_origin"])
        b = host.make_tensor(L(row["dst"]).lower(), t.data_ptr(), row["cells"], 8, row["dst_origin"])
        plan = host.copy((a, None), (b, None))
        torch.cuda.synchronize()
        assert t.cpu().numpy().tolist() == row["result"], (row["src"], row["dst"], plan)
        assert plan in ("aliased", "serial")
    n = 1 << 18
    assert _alias_case(f"{n}:1", f"{n}:1", 0, 1, n + 1) == "aliased"      # shift right: a read-after-write chain of length n
    assert _alias_case(f"{n}:1", f"{n}:1", 1, 0, n + 1, eb=4) == "aliased"  # shift left: a plain move
    assert _alias_case(f"{n}:1", f"{n}:1", 0, 7, n + 7, eb=2) == "aliased"  # period-7 propagation
    assert _alias_case("(512,512):(512,1)", "(512,512):(1,512)", 0, 0, 512 * 512, eb=4) == "aliased"   # in-place transpose
    assert _alias_case("(512,512):(512,1)", "(512,512):(1,512)", 0, 0, 512 * 512, eb=16) == "aliased"
    assert _alias_case("(256,128):(128,1)", "(256,128):(1,256)", 5, 1000, 256 * 128 + 1000, eb=1) == "aliased"
    assert _alias_case("(64,64):(1,64)", "(64,64):(1,0)", 0, 10, 4096 + 64) == "serial"    # non-injective destination too
    # disjoint halves of one allocation are NOT aliased: the planned kernels keep running
    assert _alias_case("(256,128):(128,1)", "(256,128):(1,256)", 0, 256 * 128, 2 * 256 * 128, eb=4) == "tiled"


def test_copy_subranges_tile_aligned_and_ragged():
    s, d = "(256,128):(128,1)", "(256,128):(1,256)"
    n = 256 * 128
    src = cells(n, 4, 2)
    for (b, e) in [(0, n // 2), (n // 2, n), (256 * 32, 256 * 96), (5, 777), (0, 0), (n, n + 5)]:
        want = cells(n, 4, fill=-1)
        assert ou.orc_copy(s, src, d, want, i_begin=b, i_end=min(e, n)) == 0
        tsrc, tdst = dev(src), dev(cells(n, 4, fill=-1))
        a = host.make_tensor(L(s).lower(), tsrc.data_ptr(), n, 4)
        bb = host.make_tensor(L(d).lower(), tdst.data_ptr(), n, 4)
        host.copy((a, None), (bb, None), b, e)
        torch.cuda.synchronize()
        assert (tdst.cpu().numpy() == want).all(), (b, e)


def test_copy_error_contracts_write_nothing():
    buf = dev(np.arange(8, dtype=np.int64))
    out = dev(np.full(8, -1, dtype=np.int64))
    src = host.make_tensor(L("4:3").lower(), buf.data_ptr(), 8, 8)
    dst = host.make_tensor(L("4:1").lower(), out.data_ptr(), 8, 8)
    with pytest.raises(TlbError) as e:            # 4:3 reads cell 9 of 8 -> bounds_error (test_tensor.cpp:34-40)
        host.copy((src, None), (dst, None))
    assert e.value.status == abi.TLB_ERR_BOUNDS
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == -1).all()         # pre-flight: nothing was written (documented difference)
    neg = host.make_tensor(L("1:0").lower(), buf.data_ptr(), 8, 8, -1)
    with pytest.raises(TlbError) as e:            # origin -1 (test_tensor.cpp:39)
        host.copy((neg, None), (host.make_tensor(L("1:0").lower(), out.data_ptr(), 8, 8), None))
    assert e.value.status == abi.TLB_ERR_BOUNDS
    with pytest.raises(TlbError) as e:
        host.copy((host.make_tensor(L("8:1").lower(), buf.data_ptr(), 8, 8), None), (dst, None))
    assert e.value.status == abi.TLB_ERR_CONTRACT
    with pytest.raises(TlbError) as e:
        host.copy((host.make_tensor(L("(2,2):(e0,e1)").lower(), buf.data_ptr(), 8, 8), None), (dst, None))
    assert e.value.status == abi.TLB_ERR_SEMIMODULE
    # Xor layout whose OR-bound exceeds the buffer but whose exact image fits: (3):(f4) touches {0,4,8}
    small = dev(np.arange(9, dtype=np.int64))
    o3 = dev(np.full(3, -1, dtype=np.int64))
    host.copy((host.make_tensor(L("3:f4").lower(), small.data_ptr(), 9, 8), None),
              (host.make_tensor(L("3:1").lower(), o3.data_ptr(), 3, 8), None))
    torch.cuda.synchronize()
    assert o3.cpu().numpy().tolist() == [0, 4, 8]


def test_copy_host_entry_point():
    s, d = "(256,128):(128,1)", "(256,128):(1,256)"
    n = 256 * 128
    src = torch.from_numpy(cells(n, 4, 9)).pin_memory()
    dst = torch.full((n,), -1, dtype=torch.int32).pin_memory()
    want = np.full(n, -1, dtype=np.int32)
    assert ou.orc_copy(s, src.numpy(), d, want) == 0
    a = host.make_tensor(L(s).lower(), src.data_ptr(), n, 4)
    b = host.make_tensor(L(d).lower(), dst.data_ptr(), n, 4)
    host.copy_host((a, None), (b, None))
    assert (dst.numpy() == want).all()
    # a destination the copy only partly covers keeps its other cells
    dst2 = torch.full((2 * n,), -7, dtype=torch.int32)
    want2 = np.full(2 * n, -7, dtype=np.int32)
    d2 = "(256,128):(2,512)"
    assert ou.orc_copy(s, src.numpy(), d2, want2) == 0
    host.copy_host((a, None), (host.make_tensor(L(d2).lower(), dst2.data_ptr(), 2 * n, 4), None))
    assert (dst2.numpy() == want2).all()


def test_c1_transpose_full_size_properties():
    """Config C1 at BASELINE size (8192^2 fp32): involution + spot rows vs the oracle on a sub-block."""
    n = 8192
    src = torch.arange(n * n, dtype=torch.int32, device="cuda")          # element-index bit patterns
    dst = torch.full((n * n,), -1, dtype=torch.int32, device="cuda")
    s, d = f"({n},{n}):({n},1)", f"({n},{n}):(1,{n})"
    a, ka = host.tensor_of(s, src)
    b, kb = host.tensor_of(d, dst)
    assert host.copy((a, ka), (b, kb)) == "tiled"
    torch.cuda.synchronize()
    # dst viewed as (n,n) row-major must equal src viewed row-major, transposed
    assert torch.equal(dst.view(n, n), src.view(n, n).t())
    # the TMA-fed variant produces the same bytes
    dst2 = torch.full((n * n,), -1, dtype=torch.int32, device="cuda")
    b_t, kb_t = host.tensor_of(d, dst2)
    abi.load().tlb_copy_set_path(3)
    try:
        assert host.copy((a, ka), (b_t, kb_t)) == "tiled_tma"
    finally:
        abi.load().tlb_copy_set_path(0)
    torch.cuda.synchronize()
    assert torch.equal(dst2, dst)
    del dst2
    # involution: transposing back restores the source bit for bit
    back = torch.full((n * n,), -1, dtype=torch.int32, device="cuda")
    a2, k2 = host.tensor_of(s, dst)
    b2, k3 = host.tensor_of(d, back)
    host.copy((a2, k2), (b2, k3))
    torch.cuda.synchronize()
    assert torch.equal(back, src)


def test_c3_permute_full_size_properties():
    """Config C3 at BASELINE size (2^30 fp32 = 4 GiB each way): the destination is a permutation of the
    source (checksum of checksums), sampled tiles equal the oracle, and the inverse permutation restores it."""
    T = 4096
    s = f"((8,128),(4,64),{T}):((1,2048),(8,32),262144)"
    d = f"((8,128),(4,64),{T}):((128,1),(65536,1024),262144)"
    n = 262144 * T
    src = torch.arange(n, dtype=torch.int32, device="cuda")
    dst = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    a, ka = host.tensor_of(s, src)
    b, kb = host.tensor_of(d, dst)
    assert host.copy((a, ka), (b, kb)) == "tiled"
    torch.cuda.synchronize()
    # per-tile checksums: every tile permutes its own 262144 cells
    assert torch.equal(dst.view(T, -1).sum(dim=1, dtype=torch.int64), src.view(T, -1).sum(dim=1, dtype=torch.int64))
    # tiles 0, 1234 and T-1 against the oracle
    tile_s = "((8,128),(4,64)):((1,2048),(8,32))"
    tile_d = "((8,128),(4,64)):((128,1),(65536,1024))"
    for t in (0, 1234, T - 1):
        want = np.full(262144, -1, dtype=np.int32)
        assert ou.orc_copy(tile_s, src[t * 262144:(t + 1) * 262144].cpu().numpy(), tile_d, want) == 0
        assert (dst[t * 262144:(t + 1) * 262144].cpu().numpy() == want).all()
    # inverse: copy with the roles of the layouts swapped restores the source
    back = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    a2, k2 = host.tensor_of(d, dst)
    b2, k3 = host.tensor_of(s, back)
    host.copy((a2, k2), (b2, k3))
    torch.cuda.synchronize()
    assert torch.equal(back, src)


def test_tensormap_from_divided_fetches_the_tile_the_layout_names():
    """tlb_tensormap_from_divided: the box TMA delivers for tile (i, j) of zipped_divide(parent, tiler) equals the cells
    the divided layout addresses (oracle evaluation), for every hardware swizzle mode: the de-swizzle is
    Swizzle<B,4,3> on byte offsets, i.e. the reference's Xor layouts."""
    import oracle_util as ou
    parent = "(96,192):(192,1)"
    buf = torch.arange(96 * 192, dtype=torch.int32, device="cuda") * 3 + 1
    hbuf = buf.cpu().numpy()
    # the inner box extent may not exceed the swizzle span (32 / 64 / 128 bytes): 8 / 16 / 32 int32 columns
    width = {0: 32, 1: 8, 2: 16, 3: 32}
    for (ti, tj) in [(0, 0), (2, 5), (1, 3)]:
        base = ti * 32 * 192 + tj * 32
        for swz in (0, 1, 2, 3):
            w = width[swz]
            tile = f"(32,{w}):(192,1)"                                   # zipped_divide(parent, [32,w]) tile mode
            tile_off = ou.orc_eval_range(tile, 0, 32 * w).reshape(w, 32)    # [col][row]: colex, mode 0 = rows
            want = hbuf[base + tile_off].T                                   # TMA box order: dim0 (stride 1) fastest
            got = host.tensormap_fetch(parent, tile, buf, (tj * 32, ti * 32), swizzle=swz)
            torch.cuda.synchronize()
            assert (got.cpu().numpy().view(np.int32).reshape(32, w) == want).all(), (ti, tj, swz)
    # config C3 source tile: box 32 x 128 (16 KiB) at tile 2, 128-byte swizzle
    T = 4
    s3 = f"((8,128),(4,64),{T}):((1,2048),(8,32),262144)"
    b3 = torch.arange(262144 * T, dtype=torch.int32, device="cuda")
    got = host.tensormap_fetch(s3, "((8,128),4):((1,2048),8)", b3, (64, 2 * 128), swizzle=3)
    torch.cuda.synchronize()
    want = (2 * 262144 + 64 + np.arange(32)[None, :] + 2048 * np.arange(128)[:, None]).astype(np.int32)
    assert (got.cpu().numpy().view(np.int32).reshape(128, 32) == want).all()


def test_tma_coordinates_come_from_the_tiled_coordinate_identity():
    """TMA coordinates are produced from tiled identity tensors. coordinate_identity((96,192)) =
    (96,192):(e0,e1) (layout.hpp:253); zipped_divide by [32,32] gives ((32,32),(3,6)):((e0,e1),(32*e0,32*e1)), whose rest
    mode evaluated ON THE DEVICE (tlb_eval_axes_range over the tile index) is the (row, column) where each tile starts.
    Those per-axis coordinates, reversed to TMA order (dimension 0 = the stride-1 column axis), fetch every tile of the
    divided layout through the tensor map; each box must hold exactly the cells the divided layout addresses (oracle)."""
    parent = "(96,192):(192,1)"
    buf = torch.arange(96 * 192, dtype=torch.int32, device="cuda") * 3 + 1
    hbuf = buf.cpu().numpy()
    rest = "(3,6):(32*e0,32*e1)"                                   # rest mode of the divided coordinate identity
    crd = torch.empty(18, 2, dtype=torch.int64, device="cuda")
    host.eval_axes_range(rest, 2, 0, 18, crd)
    torch.cuda.synchronize()
    coords = crd.cpu().numpy()
    assert (coords == ou.orc_eval_axes_range(rest, 2, 0, 18)).all()
    tile = "(32,32):(192,1)"
    tile_off = ou.orc_eval_range(tile, 0, 32 * 32).reshape(32, 32)   # [col][row]
    for t in range(18):
        row0, col0 = int(coords[t, 0]), int(coords[t, 1])
        got = host.tensormap_fetch(parent, tile, buf, (col0, row0), swizzle=3)
        torch.cuda.synchronize()
        want = hbuf[row0 * 192 + col0 + tile_off].T
        assert (got.cpu().numpy().view(np.int32).reshape(32, 32) == want).all(), t


def _copy_tv_case(s, d, eb, tv, seed=0, expect_all=True):
    """tlb_copy_tv against the oracle: with a thread-value layout that covers every coordinate once the result is
    tla::copy's; cells no (thread, value) pair maps to must keep their pre-fill."""
    ns, nd = ou.cosize_of(s), ou.cosize_of(d)
    src, dst0 = cells(ns, eb, seed), cells(nd, eb, fill=-1 if eb != 1 else 255)
    want = dst0.copy()
    n = L(s).size
    covered = np.unique(ou.orc_eval_range(tv, 0, L(tv).size))
    covered = covered[covered < n]
    if expect_all:
        assert covered.size == n
        assert ou.orc_copy(s, src, d, want) == 0
    else:
        so, do = ou.orc_eval_range(s, 0, n), ou.orc_eval_range(d, 0, n)
        want[do[covered]] = src[so[covered]]
    tsrc, tdst = dev(src), dev(dst0)
    a = host.make_tensor(L(s).lower(), tsrc.data_ptr(), ns, eb)
    b = host.make_tensor(L(d).lower(), tdst.data_ptr(), nd, eb)
    plan = host.copy_tv((a, None), (b, None), tv)
    torch.cuda.synchronize()
    got = tdst.cpu().numpy()
    assert (got == want).all(), f"copy_tv {s} -> {d} tv={tv}: {int((got != want).sum())} cells differ"
    return plan


@pytest.mark.parametrize("eb", [1, 2, 4, 8])
def test_copy_partitioned_by_thread_value_layouts(eb):
    """local_partition-style copies (partition_demo.cpp:26-40): the library-derived raked TV layout on
    contiguous, transposed, strided and swizzled pairs (vectors where max_common_vector allows), thread-value maps built
    with the reference's products, and a TV layout that covers only part of the tensor."""
    pairs = [("4096:1", "4096:1"), ("(64,64):(64,1)", "(64,64):(1,64)"), ("(8,16,8):(1,8,128)", "(8,16,8):(1,64,8)"),
             ("(128,8,4):(1,128,1024)", "(128,8,4):(f1,f144,f1024)"), ("1000:1", "1000:1"), ("(30,20):(3,91)", "(30,20):(20,1)")]
    plans = set()
    for k, (s, d) in enumerate(pairs):
        tv = host.copy_tv_auto(s, d, eb, threads=64)
        plans.add(_copy_tv_case(s, d, eb, tv, seed=k))
    # digit-permutation TV layouts run as the copy between src o TV and dst o TV ("tv:<plan>"); 1000 = 2^3 5^3 elements with
    # 64 threads is over-covered by its TV layout and keeps the per-thread kernel, as do the Xor destination's pairs
    assert plans & {"tv", "tv_vec"} and any(p.startswith("tv:") for p in plans), plans
    assert all(p in ("tv", "tv_vec") or p.startswith("tv:") for p in plans), plans
    # partition_demo.cpp: 32 threads in a (4,8) arrangement, 2 values each, over an 8 x 8 tile stored column-major
    _copy_tv_case("(8,8):(1,8)", "(8,8):(8,1)", eb, "((4,8),2):((16,1),8)", seed=7)
    # blocked_product((2,2):(1,2), (4,4):(1,4)) as a TV layout: each of 16 threads owns a 2 x 2 block of a 8 x 8 tile
    _copy_tv_case("(8,8):(1,8)", "(8,8):(1,8)", eb, "((4,4),(2,2)):((2,16),(1,8))", seed=8)
    # half of the threads only: the other cells keep their pre-fill
    _copy_tv_case("(8,8):(1,8)", "(8,8):(8,1)", eb, "((4,4),2):((16,1),8)", seed=9, expect_all=False)


@pytest.mark.parametrize("eb", [2, 4])
def test_copy_tv_runs_as_the_copy_between_the_compositions(eb):
    """Partitioning is composition (compose, algebra.hpp:235): a TV layout that permutes the digits of the
    integral coordinate turns tlb_copy_tv into tlb_copy between src o TV and dst o TV, so the planner's staged and
    vectorised plans apply. Same cells as the per-thread kernel (COPY_TV_COMPOSE=0) and as tla::copy."""
    cases = [("(256,256):(1,256)", "(256,256):(1,256)", None, "tv:vec"),                      # contiguous: vectors
             ("(256,256):(256,1)", "(256,256):(1,256)", None, "tv:tiled"),                    # transpose: staged tile
             ("(8,128,64):(1,512,8)", "(8,128,64):(128,1,1024)", None, "tv:"),                # hierarchical permute
             ("(64,64):(1,64)", "(64,64):(64,1)", "((4,8,2),(2,32)):((16,1,8),(64,128))", "tv:"),  # a hand-built digit permutation
             ("(96,40):(1,96)", "(96,40):(40,1)", "((32,3),40):((1,32),96)", "tv:")]          # non-power-of-two digits
    for k, (sl, dl, tv, want) in enumerate(cases):
        tv = tv or host.copy_tv_auto(sl, dl, eb, threads=256)
        plan = _copy_tv_case(sl, dl, eb, tv, seed=20 + k)
        assert plan.startswith(want), (sl, dl, tv, plan)
        host.config("COPY_TV_COMPOSE", "0")
        try:
            assert _copy_tv_case(sl, dl, eb, tv, seed=20 + k) in ("tv", "tv_vec")
        finally:
            host.config("COPY_TV_COMPOSE", None)
    # digits of extent 3, 2, 2 in two different thread / value arrangements over a 12-cell tensor whose destination splits 3 x 4
    assert _copy_tv_case("12:1", "(3,4):(4,1)", eb, "(3,(2,2)):(1,(3,6))", seed=31).startswith("tv:")
    assert _copy_tv_case("12:1", "(3,4):(4,1)", eb, "(2,(3,2)):(3,(1,6))", seed=32).startswith("tv:")
    # a digit of extent 4 splits across the source's leaves 6 and 2 (stride-3 half, then the second leaf)
    assert _copy_tv_case("(6,2):(1,6)", "(6,2):(2,1)", eb, "(4,3):(3,1)", seed=33).startswith("tv:")
    # a digit that would straddle a leaf (i = c0 + 4 c1 against a leaf of extent 6): not a composition, per-thread kernel
    assert _copy_tv_case("(6,2):(1,6)", "(6,2):(2,1)", eb, "(4,3):(1,4)", seed=34) in ("tv", "tv_vec")


def test_copy_tv_contracts():
    src, dst = dev(cells(64, 8, 1)), dev(cells(64, 8, fill=-1))
    a = host.make_tensor(L("(8,8):(1,8)").lower(), src.data_ptr(), 64, 8)
    b = host.make_tensor(L("(8,8):(8,1)").lower(), dst.data_ptr(), 64, 8)
    for tv, status in [("64:1", abi.TLB_ERR_CONTRACT),                       # rank 1: no (thread, value) structure
                       ("((4,8),2):((16,1),1)", abi.TLB_ERR_UNSUPPORTED),    # two (thread, value) pairs on one coordinate
                       ("(32,2):(f1,f32)", abi.TLB_ERR_SEMIMODULE)]:
        with pytest.raises(TlbError) as e:
            host.copy_tv((a, None), (b, None), tv)
        assert e.value.status == status, tv
    torch.cuda.synchronize()
    assert (dst.cpu().numpy() == -1).all()                                   # nothing was written

"""Thin Python driver over the C ABI, used by tests/, bench.py and smoke().

The reference (`tla`, header-only C++) has no Python surface; its C++ surface is mirrored by
include/tla/ (see INTEGRATION.md). This module only does what a C++ caller would do before
calling libtlb: spell a layout (the reference's own text syntax, text.hpp:130: `shape:stride`
with `f9`-style Xor strides and `2*e1`-style Basis strides), flatten it to leaves (flat_modes,
layout.hpp:111), lower it, and pass device pointers of torch tensors. No arithmetic on tensor
contents happens here.
"""
from __future__ import annotations

import ctypes as C
import re
from dataclasses import dataclass

from . import abi

_TOK = re.compile(r"\s*(\(|\)|,|:|\*|-?\d+|e\d+|f\d+)")


def _tokens(text: str):
    pos, out = 0, []
    text = text.strip()
    while pos < len(text):
        m = _TOK.match(text, pos)
        if not m:
            raise ValueError(f"cannot parse layout text at {text[pos:]!r}")
        out.append(m.group(1))
        pos = m.end()
    return out


def _parse_tree(toks, i, leaf):
    if toks[i] == "(":
        kids = []
        i += 1
        while True:
            node, i = _parse_tree(toks, i, leaf)
            kids.append(node)
            if toks[i] == ",":
                i += 1
                continue
            if toks[i] == ")":
                return tuple(kids), i + 1
            raise ValueError("expected , or )")
    return leaf(toks, i)


def _shape_leaf(toks, i):
    return int(toks[i]), i + 1


def _stride_leaf(toks, i):
    t = toks[i]
    if t[0] == "f":
        m = int(t[1:])
        return ((abi.KIND_XOR, m, 0) if m else (abi.KIND_INT, 0, 0)), i + 1
    if t[0] == "e":
        return (abi.KIND_BASIS, 1, int(t[1:])), i + 1
    v = int(t)
    if i + 1 < len(toks) and toks[i + 1] == "*":
        return ((abi.KIND_BASIS, v, int(toks[i + 2][1:])) if v else (abi.KIND_INT, 0, 0)), i + 3
    if i + 1 < len(toks) and toks[i + 1][0] == "e":
        return ((abi.KIND_BASIS, v, int(toks[i + 1][1:])) if v else (abi.KIND_INT, 0, 0)), i + 2
    return (abi.KIND_INT, v, 0), i + 1


def _flat_shape(tree):
    if isinstance(tree, tuple):
        out = []
        for k in tree:
            out.extend(_flat_shape(k))
        return out
    return [tree]


def _flat_stride(tree):
    # stride leaves are (kind, value, axis) triples; inner nodes are tuples of nodes
    if isinstance(tree, tuple) and len(tree) == 3 and all(isinstance(x, int) for x in tree):
        return [tree]
    out = []
    for k in tree:
        out.extend(_flat_stride(k))
    return out


def _is_stride_leaf(t):
    return isinstance(t, tuple) and len(t) == 3 and all(isinstance(x, int) for x in t)


def _expand(shape, stride):
    """Pairs shape leaves with stride leaves; a leaf stride under a tuple shape is not congruent."""
    if isinstance(shape, tuple):
        if _is_stride_leaf(stride) or len(stride) != len(shape):
            raise ValueError("shape and stride are not congruent")
        out = []
        for s, d in zip(shape, stride):
            out.extend(_expand(s, d))
        return out
    if not _is_stride_leaf(stride):
        raise ValueError("shape and stride are not congruent")
    return [(shape, stride)]


@dataclass
class Layout:
    """A parsed layout: flat leaves in left-to-right order plus the top-level grouping."""
    text: str
    modes: list      # [(extent, kind, value, axis)]
    top_leaves: list  # leaves per top-level mode

    @staticmethod
    def parse(text: str) -> "Layout":
        toks = _tokens(text)
        shape, i = _parse_tree(toks, 0, _shape_leaf)
        if toks[i] != ":":
            raise ValueError("expected ':' between shape and stride")
        stride, i = _parse_tree(toks, i + 1, _stride_leaf)
        if i != len(toks):
            raise ValueError("trailing text after layout")
        pairs = _expand(shape, stride)
        modes = [(e, k, v, ax) for (e, (k, v, ax)) in pairs]
        if isinstance(shape, tuple):
            top = [len(_flat_shape(s)) for s in shape]
        else:
            top = [1]
        return Layout(text, modes, top)

    @property
    def size(self) -> int:
        n = 1
        for e, *_ in self.modes:
            n *= e
        return n

    @property
    def cosize(self) -> int:
        """Buffer extent the layout addresses (cosize, layout.hpp:277), from the lowered descriptor."""
        return int(self.lower().cosize)

    def top_sizes(self) -> list:
        """Size of every top-level mode (product of its leaves)."""
        out, r = [], 0
        for n in self.top_leaves:
            s = 1
            for e, *_ in self.modes[r:r + n]:
                s *= e
            out.append(s)
            r += n
        return out

    def mode_array(self):
        arr = (abi.tlb_mode * len(self.modes))()
        for r, (e, k, v, ax) in enumerate(self.modes):
            arr[r].extent, arr[r].kind, arr[r].stride, arr[r].axis = e, k, v, ax
        return arr

    def lower(self, ranked: bool = False) -> abi.tlb_layout_desc:
        lib = abi.load()
        d = abi.tlb_layout_desc()
        arr = self.mode_array()
        if ranked:
            tl = (C.c_int32 * len(self.top_leaves))(*self.top_leaves)
            abi.check(lib.tlb_layout_lower_ranked(arr, len(self.modes), tl, len(self.top_leaves), C.byref(d)))
        else:
            abi.check(lib.tlb_layout_lower(arr, len(self.modes), C.byref(d)))
        return d


def L(text: str) -> Layout:
    return Layout.parse(text)


def config(name: str, value: str | None) -> None:
    """tlb_config_set: change a library knob (the TLB_* environment is only read once, at first use)."""
    abi.check(abi.load().tlb_config_set(name.encode(), None if value is None else str(value).encode()))


def make_tensor(desc: abi.tlb_layout_desc, data_ptr: int | None, capacity: int, elem_bytes: int, origin: int = 0,
                counting: bool = False) -> abi.tlb_tensor:
    t = abi.tlb_tensor()
    t.layout = C.pointer(desc)
    t.data = C.c_void_p(data_ptr) if data_ptr else None
    t.origin = origin
    t.capacity = capacity
    t.elem_bytes = elem_bytes
    t.accessor = abi.ACC_COUNTING if counting else abi.ACC_BUFFER
    return t


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def tensor_of(layout: Layout | str, buf, origin: int = 0, ranked: bool = False):
    """(tlb_tensor, keepalive) over a torch tensor (device or host) viewed as a flat buffer of cells."""
    lay = L(layout) if isinstance(layout, str) else layout
    desc = lay.lower(ranked=ranked)
    t = make_tensor(desc, buf.data_ptr(), buf.numel(), buf.element_size(), origin)
    return t, (desc, buf)


def counting_tensor(layout: Layout | str, base: int = 0):
    lay = L(layout) if isinstance(layout, str) else layout
    desc = lay.lower()
    return make_tensor(desc, None, 0, 8, base, counting=True), (desc,)


def copy(src, dst, i_begin: int = 0, i_end: int = 2**64 - 1, stream=None) -> str:
    """tla::copy on device tensors built by tensor_of(); returns the plan the library chose."""
    lib = abi.load()
    abi.check(lib.tlb_copy(C.byref(src[0]), C.byref(dst[0]), i_begin, i_end, _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def copy_plan(src_layout, dst_layout, elem_bytes: int, i_begin: int = 0, i_end: int = 2**64 - 1, src_align: int = 256,
              dst_align: int = 256) -> str:
    """The plan tlb_copy would choose for two compact buffers at the given pointer alignments (no device needed)."""
    lib = abi.load()
    ls = L(src_layout) if isinstance(src_layout, str) else src_layout
    ld = L(dst_layout) if isinstance(dst_layout, str) else dst_layout
    ds, dd = ls.lower(), ld.lower()
    big = 1 << 40
    # two disjoint fake buffers (overlapping byte ranges would select the aliased plan)
    a = make_tensor(ds, src_align + (1 << 48), big, elem_bytes)
    b = make_tensor(dd, dst_align + (1 << 52), big, elem_bytes)
    abi.check(lib.tlb_copy_plan(C.byref(a), C.byref(b), i_begin, i_end))
    return lib.tlb_last_plan().decode()


def max_common_vector(a: Layout | str, b: Layout | str) -> int:
    da = (L(a) if isinstance(a, str) else a).lower()
    db = (L(b) if isinstance(b, str) else b).lower()
    k = C.c_int64(0)
    abi.check(abi.load().tlb_max_common_vector(C.byref(da), C.byref(db), C.byref(k)))
    return k.value


def copy_tv(src, dst, tv: Layout | str, stream=None) -> str:
    """tlb_copy_tv: thread-value partitioned copy; tv is a rank-2 layout (thread, value) -> integral coordinate."""
    lib = abi.load()
    d = (L(tv) if isinstance(tv, str) else tv).lower(ranked=True)
    abi.check(lib.tlb_copy_tv(C.byref(src[0]), C.byref(dst[0]), C.byref(d), _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def copy_tv_auto(src_layout: Layout | str, dst_layout: Layout | str, elem_bytes: int, threads: int = 256) -> str:
    """The thread-value layout the library derives for a copy, in the reference's text syntax."""
    ds = (L(src_layout) if isinstance(src_layout, str) else src_layout).lower()
    dd = (L(dst_layout) if isinstance(dst_layout, str) else dst_layout).lower()
    modes = (abi.tlb_mode * 16)()
    n = C.c_int32(0)
    tops = (C.c_int32 * 2)()
    abi.check(abi.load().tlb_copy_tv_auto(C.byref(ds), C.byref(dd), elem_bytes, threads, modes, C.byref(n), tops))
    assert n.value == 3 and list(tops) == [1, 2]
    (t, v, r) = [(int(modes[k].extent), int(modes[k].stride)) for k in range(3)]
    return f"({t[0]},({v[0]},{r[0]})):({t[1]},({v[1]},{r[1]}))"


def copy_host(src, dst) -> None:
    abi.check(abi.load().tlb_copy_host(C.byref(src[0]), C.byref(dst[0])))


def gemm_bf16(a, b, c, tile_begin: int = 0, tile_end: int = 2**32 - 1, stream=None) -> str:
    lib = abi.load()
    abi.check(lib.tlb_gemm_bf16(C.byref(a[0]), C.byref(b[0]), C.byref(c[0]), tile_begin, tile_end, _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def gemm_f16(a, b, c, tile_begin: int = 0, tile_end: int = 2**32 - 1, stream=None) -> str:
    lib = abi.load()
    abi.check(lib.tlb_gemm_f16(C.byref(a[0]), C.byref(b[0]), C.byref(c[0]), tile_begin, tile_end, _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def gemm_bf16_tiled(a, b, c, tiler, stream=None) -> str:
    """tlb_gemm_bf16_tiled: tiler = (bm, bn, bk), the CTA (pair) tile of zipped_divide(C, [bm, bn]) and the k-block."""
    lib = abi.load()
    t = abi.tlb_gemm_tiler(*tiler)
    abi.check(lib.tlb_gemm_bf16_tiled(C.byref(a[0]), C.byref(b[0]), C.byref(c[0]), C.addressof(t), _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def locate_offsets(a: Layout | str, t: Layout | str, stream=None) -> list:
    """tlb_locate_offsets: flat modes [(extent, stride), ...] of R = left_inverse(A) o T; raises admissibility_error."""
    da = (L(a) if isinstance(a, str) else a).lower()
    dt = (L(t) if isinstance(t, str) else t).lower()
    modes = (abi.tlb_mode * abi.TLB_MAX_MODES)()
    n = C.c_int32(0)
    abi.check(abi.load().tlb_locate_offsets(C.byref(da), C.byref(dt), modes, C.byref(n), _stream_ptr(stream)))
    return [(modes[i].extent, modes[i].stride) for i in range(n.value)]


def tensormap_cache_stats():
    h, m = C.c_uint64(0), C.c_uint64(0)
    abi.check(abi.load().tlb_tensormap_cache_stats(C.byref(h), C.byref(m)))
    return h.value, m.value


def gemm_tile_count(a, b, c) -> int:
    n = C.c_uint32(0)
    abi.check(abi.load().tlb_gemm_tile_count(C.byref(a[0]), C.byref(b[0]), C.byref(c[0]), C.byref(n)))
    return n.value


def gemm_bf16_batched(a, b, c, a_bs: int, b_bs: int, c_bs: int, batch_begin: int, batch_end: int, stream=None) -> str:
    lib = abi.load()
    abi.check(lib.tlb_gemm_bf16_batched(C.byref(a[0]), C.byref(b[0]), C.byref(c[0]), a_bs, b_bs, c_bs, batch_begin,
                                        batch_end, _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def gemm_bf16_host(a, b, c) -> None:
    abi.check(abi.load().tlb_gemm_bf16_host(C.byref(a[0]), C.byref(b[0]), C.byref(c[0])))


def gemm_i64(a, b, c, status_buf=None, stream=None) -> str:
    lib = abi.load()
    sp = status_buf.data_ptr() if status_buf is not None else None
    abi.check(lib.tlb_gemm_i64(C.byref(a[0]), C.byref(b[0]), C.byref(c[0]), sp, _stream_ptr(stream)))
    return lib.tlb_last_plan().decode()


def eval_range(layout: Layout | str, i0: int, n: int, out, stream=None) -> None:
    lay = L(layout) if isinstance(layout, str) else layout
    d = lay.lower()
    abi.check(abi.load().tlb_eval_range(C.byref(d), i0, n, out.data_ptr(), _stream_ptr(stream)))


def eval_range_host(layout: Layout | str, i0: int, n: int, out) -> None:
    """tlb_eval_range_host: `out` is a HOST int64 tensor / array (pinned memory makes the download asynchronous)."""
    lay = L(layout) if isinstance(layout, str) else layout
    d = lay.lower()
    ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
    abi.check(abi.load().tlb_eval_range_host(C.byref(d), i0, n, ptr))


def idx2crd_range(layout: Layout | str, i0: int, n: int, out, stream=None) -> None:
    lay = L(layout) if isinstance(layout, str) else layout
    d = lay.lower()
    abi.check(abi.load().tlb_idx2crd_range(C.byref(d), i0, n, out.data_ptr(), _stream_ptr(stream)))


def crd2idx_range(layout: Layout | str, crd, n: int, out, stream=None, status_buf=None) -> None:
    """tla::crd2idx over n natural coordinates; with status_buf (int32 on device, zeroed) a checked_mul / checked_add
    wrap is reported there as TLB_ERR_OVERFLOW."""
    lay = L(layout) if isinstance(layout, str) else layout
    d = lay.lower()
    sp = status_buf.data_ptr() if status_buf is not None else None
    abi.check(abi.load().tlb_crd2idx_range_checked(C.byref(d), crd.data_ptr(), n, out.data_ptr(), sp, _stream_ptr(stream)))


def rinv_check_range(layout, rinv, k0: int, n: int, counter, stream=None) -> None:
    dl = (L(layout) if isinstance(layout, str) else layout).lower()
    dr = (L(rinv) if isinstance(rinv, str) else rinv).lower()
    abi.check(abi.load().tlb_rinv_check_range(C.byref(dl), C.byref(dr), k0, n, counter.data_ptr(), _stream_ptr(stream)))


def compose_check_range(a, b, r, i0: int, n: int, counter, stream=None) -> None:
    da, db, dr = ((L(x) if isinstance(x, str) else x).lower() for x in (a, b, r))
    abi.check(abi.load().tlb_compose_check_range(C.byref(da), C.byref(db), C.byref(dr), i0, n, counter.data_ptr(),
                                                 _stream_ptr(stream)))


def eval_axes_range(layout: Layout | str, n_axes: int, i0: int, n: int, out, stream=None) -> None:
    lay = L(layout) if isinstance(layout, str) else layout
    arr = lay.mode_array()
    abi.check(abi.load().tlb_eval_axes_range(arr, len(lay.modes), n_axes, i0, n, out.data_ptr(), _stream_ptr(stream)))


def tensormap_describe(parent: Layout | str, tile: Layout | str):
    """(rank, dims, strides, box) of the TMA dimensions derived from a divided layout (host only)."""
    lp = (L(parent) if isinstance(parent, str) else parent).lower()
    lt = (L(tile) if isinstance(tile, str) else tile).lower()
    rank = C.c_int32(0)
    dims, strides, box = (C.c_uint64 * 5)(), (C.c_uint64 * 5)(), (C.c_uint32 * 5)()
    abi.check(abi.load().tlb_tensormap_describe(C.byref(lp), C.byref(lt), C.byref(rank), dims, strides, box))
    r = rank.value
    return r, list(dims)[:r], list(strides)[:r], list(box)[:r]


def tensormap_fetch(parent: Layout | str, tile: Layout | str, buf, coords, swizzle: int = 0, stream=None):
    """Builds the tensor map of (parent, tile) over `buf`, fetches the box at `coords` and returns it as a torch
    uint8 tensor on the device (de-swizzled, dimension 0 fastest)."""
    import torch
    lib = abi.load()
    lp = (L(parent) if isinstance(parent, str) else parent).lower()
    lt = (L(tile) if isinstance(tile, str) else tile).lower()
    eb = buf.element_size()
    raw = C.create_string_buffer(128 + 64)
    addr = (C.addressof(raw) + 63) & ~63
    abi.check(lib.tlb_tensormap_from_divided(C.byref(lp), C.byref(lt), eb, swizzle, buf.data_ptr(), addr))
    rank, dims, strides, box = tensormap_describe(parent, tile)
    nbytes = eb
    for b in box:
        nbytes *= b
    out = torch.empty(nbytes, dtype=torch.uint8, device=buf.device)
    cc = (C.c_int32 * 5)(*([int(c) for c in coords] + [0] * (5 - len(coords))))
    abi.check(lib.tlb_tensormap_fetch_tile(addr, rank, cc, nbytes, swizzle, out.data_ptr(), _stream_ptr(stream)))
    return out

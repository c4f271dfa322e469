// tla/device.hpp — the C++ host side of the sm_100a hot path: device tensors for the `tla` layout algebra.
//
// This header is ADDITIVE to the reference library (arXiv 2603.02298 artifact, proj/include/tla): include it
// after the reference's own headers (-I <reference>/proj/include -I <this repo>/include) and link libtlb.
// Layouts keep being built by the reference's host algebra (compose, logical_divide, zipped_divide,
// right_inverse, ... algebra.hpp); this header only lowers them (flat_modes, layout.hpp:111) and dispatches
//   tla::copy  (tensor.hpp:195)   -> tlb_copy
//   tla::gemm  (tensor.hpp:214)   -> tlb_gemm_bf16 / tlb_gemm_f16 / tlb_gemm_i64
//   tla::eval_int over a range (layout.hpp:74) -> tlb_eval_range
// to the C ABI of include/tlb.h when the cells live in device memory. Same argument meaning, same exception
// types (common.hpp:13-97). Device pointers are borrowed, never owned.
#pragma once

#include <cstdint>
#include <vector>

#include "tla/algebra.hpp"
#include "tla/layout.hpp"
#include "tla/tensor.hpp"

#include "tlb.h"

namespace tla {

// A tensor over device cells, seen through the reference's own Tensor type. The VIEW is a reference Tensor over a
// COUNTING accessor (tensor.hpp:22): its accessor position is the cell index of the view's origin inside the device
// buffer, so the reference's own slice / keep / fix (tensor.hpp:145-192) compose views of device memory exactly as they
// do for host tensors: nothing about slicing is re-implemented here, and a sliced device tensor goes straight back into
// tla::copy / tla::gemm below. It is the device flavour of Tensor(Accessor::buffer(storage, origin), layout).
struct DeviceTensor {
    Tensor view;            // counting accessor at the view's origin + the view's layout
    void* data = nullptr;   // device pointer to cell 0 of the buffer (borrowed)
    Int capacity = 0;       // buffer length in cells; every access is bounds-checked against it before launch
    int elem_bytes = 8;     // 1, 2, 4, 8 or 16; the reference's own cells are 8-byte Int
    void* stream = nullptr; // cudaStream_t

    DeviceTensor(void* d, Int cap, int eb, Layout l, Int org = 0, void* s = nullptr)
        : view(Accessor::counting(org), std::move(l)), data(d), capacity(cap), elem_bytes(eb), stream(s) {}
    // the same storage behind another view (what slice returns)
    DeviceTensor(const DeviceTensor& storage, Tensor v)
        : view(std::move(v)), data(storage.data), capacity(storage.capacity), elem_bytes(storage.elem_bytes), stream(storage.stream) {
        if (view.accessor().tag() != Accessor::Tag::Counting) throw contract_error("device views are tracked by counting accessors");
    }
    [[nodiscard]] const Layout& layout() const { return view.layout(); }
    [[nodiscard]] Int origin() const { return view.accessor().position(); }
};

// slice (tensor.hpp:187): partial evaluation of a device tensor; the fixed part advances the origin, the kept part is the
// sliced layout. Same coordinates, same exceptions (index_error, structural_error) as on the host: it IS the host code.
inline DeviceTensor slice(const DeviceTensor& t, const SliceCoord& sc) { return DeviceTensor(t, slice(t.view, sc)); }

// local_tile(t, tiler, blk) = slice(zipped_divide(t, tiler), (_, blk)) (partition_demo.cpp): the blk-th tile.
inline DeviceTensor local_tile(const DeviceTensor& t, const Tiler& tiler, const SliceCoord& blk) {
    Tensor divided(t.view.accessor(), zipped_divide(t.layout(), tiler));
    std::vector<SliceCoord> sc{keep(), blk};
    return DeviceTensor(t, slice(divided, SliceCoord(std::move(sc))));
}

namespace device_detail {

inline void rethrow(int st) {
    if (st == TLB_OK) return;
    const std::string m = tlb_last_error();
    switch (st) {
    case TLB_ERR_CONTRACT: throw contract_error(m);
    case TLB_ERR_BOUNDS: throw bounds_error(m);
    case TLB_ERR_STRUCTURAL: throw structural_error(m);
    case TLB_ERR_SEMIMODULE: throw semimodule_error(m);
    case TLB_ERR_OVERFLOW: throw overflow_error(m);
    case TLB_ERR_INDEX: throw index_error(m);
    case TLB_ERR_ADMISSIBILITY: throw admissibility_error(m);
    default: throw resource_error(m); // CUDA failure / no device / no kernel for this request
    }
}

inline tlb_layout_desc lower(const Layout& l, bool ranked) {
    std::vector<tlb_mode> modes;
    for (const FlatMode& m : flat_modes(l)) {
        tlb_mode t{m.first, 0, TLB_KIND_INT, 0};
        if (m.second.is_int()) {
            t.stride = m.second.value();
        } else if (m.second.is_xor()) {
            t.stride = m.second.mask();
            t.kind = TLB_KIND_XOR;
        } else {
            t.stride = m.second.scale();
            t.axis = static_cast<int32_t>(m.second.axis());
            t.kind = TLB_KIND_BASIS;
        }
        modes.push_back(t);
    }
    tlb_layout_desc d;
    if (ranked) {
        std::vector<int32_t> tops;
        for (Int i = 0; i < l.rank(); ++i)
            tops.push_back(static_cast<int32_t>(flat_leaves(l.shape()[static_cast<std::size_t>(i)]).size()));
        rethrow(tlb_layout_lower_ranked(modes.data(), static_cast<int>(modes.size()), tops.data(),
                                        static_cast<int>(tops.size()), &d));
    } else {
        rethrow(tlb_layout_lower(modes.data(), static_cast<int>(modes.size()), &d));
    }
    return d;
}

inline tlb_tensor view(const tlb_layout_desc& d, const DeviceTensor& t) {
    return tlb_tensor{&d, t.data, t.origin(), t.capacity, t.elem_bytes, TLB_ACC_BUFFER};
}

} // namespace device_detail

// dst(i) = src(i) over the shared integral coordinate space (tensor.hpp:195). [i_begin, i_end) restricts the
// coordinate range (multi-GPU sharding); the default is the whole domain.
inline void copy(const DeviceTensor& src, const DeviceTensor& dst, Int i_begin = 0, Int i_end = -1) {
    tlb_layout_desc ds = device_detail::lower(src.layout(), false), dd = device_detail::lower(dst.layout(), false);
    tlb_tensor s = device_detail::view(ds, src), d = device_detail::view(dd, dst);
    device_detail::rethrow(tlb_copy(&s, &d, static_cast<uint64_t>(i_begin),
                                    i_end < 0 ? UINT64_MAX : static_cast<uint64_t>(i_end), dst.stream));
}

// Thread-value partitioned copy: `tv` is a rank-2 layout (thread, value) -> integral coordinate, built with the
// reference's own products (raked_product / blocked_product, algebra.hpp:629-635; the thread-value maps of
// proj/demo/partition_demo.cpp:26-40). Logical thread t moves dst(tv(t, v)) = src(tv(t, v)) for every value v.
inline void copy(const DeviceTensor& src, const DeviceTensor& dst, const Layout& tv) {
    tlb_layout_desc ds = device_detail::lower(src.layout(), false), dd = device_detail::lower(dst.layout(), false),
                    dt = device_detail::lower(tv, true);
    tlb_tensor s = device_detail::view(ds, src), d = device_detail::view(dd, dst);
    device_detail::rethrow(tlb_copy_tv(&s, &d, &dt, dst.stream));
}

// A counting source (Accessor::counting(base), tensor.hpp:22): dst(i) = base + src_layout(i).
inline void copy_counting(const Layout& src_layout, Int base, const DeviceTensor& dst) {
    tlb_layout_desc ds = device_detail::lower(src_layout, false), dd = device_detail::lower(dst.layout(), false);
    tlb_tensor s{&ds, nullptr, base, 0, 8, TLB_ACC_COUNTING}, d = device_detail::view(dd, dst);
    device_detail::rethrow(tlb_copy(&s, &d, 0, UINT64_MAX, dst.stream));
}

// C(m,n) += A(m,k) * B(n,k), rank-2 tensors with modes addressed by 1-D coordinates (tensor.hpp:214).
// elem_bytes 8/8/8: the reference's checked int64 arithmetic; the call waits for the kernel and throws overflow_error
// on a wrap (tlb_gemm_i64 with a NULL status word is synchronous), and takes no tile range (contract_error otherwise).
// elem_bytes 2/2/4: bf16 operands, fp32 accumulator starting from C, asynchronous on c.stream.
inline void gemm(const DeviceTensor& a, const DeviceTensor& b, const DeviceTensor& c, std::uint32_t tile_begin = 0,
                 std::uint32_t tile_end = UINT32_MAX) {
    tlb_layout_desc da = device_detail::lower(a.layout(), true), db = device_detail::lower(b.layout(), true),
                    dc = device_detail::lower(c.layout(), true);
    tlb_tensor ta = device_detail::view(da, a), tb = device_detail::view(db, b), tc = device_detail::view(dc, c);
    if (c.elem_bytes == 8) {
        if (tile_begin != 0 || tile_end != UINT32_MAX) throw contract_error("gemm: tile ranges apply to the bf16 / fp16 paths only");
        device_detail::rethrow(tlb_gemm_i64(&ta, &tb, &tc, nullptr, c.stream));
    } else device_detail::rethrow(tlb_gemm_bf16(&ta, &tb, &tc, tile_begin, tile_end, c.stream));
}

// The same GEMM partitioned by a caller-chosen tiler [bm, bn, bk] (tlb_gemm_bf16_tiled): bf16 operands only.
inline void gemm(const DeviceTensor& a, const DeviceTensor& b, const DeviceTensor& c, const tlb_gemm_tiler& tiler) {
    tlb_layout_desc da = device_detail::lower(a.layout(), true), db = device_detail::lower(b.layout(), true),
                    dc = device_detail::lower(c.layout(), true);
    tlb_tensor ta = device_detail::view(da, a), tb = device_detail::view(db, b), tc = device_detail::view(dc, c);
    device_detail::rethrow(tlb_gemm_bf16_tiled(&ta, &tb, &tc, &tiler, c.stream));
}

// Same contract with IEEE fp16 operands (elem_bytes 2/2/4).
inline void gemm_f16(const DeviceTensor& a, const DeviceTensor& b, const DeviceTensor& c, std::uint32_t tile_begin = 0,
                     std::uint32_t tile_end = UINT32_MAX) {
    tlb_layout_desc da = device_detail::lower(a.layout(), true), db = device_detail::lower(b.layout(), true),
                    dc = device_detail::lower(c.layout(), true);
    tlb_tensor ta = device_detail::view(da, a), tb = device_detail::view(db, b), tc = device_detail::view(dc, c);
    device_detail::rethrow(tlb_gemm_f16(&ta, &tb, &tc, tile_begin, tile_end, c.stream));
}

// compose (algebra.hpp:235-250) with its O(size(B)) re-check on the device. The reference composes leaf by leaf and then
// verifies R(i) == A(B(i)) for EVERY i on the host (detail::verify_distributed, algebra.hpp:211-228): about 0.27 us per
// element, 18 s for the 8192 x 8192 transpose map of config C1. This is the same function, with the same per-leaf
// composition (the reference's own detail:: helpers) and the same exceptions, and the pointwise check in libtlb.
inline Layout compose_device(const Layout& a, const Layout& b, void* stream = nullptr) {
    Kind bk = b.kind();
    if (bk == Kind::Xor) throw semimodule_error("xor strides are not admissible on the right of composition");
    std::vector<FlatMode> modes = detail::compose_lhs_modes(a);
    std::size_t b_leaves = 0;
    for (const FlatMode& m : flat_modes(b))
        if (m.first > 1) ++b_leaves;
    if (bk == Kind::Int && modes.size() >= 2) detail::check_distributive(b);
    detail::ComposeRec rec{a, modes};
    Layout r = rec.run(b.shape(), b.stride());
    if (bk == Kind::Int && b_leaves >= 2) {
        if (a.kind() == Kind::Basis) {
            detail::verify_distributed(a, b, r); // coordinate codomain: stays on the host
        } else {
            tlb_layout_desc da = device_detail::lower(a, false), db = device_detail::lower(b, false), dr = device_detail::lower(r, false);
            uint64_t bad = 0;
            device_detail::rethrow(tlb_compose_check(&da, &db, &dr, &bad, stream));
            if (bad) throw non_distributive_error("composition does not distribute: mode images interleave");
        }
    }
    return r;
}

// locate_offsets (analysis.hpp:40-56) with the O(size(T)) admissibility loop on the device; returns R like the reference.
inline Layout locate_offsets_device(const Layout& a, const Layout& t, void* stream = nullptr) {
    tlb_layout_desc da = device_detail::lower(a, false), dt = device_detail::lower(t, false);
    tlb_mode r[TLB_MAX_MODES];
    int32_t n = 0;
    device_detail::rethrow(tlb_locate_offsets(&da, &dt, r, &n, stream));
    std::vector<FlatMode> modes;
    for (int32_t i = 0; i < n; ++i) modes.emplace_back(r[i].extent, StrideElem(r[i].stride));
    return from_flat_modes(modes);
}

// d_out[k] = L(i0 + k), k < n: eval_int (layout.hpp:74) over a range, int64 out, extended domain allowed.
inline void eval_range(const Layout& l, Int i0, Int n, Int* d_out, void* stream = nullptr) {
    tlb_layout_desc d = device_detail::lower(l, false);
    device_detail::rethrow(tlb_eval_range(&d, static_cast<uint64_t>(i0), static_cast<uint64_t>(n), d_out, stream));
}

} // namespace tla

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

#include "tla/layout.hpp"
#include "tla/tensor.hpp"

#include "tlb.h"

namespace tla {

// A tensor over device cells: the device flavour of Tensor(Accessor::buffer(storage, origin), layout).
struct DeviceTensor {
    void* data = nullptr;   // device pointer to cell 0 of the buffer (borrowed)
    Int capacity = 0;       // buffer length in cells; every access is bounds-checked against it before launch
    int elem_bytes = 8;     // 1, 2, 4, 8 or 16; the reference's own cells are 8-byte Int
    Layout layout;
    Int origin = 0;         // accessor position before the layout offset is applied
    void* stream = nullptr; // cudaStream_t

    DeviceTensor(void* d, Int cap, int eb, Layout l, Int org = 0, void* s = nullptr)
        : data(d), capacity(cap), elem_bytes(eb), layout(std::move(l)), origin(org), stream(s) {}
};

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
    return tlb_tensor{&d, t.data, t.origin, t.capacity, t.elem_bytes, TLB_ACC_BUFFER};
}

} // namespace device_detail

// dst(i) = src(i) over the shared integral coordinate space (tensor.hpp:195). [i_begin, i_end) restricts the
// coordinate range (multi-GPU sharding); the default is the whole domain.
inline void copy(const DeviceTensor& src, const DeviceTensor& dst, Int i_begin = 0, Int i_end = -1) {
    tlb_layout_desc ds = device_detail::lower(src.layout, false), dd = device_detail::lower(dst.layout, false);
    tlb_tensor s = device_detail::view(ds, src), d = device_detail::view(dd, dst);
    device_detail::rethrow(tlb_copy(&s, &d, static_cast<uint64_t>(i_begin),
                                    i_end < 0 ? UINT64_MAX : static_cast<uint64_t>(i_end), dst.stream));
}

// A counting source (Accessor::counting(base), tensor.hpp:22): dst(i) = base + src_layout(i).
inline void copy_counting(const Layout& src_layout, Int base, const DeviceTensor& dst) {
    tlb_layout_desc ds = device_detail::lower(src_layout, false), dd = device_detail::lower(dst.layout, false);
    tlb_tensor s{&ds, nullptr, base, 0, 8, TLB_ACC_COUNTING}, d = device_detail::view(dd, dst);
    device_detail::rethrow(tlb_copy(&s, &d, 0, UINT64_MAX, dst.stream));
}

// C(m,n) += A(m,k) * B(n,k), rank-2 tensors with modes addressed by 1-D coordinates (tensor.hpp:214).
// elem_bytes 8/8/8: the reference's checked int64 arithmetic; the call waits for the kernel and throws overflow_error
// on a wrap (tlb_gemm_i64 with a NULL status word is synchronous), and takes no tile range (contract_error otherwise).
// elem_bytes 2/2/4: bf16 operands, fp32 accumulator starting from C, asynchronous on c.stream.
inline void gemm(const DeviceTensor& a, const DeviceTensor& b, const DeviceTensor& c, std::uint32_t tile_begin = 0,
                 std::uint32_t tile_end = UINT32_MAX) {
    tlb_layout_desc da = device_detail::lower(a.layout, true), db = device_detail::lower(b.layout, true),
                    dc = device_detail::lower(c.layout, true);
    tlb_tensor ta = device_detail::view(da, a), tb = device_detail::view(db, b), tc = device_detail::view(dc, c);
    if (c.elem_bytes == 8) {
        if (tile_begin != 0 || tile_end != UINT32_MAX) throw contract_error("gemm: tile ranges apply to the bf16 / fp16 paths only");
        device_detail::rethrow(tlb_gemm_i64(&ta, &tb, &tc, nullptr, c.stream));
    } else device_detail::rethrow(tlb_gemm_bf16(&ta, &tb, &tc, tile_begin, tile_end, c.stream));
}

// Same contract with IEEE fp16 operands (elem_bytes 2/2/4).
inline void gemm_f16(const DeviceTensor& a, const DeviceTensor& b, const DeviceTensor& c, std::uint32_t tile_begin = 0,
                     std::uint32_t tile_end = UINT32_MAX) {
    tlb_layout_desc da = device_detail::lower(a.layout, true), db = device_detail::lower(b.layout, true),
                    dc = device_detail::lower(c.layout, true);
    tlb_tensor ta = device_detail::view(da, a), tb = device_detail::view(db, b), tc = device_detail::view(dc, c);
    device_detail::rethrow(tlb_gemm_f16(&ta, &tb, &tc, tile_begin, tile_end, c.stream));
}

// d_out[k] = L(i0 + k), k < n: eval_int (layout.hpp:74) over a range, int64 out, extended domain allowed.
inline void eval_range(const Layout& l, Int i0, Int n, Int* d_out, void* stream = nullptr) {
    tlb_layout_desc d = device_detail::lower(l, false);
    device_detail::rethrow(tlb_eval_range(&d, static_cast<uint64_t>(i0), static_cast<uint64_t>(n), d_out, stream));
}

} // namespace tla

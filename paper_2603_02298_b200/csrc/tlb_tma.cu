// TMA tensor-map builder. Tensor maps are derived from layouts: the parent layout's flat
// Int leaves give globalDim / globalStrides, the tile mode of zipped_divide(parent, tiler)
// (algebra.hpp:595) gives boxDim / elementStrides, and the staging swizzle is one of the
// hardware modes (128 B = Swizzle<3,4,3> on byte offsets = reference layout (128,8):(f1,f144)).
// cuTensorMapEncodeTiled is resolved through cudaGetDriverEntryPoint so libtlb.so carries no
// link-time dependency on libcuda (it must load on the GPU-less build host).
#include <algorithm>
#include <cstring>
#include <vector>

#include <cuda.h>

#include "tlb_internal.h"

namespace tlb {

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        (void)cudaGetLastError();
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}
} // namespace

int tma_encode(TmaDesc* out, int dtype_bytes, bool is_float, int rank, void* base, const uint64_t* dims,
               const uint64_t* strides_bytes, const uint32_t* box, int swizzle, int l2_promotion_bytes) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(TLB_ERR_CUDA, "cuTensorMapEncodeTiled is not available from this driver");
    if (rank < 1 || rank > 5) return fail(TLB_ERR_UNSUPPORTED, "TMA tensor maps have rank 1..5");
    CUtensorMapDataType dt;
    switch (dtype_bytes) {
    case 1: dt = CU_TENSOR_MAP_DATA_TYPE_UINT8; break;
    case 2: dt = is_float ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT16; break;
    case 4: dt = is_float ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT32; break;
    case 8: dt = CU_TENSOR_MAP_DATA_TYPE_UINT64; break;
    default: return fail(TLB_ERR_UNSUPPORTED, "TMA element size must be 1, 2, 4 or 8 bytes");
    }
    if (reinterpret_cast<uintptr_t>(base) & 15) return fail(TLB_ERR_UNSUPPORTED, "TMA base address must be 16-byte aligned");
    cuuint64_t gdim[5];
    cuuint64_t gstr[4];
    cuuint32_t bdim[5];
    cuuint32_t estr[5];
    for (int d = 0; d < rank; ++d) {
        gdim[d] = dims[d];
        bdim[d] = box[d];
        estr[d] = 1;
        if (box[d] < 1 || box[d] > 256) return fail(TLB_ERR_UNSUPPORTED, "TMA box extents must be 1..256");
        if (d > 0) {
            gstr[d - 1] = strides_bytes[d - 1];
            if (gstr[d - 1] & 15) return fail(TLB_ERR_UNSUPPORTED, "TMA strides must be multiples of 16 bytes");
        }
    }
    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
    if (swizzle == TMA_SW_32) sw = CU_TENSOR_MAP_SWIZZLE_32B;
    else if (swizzle == TMA_SW_64) sw = CU_TENSOR_MAP_SWIZZLE_64B;
    else if (swizzle == TMA_SW_128) sw = CU_TENSOR_MAP_SWIZZLE_128B;
    CUtensorMapL2promotion l2 = CU_TENSOR_MAP_L2_PROMOTION_NONE;
    if (l2_promotion_bytes == 128) l2 = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    else if (l2_promotion_bytes == 256) l2 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap is 128 bytes");
    CUresult r = fn(reinterpret_cast<CUtensorMap*>(out->bytes), dt, static_cast<cuuint32_t>(rank), base, gdim, gstr,
                    bdim, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TLB_ERR_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string(int(r)));
    return TLB_OK;
}

} // namespace tlb

using namespace tlb;

// Public builder: parent = full layout (Int kind, non-negative strides), tile = the tile mode
// of zipped_divide(parent, tiler). The parent is coalesced into TMA dimensions sorted by
// stride (dimension 0 must have stride 1); every tile leaf must lie inside exactly one of them
// (its stride a multiple of the dimension's, staying inside the dimension's extent), and
// contributes extent -> boxDim, stride/dim_stride -> elementStrides.
extern "C" int tlb_tensormap_from_divided(const tlb_layout_desc* parent, const tlb_layout_desc* tile, int elem_bytes,
                                          int swizzle, void* d_base, void* out_tensormap_128B) {
    if (!parent || !tile || !out_tensormap_128B) return fail(TLB_ERR_CONTRACT, "tlb_tensormap_from_divided: null argument");
    if (parent->kind != TLB_KIND_INT || tile->kind != TLB_KIND_INT)
        return fail(TLB_ERR_SEMIMODULE, "tensor maps require integer strides");
    if (parent->flags & TLB_LF_HAS_NEG) return fail(TLB_ERR_UNSUPPORTED, "tensor maps require non-negative strides");
    if (reinterpret_cast<uintptr_t>(out_tensormap_128B) & 63)
        return fail(TLB_ERR_CONTRACT, "tensor map storage must be 64-byte aligned");
    // Parent leaves sorted by stride, merged when contiguous (coalesce, layout.hpp:206, after sorting).
    struct Dim { uint64_t extent, stride; uint32_t box, estride; bool used; };
    std::vector<std::pair<uint64_t, uint64_t>> leaves; // stride, extent
    for (int r = 0; r < parent->n_modes; ++r)
        if (parent->extent[r] > 1) {
            if (parent->stride[r] == 0) return fail(TLB_ERR_UNSUPPORTED, "tensor maps cannot express stride-0 (broadcast) modes");
            leaves.emplace_back(static_cast<uint64_t>(parent->stride[r]), static_cast<uint64_t>(parent->extent[r]));
        }
    std::sort(leaves.begin(), leaves.end());
    std::vector<Dim> dims;
    for (auto& [st, ex] : leaves) {
        if (!dims.empty() && dims.back().stride * dims.back().extent == st) dims.back().extent *= ex;
        else dims.push_back({ex, st, 1, 1, false});
    }
    if (dims.empty()) dims.push_back({1, 1, 1, 1, false});
    if (dims[0].stride != 1) return fail(TLB_ERR_UNSUPPORTED, "tensor maps need a stride-1 innermost dimension");
    if (dims.size() > 5) return fail(TLB_ERR_UNSUPPORTED, "layout needs more than 5 TMA dimensions");
    for (int r = 0; r < tile->n_modes; ++r) {
        uint64_t e = static_cast<uint64_t>(tile->extent[r]);
        if (e == 1) continue;
        if (tile->stride[r] <= 0) return fail(TLB_ERR_UNSUPPORTED, "tile leaves must have positive strides");
        uint64_t s = static_cast<uint64_t>(tile->stride[r]);
        Dim* hit = nullptr;
        for (auto it = dims.rbegin(); it != dims.rend(); ++it)
            if (s >= it->stride && s % it->stride == 0) { hit = &*it; break; }
        if (!hit || hit->used) return fail(TLB_ERR_UNSUPPORTED, "tile leaf does not map onto one TMA dimension");
        uint64_t es = s / hit->stride;
        if (es > 8 || (e - 1) * es >= hit->extent) return fail(TLB_ERR_UNSUPPORTED, "tile leaf exceeds its TMA dimension");
        // the driver's boxDim counts the traversed extent; elementStrides subsample it
        hit->box = static_cast<uint32_t>(e * es);
        hit->estride = static_cast<uint32_t>(es);
        hit->used = true;
    }
    for (auto& d : dims) if (d.estride != 1) return fail(TLB_ERR_UNSUPPORTED, "strided (elementStrides > 1) tiles are not built yet");
    uint64_t gd[5], gs[4];
    uint32_t bx[5];
    for (size_t d = 0; d < dims.size(); ++d) {
        gd[d] = dims[d].extent;
        bx[d] = dims[d].box;
        if (d > 0) gs[d - 1] = dims[d].stride * static_cast<uint64_t>(elem_bytes);
    }
    TmaDesc tmp;
    TLB_TRY(tma_encode(&tmp, elem_bytes, false, static_cast<int>(dims.size()), d_base, gd, gs, bx, swizzle, 128));
    std::memcpy(out_tensormap_128B, tmp.bytes, 128);
    return TLB_OK;
}

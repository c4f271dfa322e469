// TMA tensor-map builder. Tensor maps are derived from layouts: the parent layout's flat
// Int leaves give globalDim / globalStrides, the tile mode of zipped_divide(parent, tiler)
// (algebra.hpp:595) gives boxDim / elementStrides, and the staging swizzle is one of the
// hardware modes (128 B = Swizzle<3,4,3> on byte offsets = reference layout (128,8):(f1,f144)).
// cuTensorMapEncodeTiled is resolved through cudaGetDriverEntryPoint so libtlb.so carries no
// link-time dependency on libcuda (it must load on the GPU-less build host).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda.h>

#include "tlb_internal.h"
#include "tlb_gemm.h"

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

namespace {
// Cache of encoded tensor maps, keyed by everything that goes into cuTensorMapEncodeTiled plus the device: a GEMM or a
// TMA-fed copy issued again on the same buffers (the steady state of a training / serving loop, and every step of
// bench.py) reuses its maps instead of re-encoding three of them per call. Mutex-guarded; 256 entries, round-robin
// replacement; the only state the library shares between host threads besides the launch counter and the knobs.
struct MapKey {
    int32_t device, dtype_bytes, is_float, rank, swizzle, l2;
    uint64_t base;
    uint64_t dims[5];
    uint64_t strides[4];
    uint32_t box[5];
    uint32_t pad_;
};
struct MapEntry {
    MapKey key;
    TmaDesc desc;
};
constexpr int kMapCache = 256;
std::mutex g_map_mu;
std::vector<MapEntry> g_map_cache;
unsigned g_map_next = 0;
std::atomic<uint64_t> g_map_hits{0}, g_map_misses{0};
} // namespace

uint64_t tma_cache_hits() { return g_map_hits.load(std::memory_order_relaxed); }
uint64_t tma_cache_misses() { return g_map_misses.load(std::memory_order_relaxed); }

int tma_encode(TmaDesc* out, int dtype_bytes, int is_float, int rank, void* base, const uint64_t* dims,
               const uint64_t* strides_bytes, const uint32_t* box, int swizzle, int l2_promotion_bytes) {
    if (rank < 1 || rank > 5) return fail(TLB_ERR_UNSUPPORTED, "TMA tensor maps have rank 1..5");
    MapKey key;
    std::memset(&key, 0, sizeof(key));
    if (cudaGetDevice(&key.device) != cudaSuccess) key.device = -1;
    key.dtype_bytes = dtype_bytes;
    key.is_float = is_float;
    key.rank = rank;
    key.swizzle = swizzle;
    key.l2 = l2_promotion_bytes;
    key.base = reinterpret_cast<uint64_t>(base);
    for (int d = 0; d < rank; ++d) {
        key.dims[d] = dims[d];
        key.box[d] = box[d];
        if (d > 0) key.strides[d - 1] = strides_bytes[d - 1];
    }
    {
        std::lock_guard<std::mutex> lock(g_map_mu);
        for (const MapEntry& e : g_map_cache)
            if (std::memcmp(&e.key, &key, sizeof(key)) == 0) {
                *out = e.desc;
                g_map_hits.fetch_add(1, std::memory_order_relaxed);
                return TLB_OK;
            }
    }
    const int st = tma_encode_uncached(out, dtype_bytes, is_float, rank, base, dims, strides_bytes, box, swizzle, l2_promotion_bytes);
    if (st != TLB_OK) return st;
    g_map_misses.fetch_add(1, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lock(g_map_mu);
    if (g_map_cache.size() < static_cast<size_t>(kMapCache)) g_map_cache.push_back({key, *out});
    else g_map_cache[g_map_next++ % kMapCache] = {key, *out};
    return TLB_OK;
}

int tma_encode_uncached(TmaDesc* out, int dtype_bytes, int is_float, int rank, void* base, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box, int swizzle, int l2_promotion_bytes) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(TLB_ERR_CUDA, "cuTensorMapEncodeTiled is not available from this driver");
    if (rank < 1 || rank > 5) return fail(TLB_ERR_UNSUPPORTED, "TMA tensor maps have rank 1..5");
    CUtensorMapDataType dt;
    switch (dtype_bytes) {
    case 1: dt = CU_TENSOR_MAP_DATA_TYPE_UINT8; break;
    case 2: dt = is_float == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : is_float ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT16; break;
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

namespace tlb {

int mode_leaves(const tlb_layout_desc& L, int top, int64_t* extent, int64_t* stride, int cap) {
    int n = 0;
    for (int r = L.top_start[top]; r < L.top_start[top + 1]; ++r) {
        if (L.extent[r] == 1) continue;
        if (n > 0 && stride[n - 1] * extent[n - 1] == L.stride[r]) {
            extent[n - 1] *= L.extent[r]; // coalesce (layout.hpp:206): the two leaves walk one stride chain
            continue;
        }
        if (n == cap) return -1;
        extent[n] = L.extent[r];
        stride[n] = L.stride[r];
        ++n;
    }
    return n;
}

// The tensor map of the tiles of zipped_divide(L, [box_inner, box_outer]) (see tlb_gemm.h). Dimension order: the leaves of
// the inner mode, the leaves of the outer mode, the batch; so a box lands in shared memory as [outer tile][inner tile] with
// both tiles in the colex order of their modes, which is the order the UMMA descriptors and the epilogue expect.
int tile_dims_derive(const tlb_layout_desc& L, int inner_top, int outer_top, int64_t box_inner, int64_t box_outer,
                     int inner_src, int outer_src, int batch, int64_t batch_stride, int elem_bytes, TileDims* out) {
    if (L.kind != TLB_KIND_INT) return fail(TLB_ERR_UNSUPPORTED, "tensor maps require integer strides");
    const int64_t align = 16 / elem_bytes; // strides of dimensions 1.. must be multiples of 16 bytes
    uint64_t* dims = out->dims;
    uint64_t* strides = out->strides;
    uint32_t* box = out->box;
    TmaCoord* cc = out->c;
    int rank = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int top = pass == 0 ? inner_top : outer_top;
        int64_t e[4], st[4];
        int n = mode_leaves(L, top, e, st, 4);
        if (n < 0) return fail(TLB_ERR_UNSUPPORTED, "tensor map: a mode folds into more than 4 leaves");
        if (n == 0) { // extent-1 mode: a unit dimension
            n = 1;
            e[0] = 1;
            st[0] = pass == 0 ? 1 : align;
        }
        if (pass == 0 && st[0] != 1 && !(n == 1 && e[0] == 1))
            return fail(TLB_ERR_UNSUPPORTED, "tensor map: the inner mode does not start with a unit-stride leaf");
        int64_t t = pass == 0 ? box_inner : box_outer;
        uint64_t prefix = 1;
        for (int j = 0; j < n; ++j) {
            // five dimensions in all: a single problem may spend the batch dimension on a fifth leaf (im2col operands:
            // three row leaves (q, p, n) and two k leaves (c s, r))
            if (rank == (batch > 1 ? 4 : 5)) return fail(TLB_ERR_UNSUPPORTED, "tensor map: layout needs more than 5 TMA dimensions");
            if (st[j] <= 0) return fail(TLB_ERR_UNSUPPORTED, "tensor map: strides must be positive");
            if (!(pass == 0 && j == 0) && (st[j] % align != 0 && e[j] > 1))
                return fail(TLB_ERR_UNSUPPORTED, "tensor map: strides must be multiples of 16 bytes");
            if (e[j] >= (1ll << 32)) return fail(TLB_ERR_UNSUPPORTED, "tensor map: extent exceeds 2^32");
            const bool last = j + 1 == n;
            int64_t b;
            if (t == 1) b = 1;
            else if (last) b = t; // ragged / short outermost leaf: the TMA unit clips and zero-fills
            else if (t <= e[j]) {
                if (e[j] % t != 0) return fail(TLB_ERR_UNSUPPORTED, "tensor map: tile straddles a leaf boundary");
                b = t;
            } else {
                if (t % e[j] != 0) return fail(TLB_ERR_UNSUPPORTED, "tensor map: tile straddles a leaf boundary");
                b = e[j];
            }
            // the swizzled staging layouts need the whole inner tile in ONE dimension (rows of box_inner elements)
            if (pass == 0 && j == 0 && b != box_inner && !(last))
                return fail(TLB_ERR_UNSUPPORTED, "tensor map: the inner tile does not fit the unit-stride leaf");
            if (b > 256) return fail(TLB_ERR_UNSUPPORTED, "tensor map: box extents must be 1..256");
            t = t == 1 ? 1 : (last ? 1 : (t <= e[j] ? 1 : t / e[j]));
            dims[rank] = static_cast<uint64_t>(e[j]);
            strides[rank] = static_cast<uint64_t>(st[j]);
            box[rank] = static_cast<uint32_t>(b);
            if (prefix >= (1ull << 31)) return fail(TLB_ERR_UNSUPPORTED, "tensor map: mode extent exceeds 2^31");
            cc[rank] = tma_coord(static_cast<uint32_t>(pass == 0 ? inner_src : outer_src), static_cast<uint32_t>(prefix),
                                 last ? 0u : static_cast<uint32_t>(e[j]));
            prefix *= static_cast<uint64_t>(e[j]);
            ++rank;
        }
    }
    // batch: the last dimension (a unit dimension for a single problem, dropped when the leaves need all five)
    if (rank == 5) {
        out->rank = rank;
        return TLB_OK;
    }
    dims[rank] = static_cast<uint64_t>(std::max(batch, 1));
    if (batch > 1) {
        if (batch_stride <= 0 || batch_stride % align != 0) return fail(TLB_ERR_UNSUPPORTED, "tensor map: batch stride must be a positive multiple of 16 bytes");
        strides[rank] = static_cast<uint64_t>(batch_stride);
    } else {
        uint64_t span = 1;
        for (int d = 0; d < rank; ++d) span = std::max<uint64_t>(span, strides[d] * dims[d]);
        strides[rank] = (span + align - 1) / align * align;
    }
    box[rank] = 1;
    cc[rank] = tma_coord(2u, 1u, 0u);
    ++rank;
    out->rank = rank;
    for (int d = rank; d < 5; ++d) {
        dims[d] = 1;
        strides[d] = 0;
        box[d] = 1;
        cc[d] = tma_coord(2u, 1u, 0u);
    }
    return TLB_OK;
}

int tensormap_for_tile(const tlb_layout_desc& L, int inner_top, int outer_top, int64_t box_inner, int64_t box_outer,
                       int inner_src, int outer_src, const void* base, int batch, int64_t batch_stride, int elem_bytes,
                       int is_float, int swizzle, int l2_promotion, TmaTileMap* out) {
    TileDims td;
    TLB_TRY(tile_dims_derive(L, inner_top, outer_top, box_inner, box_outer, inner_src, outer_src, batch, batch_stride, elem_bytes, &td));
    uint64_t sb[4];
    for (int d = 1; d < td.rank; ++d) sb[d - 1] = td.strides[d] * static_cast<uint64_t>(elem_bytes);
    TmaDesc tmp;
    TLB_TRY(tma_encode(&tmp, elem_bytes, is_float, td.rank, const_cast<void*>(base), td.dims, sb, td.box, swizzle, l2_promotion));
    std::memcpy(out->desc, tmp.bytes, 128);
    out->rank = td.rank;
    for (int d = 0; d < 5; ++d) out->c[d] = td.c[d];
    return TLB_OK;
}

} // namespace tlb

using namespace tlb;

// Shared derivation: parent = full layout (Int kind, non-negative strides), tile = the tile mode of
// zipped_divide(parent, tiler). The parent is coalesced into TMA dimensions sorted by stride (dimension 0
// must have stride 1); every tile leaf must lie inside exactly one of them (its stride a multiple of the
// dimension's, staying inside the dimension's extent) and contributes its extent to boxDim.
namespace tlb {
namespace {
struct Dim {
    uint64_t extent, stride;
    uint32_t box, estride;
    bool used;
};

int derive_dims(const tlb_layout_desc* parent, const tlb_layout_desc* tile, std::vector<Dim>* out) {
    if (!parent || !tile) return fail(TLB_ERR_CONTRACT, "tensor map derivation: null layout");
    if (parent->kind != TLB_KIND_INT || tile->kind != TLB_KIND_INT)
        return fail(TLB_ERR_SEMIMODULE, "tensor maps require integer strides");
    if (parent->flags & TLB_LF_HAS_NEG) return fail(TLB_ERR_UNSUPPORTED, "tensor maps require non-negative strides");
    // Tile leaves sorted by stride and coalesced: each surviving leaf needs a TMA dimension that STARTS at its stride.
    std::vector<std::pair<uint64_t, uint64_t>> tl; // stride, extent
    for (int r = 0; r < tile->n_modes; ++r) {
        if (tile->extent[r] == 1) continue;
        if (tile->stride[r] <= 0) return fail(TLB_ERR_UNSUPPORTED, "tile leaves must have positive strides");
        tl.emplace_back(static_cast<uint64_t>(tile->stride[r]), static_cast<uint64_t>(tile->extent[r]));
    }
    std::sort(tl.begin(), tl.end());
    std::vector<std::pair<uint64_t, uint64_t>> tiles;
    for (auto& [st, ex] : tl) {
        if (!tiles.empty() && tiles.back().first * tiles.back().second == st) tiles.back().second *= ex;
        else tiles.emplace_back(st, ex);
    }
    auto tile_starts_at = [&](uint64_t st) {
        for (auto& t : tiles) if (t.first == st) return true;
        return false;
    };
    // Parent leaves sorted by stride, merged when contiguous (coalesce, layout.hpp:206, after sorting) unless a
    // tile leaf starts there (the box needs that dimension boundary).
    std::vector<std::pair<uint64_t, uint64_t>> leaves; // stride, extent
    for (int r = 0; r < parent->n_modes; ++r)
        if (parent->extent[r] > 1) {
            if (parent->stride[r] == 0) return fail(TLB_ERR_UNSUPPORTED, "tensor maps cannot express stride-0 (broadcast) modes");
            leaves.emplace_back(static_cast<uint64_t>(parent->stride[r]), static_cast<uint64_t>(parent->extent[r]));
        }
    std::sort(leaves.begin(), leaves.end());
    std::vector<Dim>& dims = *out;
    for (auto& [st, ex] : leaves) {
        if (!dims.empty() && dims.back().stride * dims.back().extent == st && !tile_starts_at(st)) dims.back().extent *= ex;
        else dims.push_back({ex, st, 1, 1, false});
    }
    if (dims.empty()) dims.push_back({1, 1, 1, 1, false});
    if (dims[0].stride != 1) return fail(TLB_ERR_UNSUPPORTED, "tensor maps need a stride-1 innermost dimension");
    if (dims.size() > 5) return fail(TLB_ERR_UNSUPPORTED, "layout needs more than 5 TMA dimensions");
    for (auto& [s, e] : tiles) {
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
    return TLB_OK;
}

// One-box fetch used to validate tensor maps: the box lands in shared memory (hardware swizzle as encoded in
// the map) and is written out de-swizzled, dimension 0 fastest. The de-swizzle is Swizzle<B,4,3> on the byte
// offset (B = 1, 2, 3 for the 32 / 64 / 128-byte modes), i.e. the reference's Xor layouts (stride.hpp:142).
template <int RANK>
__global__ void __launch_bounds__(128) fetch_tile_kernel(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2,
                                                         int c3, int c4, uint32_t bytes, int swizzle_bits,
                                                         unsigned char* __restrict__ out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    const uint32_t bar = base + 32768;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        if constexpr (RANK == 1)
            asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3}], [%2];" ::"r"(base), "l"(&map), "r"(bar), "r"(c0) : "memory");
        else if constexpr (RANK == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(base), "l"(&map), "r"(bar), "r"(c0), "r"(c1) : "memory");
        else if constexpr (RANK == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(base), "l"(&map), "r"(bar), "r"(c0), "r"(c1), "r"(c2) : "memory");
        else if constexpr (RANK == 4)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(base), "l"(&map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(base), "l"(&map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4) : "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    for (;;) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar) : "memory");
        if (ok) break;
        if (clock64() - t0 > 4000000000ll) __trap();
    }
    const uint32_t xor_mask = (1u << swizzle_bits) - 1u;
    for (uint32_t o = threadIdx.x; o < bytes; o += blockDim.x) {
        const uint32_t phys = o ^ (((o >> 7) & xor_mask) << 4);
        unsigned int v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(base + phys));
        out[o] = static_cast<unsigned char>(v);
    }
}
} // namespace
} // namespace tlb

extern "C" int tlb_tensormap_from_divided(const tlb_layout_desc* parent, const tlb_layout_desc* tile, int elem_bytes,
                                          int swizzle, void* d_base, void* out_tensormap_128B) {
    if (!out_tensormap_128B) return fail(TLB_ERR_CONTRACT, "tlb_tensormap_from_divided: null argument");
    if (reinterpret_cast<uintptr_t>(out_tensormap_128B) & 63)
        return fail(TLB_ERR_CONTRACT, "tensor map storage must be 64-byte aligned");
    std::vector<Dim> dims;
    TLB_TRY(derive_dims(parent, tile, &dims));
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

extern "C" int tlb_tensormap_cache_stats(uint64_t* hits, uint64_t* misses) {
    if (hits) *hits = tma_cache_hits();
    if (misses) *misses = tma_cache_misses();
    return TLB_OK;
}

extern "C" int tlb_tensormap_describe(const tlb_layout_desc* parent, const tlb_layout_desc* tile, int32_t* rank,
                                      uint64_t* dims5, uint64_t* strides5, uint32_t* box5) {
    if (!rank || !dims5 || !strides5 || !box5) return fail(TLB_ERR_CONTRACT, "tlb_tensormap_describe: null output");
    std::vector<Dim> dims;
    TLB_TRY(derive_dims(parent, tile, &dims));
    *rank = static_cast<int32_t>(dims.size());
    for (size_t d = 0; d < 5; ++d) {
        dims5[d] = d < dims.size() ? dims[d].extent : 1;
        strides5[d] = d < dims.size() ? dims[d].stride : 0;
        box5[d] = d < dims.size() ? dims[d].box : 1;
    }
    return TLB_OK;
}

extern "C" int tlb_tensormap_fetch_tile(const void* tensormap_128B, int rank, const int32_t* coords, uint32_t box_bytes,
                                        int swizzle, void* d_out, void* stream) {
    if (!tensormap_128B || !coords || !d_out) return fail(TLB_ERR_CONTRACT, "tlb_tensormap_fetch_tile: null argument");
    if (rank < 1 || rank > 5) return fail(TLB_ERR_CONTRACT, "tensor maps have rank 1..5");
    if (box_bytes == 0 || box_bytes > 32768 || (box_bytes & 15)) return fail(TLB_ERR_UNSUPPORTED, "box must be 16..32768 bytes, a multiple of 16");
    if (swizzle < 0 || swizzle > 3) return fail(TLB_ERR_CONTRACT, "swizzle mode is 0..3");
    TLB_TRY(require_device());
    CUtensorMap map;
    std::memcpy(&map, tensormap_128B, 128);
    int c[5] = {0, 0, 0, 0, 0};
    for (int d = 0; d < rank; ++d) c[d] = coords[d];
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t smem = 32768 + 1024 + 64;
    unsigned char* out = static_cast<unsigned char*>(d_out);
#define TLB_FETCH(R)                                                                                               \
    do {                                                                                                           \
        TLB_CUDA(cudaFuncSetAttribute(fetch_tile_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
        fetch_tile_kernel<R><<<1, 128, smem, s>>>(map, c[0], c[1], c[2], c[3], c[4], box_bytes, swizzle, out);      \
    } while (0)
    switch (rank) {
    case 1: TLB_FETCH(1); break;
    case 2: TLB_FETCH(2); break;
    case 3: TLB_FETCH(3); break;
    case 4: TLB_FETCH(4); break;
    default: TLB_FETCH(5); break;
    }
#undef TLB_FETCH
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

// Internal declarations shared by the translation units of libtlb.so.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "tlb.h"

#include <cstdlib>
#include <utility>

namespace tlb {

// ---- error plumbing ---------------------------------------------------------
int fail(int status, const std::string& msg);   // records tlb_last_error(), returns status
int cuda_fail(cudaError_t e, const char* what); // TLB_ERR_CUDA with the runtime's message
void set_plan(const char* name);                // records tlb_last_plan()
void count_launch(uint64_t n = 1);              // bumps tlb_launch_count()

#define TLB_CUDA(expr)                                              \
    do {                                                            \
        cudaError_t e__ = (expr);                                   \
        if (e__ != cudaSuccess) return ::tlb::cuda_fail(e__, #expr); \
    } while (0)

#define TLB_TRY(expr)                \
    do {                             \
        int s__ = (expr);            \
        if (s__ != TLB_OK) return s__; \
    } while (0)

// ---- configuration knobs ---------------------------------------------------------
// Every tuning / debugging switch of the library. The environment (TLB_<NAME>) is read ONCE, at the first use of any
// knob; after that a knob only changes through tlb_config_set(). Reading a knob on a launch path is one relaxed atomic
// load: no getenv, no locks, no allocation.
enum KnobId {
    K_GEMM_WIDE,        // -1 auto, 0 never, 1 always take the 512 x 256 plan when it applies
    K_GEMM_SPLIT_TAIL,  // 1: cut the partial wave into k-ranges (default), 0: bitwise reproducible sums
    K_GEMM_EPILOGUE,    // 0 auto, 1 "regs": register epilogue
    K_GEMM_GROUP_M,     // rasterisation group (m-blocks)
    K_GEMM_BACKOFF_NS,
    K_GEMM_DEBUG,       // timing experiments (garbage results)
    K_GEMM_HINTS,       // L2 hints
    K_GEMM_PDL,         // programmatic dependent launch of the GEMM kernels
    K_GEMM_PREFETCH_C,
    K_GEMM_WORKERS,     // cap on CTA pairs (0 = all)
    K_GEMM_C16_SK,
    K_GEMM_SK_PCT,
    K_GEMM_EPI_KB,
    K_GEMM_CLOCK,       // record {clock64, globaltimer} per launch
    K_PDL,              // programmatic stream serialisation of the copy / eval kernels
    K_COPY_TMA,         // TMA-fed tiled copy as the default
    K_COPY_LB256,
    K_COPY_PERSIST,     // persistent ring variant of the tiled copy
    K_EVAL_NO_WARP,
    K_HOST_PIPELINE,
    K_HOST_PANEL,
    K_COPY_TMA_STAGES,  // staged tiles per CTA of the TMA-fed tiled copy
    K_COPY_TMA_CTAS,    // its CTAs per SM
    K_GEMM_CHUNK_WAVES, // waves of pair tiles per launch of the wide plan (0: one launch whatever the range)
    K_GEMM_MCAST,       // wide plan in clusters of 4 with A multicast between two pair tiles: 0 never, 1 when it applies, -1 auto
    K_GEMM_EARLY_RELEASE, // wide plan, fp32 C: accumulator halves go to registers and are released before their reductions
    K_GEMM_PACK,        // 1: operands / C that no tensor map can address are packed and run on tcgen05 (default), 0: SIMT plan
    K_GEMM_PACK_MIN,    // log2 of the smallest M*N*K that takes the packed plan
    K_COPY_TV_COMPOSE,  // tlb_copy_tv: run digit-permutation TV layouts as the copy between src o TV and dst o TV (1), or always the per-thread kernel (0)
    K_COPY_GATHER_RUN,  // gather fallback: 32 / 64-byte runs per evaluation with 256-bit accesses (1), or 16-byte vectors only (0)
    K_COPY_RAGGED,      // staged copy of ragged extents as a whole-tile body plus edge strips: log2 of the smallest element count that is cut (22), 0 = never
    K_COPY_INTERLEAVE,  // AoS <-> SoA copies on the register-permuting interleave plan (1) or the gather (0)
    K_COPY_CELL_TILES,  // tiled_u: consecutive lanes on consecutive cells, padded staging (1), or the vector-shaped lane assignment with cell-sized accesses (0)
    K_EVAL_ODOMETER,    // tlb_eval_range: leading leaves no group size divides are walked by odometer, 8 indices per thread (1), or peeled per index (0)
    K_COPY_TILES_PER_CTA, // aligned staged copy, 32 / 64-row tiles: 256 / rows tiles per CTA when there are many tiles (1), always one (0)
    K_COPY_ODD_TILES,   // staged copy: 96 / 160 / 192 / 224-row tiles for destination runs of that many cells (1), powers of two only (0)
    K_HOST_TAPER,       // pipelined host GEMM: the last panel is cut into 1/2, 1/4, 1/4 so that little is left after the last upload
    K_COUNT
};
int knob(KnobId id);

// One device is required; there is no CPU fallback anywhere in this library.
int require_device();
// Stream-ordered workspace (winner arrays, packed GEMM panels, status words): cudaMallocFromPoolAsync on a per-device pool
// of the library's own whose release threshold is unlimited, so a call that allocates the same workspace every time (a
// copy in a loop) reuses the pool's memory instead of returning it to the driver at every synchronisation. Freed with
// cudaFreeAsync. The process's default pool is left alone.
cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t stream);
cudaError_t ws_trim(size_t keep_bytes);
int sm_count();

// ---- host helpers over descriptors -------------------------------------------
// Exact min/max of origin (+|^) L(i) over i in [0, size): used by the bounds pre-flight.
struct Span {
    int64_t lo, hi;
};
int position_span(const tlb_layout_desc& L, int64_t origin, Span* out);
// Conservative proof that no checked_add/checked_mul of the reference (common.hpp:99-109)
// can overflow while evaluating L on [0, max_index].
int overflow_preflight(const tlb_layout_desc& L, int64_t origin, uint64_t max_index);
// Upper bound of |L(i)| over 0 <= i <= max_index (extended domain), saturating at INT64_MAX.
uint64_t max_abs_offset(const tlb_layout_desc& L, uint64_t max_index);
bool provably_injective(const tlb_layout_desc& L);
// Argument contract of one tensor (null pointers, accessor, element size).
int check_tensor(const tlb_tensor* t, const char* who, bool writable);
// Bounds pre-flight of tensor.hpp:99 for the positions origin (+|^) L(i), i in [i0, i0+n).
int bounds_preflight(const tlb_tensor& t, uint64_t i0, uint64_t n, const char* who, cudaStream_t stream, Span* out);
// Shared by the device-pointer and host-pointer entry points.
int copy_impl(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end, cudaStream_t stream);
int gemm_bf16_impl(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int64_t a_bs, int64_t b_bs, int64_t c_bs,
                   int batch_begin, int batch_end, uint32_t tile_begin, uint32_t tile_end, cudaStream_t stream);

// Flat view of a GEMM whose every mode coalesces to one stride (what the tcgen05 plans and the pipelined host path
// need): extents, the two strides of every operand, in elements.
struct GemmFlat {
    int64_t M, N, K;
    int64_t a_sm, a_sk, b_sn, b_sk, c_sm, c_sn;
};
bool gemm_flat_view(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, GemmFlat* out);

// Launch with programmatic stream serialisation: the kernel may be scheduled while the previous kernel of the stream
// drains. Kernels launched this way execute pdl_wait() before their first global-memory access, which blocks until
// that previous kernel has completed and flushed; without the attribute pdl_wait() is a no-op. Hides the 2-4 us of
// launch latency and scheduling ramp between back-to-back kernels (TLB_PDL=0 turns it off).
inline bool pdl_enabled() { return knob(K_PDL) != 0; }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

// ---- joint descriptor: one peel, two offsets ------------------------------------
// The common refinement of a source and a destination layout over the same integral domain:
// refined mode r has one extent and one stride on each side, so a single division chain
// yields both offsets (the copy kernels' replacement for two eval_rec walks, layout.hpp:49).
struct JointDesc {
    int32_t n;
    int32_t pad_;
    int64_t extent[TLB_MAX_MODES];
    int64_t ss[TLB_MAX_MODES]; // source stride (elements)
    int64_t ds[TLB_MAX_MODES]; // destination stride (elements)
    uint64_t magic[TLB_MAX_MODES];
    uint8_t shift[TLB_MAX_MODES];
    uint8_t log2e[TLB_MAX_MODES];
};
void joint_set_mode(JointDesc* J, int r, int64_t extent, int64_t ss, int64_t ds);

// ---- TMA tensor maps (driver entry point resolved at run time; no libcuda link) ----
struct TmaDesc {
    alignas(64) unsigned char bytes[128];
};
enum TmaSwizzle { TMA_SW_NONE = 0, TMA_SW_32 = 1, TMA_SW_64 = 2, TMA_SW_128 = 3 };
// dtype_bytes: 1,2,4,8; is_float: 0 unsigned integers, 1 bf16 / fp32, 2 fp16 (the element type matters to TMA reductions).
// Served from a mutex-guarded cache keyed by (device, base, dtype, rank, dims, strides, box, swizzle, promotion).
int tma_encode(TmaDesc* out, int dtype_bytes, int is_float, int rank, void* base, const uint64_t* dims,
               const uint64_t* strides_bytes /* rank-1 entries, dims 1.. */, const uint32_t* box,
               int swizzle, int l2_promotion_bytes);
int tma_encode_uncached(TmaDesc* out, int dtype_bytes, int is_float, int rank, void* base, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box, int swizzle, int l2_promotion_bytes);
uint64_t tma_cache_hits();
uint64_t tma_cache_misses();

} // namespace tlb

// ---- device-side layout evaluator ----------------------------------------------
// The flat peel of oracle::oracle_eval (oracle.hpp:58-69) == layout_eval on an integral
// coordinate (layout.hpp:66-71): c_r = i mod e_r, i /= e_r, last leaf unbounded; Int leaves
// contribute c*d (eval_leaf stride.hpp:138), Xor leaves the XOR of mask<<bit over the set bits
// of c (stride.hpp:142-151), which is the carry-less product clmul(c, mask).
#ifdef __CUDACC__
namespace tlb {

__device__ __forceinline__ uint64_t dev_div(const tlb_layout_desc& L, int r, uint64_t i) {
    const unsigned l2 = L.log2e[r];
    if (l2 != 0xffu) return i >> l2;
    return __umul64hi(i, L.magic[r]) >> L.shift[r];
}

__device__ __forceinline__ int64_t dev_clmul(uint64_t c, uint64_t mask) {
    uint64_t acc = 0;
    while (mask) {
        const int b = __ffsll(static_cast<long long>(mask)) - 1;
        acc ^= c << b;
        mask &= mask - 1;
    }
    return static_cast<int64_t>(acc);
}

// Offset of integral coordinate i (extended domain allowed).
__device__ __forceinline__ int64_t dev_eval(const tlb_layout_desc& L, uint64_t i) {
    int64_t acc = 0;
    const int n = L.n_modes;
    const bool is_xor = L.kind == TLB_KIND_XOR;
    for (int r = 0; r < n; ++r) {
        uint64_t c;
        if (r + 1 < n) {
            const uint64_t q = dev_div(L, r, i);
            c = i - q * static_cast<uint64_t>(L.extent[r]);
            i = q;
        } else {
            c = i;
        }
        if (is_xor) acc ^= dev_clmul(c, static_cast<uint64_t>(L.stride[r]));
        else acc += static_cast<int64_t>(c) * L.stride[r];
    }
    return acc;
}

// Offset of a 1-D coordinate inside top-level mode t only (gemm addresses each of the two
// top-level modes by one integer, tensor.hpp:203 + layout.hpp:54).
__device__ __forceinline__ int64_t dev_eval_top(const tlb_layout_desc& L, int t, uint64_t i) {
    int64_t acc = 0;
    const int lo = L.top_start[t], hi = L.top_start[t + 1];
    const bool is_xor = L.kind == TLB_KIND_XOR;
    for (int r = lo; r < hi; ++r) {
        uint64_t c;
        if (r + 1 < hi) {
            const uint64_t q = dev_div(L, r, i);
            c = i - q * static_cast<uint64_t>(L.extent[r]);
            i = q;
        } else {
            c = i;
        }
        if (is_xor) acc ^= dev_clmul(c, static_cast<uint64_t>(L.stride[r]));
        else acc += static_cast<int64_t>(c) * L.stride[r];
    }
    return acc;
}

// One peel of idx through the joint modes (last mode unbounded): both offsets at once.
__device__ __forceinline__ void dev_joint(const JointDesc& J, uint64_t i, int64_t* so, int64_t* dof) {
    int64_t a = 0, b = 0;
    const int n = J.n;
    for (int r = 0; r < n; ++r) {
        uint64_t c;
        if (r + 1 < n) {
            const unsigned l2 = J.log2e[r];
            const uint64_t q = (l2 != 0xffu) ? (i >> l2) : (__umul64hi(i, J.magic[r]) >> J.shift[r]);
            c = i - q * static_cast<uint64_t>(J.extent[r]);
            i = q;
        } else {
            c = i;
        }
        a += static_cast<int64_t>(c) * J.ss[r];
        b += static_cast<int64_t>(c) * J.ds[r];
    }
    *so = a;
    *dof = b;
}

// Accessor::offset (tensor.hpp:48-60): Int adds, Xor XORs into the absolute position.
__device__ __forceinline__ int64_t dev_position(const tlb_layout_desc& L, int64_t origin, int64_t off) {
    return L.kind == TLB_KIND_XOR ? (origin ^ off) : (origin + off);
}

} // namespace tlb
#endif

// Layout-driven copy: tla::copy(src, dst) (tensor.hpp:195-199) on device.
//
//   for i in [0, size) ascending:  dst(i) = src(i)
//
// Kernels chosen by a host planner that works on the COMMON REFINEMENT of the two layouts (every refined mode has one
// extent, one source stride, one destination stride). The first four are round 1's; round 2 added, for the ordinary
// layout pairs that fell to the gather: tiled_u / tiled_s / tiled_n (cell-granular staged tiles: unaligned bases, strided
// runs, a whole short mode as one of the runs), interleave (AoS <-> SoA by register permutation), gather_vec / gather_run
// (one evaluation per vector / per 32-64-byte run: swizzled layouts), last_writer (broadcast destinations), ragged:<plan>
// (extents that are not whole tiles: a whole-tile body plus edge strips, cut on the refined modes), and tv:<plan>
// (tlb_copy_tv of a digit-permutation thread-value layout = this copy between src o TV and dst o TV). DESIGN.md 3.2.
//
//   vec     one refined mode is contiguous on both sides: 16-byte (or narrower) vectors along
//           it, one joint peel per vector.                                  [memcpy, row permutes]
//   tiled   the source-contiguous run A and the destination-contiguous run B are different
//           modes (transpose / permute): a CTA stages a (|B| rows x 128 B of A) tile in shared
//           memory with the 128-byte XOR swizzle (Swizzle<3,4,3> on byte offsets, i.e. the
//           reference layout (128,8):(f1,f144) per 1 KiB, stride.hpp:142), so that BOTH the
//           global loads along A and the global stores along B are full 128-bit, fully
//           coalesced accesses and every shared-memory access is a conflict-free 128-bit one.
//           The V x V element blocks are transposed in registers in between.   [configs C1, C3]
//   gather  anything else (Xor strides, non-refinable shapes, misalignment, counting source):
//           one element per thread through the device evaluator. Always correct, never fast.
//   ordered non-injective destinations: last writer wins in ascending i (tensor.hpp:198), kept
//           by a two-pass winner election (atomicMax of i per destination cell).
//   aliased source and destination ranges overlap in one buffer (views share storage, tensor.hpp:29):
//           the serial read-after-write chains are resolved by pointer jumping, then one snapshot
//           and one scatter ("serial", one thread, when the destination is also non-injective).
//
// All contract / bounds / overflow checks happen on the host before any launch.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>

#include "tlb_internal.h"

namespace tlb {
namespace {

thread_local int g_copy_path = 0; // 0 auto, 1 gather, 2 tiled (LDG), 3 tiled TMA
thread_local bool g_dry_run = false; // tlb_copy_plan: run the planner, launch nothing
thread_local int g_ragged_depth = 0;   // recursion depth of the ragged cut (try_ragged)
thread_local bool g_defer_narrow = false, g_narrow_deferred = false; // copy_impl: the ragged interleave cut goes before narrow tiles
thread_local std::string g_ragged_plan;

// TLB_COPY_TMA=1 makes the TMA-fed tiled kernel the default for layouts that admit a tensor map.
bool tma_default() { return knob(K_COPY_TMA) == 1; }

constexpr int kThreads = 256;

// The tiled plan prefers 256-row tiles (1 KiB destination segments, 32 KiB of smem per CTA; C1 5.90 -> 6.09 TB/s);
// TLB_COPY_LB256=0 caps the tile at 128 rows (A/B comparisons).
bool lb256_enabled() { return knob(K_COPY_LB256) != 0; }
// Short-mode extents the register-permuting interleave plan is compiled for: 2 .. 26, 28, 30, 32 for 2- and 4-byte cells
// (bf16 / fp32: tall-skinny transposes of any width up to 32), the common ones for 1- and 8-byte cells.
bool interleave_size(int64_t e, int eb) {
    if (e < 2 || e > 32) return false;
    if (eb == 2 || eb == 4) return e % 2 == 0 || e <= 25;   // odd extents own two lane pieces (G = 2): 27, 29 and 31 cells would spill
    return e <= 10 || e == 12 || e == 16 || e == 24 || e == 32;
}

// ---------------------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------------------
template <int BYTES> struct Cell;
template <> struct Cell<1> { using type = uint8_t; };
template <> struct Cell<2> { using type = uint16_t; };
template <> struct Cell<4> { using type = uint32_t; };
template <> struct Cell<8> { using type = uint64_t; };
template <> struct Cell<16> { using type = uint4; };

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void stg_stream(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// ---------------------------------------------------------------------------------------
// gather: dst(i) = src(i), one element per thread, both layouts through the evaluator
// ---------------------------------------------------------------------------------------
template <int EB>
__global__ void __launch_bounds__(kThreads)
gather_kernel(const __grid_constant__ tlb_layout_desc S, const __grid_constant__ tlb_layout_desc D,
              const void* __restrict__ src, void* __restrict__ dst, int64_t s_origin, int64_t d_origin, uint64_t i0,
              uint64_t n, int counting) {
    using T = typename Cell<EB>::type;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t i = i0 + k;
        const int64_t sp = dev_position(S, s_origin, dev_eval(S, i));
        const int64_t dp = dev_position(D, d_origin, dev_eval(D, i));
        if constexpr (EB == 8) {
            if (counting) {
                static_cast<uint64_t*>(dst)[dp] = static_cast<uint64_t>(sp); // Accessor::deref of a counting accessor
                continue;
            }
        }
        static_cast<T*>(dst)[dp] = static_cast<const T*>(src)[sp];
    }
}

// gather, vectorised: when both layouts keep V consecutive integral coordinates in V consecutive cells (the low run of
// tla::max_common_vector, analysis.hpp:18-28, here also for Xor layouts: leaf 0 is the identity on the low bits and no
// other leaf touches them) a thread evaluates both layouts ONCE per vector and moves VB = V * elem_bytes bytes.
template <int VB>
__global__ void __launch_bounds__(kThreads)
gather_vec_kernel(const __grid_constant__ tlb_layout_desc S, const __grid_constant__ tlb_layout_desc D,
                  const char* __restrict__ src, char* __restrict__ dst, int64_t s_origin, int64_t d_origin, uint64_t i0,
                  uint64_t n_vec, int v_elems, int elem_bytes) {
    using T = typename Cell<VB>::type;
    pdl_wait();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n_vec; k += stride) {
        const uint64_t i = i0 + k * static_cast<uint64_t>(v_elems);
        const int64_t sp = dev_position(S, s_origin, dev_eval(S, i));
        const int64_t dp = dev_position(D, d_origin, dev_eval(D, i));
        *reinterpret_cast<T*>(dst + dp * elem_bytes) = *reinterpret_cast<const T*>(src + sp * elem_bytes);
    }
}

// Same fallback when both layouts keep LONGER runs: a thread moves one run of RB = 32 or 64 bytes per evaluation of the
// two layouts, as 256-bit accesses (LDG.E.256 / STG.E.256: every request covers whole 32-byte sectors; 16-byte lanes 64
// bytes apart would ask for every sector twice).
template <int RB>
__global__ void __launch_bounds__(kThreads)
gather_run_kernel(const __grid_constant__ tlb_layout_desc S, const __grid_constant__ tlb_layout_desc D,
                  const char* __restrict__ src, char* __restrict__ dst, int64_t s_origin, int64_t d_origin, uint64_t i0,
                  uint64_t n_runs, int run_elems, int elem_bytes) {
    pdl_wait();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n_runs; k += stride) {
        const uint64_t i = i0 + k * static_cast<uint64_t>(run_elems);
        const char* sp = src + dev_position(S, s_origin, dev_eval(S, i)) * elem_bytes;
        char* dp = dst + dev_position(D, d_origin, dev_eval(D, i)) * elem_bytes;
        uint64_t v[RB / 8];
#pragma unroll
        for (int j = 0; j < RB / 32; ++j)
            asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0, %1, %2, %3}, [%4];"
                         : "=l"(v[4 * j]), "=l"(v[4 * j + 1]), "=l"(v[4 * j + 2]), "=l"(v[4 * j + 3])
                         : "l"(sp + 32 * j));
#pragma unroll
        for (int j = 0; j < RB / 32; ++j)
            asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dp + 32 * j), "l"(v[4 * j]), "l"(v[4 * j + 1]),
                         "l"(v[4 * j + 2]), "l"(v[4 * j + 3])
                         : "memory");
    }
}

// Thread-value partitioned copy (local_partition; partition_demo.cpp:26-40): TV is a rank-2 layout
// (thread, value) -> integral coordinate. GPU thread t is logical thread t; it walks its values in chunks of `vec` cells
// that the host has proven contiguous and aligned in TV, source and destination (vec = 1: cell by cell).
template <int VB>
__global__ void __launch_bounds__(kThreads)
copy_tv_kernel(const __grid_constant__ tlb_layout_desc TV, const __grid_constant__ tlb_layout_desc S,
               const __grid_constant__ tlb_layout_desc D, const char* __restrict__ src, char* __restrict__ dst,
               int64_t s_origin, int64_t d_origin, uint64_t n_threads, uint64_t n_values, uint64_t size, int vec, int elem_bytes) {
    using T = typename Cell<VB>::type;
    pdl_wait();
    const uint64_t n_chunks = n_values / static_cast<uint64_t>(vec);
    const uint64_t total = n_threads * n_chunks, stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    // consecutive GPU threads are consecutive logical threads of one value chunk (the coalescing a raked TV layout is built for)
    for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < total; w += stride) {
        const uint64_t t = w % n_threads, c = w / n_threads;
        const int64_t i = dev_eval_top(TV, 0, t) + dev_eval_top(TV, 1, c * static_cast<uint64_t>(vec));
        if (i < 0 || static_cast<uint64_t>(i) >= size) continue; // a TV layout may over-cover the tensor (predicated tail)
        const int64_t sp = dev_position(S, s_origin, dev_eval(S, static_cast<uint64_t>(i)));
        const int64_t dp = dev_position(D, d_origin, dev_eval(D, static_cast<uint64_t>(i)));
        *reinterpret_cast<T*>(dst + dp * elem_bytes) = *reinterpret_cast<const T*>(src + sp * elem_bytes);
    }
}

// gather over the common refinement: one peel yields both offsets (half the index arithmetic of two evaluations), and,
// the destination being injective, the refined modes may be walked in any order: the host sorts them by destination
// stride so that consecutive threads store to neighbouring cells.
template <int EB>
__global__ void __launch_bounds__(kThreads)
gather_joint_kernel(const __grid_constant__ JointDesc J, const char* __restrict__ src, char* __restrict__ dst, uint64_t n) {
    using T = typename Cell<EB>::type;
    pdl_wait();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        int64_t so, dof;
        dev_joint(J, k, &so, &dof);
        reinterpret_cast<T*>(dst)[dof] = reinterpret_cast<const T*>(src)[so];
    }
}

// ordered pass 1: winner[dp - lo] = max(i + 1) over the i that store to dp
// W: 32-bit winners (k + 1, relative to the call's range) when the range has fewer than 2^32 - 1 elements (half the winner
// traffic), 64-bit otherwise and for the aliased plan's writer table.
template <typename W>
__global__ void __launch_bounds__(kThreads)
winner_kernel(const __grid_constant__ tlb_layout_desc D, int64_t d_origin, int64_t lo, uint64_t i0, uint64_t n,
              W* __restrict__ winner) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t i = i0 + k;
        const int64_t dp = dev_position(D, d_origin, dev_eval(D, i));
        if constexpr (sizeof(W) == 4) atomicMax(winner + (dp - lo), static_cast<unsigned int>(k + 1));
        else atomicMax(winner + (dp - lo), static_cast<unsigned long long>(i + 1));
    }
}

// ordered pass 2: only the last writer of each destination cell stores
template <int EB, typename W>
__global__ void __launch_bounds__(kThreads)
ordered_kernel(const __grid_constant__ tlb_layout_desc S, const __grid_constant__ tlb_layout_desc D,
               const void* __restrict__ src, void* __restrict__ dst, int64_t s_origin, int64_t d_origin, int64_t lo,
               uint64_t i0, uint64_t n, int counting, const W* __restrict__ winner) {
    using T = typename Cell<EB>::type;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t i = i0 + k;
        const int64_t dp = dev_position(D, d_origin, dev_eval(D, i));
        if (static_cast<uint64_t>(winner[dp - lo]) != (sizeof(W) == 4 ? k + 1 : i + 1)) continue;
        const int64_t sp = dev_position(S, s_origin, dev_eval(S, i));
        if constexpr (EB == 8) {
            if (counting) {
                static_cast<uint64_t*>(dst)[dp] = static_cast<uint64_t>(sp);
                continue;
            }
        }
        static_cast<T*>(dst)[dp] = static_cast<const T*>(src)[sp];
    }
}

// ---------------------------------------------------------------------------------------
// aliased: source and destination position spans overlap inside one buffer. The reference copies serially in
// ascending i over shared storage (tensor.hpp:29,195-199), so src(i) may read what an earlier dst(j) wrote:
//   value(i) = value(pred(i))   where pred(i) = the writer j < i of the cell src(i) reads   (else the original cell)
// Injective destinations have at most one writer per cell, so pred is a forest; pointer jumping resolves every i to
// the root whose ORIGINAL cell it ends up copying. Values are snapshotted before anything is stored.
// ---------------------------------------------------------------------------------------
// pass 2 (pass 1 is winner_kernel: writer[dp - lo] = i + 1): root[k] = pred(i0 + k) - i0, or k when there is none.
// `shift` = (src.data - dst.data) / elem_bytes converts a source position into the destination buffer's cell index.
__global__ void __launch_bounds__(kThreads)
alias_pred_kernel(const __grid_constant__ tlb_layout_desc S, int64_t s_origin, int64_t shift, int64_t dlo, int64_t dhi,
                  uint64_t i0, uint64_t n, const unsigned long long* writer, unsigned long long* root) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t i = i0 + k;
        const int64_t p = dev_position(S, s_origin, dev_eval(S, i)) + shift;
        unsigned long long r = k;
        if (p >= dlo && p <= dhi) {
            const unsigned long long w = writer[p - dlo];
            if (w != 0 && w - 1 < i) r = w - 1 - i0;
        }
        root[k] = r;
    }
}
// pass 3, ceil(log2 n) times: root[k] = root[root[k]] (in place: a concurrently updated entry is still an ancestor)
__global__ void __launch_bounds__(kThreads) alias_jump_kernel(uint64_t n, unsigned long long* root) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const unsigned long long r = root[k];
        const unsigned long long rr = root[r];
        if (rr != r) root[k] = rr;
    }
}
// pass 4: vals[k] = original source cell of the root; pass 5: dst(i0 + k) = vals[k]
template <int EB>
__global__ void __launch_bounds__(kThreads)
alias_fetch_kernel(const __grid_constant__ tlb_layout_desc S, const void* src, int64_t s_origin, uint64_t i0, uint64_t n,
                   const unsigned long long* root, void* vals) {
    using T = typename Cell<EB>::type;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride)
        static_cast<T*>(vals)[k] = static_cast<const T*>(src)[dev_position(S, s_origin, dev_eval(S, i0 + root[k]))];
}
template <int EB>
__global__ void __launch_bounds__(kThreads)
alias_store_kernel(const __grid_constant__ tlb_layout_desc D, void* dst, int64_t d_origin, uint64_t i0, uint64_t n,
                   const void* vals) {
    using T = typename Cell<EB>::type;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride)
        static_cast<T*>(dst)[dev_position(D, d_origin, dev_eval(D, i0 + k))] = static_cast<const T*>(vals)[k];
}
// Non-injective destination AND aliasing: the reference's loop itself, one thread, ascending i (small copies only).
template <int EB>
__global__ void serial_kernel(const __grid_constant__ tlb_layout_desc S, const __grid_constant__ tlb_layout_desc D,
                              const void* src, void* dst, int64_t s_origin, int64_t d_origin, uint64_t i0, uint64_t n) {
    using T = typename Cell<EB>::type;
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (uint64_t k = 0; k < n; ++k) {
        const uint64_t i = i0 + k;
        // src and dst are not __restrict__: program order of one thread's loads and stores is kept
        const T v = static_cast<const T*>(src)[dev_position(S, s_origin, dev_eval(S, i))];
        static_cast<T*>(dst)[dev_position(D, d_origin, dev_eval(D, i))] = v;
    }
}

// exact min/max position of an Xor-kind tensor over [i0, i0+n) (used when the OR-bound is too loose)
__global__ void __launch_bounds__(kThreads)
span_kernel(const __grid_constant__ tlb_layout_desc L, int64_t origin, uint64_t i0, uint64_t n,
            long long* __restrict__ lohi) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    long long lo = INT64_MAX, hi = INT64_MIN;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const long long p = dev_position(L, origin, dev_eval(L, i0 + k));
        lo = p < lo ? p : lo;
        hi = p > hi ? p : hi;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(lohi, lo);
        atomicMax(lohi + 1, hi);
    }
}

// ---------------------------------------------------------------------------------------
// vec: one refined mode contiguous on both sides. J's mode 0 is that mode, counted in vectors.
// ---------------------------------------------------------------------------------------
template <int VB>
__global__ void __launch_bounds__(kThreads)
vec_kernel(const __grid_constant__ JointDesc J, const char* __restrict__ src, char* __restrict__ dst, int eb,
           uint64_t n_vec) {
    using T = typename Cell<VB>::type;
    pdl_wait();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if constexpr (VB == 16) {
        // four independent 16-byte loads in flight per thread before the first store (memory-level parallelism)
        constexpr int U = 4;
        for (; v + (U - 1) * stride < n_vec; v += U * stride) {
            int64_t so[U], dof[U];
            uint4 val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) dev_joint(J, v + u * stride, &so[u], &dof[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) val[u] = ldg_stream(src + so[u] * eb);
#pragma unroll
            for (int u = 0; u < U; ++u) stg_stream(dst + dof[u] * eb, val[u]);
        }
    }
    for (; v < n_vec; v += stride) {
        int64_t so, dof;
        dev_joint(J, v, &so, &dof); // offsets in elements
        if constexpr (VB == 16) {
            stg_stream(dst + dof * eb, ldg_stream(src + so * eb));
        } else {
            *reinterpret_cast<T*>(dst + dof * eb) = *reinterpret_cast<const T*>(src + so * eb);
        }
    }
}

// ---------------------------------------------------------------------------------------
// interleave: AoS <-> SoA. A short mode c (2 .. 26, 28, 30 or 32 cells for 2- / 4-byte cells, the common extents otherwise: channels, the parts of a complex number, the short side of a
// tall-skinny transpose) and a long mode j
// where one side keeps (c, j) jointly contiguous (cell j * EC + c: interleaved) and the other keeps j contiguous for each
// c (planar, rows `planar_stride` apart). The staged plan has no whole 128-byte A run that leaves a unit-stride B run here.
// A lane owns NJ = G * 16 / EB consecutive j: on the interleaved side that is one contiguous piece of EC * G * 16 bytes, on
// the planar side EC pieces of G * 16 bytes, and the permutation between them happens in registers. Consecutive lanes own
// consecutive pieces, so every warp-level access covers whole sectors on both sides (256-bit accesses on the interleaved
// side, where a lane's piece is a multiple of 32 bytes: G = 2 for odd EC); no shared memory, no barriers.
// ---------------------------------------------------------------------------------------
struct InterParams {
    JointDesc rest;          // unit index / nJ -> base offsets (elements) of the other modes on both sides
    int64_t nJ;              // units along j
    int64_t planar_stride;   // elements between the rows of consecutive c on the planar side
    uint64_t n_units;
    int32_t wide_i, wide_p;  // 256-bit accesses allowed on the interleaved / planar side (32-byte alignment proven)
};

__device__ __forceinline__ void ld32(const char* p, uint4* lo, uint4* hi) {
    uint64_t a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    lo->x = static_cast<uint32_t>(a); lo->y = static_cast<uint32_t>(a >> 32); lo->z = static_cast<uint32_t>(b); lo->w = static_cast<uint32_t>(b >> 32);
    hi->x = static_cast<uint32_t>(c); hi->y = static_cast<uint32_t>(c >> 32); hi->z = static_cast<uint32_t>(d); hi->w = static_cast<uint32_t>(d >> 32);
}
__device__ __forceinline__ void st32(char* p, const uint4& lo, const uint4& hi) {
    const uint64_t a = lo.x | (static_cast<uint64_t>(lo.y) << 32), b = lo.z | (static_cast<uint64_t>(lo.w) << 32);
    const uint64_t c = hi.x | (static_cast<uint64_t>(hi.y) << 32), d = hi.z | (static_cast<uint64_t>(hi.w) << 32);
    asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

template <int EB, int EC, bool DEINT>
__global__ void __launch_bounds__(kThreads)
interleave_kernel(const __grid_constant__ InterParams P, const char* __restrict__ src, char* __restrict__ dst) {
    using T = typename Cell<EB>::type;
    constexpr int V = 16 / EB, G = (EC % 2) ? 2 : 1, NJ = G * V, NE = EC * NJ, NV = EC * G; // NV 16-byte vectors per unit
    pdl_wait();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < P.n_units; w += stride) {
        const uint64_t t = w / static_cast<uint64_t>(P.nJ), u = w - t * static_cast<uint64_t>(P.nJ);
        int64_t bs, bd;
        dev_joint(P.rest, t, &bs, &bd);
        union { uint4 v[NV]; T e[NE]; } inter;   // cell jj * EC + c
        union { uint4 v[G]; T e[NJ]; } row;      // cells jj of one c
        if constexpr (DEINT) {
            const char* sp = src + (bs + static_cast<int64_t>(u) * NE) * EB;
            if (P.wide_i) {
#pragma unroll
                for (int k = 0; k < NV; k += 2) ld32(sp + 16 * k, &inter.v[k], &inter.v[k + 1]);
            } else {
#pragma unroll
                for (int k = 0; k < NV; ++k) inter.v[k] = ldg_stream(sp + 16 * k);
            }
#pragma unroll
            for (int c = 0; c < EC; ++c) {
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) row.e[jj] = inter.e[jj * EC + c];
                char* dp = dst + (bd + static_cast<int64_t>(u) * NJ + c * P.planar_stride) * EB;
                if (G == 2 && P.wide_p) st32(dp, row.v[0], row.v[G - 1]);
                else {
#pragma unroll
                    for (int g = 0; g < G; ++g) stg_stream(dp + 16 * g, row.v[g]);
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < EC; ++c) {
                const char* sp = src + (bs + static_cast<int64_t>(u) * NJ + c * P.planar_stride) * EB;
                if (G == 2 && P.wide_p) ld32(sp, &row.v[0], &row.v[G - 1]);
                else {
#pragma unroll
                    for (int g = 0; g < G; ++g) row.v[g] = ldg_stream(sp + 16 * g);
                }
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) inter.e[jj * EC + c] = row.e[jj];
            }
            char* dp = dst + (bd + static_cast<int64_t>(u) * NE) * EB;
            if (P.wide_i) {
#pragma unroll
                for (int k = 0; k < NV; k += 2) st32(dp + 16 * k, inter.v[k], inter.v[k + 1]);
            } else {
#pragma unroll
                for (int k = 0; k < NV; ++k) stg_stream(dp + 16 * k, inter.v[k]);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// tiled: swizzled shared-memory staging between a source-contiguous run A and a
// destination-contiguous run B.
// ---------------------------------------------------------------------------------------
constexpr int kMaxPieces = 6;

struct TileParams {
    JointDesc rest;         // tile index -> base offsets (elements) on both sides
    int32_t nA, nB;         // pieces of the two runs
    int64_t eA[kMaxPieces]; // A pieces: extents (product = La) ...
    int64_t dA[kMaxPieces]; // ... and DESTINATION strides (the source stride chain is 1, e0, e0*e1, ...)
    int64_t eB[kMaxPieces]; // B pieces: extents (product = Lb) ...
    int64_t sB[kMaxPieces]; // ... and SOURCE strides
    int32_t La, Lb;         // elements; La * EB = 128 bytes (one swizzle row), Lb rows
    int32_t ua, ub;         // element stride of the A run on the source / of the B run on the destination (1: contiguous;
                            // > 1: "tiled_s", runs along the smallest-stride modes of layouts without a unit stride)
    uint64_t n_tiles;
    int32_t tpc;            // tiles per CTA of the aligned staged kernel (1 .. tiles_per_cta(Lb)); 0 reads as 1
};

// byte offset of 16-byte chunk `c` of row `r` in the staged tile: 128 B rows, chunk index XORed
// with the row index mod 8 == Swizzle<3,4,3> on the byte offset r*128 + c*16.
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) { return (r << 7) | ((c ^ (r & 7u)) << 4); }

// phase 2 of the tiled copy: each lane owns V x V element blocks; conflict-free 128-bit smem reads, register
// transpose, 128-bit stores along B (lanes sharing a chunk cover 32 consecutive b).
// 16 staged bytes -> global: one 128-bit store when the layouts guarantee 16-byte alignment (AL), V cell-sized stores
// otherwise (unaligned bases / leading dimensions: the L2 merges them into full sectors before they reach HBM).
template <int EB, bool AL> __device__ __forceinline__ void store_vec(char* p, const uint4& v, int ub = 1) {
    if constexpr (AL) {
        stg_stream(p, v);
    } else {
        using T = typename Cell<EB>::type;
        union { uint4 v; T e[16 / EB]; } u;
        u.v = v;
#pragma unroll
        for (int k = 0; k < 16 / EB; ++k) reinterpret_cast<T*>(p)[static_cast<int64_t>(k) * ub] = u.e[k];
    }
}

template <int EB, int LB, bool AL = true>
__device__ __forceinline__ void tile_phase2(const unsigned char* tile, const int64_t* s_offA, char* __restrict__ dst,
                                            int64_t base_d, int ub = 1) {
    using T = typename Cell<EB>::type;
    constexpr int V = 16 / EB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr ((EB == 2 && LB % 64 == 0) || (EB == 1 && LB % 128 == 0)) {
        // 1- and 2-byte cells: 8 lanes x V b are one full 128-byte destination line, so the 8 lanes that share a chunk
        // must sit in ONE shared-memory phase. Their rows r0 + j agree mod 8 (an 8-way bank conflict under the
        // swizzle), so lane bb reads its rows rotated, r0 + ((j + bb) mod V), which makes the phase conflict free, and
        // a 3-stage barrel rotation of the V vectors puts them back in row order before the register transpose.
        const int bb = lane & 7, cg = lane >> 3;
        constexpr int NWT2 = (LB / (8 * V)) * 2;       // 8 V rows x 4 chunks per warp-tile
        for (int wt = warp; wt < NWT2; wt += kThreads / 32) {
            const int c = (wt & 1) * 4 + cg;
            const int r0 = (wt >> 1) * (8 * V) + bb * V;
            union { uint4 v; T e[V]; } in[V], out;
#pragma unroll
            for (int j = 0; j < V; ++j) in[j].v = *reinterpret_cast<const uint4*>(tile + swz(r0 + ((j + bb) & (V - 1)), c));
            // in[j] holds row r0 + ((j + bb) mod V); rotate so that in[k] holds row r0 + k: new[k] = old[(k - bb) mod V]
#pragma unroll
            for (int s = 1; s < 8; s <<= 1) {
                if (bb & s) {
                    uint4 t[V];
#pragma unroll
                    for (int k = 0; k < V; ++k) t[k] = in[(k - s) & (V - 1)].v;
#pragma unroll
                    for (int k = 0; k < V; ++k) in[k].v = t[k];
                }
            }
#pragma unroll
            for (int i = 0; i < V; ++i) {
#pragma unroll
                for (int j = 0; j < V; ++j) out.e[j] = in[j].e[i];
                store_vec<EB, AL>(dst + (base_d + s_offA[c * V + i] + static_cast<int64_t>(r0) * ub) * EB, out.v, ub);
            }
        }
        return;
    }
    static_assert(EB != 1 || LB % 128 == 0, "1-byte cells need 128-row tiles");
    if constexpr (EB == 16) {
        // 16-byte cells are their own vectors: nothing to transpose in registers. A warp reads chunk c of 32
        // consecutive rows (conflict free under the swizzle) and writes 512 contiguous destination bytes.
        for (int wt = warp; wt < 8 * (LB / 32); wt += kThreads / 32) {
            const int c = wt & 7, r = (wt >> 3) * 32 + lane;
            const uint4 v = *reinterpret_cast<const uint4*>(tile + swz(r, c));
            store_vec<EB, AL>(dst + (base_d + s_offA[c] + r) * 16, v);
        }
        return;
    }
    constexpr int LOGV = (V == 2) ? 1 : (V == 4) ? 2 : 3;
    constexpr int NR = (EB == 1 || EB == 16) ? 0 : 3 - LOGV;
    constexpr int CW = 8 >> NR;
    const int q = lane & 7, p = lane >> 3;
    const int bb = (q & ((1 << NR) - 1)) | (p << NR);
    const int cl = q >> NR;
    constexpr int GROUPS = 1 << NR;                    // warp-tiles per 128 B of A
    constexpr int NWT = GROUPS * (LB / 32);
    for (int wt = warp; wt < NWT; wt += kThreads / 32) {
        const int c = (wt % GROUPS) * CW + cl;
        const int r0 = (wt / GROUPS) * 32 + bb * V;
        union { uint4 v; T e[V]; } in[V], out;
#pragma unroll
        for (int j = 0; j < V; ++j) in[j].v = *reinterpret_cast<const uint4*>(tile + swz(r0 + j, c));
#pragma unroll
        for (int i = 0; i < V; ++i) {
#pragma unroll
            for (int j = 0; j < V; ++j) out.e[j] = in[j].e[i];
            store_vec<EB, AL>(dst + (base_d + s_offA[c * V + i] + static_cast<int64_t>(r0) * ub) * EB, out.v, ub);
        }
    }
}

// Tiles per CTA of the aligned staged kernel: short tiles (32 / 64 rows: a destination run of 32 .. 127 cells) are only 4 / 8
// KiB, and one tile per CTA leaves the per-CTA work (offset tables, two barriers, the launch of 8 warps) unamortised: a
// 4M x 96 fp32 planar -> interleaved transpose ran 3.65 TB/s. A CTA of such a plan walks 256 / LB consecutive tiles with the
// tables computed once and the loads of tile k + 1 issued before the stores of tile k.
__host__ __device__ constexpr int tiles_per_cta(int lb, bool aligned) { return (aligned && lb <= 64) ? 256 / lb : 1; }

template <int EB, int LB, bool AL = true>
__global__ void __launch_bounds__(kThreads)
tiled_kernel(const __grid_constant__ TileParams P, const char* __restrict__ src, char* __restrict__ dst) {
    constexpr int V = 16 / EB;                         // elements per 16-byte vector
    constexpr int LA = 128 / EB;                       // elements of A per row
    constexpr int TPC = tiles_per_cta(LB, AL);
    __shared__ __align__(1024) unsigned char tile[LB * 128];
    __shared__ int64_t s_offB[LB];                     // source offset of row b
    __shared__ int64_t s_offA[LA];                     // destination offset of column a

    pdl_wait();
    // (the first tile's base offsets before the tables and their barrier, as in the one-tile kernel: computing them after the
    // barrier cost C3 1.5 %)
    const int tpc = TPC == 1 ? 1 : max(1, min(TPC, P.tpc));   // run time: few tiles stay one per CTA (parallelism first)
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * tpc;
    int64_t base_s0, base_d;
    dev_joint(P.rest, t0, &base_s0, &base_d);
    for (int t = threadIdx.x; t < LB + LA; t += kThreads) {
        const bool isB = t < LB;
        uint32_t i = isB ? t : t - LB;
        const int np = isB ? P.nB : P.nA;
        int64_t acc = 0;
        for (int p = 0; p < np; ++p) {
            const uint32_t e = static_cast<uint32_t>(isB ? P.eB[p] : P.eA[p]);
            const uint32_t c = (p + 1 < np) ? i % e : i;
            i /= e;
            acc += static_cast<int64_t>(c) * (isB ? P.sB[p] : P.dA[p]);
        }
        if (isB) s_offB[t] = acc;
        else s_offA[t - LB] = acc;
    }
    __syncthreads();

    // phase 1: 128-bit loads along A (8 lanes = one 128 B line), swizzled 128-bit stores
    constexpr int NVEC = LB * 8;
    constexpr int PER = (NVEC + kThreads - 1) / kThreads;
    uint4 stage[PER];
    auto load_tile = [&](int64_t base_s) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int v = threadIdx.x + u * kThreads;
            if (NVEC % kThreads == 0 || v < NVEC) {
                const int c = v & 7, b = v >> 3;
                if constexpr (AL) {
                    stage[u] = ldg_stream(src + (base_s + s_offB[b] + c * V) * EB);
                } else {
                    using T = typename Cell<EB>::type;
                    const char* gp = src + (base_s + s_offB[b] + static_cast<int64_t>(c * V) * P.ua) * EB;
                    union { uint4 v; T e[V]; } tt;
#pragma unroll
                    for (int k = 0; k < V; ++k) tt.e[k] = reinterpret_cast<const T*>(gp)[static_cast<int64_t>(k) * P.ua];
                    stage[u] = tt.v;
                }
            }
        }
    };
    int64_t next_d = 0;
    load_tile(base_s0);
    if constexpr (TPC == 1) {   // one tile per CTA: straight-line code (C1, C3)
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int v = threadIdx.x + u * kThreads;
            if (NVEC % kThreads == 0 || v < NVEC) {
                const int c = v & 7, b = v >> 3;
                *reinterpret_cast<uint4*>(tile + swz(b, c)) = stage[u];
            }
        }
        __syncthreads();
        tile_phase2<EB, LB, AL>(tile, s_offA, dst, base_d, AL ? 1 : P.ub);
        return;
    }
#pragma unroll 1
    for (int k = 0; k < tpc; ++k) {
        const uint64_t t = t0 + k;
        if (t >= P.n_tiles) break;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int v = threadIdx.x + u * kThreads;
            if (NVEC % kThreads == 0 || v < NVEC) {
                const int c = v & 7, b = v >> 3;
                *reinterpret_cast<uint4*>(tile + swz(b, c)) = stage[u];
            }
        }
        __syncthreads();
        const bool more = k + 1 < tpc && t + 1 < P.n_tiles;
        if (more) {                                    // the next tile's loads are in flight while this tile is written out
            int64_t bs;
            dev_joint(P.rest, t + 1, &bs, &next_d);
            load_tile(bs);
        }
        tile_phase2<EB, LB, AL>(tile, s_offA, dst, base_d, AL ? 1 : P.ub);
        __syncthreads();                               // the staged tile is free again
        base_d = next_d;
    }
}

// tiled, cell-sized accesses ("tiled_u": bases or leading dimensions that are not multiples of 16 bytes, so no 128-bit
// access is aligned). Consecutive lanes take consecutive CELLS: along A when loading (a warp instruction reads one
// contiguous 128-byte piece of a source row), along B when storing (one contiguous piece of a destination run); the tile is
// staged with a padded row pitch (33 words), which makes both the row-wise stores and the column-wise loads of shared
// memory conflict free. The first version gave every lane the V cells of a 16-byte vector (four accesses 16 bytes apart per
// lane: every instruction touched four times the sectors it used): 8001 x 6001 fp32 transpose 2.95 TB/s.
template <int EB, int LB>
__global__ void __launch_bounds__(kThreads)
tiled_cell_kernel(const __grid_constant__ TileParams P, const char* __restrict__ src, char* __restrict__ dst) {
    using T = typename Cell<EB>::type;
    constexpr int LA = 128 / EB;
    constexpr int PITCH = 128 + (EB > 4 ? EB : 4);     // bytes per staged row
#ifndef TLB_CELL_U
#define TLB_CELL_U 32
#endif
    constexpr int N = LB * LA;                         // cells per tile
    constexpr int U = (N / kThreads) < TLB_CELL_U ? (N / kThreads) : TLB_CELL_U;   // loads in flight per thread: narrow cells need many
                                                       // (2-byte cells, 8 in flight: 4 KiB per CTA, latency bound at 3.5 TB/s)
    static_assert(N % (kThreads * U) == 0, "tile size");
    __shared__ __align__(16) unsigned char tile[LB * PITCH];
    __shared__ int64_t s_offB[LB];
    __shared__ int64_t s_offA[LA];
    pdl_wait();
    int64_t base_s, base_d;
    dev_joint(P.rest, blockIdx.x, &base_s, &base_d);
    for (int t = threadIdx.x; t < LB + LA; t += kThreads) {
        const bool isB = t < LB;
        uint32_t i = isB ? t : t - LB;
        const int np = isB ? P.nB : P.nA;
        int64_t acc = 0;
        for (int p = 0; p < np; ++p) {
            const uint32_t e = static_cast<uint32_t>(isB ? P.eB[p] : P.eA[p]);
            const uint32_t c = (p + 1 < np) ? i % e : i;
            i /= e;
            acc += static_cast<int64_t>(c) * (isB ? P.sB[p] : P.dA[p]);
        }
        if (isB) s_offB[t] = acc;
        else s_offA[t - LB] = acc;
    }
    __syncthreads();
    const T* s = reinterpret_cast<const T*>(src) + base_s;
    T* d = reinterpret_cast<T*>(dst) + base_d;
    const int ua = P.ua, ub = P.ub;                    // > 1: "tiled_s", runs along the smallest-stride modes
    constexpr int STEP = U;
    for (int i0 = threadIdx.x; i0 < N; i0 += kThreads * STEP) {
        T v[STEP];
#pragma unroll
        for (int u = 0; u < STEP; ++u) {
            const int i = i0 + u * kThreads, b = i / LA, a = i % LA;
            v[u] = s[s_offB[b] + static_cast<int64_t>(a) * ua];
        }
#pragma unroll
        for (int u = 0; u < STEP; ++u) {
            const int i = i0 + u * kThreads, b = i / LA, a = i % LA;
            *reinterpret_cast<T*>(tile + b * PITCH + a * EB) = v[u];
        }
    }
    __syncthreads();
    for (int i0 = threadIdx.x; i0 < N; i0 += kThreads * STEP) {
#pragma unroll
        for (int u = 0; u < STEP; ++u) {
            const int i = i0 + u * kThreads, a = i / LB, b = i % LB;
            d[s_offA[a] + static_cast<int64_t>(b) * ub] = *reinterpret_cast<const T*>(tile + b * PITCH + a * EB);
        }
    }
}

// tiled, narrow runs ("tiled_n"): one of the two runs is a whole SHORT mode that no 128-byte row / 32-row tile can be assembled
// from: a source-contiguous mode of la < 128 / EB cells (a 4M x 24 transpose, AoS with 9 or 24 fields: what the register-
// permuting interleave plan does not cover), or a destination-contiguous mode of lb < 32 cells (the opposite direction).
// Same cell-granular scheme as tiled_cell_kernel with run-time tile extents: consecutive lanes walk the tile in (b, a)
// order when loading and in (a, b) order when storing (for an interleaved side that is one contiguous stream); the staged
// row pitch is an odd number of words, so the column-wise accesses are conflict free for every extent.
constexpr int kNarrowTileBytes = 256 * 132, kNarrowMaxRun = 256;
template <int EB>
__global__ void __launch_bounds__(kThreads)
tiled_narrow_kernel(const __grid_constant__ TileParams P, const char* __restrict__ src, char* __restrict__ dst) {
    using T = typename Cell<EB>::type;
    __shared__ __align__(16) unsigned char tile[kNarrowTileBytes];
    __shared__ int64_t s_offB[kNarrowMaxRun];
    __shared__ int64_t s_offA[kNarrowMaxRun];
    pdl_wait();
    const int la = P.La, lb = P.Lb;
    const int pitch = ((((la * EB + 3) >> 2) | 1) + (EB == 8 ? 1 : 0)) << 2;   // bytes; 8-byte cells keep 8-byte alignment (even word count)
    int64_t base_s, base_d;
    dev_joint(P.rest, blockIdx.x, &base_s, &base_d);
    for (int t = threadIdx.x; t < lb + la; t += kThreads) {
        const bool isB = t < lb;
        uint32_t i = isB ? t : t - lb;
        const int np = isB ? P.nB : P.nA;
        int64_t acc = 0;
        for (int p = 0; p < np; ++p) {
            const uint32_t e = static_cast<uint32_t>(isB ? P.eB[p] : P.eA[p]);
            const uint32_t c = (p + 1 < np) ? i % e : i;
            i /= e;
            acc += static_cast<int64_t>(c) * (isB ? P.sB[p] : P.dA[p]);
        }
        if (isB) s_offB[t] = acc;
        else s_offA[t - lb] = acc;
    }
    __syncthreads();
    const T* s = reinterpret_cast<const T*>(src) + base_s;
    T* d = reinterpret_cast<T*>(dst) + base_d;
    const int n = lb * la;
#ifndef TLB_NARROW_U
#define TLB_NARROW_U 4
#endif
    constexpr int U = TLB_NARROW_U;   // cells in flight per thread
    {
        // (b, a) of the thread's k-th cell advance by (256 / la, 256 % la) with one carry: no division in the loop
        const int db = kThreads / la, da = kThreads % la;
        int b = threadIdx.x / la, a = threadIdx.x % la;
        int i = threadIdx.x;
        for (; i + (U - 1) * kThreads < n; i += U * kThreads) {
            T v[U];
            int off[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = s[s_offB[b] + a];
                off[u] = b * pitch + a * EB;
                a += da;
                b += db;
                if (a >= la) { a -= la; ++b; }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) *reinterpret_cast<T*>(tile + off[u]) = v[u];
        }
        for (; i < n; i += kThreads) {
            *reinterpret_cast<T*>(tile + b * pitch + a * EB) = s[s_offB[b] + a];
            a += da;
            b += db;
            if (a >= la) { a -= la; ++b; }
        }
    }
    __syncthreads();
    {
        const int da = kThreads / lb, db = kThreads % lb;
        int a = threadIdx.x / lb, b = threadIdx.x % lb;
        int i = threadIdx.x;
        for (; i + (U - 1) * kThreads < n; i += U * kThreads) {
            T v[U];
            int64_t off[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = *reinterpret_cast<const T*>(tile + b * pitch + a * EB);
                off[u] = s_offA[a] + b;
                b += db;
                a += da;
                if (b >= lb) { b -= lb; ++a; }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) d[off[u]] = v[u];
        }
        for (; i < n; i += kThreads) {
            d[s_offA[a] + b] = *reinterpret_cast<const T*>(tile + b * pitch + a * EB);
            b += db;
            a += da;
            if (b >= lb) { b -= lb; ++a; }
        }
    }
}

// ---------------------------------------------------------------------------------------
// tiled, TMA-fed: phase 1 is a cp.async.bulk.tensor load through a tensor map derived from the source layout
// (tlb_tensormap_describe: parent = the source's refined modes, tile = the A and B runs) with the hardware
// 128-byte swizzle, which is the staging layout phase 2 already expects. PERSISTENT: a few CTAs per SM, CTA c walks the
// tiles c, c + grid, c + 2 grid, ... through a ring of staged tiles, so loads run `stages` tiles ahead of the stores and
// the CTAs that run together read NEIGHBOURING tiles (consecutive tile ids are adjacent 128-byte pieces of the same
// source rows: walking consecutive tiles inside one CTA instead touches every DRAM page at eight different times).
// ---------------------------------------------------------------------------------------
constexpr int kTmaMaxStages = 8;

struct TmaTileParams {
    TileParams t;
    int32_t ndim;
    int32_t pad_;
    int64_t dim_stride[5]; // source strides (elements) of the TMA dimensions, innermost first
};

__device__ __forceinline__ void tma_issue_tile(const CUtensorMap* map, uint32_t dst, uint32_t bar, int ndim, const int* c) {
    switch (ndim) {
    case 2:
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]) : "memory");
        break;
    case 3:
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
        break;
    case 4:
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
        break;
    default:
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
        break;
    }
}

template <int EB, int LB>
__global__ void __launch_bounds__(kThreads)
tiled_tma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ TmaTileParams P, char* __restrict__ dst, int stages) {
    constexpr int LA = 128 / EB;
    constexpr uint32_t kTileBytes = LB * 128;
    extern __shared__ unsigned char smem_dyn[];
    __shared__ int64_t s_offA[LA];
    __shared__ int64_t s_base_d[kTmaMaxStages];
    __shared__ __align__(8) unsigned long long s_bar[kTmaMaxStages];
    const uint32_t smem0 = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_dyn)) + 1023u) & ~1023u;
    unsigned char* tiles = smem_dyn + (smem0 - static_cast<uint32_t>(__cvta_generic_to_shared(smem_dyn)));
    const uint64_t first = blockIdx.x, step = gridDim.x;
    const int count = first < P.t.n_tiles ? static_cast<int>((P.t.n_tiles - first + step - 1) / step) : 0;

    auto issue = [&](int i) { // thread 0 only: tile first + i * step -> stage i % stages
        const int stage = i % stages;
        int64_t base_s, base_d;
        dev_joint(P.t.rest, first + static_cast<uint64_t>(i) * step, &base_s, &base_d);
        s_base_d[stage] = base_d;
        int c[5];
        int64_t off = base_s;
        for (int d = P.ndim - 1; d >= 1; --d) {
            const int64_t q = off / P.dim_stride[d];
            c[d] = static_cast<int>(q);
            off -= q * P.dim_stride[d];
        }
        c[0] = static_cast<int>(off);
        const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar[stage]));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kTileBytes) : "memory");
        tma_issue_tile(&map, smem0 + stage * kTileBytes, bar, P.ndim, c);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar[s]))) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int t = threadIdx.x; t < LA; t += kThreads) {
        uint32_t i = t;
        int64_t acc = 0;
        for (int p = 0; p < P.t.nA; ++p) {
            const uint32_t e = static_cast<uint32_t>(P.t.eA[p]);
            const uint32_t c = (p + 1 < P.t.nA) ? i % e : i;
            i /= e;
            acc += static_cast<int64_t>(c) * P.t.dA[p];
        }
        s_offA[t] = acc;
    }
    // everything above overlaps the previous kernel's tail; no global access before this point
    pdl_wait();
    if (threadIdx.x == 0)
        for (int i = 0; i < min(count, stages); ++i) issue(i);
    __syncthreads();

    for (int i = 0; i < count; ++i) {
        const int stage = i % stages;
        const uint32_t parity = (i / stages) & 1;
        const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar[stage]));
        const long long t_start = clock64();
        for (;;) {
            uint32_t ok;
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
            if (ok) break;
            if (clock64() - t_start > 4000000000ll) __trap();
        }
        tile_phase2<EB, LB>(tiles + stage * kTileBytes, s_offA, dst, s_base_d[stage]);
        __syncthreads(); // every lane is done reading this stage
        if (threadIdx.x == 0 && i + stages < count) issue(i + stages);
    }
}

// ---------------------------------------------------------------------------------------
// host planner
// ---------------------------------------------------------------------------------------
struct JM {
    int64_t e, ss, ds;
};

bool mul_ok(int64_t a, int64_t b, int64_t* r) { return !__builtin_mul_overflow(a, b, r); }

// Common refinement of the two flat extent lists (both are mixed-radix splittings of the same
// integral domain). Fails when some pair of radices is not nested (e.g. 6 against 4).
bool refine_modes(const tlb_layout_desc& S, const tlb_layout_desc& D, std::vector<JM>* out) {
    int i = 0, j = 0;
    int64_t rs = S.extent[0], rd = D.extent[0], fs = 1, fd = 1;
    int guard = 0;
    while (i < S.n_modes || j < D.n_modes) {
        if (++guard > 4 * TLB_MAX_MODES) return false;
        const int64_t es = i < S.n_modes ? rs : 1, ed = j < D.n_modes ? rd : 1;
        const int64_t g = std::min(es, ed);
        if (std::max(es, ed) % g != 0) return false;
        JM m{g, 0, 0};
        if (i < S.n_modes && !mul_ok(S.stride[i], fs, &m.ss)) return false;
        if (j < D.n_modes && !mul_ok(D.stride[j], fd, &m.ds)) return false;
        if (g > 1) {
            if (i >= S.n_modes || j >= D.n_modes) return false; // sizes differ (checked earlier)
            out->push_back(m);
        }
        if (i < S.n_modes) {
            rs /= g;
            fs *= g;
            if (rs == 1) {
                ++i;
                fs = 1;
                if (i < S.n_modes) rs = S.extent[i];
            }
        }
        if (j < D.n_modes) {
            rd /= g;
            fd *= g;
            if (rd == 1) {
                ++j;
                fd = 1;
                if (j < D.n_modes) rd = D.extent[j];
            }
        }
    }
    return true;
}

void joint_coalesce(std::vector<JM>* m) {
    std::vector<JM> r;
    for (const JM& x : *m) {
        if (x.e == 1) continue;
        if (!r.empty()) {
            JM& b = r.back();
            int64_t ns, nd;
            if (mul_ok(b.ss, b.e, &ns) && mul_ok(b.ds, b.e, &nd) && ns == x.ss && nd == x.ds) {
                b.e *= x.e;
                continue;
            }
        }
        r.push_back(x);
    }
    *m = r;
}

int launch_grid(uint64_t work_items, int threads, int waves) {
    const uint64_t per_wave = static_cast<uint64_t>(sm_count()) * (2048 / threads);
    uint64_t blocks = (work_items + threads - 1) / threads;
    blocks = std::min<uint64_t>(blocks, per_wave * waves);
    return static_cast<int>(std::max<uint64_t>(blocks, 1));
}

int fill_joint(const std::vector<JM>& m, JointDesc* J) {
    std::memset(J, 0, sizeof(*J));
    if (m.size() > TLB_MAX_MODES) return fail(TLB_ERR_UNSUPPORTED, "too many refined modes");
    J->n = static_cast<int>(m.size());
    for (size_t r = 0; r < m.size(); ++r) joint_set_mode(J, static_cast<int>(r), m[r].e, m[r].ss, m[r].ds);
    if (J->n == 0) {
        J->n = 1;
        joint_set_mode(J, 0, 1, 0, 0);
    }
    return TLB_OK;
}

// Takes a run of total length L (elements) along the stride chain of one side, starting at the
// mode whose stride on that side is 1. Pieces are split off `modes` (partial modes leave their
// outer part behind). `src_side` selects which stride forms the chain.
bool take_run(std::vector<JM>* modes, bool src_side, int64_t L, std::vector<JM>* pieces, int64_t unit = 1) {
    int64_t want = L, next = unit;
    while (want > 1) {
        int hit = -1;
        for (size_t r = 0; r < modes->size(); ++r)
            if ((src_side ? (*modes)[r].ss : (*modes)[r].ds) == next && (*modes)[r].e > 1) {
                hit = static_cast<int>(r);
                break;
            }
        if (hit < 0) return false;
        JM& m = (*modes)[hit];
        if (m.e >= want) {
            if (m.e % want != 0) return false;
            pieces->push_back({want, m.ss, m.ds});
            m.e /= want;
            m.ss *= want;
            m.ds *= want;
            want = 1;
        } else {
            if (want % m.e != 0) return false;
            pieces->push_back(m);
            want /= m.e;
            next *= m.e;
            m.e = 1;
        }
    }
    return true;
}

struct CopyCall {
    const tlb_tensor* src;
    const tlb_tensor* dst;
    uint64_t i0, n;
    cudaStream_t stream;
};

// Largest power-of-two V (elements) such that every aligned block of V consecutive integral coordinates lands in V
// consecutive cells of the tensor: leaf 0 is the identity on the low coordinate bits (Int stride 1 / Xor mask 1, extent a
// multiple of V), no other leaf reaches below V (Int stride a multiple of V, Xor mask without bits below V), and the
// origin and the base pointer are V-aligned.
int low_run(const tlb_tensor& t, int vmax) {
    const tlb_layout_desc& L = *t.layout;
    if (L.kind != TLB_KIND_INT && L.kind != TLB_KIND_XOR) return 1;
    int lead = 0;
    while (lead < L.n_modes && L.extent[lead] == 1) ++lead;
    if (lead == L.n_modes || L.stride[lead] != 1) return 1;
    int v = vmax;
    while (v > 1) {
        bool ok = L.extent[lead] % v == 0 && t.origin % v == 0 &&
                  reinterpret_cast<uintptr_t>(t.data) % (static_cast<uintptr_t>(v) * t.elem_bytes) == 0;
        for (int r = lead + 1; ok && r < L.n_modes; ++r) {
            if (L.extent[r] == 1) continue;
            ok = L.kind == TLB_KIND_INT ? (L.stride[r] % v == 0) : ((L.stride[r] & (v - 1)) == 0);
        }
        if (ok) break;
        v >>= 1;
    }
    return v;
}

int launch_gather(const CopyCall& c) {
    const tlb_layout_desc& S = *c.src->layout;
    const tlb_layout_desc& D = *c.dst->layout;
    const int counting = c.src->accessor == TLB_ACC_COUNTING;
    const int eb = c.dst->elem_bytes;
    int V = 1;
    if (!counting && eb < 16 && c.src->data) {
        V = std::min(low_run(*c.src, 16 / eb), low_run(*c.dst, 16 / eb));
        while (V > 1 && (c.i0 % V != 0 || c.n % V != 0)) V >>= 1;
    }
    // runs of 32 or 64 bytes that both layouts keep contiguous and aligned: one evaluation per run, 256-bit accesses
    int R = 1;
    if (V * eb == 16 && knob(K_COPY_GATHER_RUN) != 0) {
        R = std::min(low_run(*c.src, 64 / eb), low_run(*c.dst, 64 / eb));
        while (R * eb > 16 && (c.i0 % R != 0 || c.n % R != 0)) R >>= 1;
        if (R * eb < 32) R = 1;
    }
    if (g_dry_run) {
        set_plan(R > 1 ? "gather_run" : V > 1 ? "gather_vec" : "gather");
        return TLB_OK;
    }
    if (R > 1) {
        const uint64_t n_runs = c.n / R;
        const int gridr = launch_grid(n_runs, kThreads, 8);
        const char* sb = static_cast<const char*>(c.src->data);
        char* db = static_cast<char*>(c.dst->data);
        if (R * eb == 64)
            TLB_CUDA(launch_pdl(gather_run_kernel<64>, dim3(gridr), dim3(kThreads), 0, c.stream, S, D, sb, db, c.src->origin, c.dst->origin, c.i0, n_runs, R, eb));
        else
            TLB_CUDA(launch_pdl(gather_run_kernel<32>, dim3(gridr), dim3(kThreads), 0, c.stream, S, D, sb, db, c.src->origin, c.dst->origin, c.i0, n_runs, R, eb));
        count_launch();
        set_plan("gather_run");
        return TLB_OK;
    }
    if (V > 1) {
        const uint64_t n_vec = c.n / V;
        const int gridv = launch_grid(n_vec, kThreads, 8);
        const char* sb = static_cast<const char*>(c.src->data);
        char* db = static_cast<char*>(c.dst->data);
#define TLB_GV(VB) TLB_CUDA(launch_pdl(gather_vec_kernel<VB>, dim3(gridv), dim3(kThreads), 0, c.stream, S, D, sb, db, c.src->origin, c.dst->origin, c.i0, n_vec, V, eb))
        switch (V * eb) {
        case 2: TLB_GV(2); break;
        case 4: TLB_GV(4); break;
        case 8: TLB_GV(8); break;
        default: TLB_GV(16); break;
        }
#undef TLB_GV
        count_launch();
        set_plan("gather_vec");
        return TLB_OK;
    }
    const int grid = launch_grid(c.n, kThreads, 8);
#define TLB_GATHER(EB)                                                                                        \
    gather_kernel<EB><<<grid, kThreads, 0, c.stream>>>(S, D, c.src->data, c.dst->data, c.src->origin, c.dst->origin, \
                                                       c.i0, c.n, counting)
    switch (eb) {
    case 1: TLB_GATHER(1); break;
    case 2: TLB_GATHER(2); break;
    case 4: TLB_GATHER(4); break;
    case 8: TLB_GATHER(8); break;
    default: TLB_GATHER(16); break;
    }
#undef TLB_GATHER
    count_launch();
    TLB_CUDA(cudaGetLastError());
    set_plan("gather");
    return TLB_OK;
}

// The refined modes of a call restricted to its index range, for the joint gather fallback.
struct Refined {
    bool ok = false;
    std::vector<JM> modes;
    int64_t base_s = 0, base_d = 0;
};

int launch_gather_joint(const CopyCall& c, const Refined& R) {
    std::vector<JM> order = R.modes;
    std::stable_sort(order.begin(), order.end(), [](const JM& a, const JM& b) { return std::llabs(a.ds) < std::llabs(b.ds); });
    JointDesc J;
    TLB_TRY(fill_joint(order, &J));
    if (g_dry_run) {
        set_plan("gather");
        return TLB_OK;
    }
    const int eb = c.dst->elem_bytes;
    const char* sb = static_cast<const char*>(c.src->data) + R.base_s * eb;
    char* db = static_cast<char*>(c.dst->data) + R.base_d * eb;
    const int grid = launch_grid(c.n, kThreads, 8);
#define TLB_GJ(EB) TLB_CUDA(launch_pdl(gather_joint_kernel<EB>, dim3(grid), dim3(kThreads), 0, c.stream, J, sb, db, c.n))
    switch (eb) {
    case 1: TLB_GJ(1); break;
    case 2: TLB_GJ(2); break;
    case 4: TLB_GJ(4); break;
    case 8: TLB_GJ(8); break;
    default: TLB_GJ(16); break;
    }
#undef TLB_GJ
    count_launch();
    set_plan("gather");
    return TLB_OK;
}

int launch_ordered(const CopyCall& c, Span dspan) {
    const tlb_layout_desc& S = *c.src->layout;
    const tlb_layout_desc& D = *c.dst->layout;
    const int counting = c.src->accessor == TLB_ACC_COUNTING;
    const uint64_t cells = static_cast<uint64_t>(dspan.hi - dspan.lo) + 1;
    if (g_dry_run) {
        set_plan("ordered");
        return TLB_OK;
    }
    const bool w32 = c.n < 0xffffffffull;
    const size_t wbytes = w32 ? 4 : 8;
    void* winner = nullptr;
    TLB_CUDA(ws_malloc(&winner, cells * wbytes, c.stream));
    TLB_CUDA(cudaMemsetAsync(winner, 0, cells * wbytes, c.stream));
    const int grid = launch_grid(c.n, kThreads, 8);
    if (w32) winner_kernel<unsigned int><<<grid, kThreads, 0, c.stream>>>(D, c.dst->origin, dspan.lo, c.i0, c.n, static_cast<unsigned int*>(winner));
    else winner_kernel<unsigned long long><<<grid, kThreads, 0, c.stream>>>(D, c.dst->origin, dspan.lo, c.i0, c.n, static_cast<unsigned long long*>(winner));
#define TLB_ORDERED(EB)                                                                                         \
    do {                                                                                                        \
        if (w32) ordered_kernel<EB, unsigned int><<<grid, kThreads, 0, c.stream>>>(S, D, c.src->data, c.dst->data, c.src->origin, c.dst->origin, \
                                                        dspan.lo, c.i0, c.n, counting, static_cast<const unsigned int*>(winner)); \
        else ordered_kernel<EB, unsigned long long><<<grid, kThreads, 0, c.stream>>>(S, D, c.src->data, c.dst->data, c.src->origin, c.dst->origin, \
                                                        dspan.lo, c.i0, c.n, counting, static_cast<const unsigned long long*>(winner)); \
    } while (0)
    switch (c.dst->elem_bytes) {
    case 1: TLB_ORDERED(1); break;
    case 2: TLB_ORDERED(2); break;
    case 4: TLB_ORDERED(4); break;
    case 8: TLB_ORDERED(8); break;
    default: TLB_ORDERED(16); break;
    }
#undef TLB_ORDERED
    count_launch(2);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(winner, c.stream);
    TLB_CUDA(e);
    set_plan("ordered");
    return TLB_OK;
}

// Source and destination spans overlap in memory (see the alias kernels above).
int launch_aliased(const CopyCall& c, Span dspan, bool injective) {
    const tlb_layout_desc& S = *c.src->layout;
    const tlb_layout_desc& D = *c.dst->layout;
    const int eb = c.dst->elem_bytes;
    const intptr_t delta = reinterpret_cast<intptr_t>(c.src->data) - reinterpret_cast<intptr_t>(c.dst->data);
    if (delta % eb != 0)
        return fail(TLB_ERR_UNSUPPORTED, "tlb_copy: source and destination overlap at a sub-cell offset");
    if (!injective) {
        if (c.n > (1ull << 20))
            return fail(TLB_ERR_UNSUPPORTED, "tlb_copy: overlapping source and non-injective destination above 2^20 elements");
        if (g_dry_run) {
            set_plan("serial");
            return TLB_OK;
        }
#define TLB_SERIAL(EB) serial_kernel<EB><<<1, 32, 0, c.stream>>>(S, D, c.src->data, c.dst->data, c.src->origin, c.dst->origin, c.i0, c.n)
        switch (eb) {
        case 1: TLB_SERIAL(1); break;
        case 2: TLB_SERIAL(2); break;
        case 4: TLB_SERIAL(4); break;
        case 8: TLB_SERIAL(8); break;
        default: TLB_SERIAL(16); break;
        }
#undef TLB_SERIAL
        count_launch();
        TLB_CUDA(cudaGetLastError());
        set_plan("serial");
        return TLB_OK;
    }
    if (g_dry_run) {
        set_plan("aliased");
        return TLB_OK;
    }
    const uint64_t cells = static_cast<uint64_t>(dspan.hi - dspan.lo) + 1;
    unsigned long long *writer = nullptr, *root = nullptr;
    void* vals = nullptr;
    TLB_CUDA(ws_malloc(reinterpret_cast<void**>(&writer), cells * 8, c.stream));
    cudaError_t e = ws_malloc(reinterpret_cast<void**>(&root), c.n * 8, c.stream);
    if (e == cudaSuccess) e = ws_malloc(&vals, c.n * static_cast<uint64_t>(eb), c.stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(writer, 0, cells * 8, c.stream);
    int launches = 0;
    if (e == cudaSuccess) {
        const int grid = launch_grid(c.n, kThreads, 8);
        winner_kernel<unsigned long long><<<grid, kThreads, 0, c.stream>>>(D, c.dst->origin, dspan.lo, c.i0, c.n, writer);
        alias_pred_kernel<<<grid, kThreads, 0, c.stream>>>(S, c.src->origin, static_cast<int64_t>(delta / eb), dspan.lo, dspan.hi,
                                                           c.i0, c.n, writer, root);
        launches = 2;
        for (uint64_t span = 1; span < c.n; span <<= 1, ++launches) alias_jump_kernel<<<grid, kThreads, 0, c.stream>>>(c.n, root);
#define TLB_ALIAS(EB)                                                                                                   \
    do {                                                                                                                \
        alias_fetch_kernel<EB><<<grid, kThreads, 0, c.stream>>>(S, c.src->data, c.src->origin, c.i0, c.n, root, vals);  \
        alias_store_kernel<EB><<<grid, kThreads, 0, c.stream>>>(D, c.dst->data, c.dst->origin, c.i0, c.n, vals);        \
    } while (0)
        switch (eb) {
        case 1: TLB_ALIAS(1); break;
        case 2: TLB_ALIAS(2); break;
        case 4: TLB_ALIAS(4); break;
        case 8: TLB_ALIAS(8); break;
        default: TLB_ALIAS(16); break;
        }
#undef TLB_ALIAS
        launches += 2;
        e = cudaGetLastError();
    }
    count_launch(launches);
    if (writer) cudaFreeAsync(writer, c.stream);
    if (root) cudaFreeAsync(root, c.stream);
    if (vals) cudaFreeAsync(vals, c.stream);
    TLB_CUDA(e);
    set_plan("aliased");
    return TLB_OK;
}

bool aligned_to(const void* p, int64_t origin, int eb, int bytes) {
    return ((reinterpret_cast<uintptr_t>(p) + static_cast<uintptr_t>(origin) * eb) % bytes) == 0;
}

// Tries the vec and tiled plans. Returns TLB_OK with *done = true when a kernel was launched.
int try_planned(const CopyCall& c, bool* done, Refined* refined) {
    *done = false;
    const tlb_tensor& s = *c.src;
    const tlb_tensor& d = *c.dst;
    const tlb_layout_desc& S = *s.layout;
    const tlb_layout_desc& D = *d.layout;
    const int eb = d.elem_bytes;
    if (S.kind != TLB_KIND_INT || D.kind != TLB_KIND_INT || s.accessor != TLB_ACC_BUFFER) return TLB_OK;
    std::vector<JM> modes;
    if (!refine_modes(S, D, &modes)) return TLB_OK;
    joint_coalesce(&modes);
    if (modes.empty()) return TLB_OK; // single element: gather
    // Restrict to [i0, i0+n): the range must select whole slices of the outermost refined mode.
    int64_t base_s = s.origin, base_d = d.origin;
    if (c.n != static_cast<uint64_t>(S.size)) {
        JM& last = modes.back();
        const uint64_t prefix = static_cast<uint64_t>(S.size / last.e);
        if (c.i0 % prefix != 0 || c.n % prefix != 0) return TLB_OK;
        const int64_t c0 = static_cast<int64_t>(c.i0 / prefix);
        base_s += c0 * last.ss;
        base_d += c0 * last.ds;
        last.e = static_cast<int64_t>(c.n / prefix);
        if (last.e == 1) modes.pop_back();
        if (modes.empty()) return TLB_OK;
    }
    refined->ok = true;
    refined->modes = modes;
    refined->base_s = base_s;
    refined->base_d = base_d;
    int ia = -1, ib = -1;
    for (size_t r = 0; r < modes.size(); ++r) {
        if (modes[r].ss == 1 && ia < 0) ia = static_cast<int>(r);
        if (modes[r].ds == 1 && ib < 0) ib = static_cast<int>(r);
    }
    // Layouts without a unit stride on one side (BLIS-style general strides, every second element, ...) still take the
    // staged plan: the run then follows the mode with the SMALLEST positive stride on that side ("tiled_s", cell-sized
    // strided accesses: a 3-element stride reads a third of every sector instead of one cell per sector).
    int64_t ua = 1, ub = 1;
    if (ia < 0 || ib < 0) {
        if (g_copy_path == 3) return TLB_OK;
        auto smallest = [&](bool src_side, int* idx) {
            int64_t best = 0;
            for (size_t r = 0; r < modes.size(); ++r) {
                const int64_t st = src_side ? modes[r].ss : modes[r].ds;
                if (modes[r].e > 1 && st > 0 && (best == 0 || st < best)) {
                    best = st;
                    *idx = static_cast<int>(r);
                }
            }
            return best;
        };
        if (ia < 0) ua = smallest(true, &ia);
        if (ib < 0) ub = smallest(false, &ib);
        if (ia < 0 || ib < 0 || ua > 64 || ub > 64) return TLB_OK; // far-apart cells gain nothing from staging
    }
    const bool strided_runs = ua != 1 || ub != 1;
    const char* sp = static_cast<const char*>(s.data);
    char* dp = static_cast<char*>(d.data);

    if (ia == ib && !strided_runs && g_copy_path != 2 && g_copy_path != 3) {
        // ---- vec plan: widest power-of-two vector that divides the run and every other stride
        int vb = 16;
        auto fits = [&](int bytes) {
            if (bytes < eb) return false;
            const int64_t v = bytes / eb;
            if (modes[ia].e % v != 0) return false;
            for (size_t r = 0; r < modes.size(); ++r)
                if (static_cast<int>(r) != ia && (modes[r].ss % v != 0 || modes[r].ds % v != 0)) return false;
            return aligned_to(sp, base_s, eb, bytes) && aligned_to(dp, base_d, eb, bytes);
        };
        while (vb > eb && !fits(vb)) vb >>= 1;
        if (eb == 16) vb = fits(16) ? 16 : 0;
        // A run whose extent alone keeps the vectors narrow (an odd number of cells): large copies are cut into whole
        // 16-byte vectors plus the last cells of the run (try_ragged) instead of moving everything cell by cell.
        if (vb < 16 && eb < 16 && g_copy_path == 0 && g_ragged_depth == 0 && knob(K_COPY_RAGGED) != 0 &&
            c.n >= (1ull << std::min(40, knob(K_COPY_RAGGED))) && modes[ia].e >= 16 / eb) {
            // (bases off a 16-byte boundary by the SAME amount on both sides are cut as well: head cells, vectors, tail cells)
            bool wide = ((reinterpret_cast<uintptr_t>(sp) + static_cast<uintptr_t>(base_s) * eb) & 15u) ==
                        ((reinterpret_cast<uintptr_t>(dp) + static_cast<uintptr_t>(base_d) * eb) & 15u);
            for (size_t r = 0; wide && r < modes.size(); ++r)
                if (static_cast<int>(r) != ia) wide = modes[r].ss % (16 / eb) == 0 && modes[r].ds % (16 / eb) == 0;
            if (wide) return TLB_OK;
        }
        if (vb < eb || vb == 1 || !fits(vb)) return TLB_OK;
        const int64_t v = vb / eb;
        std::vector<JM> order;
        order.push_back({modes[ia].e / v, v, v});
        std::vector<JM> rest;
        for (size_t r = 0; r < modes.size(); ++r)
            if (static_cast<int>(r) != ia) rest.push_back(modes[r]);
        std::stable_sort(rest.begin(), rest.end(), [](const JM& a, const JM& b) {
            return std::min(std::llabs(a.ss), std::llabs(a.ds)) < std::min(std::llabs(b.ss), std::llabs(b.ds));
        });
        order.insert(order.end(), rest.begin(), rest.end());
        JointDesc J;
        TLB_TRY(fill_joint(order, &J));
        const uint64_t n_vec = c.n / static_cast<uint64_t>(v);
        if (g_dry_run) {
            set_plan("vec");
            *done = true;
            return TLB_OK;
        }
        const int grid = launch_grid(n_vec, kThreads, 8);
        const char* sb = sp + base_s * eb;
        char* db = dp + base_d * eb;
        switch (vb) {
        case 2: TLB_CUDA(launch_pdl(vec_kernel<2>, dim3(grid), dim3(kThreads), 0, c.stream, J, sb, db, eb, n_vec)); break;
        case 4: TLB_CUDA(launch_pdl(vec_kernel<4>, dim3(grid), dim3(kThreads), 0, c.stream, J, sb, db, eb, n_vec)); break;
        case 8: TLB_CUDA(launch_pdl(vec_kernel<8>, dim3(grid), dim3(kThreads), 0, c.stream, J, sb, db, eb, n_vec)); break;
        default: TLB_CUDA(launch_pdl(vec_kernel<16>, dim3(grid), dim3(kThreads), 0, c.stream, J, sb, db, eb, n_vec)); break;
        }
        count_launch();
        TLB_CUDA(cudaGetLastError());
        set_plan("vec");
        *done = true;
        return TLB_OK;
    }
    if (ia == ib) return TLB_OK;

    // ---- interleave plan (AoS <-> SoA): a short mode c and a long mode j, (c, j) jointly contiguous on one side, j
    // contiguous on the other
    if (!strided_runs && g_copy_path == 0 && knob(K_COPY_INTERLEAVE) != 0 && (eb == 1 || eb == 2 || eb == 4 || eb == 8)) {
        auto short_mode = [eb](int64_t e) { return interleave_size(e, eb); };
        const bool deint = modes[ib].ss == modes[ia].e && short_mode(modes[ia].e);   // source interleaved: c = ia (ss 1), j = ib (ds 1, ss = |c|)
        const bool inter = !deint && modes[ia].ds == modes[ib].e && short_mode(modes[ib].e); // destination interleaved: c = ib (ds 1), j = ia (ss 1, ds = |c|)
        if (deint || inter) {
            const int ic = deint ? ia : ib, ij = deint ? ib : ia;
            const int64_t EC = modes[ic].e, V = 16 / eb, G = (EC % 2) ? 2 : 1, NJ = G * V;
            const int64_t pstride = deint ? modes[ic].ds : modes[ic].ss;
            bool ok = short_mode(EC) && modes[ij].e % NJ == 0 && pstride % V == 0 && pstride > 0 &&
                      aligned_to(sp, base_s, eb, 16) && aligned_to(dp, base_d, eb, 16);
            bool wide = aligned_to(sp, base_s, eb, 32) && aligned_to(dp, base_d, eb, 32);
            bool wide_p = wide && pstride % (2 * V) == 0;
            std::vector<JM> rest;
            for (size_t r = 0; ok && r < modes.size(); ++r) {
                if (static_cast<int>(r) == ic || static_cast<int>(r) == ij || modes[r].e == 1) continue;
                ok = modes[r].ss % V == 0 && modes[r].ds % V == 0;
                wide = wide && modes[r].ss % (2 * V) == 0 && modes[r].ds % (2 * V) == 0;
                rest.push_back(modes[r]);
            }
            if (ok) {
                std::stable_sort(rest.begin(), rest.end(), [](const JM& a, const JM& b) {
                    return std::min(std::llabs(a.ss), std::llabs(a.ds)) < std::min(std::llabs(b.ss), std::llabs(b.ds));
                });
                InterParams P;
                std::memset(&P, 0, sizeof(P));
                TLB_TRY(fill_joint(rest, &P.rest));
                P.nJ = modes[ij].e / NJ;
                P.planar_stride = pstride;
                uint64_t units = static_cast<uint64_t>(P.nJ);
                for (const JM& m : rest) units *= static_cast<uint64_t>(m.e);
                P.n_units = units;
                P.wide_i = wide ? 1 : 0;
                P.wide_p = wide && wide_p ? 1 : 0;
                if (g_dry_run) {
                    set_plan("interleave");
                    *done = true;
                    return TLB_OK;
                }
                const int grid = launch_grid(units, kThreads, 8);
                const char* sb = sp + base_s * eb;
                char* db = dp + base_d * eb;
#define TLB_IL2(EB, EC_) do { if (deint) TLB_CUDA(launch_pdl(interleave_kernel<EB, EC_, true>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db)); \
                              else TLB_CUDA(launch_pdl(interleave_kernel<EB, EC_, false>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db)); } while (0)
#define TLB_IL(EB) do { switch (EC) { case 2: TLB_IL2(EB, 2); break; case 3: TLB_IL2(EB, 3); break; case 4: TLB_IL2(EB, 4); break; case 5: TLB_IL2(EB, 5); break; \
                                      case 6: TLB_IL2(EB, 6); break; case 7: TLB_IL2(EB, 7); break; case 8: TLB_IL2(EB, 8); break; case 9: TLB_IL2(EB, 9); break; \
                                      case 10: TLB_IL2(EB, 10); break; case 12: TLB_IL2(EB, 12); break; case 16: TLB_IL2(EB, 16); break; \
                                      case 24: TLB_IL2(EB, 24); break; default: TLB_IL2(EB, 32); break; } } while (0)
#define TLB_ILX(EB) do { switch (EC) { case 11: TLB_IL2(EB, 11); break; case 13: TLB_IL2(EB, 13); break; case 14: TLB_IL2(EB, 14); break; case 15: TLB_IL2(EB, 15); break; \
                                       case 17: TLB_IL2(EB, 17); break; case 18: TLB_IL2(EB, 18); break; case 19: TLB_IL2(EB, 19); break; case 20: TLB_IL2(EB, 20); break; \
                                       case 21: TLB_IL2(EB, 21); break; case 22: TLB_IL2(EB, 22); break; case 23: TLB_IL2(EB, 23); break; case 25: TLB_IL2(EB, 25); break; \
                                       case 26: TLB_IL2(EB, 26); break; case 28: TLB_IL2(EB, 28); break; \
                                       case 30: TLB_IL2(EB, 30); break; default: TLB_IL(EB); break; } } while (0)
                if (eb == 1) TLB_IL(1); else if (eb == 2) TLB_ILX(2); else if (eb == 4) TLB_ILX(4); else TLB_IL(8);
#undef TLB_ILX
#undef TLB_IL
#undef TLB_IL2
                count_launch();
                set_plan("interleave");
                *done = true;
                return TLB_OK;
            }
        }
    }

    // ---- tiled plan
    if (eb != 1 && eb != 2 && eb != 4 && eb != 8 && eb != 16) return TLB_OK;
    const int64_t V = 16 / eb, La = 128 / eb;
    // Negative strides (reversed modes) are fine everywhere except along the two contiguous runs themselves, which
    // take_run only builds from +1 stride chains; the offset tables and the tile index carry signed strides.
    // Bases or strides that are not multiples of 16 bytes (padded leading dimensions, odd origins) keep the tiled
    // plan with cell-sized global accesses ("tiled_u": 128- and 32-row tiles, 2-, 4- and 8-byte cells).
    const bool base_al = aligned_to(sp, base_s, eb, 16) && aligned_to(dp, base_d, eb, 16);
    // Rows per tile = cells of the destination-contiguous run per tile. Powers of two, and since round 2 the other multiples
    // of 32 up to 256 for 2-, 4- and 8-byte cells: a run of 96 / 160 / 192 / 224 cells is ONE tile (384 .. 896-byte destination
    // segments) instead of 32-row tiles with 128-byte segments.
    static const int64_t kLb[] = {256, 224, 192, 160, 128, 96, 64, 32};
    for (int64_t Lb : kLb) {
        if (Lb == 256 && !lb256_enabled()) continue;
        const bool odd_lb = Lb == 224 || Lb == 192 || Lb == 160 || Lb == 96;
        if (odd_lb && ((eb != 2 && eb != 4 && eb != 8) || g_copy_path == 3 || (g_copy_path == 0 && tma_default()) || knob(K_COPY_ODD_TILES) == 0)) continue;
        if (eb == 1 && (Lb < 128 || g_copy_path == 3 || (g_copy_path == 0 && tma_default()))) continue; // 1-byte cells: LDG-staged, 128+ rows
        if (eb == 16 && (Lb == 64 || g_copy_path == 3 || (g_copy_path == 0 && tma_default()))) continue; // 16-byte cells: LDG-staged, 256 / 128 / 32 rows
        std::vector<JM> work = modes, A, B;
        if (!take_run(&work, true, La, &A, ua)) break; // the A run does not depend on Lb
        if (!take_run(&work, false, Lb, &B, ub)) continue;
        if (A.size() > kMaxPieces || B.size() > kMaxPieces) continue;
        bool ok = base_al && !strided_runs;
        for (const JM& m : A) ok = ok && (m.ds % V == 0);
        for (const JM& m : B) ok = ok && (m.ss % V == 0);
        std::vector<JM> rest;
        for (const JM& m : work)
            if (m.e > 1) {
                ok = ok && (m.ss % V == 0) && (m.ds % V == 0);
                rest.push_back(m);
            }
        const bool unaligned = !ok;
        const bool cell_tiles = knob(K_COPY_CELL_TILES) != 0;   // 1-byte cells only have the cell-granular kernel, 128-row tiles
        if (unaligned && ((eb != 2 && eb != 4 && eb != 8 && !(eb == 1 && cell_tiles && Lb == 128)) || (Lb != 128 && Lb != 32) || g_copy_path == 3)) continue;
        // B must be contiguous on the destination (row b -> +b) and A on the source: by construction.
        TileParams P;
        std::memset(&P, 0, sizeof(P));
        // neighbouring CTAs should touch neighbouring memory: order the rest modes by locality
        std::stable_sort(rest.begin(), rest.end(), [](const JM& a, const JM& b) {
            return std::min(std::llabs(a.ss), std::llabs(a.ds)) < std::min(std::llabs(b.ss), std::llabs(b.ds));
        });
        TLB_TRY(fill_joint(rest, &P.rest));
        P.nA = static_cast<int>(A.size());
        P.nB = static_cast<int>(B.size());
        for (size_t r = 0; r < A.size(); ++r) { P.eA[r] = A[r].e; P.dA[r] = A[r].ds; }
        for (size_t r = 0; r < B.size(); ++r) { P.eB[r] = B[r].e; P.sB[r] = B[r].ss; }
        P.La = static_cast<int>(La);
        P.Lb = static_cast<int>(Lb);
        P.ua = static_cast<int32_t>(ua);
        P.ub = static_cast<int32_t>(ub);
        uint64_t tiles = 1;
        for (const JM& m : rest) tiles *= static_cast<uint64_t>(m.e);
        P.n_tiles = tiles;
        if (tiles > 0x7fffffffull) return TLB_OK;
        const char* sb = sp + base_s * eb;
        char* db = dp + base_d * eb;
        // ---- TMA-fed variant: tensor map derived from the source's refined modes (parent) and the A / B runs (tile)
        if (!unaligned && (g_copy_path == 3 || (g_copy_path == 0 && tma_default()))) {
            bool tma_ok = true;
            for (const JM& m : modes) tma_ok = tma_ok && m.ss >= 0; // tensor maps carry unsigned strides
            for (size_t r = 0; r + 1 < B.size(); ++r) tma_ok = tma_ok && B[r].ss < B[r + 1].ss; // smem row order == b order
            tlb_layout_desc parent, tdesc;
            std::memset(&parent, 0, sizeof(parent));
            std::memset(&tdesc, 0, sizeof(tdesc));
            parent.kind = tdesc.kind = TLB_KIND_INT;
            tma_ok = tma_ok && modes.size() <= TLB_MAX_MODES && A.size() + B.size() <= TLB_MAX_MODES;
            if (tma_ok) {
                parent.n_modes = static_cast<int>(modes.size());
                for (size_t r = 0; r < modes.size(); ++r) { parent.extent[r] = modes[r].e; parent.stride[r] = modes[r].ss; }
                int nt = 0;
                for (const JM& m : A) { tdesc.extent[nt] = m.e; tdesc.stride[nt++] = m.ss; }
                for (const JM& m : B) { tdesc.extent[nt] = m.e; tdesc.stride[nt++] = m.ss; }
                tdesc.n_modes = nt;
                int32_t rank = 0;
                uint64_t dims[5], strides[5];
                uint32_t box[5];
                uint64_t rows = 1;
                tma_ok = tlb_tensormap_describe(&parent, &tdesc, &rank, dims, strides, box) == TLB_OK && rank >= 2 &&
                         box[0] == static_cast<uint32_t>(La);
                for (int d2 = 1; tma_ok && d2 < rank; ++d2) rows *= box[d2];
                tma_ok = tma_ok && rows == static_cast<uint64_t>(Lb);
                for (int d2 = 0; tma_ok && d2 < rank; ++d2) tma_ok = dims[d2] < (1ull << 32);
                for (int d2 = 1; tma_ok && d2 < rank; ++d2) tma_ok = (strides[d2] * static_cast<uint64_t>(eb)) % 16 == 0;
                if (tma_ok && g_dry_run) {
                    set_plan("tiled_tma");
                    *done = true;
                    return TLB_OK;
                }
                alignas(64) unsigned char mapbytes[128];
                if (tma_ok)
                    tma_ok = tlb_tensormap_from_divided(&parent, &tdesc, eb, TMA_SW_128, const_cast<char*>(sb), mapbytes) == TLB_OK;
                if (tma_ok) {
                    TmaTileParams TP;
                    std::memset(&TP, 0, sizeof(TP));
                    TP.t = P;
                    TP.ndim = rank;
                    for (int d2 = 0; d2 < 5; ++d2) TP.dim_stride[d2] = d2 < rank ? static_cast<int64_t>(strides[d2]) : 1;
                    CUtensorMap map;
                    std::memcpy(&map, mapbytes, 128);
                    // persistent grid: ctas CTAs per SM (as many as the ring's shared memory lets co-reside), tiles dealt round-robin
                    int stages = std::max(2, std::min(kTmaMaxStages, knob(K_COPY_TMA_STAGES)));
                    while (stages > 2 && static_cast<size_t>(stages) * Lb * 128 + 2048 > 227u * 1024u) --stages;
                    const size_t smem = static_cast<size_t>(stages) * Lb * 128 + 1024;
                    const int fit = std::max(1, static_cast<int>((227u * 1024u) / (smem + 1024)));
                    const int ctas = std::max(1, std::min(fit, knob(K_COPY_TMA_CTAS)));
                    const unsigned grid_tma = static_cast<unsigned>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count()) * ctas));
#define TLB_TILED_TMA(EB, LB)                                                                                          \
    do {                                                                                                               \
        TLB_CUDA(cudaFuncSetAttribute(tiled_tma_kernel<EB, LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
        TLB_CUDA(launch_pdl(tiled_tma_kernel<EB, LB>, dim3(grid_tma), dim3(kThreads), smem, c.stream, map, TP, db, stages)); \
    } while (0)
                    if (eb == 4) {
                        if (Lb == 256) TLB_TILED_TMA(4, 256); else if (Lb == 128) TLB_TILED_TMA(4, 128); else if (Lb == 64) TLB_TILED_TMA(4, 64); else TLB_TILED_TMA(4, 32);
                    } else if (eb == 8) {
                        if (Lb == 256) TLB_TILED_TMA(8, 256); else if (Lb == 128) TLB_TILED_TMA(8, 128); else if (Lb == 64) TLB_TILED_TMA(8, 64); else TLB_TILED_TMA(8, 32);
                    } else {
                        if (Lb == 256) TLB_TILED_TMA(2, 256); else if (Lb == 128) TLB_TILED_TMA(2, 128); else if (Lb == 64) TLB_TILED_TMA(2, 64); else TLB_TILED_TMA(2, 32);
                    }
#undef TLB_TILED_TMA
                    count_launch();
                    TLB_CUDA(cudaGetLastError());
                    set_plan("tiled_tma");
                    *done = true;
                    return TLB_OK;
                }
            }
            (void)cudaGetLastError();
            if (g_copy_path == 3) continue; // this |B| has no tensor map: a shorter B run may have one
        }
        if (g_dry_run) {
            set_plan(strided_runs ? "tiled_s" : unaligned ? "tiled_u" : "tiled");
            *done = true;
            return TLB_OK;
        }
        const unsigned grid = static_cast<unsigned>(tiles);
        if (unaligned && knob(K_COPY_CELL_TILES) != 0) {
            // nothing 16-byte aligned, or runs without a unit stride: consecutive lanes on consecutive cells of the run
#define TLB_TC(EB) do { if (Lb == 128) TLB_CUDA(launch_pdl(tiled_cell_kernel<EB, 128>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db)); \
                        else TLB_CUDA(launch_pdl(tiled_cell_kernel<EB, 32>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db)); } while (0)
            if (eb == 1) TLB_CUDA(launch_pdl(tiled_cell_kernel<1, 128>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db));
            else if (eb == 2) TLB_TC(2); else if (eb == 4) TLB_TC(4); else TLB_TC(8);
#undef TLB_TC
            count_launch();
            set_plan(strided_runs ? "tiled_s" : "tiled_u");
            *done = true;
            return TLB_OK;
        }
        if (unaligned) {
            if (eb == 2) {
                if (Lb == 128) tiled_kernel<2, 128, false><<<grid, kThreads, 0, c.stream>>>(P, sb, db);
                else tiled_kernel<2, 32, false><<<grid, kThreads, 0, c.stream>>>(P, sb, db);
            } else if (eb == 4) {
                if (Lb == 128) tiled_kernel<4, 128, false><<<grid, kThreads, 0, c.stream>>>(P, sb, db);
                else tiled_kernel<4, 32, false><<<grid, kThreads, 0, c.stream>>>(P, sb, db);
            } else {
                if (Lb == 128) tiled_kernel<8, 128, false><<<grid, kThreads, 0, c.stream>>>(P, sb, db);
                else tiled_kernel<8, 32, false><<<grid, kThreads, 0, c.stream>>>(P, sb, db);
            }
            count_launch();
            TLB_CUDA(cudaGetLastError());
            set_plan(strided_runs ? "tiled_s" : "tiled_u");
            *done = true;
            return TLB_OK;
        }
        // short tiles: several per CTA once there are enough tiles to keep every SM busy with whole groups
        {
            const int tmax = tiles_per_cta(static_cast<int>(Lb), true);
            P.tpc = (knob(K_COPY_TILES_PER_CTA) != 0 && tmax > 1 && tiles >= 16ull * static_cast<uint64_t>(sm_count()) * static_cast<uint64_t>(tmax)) ? tmax : 1;
        }
#define TLB_TILED(EB, LB) TLB_CUDA(launch_pdl(tiled_kernel<EB, LB, true>, dim3((grid + P.tpc - 1) / P.tpc), dim3(kThreads), 0, c.stream, P, sb, db))
        if (eb == 1) {
            if (Lb == 256) TLB_TILED(1, 256); else TLB_TILED(1, 128);
        } else if (eb == 16) {
            if (Lb == 256) TLB_TILED(16, 256); else if (Lb == 128) TLB_TILED(16, 128); else TLB_TILED(16, 32);
        } else {
#define TLB_TILED_LB(EB) do { switch (Lb) { case 256: TLB_TILED(EB, 256); break; case 224: TLB_TILED(EB, 224); break; case 192: TLB_TILED(EB, 192); break; \
                                           case 160: TLB_TILED(EB, 160); break; case 128: TLB_TILED(EB, 128); break; case 96: TLB_TILED(EB, 96); break;   \
                                           case 64: TLB_TILED(EB, 64); break; default: TLB_TILED(EB, 32); break; } } while (0)
            if (eb == 4) TLB_TILED_LB(4); else if (eb == 8) TLB_TILED_LB(8); else TLB_TILED_LB(2);
#undef TLB_TILED_LB
        }
#undef TLB_TILED
        count_launch();
        TLB_CUDA(cudaGetLastError());
        set_plan("tiled");
        *done = true;
        return TLB_OK;
    }
    if (g_copy_path == 3) return fail(TLB_ERR_UNSUPPORTED, "tlb_copy: the source layout has no TMA tensor map for any tiling");
    // ---- narrow runs: one run is a whole short mode (fewer cells than a 128-byte row / a 32-row tile), the other as above
    if (!strided_runs && g_copy_path == 0 && knob(K_COPY_CELL_TILES) != 0 && eb <= 8) {
        if (g_defer_narrow && knob(K_COPY_RAGGED) != 0 && c.n >= (1ull << std::min(40, knob(K_COPY_RAGGED)))) {
            // an AoS <-> SoA pattern whose long mode is not whole lane pieces: let the ragged cut try the (faster) interleave body first
            auto short_mode = [eb](int64_t e) { return interleave_size(e, eb); };
            if ((modes[ib].ss == modes[ia].e && short_mode(modes[ia].e)) || (modes[ia].ds == modes[ib].e && short_mode(modes[ib].e))) {
                g_narrow_deferred = true;
                return TLB_OK;
            }
        }
        const bool narrow_a = modes[ia].e >= 2 && modes[ia].e * eb < 128;
        // (1-byte cells: the staged plan needs 128 rows; other cells: a destination run below 128 cells that is not a whole
        // number of 32-row tiles, e.g. 48, is taken whole here instead of being cut into 32 + 16)
        const bool narrow_b = !narrow_a && modes[ib].e >= 2 && (modes[ib].e < (eb == 1 ? 128 : 32) || (modes[ib].e < 128 && modes[ib].e % 32 != 0));
        // the long run's length: the staged tile (rows of an odd number of words) must fit 33 KiB
        const int64_t short_e = narrow_a ? modes[ia].e : modes[ib].e;
        // long-run candidates: tall tiles when they still give every SM a few CTAs, else shorter ones (a 16-column edge strip
        // of 8000 rows is 31 tiles of 256 rows: slower than the gather it replaces)
        const int64_t long_e = narrow_a ? modes[ib].e : modes[ia].e;
        uint64_t others = 1;
        for (size_t r = 0; r < modes.size(); ++r)
            if (static_cast<int>(r) != ia && static_cast<int>(r) != ib) others *= static_cast<uint64_t>(modes[r].e);
        std::vector<int64_t> cands;
        for (int64_t Lr : {256, 128, 64, 32})
            if (others * static_cast<uint64_t>(long_e / Lr) >= 2ull * static_cast<uint64_t>(sm_count())) cands.push_back(Lr);
        for (int64_t Lr : {32, 64, 128, 256})
            if (std::find(cands.begin(), cands.end(), Lr) == cands.end()) cands.push_back(Lr);
        for (int64_t Lr : cands) {
            if (!narrow_a && !narrow_b) break;
            const int64_t la = narrow_a ? short_e : Lr, lb = narrow_a ? Lr : short_e;
            const int64_t pitch = ((((la * eb + 3) >> 2) | 1) + (eb == 8 ? 1 : 0)) << 2;
            if (lb * pitch > kNarrowTileBytes || la > kNarrowMaxRun || lb > kNarrowMaxRun) continue;
            std::vector<JM> work = modes, A, B;
            if (narrow_a) {
                A.push_back(work[ia]);
                work[ia].e = 1;
                if (!take_run(&work, false, lb, &B, 1)) continue;
            } else {
                B.push_back(work[ib]);
                work[ib].e = 1;
                if (!take_run(&work, true, la, &A, 1)) continue;
            }
            if (A.size() > kMaxPieces || B.size() > kMaxPieces) continue;
            std::vector<JM> rest;
            for (const JM& m : work)
                if (m.e > 1) rest.push_back(m);
            std::stable_sort(rest.begin(), rest.end(), [](const JM& a, const JM& b) {
                return std::min(std::llabs(a.ss), std::llabs(a.ds)) < std::min(std::llabs(b.ss), std::llabs(b.ds));
            });
            TileParams P;
            std::memset(&P, 0, sizeof(P));
            TLB_TRY(fill_joint(rest, &P.rest));
            P.nA = static_cast<int>(A.size());
            P.nB = static_cast<int>(B.size());
            for (size_t r = 0; r < A.size(); ++r) { P.eA[r] = A[r].e; P.dA[r] = A[r].ds; }
            for (size_t r = 0; r < B.size(); ++r) { P.eB[r] = B[r].e; P.sB[r] = B[r].ss; }
            P.La = static_cast<int>(la);
            P.Lb = static_cast<int>(lb);
            P.ua = P.ub = 1;
            uint64_t tiles = 1;
            for (const JM& m : rest) tiles *= static_cast<uint64_t>(m.e);
            P.n_tiles = tiles;
            if (tiles > 0x7fffffffull) return TLB_OK;
            if (g_dry_run) {
                set_plan("tiled_n");
                *done = true;
                return TLB_OK;
            }
            const unsigned grid = static_cast<unsigned>(tiles);
            const char* sb = sp + base_s * eb;
            char* db = dp + base_d * eb;
            if (eb == 1) TLB_CUDA(launch_pdl(tiled_narrow_kernel<1>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db));
            else if (eb == 2) TLB_CUDA(launch_pdl(tiled_narrow_kernel<2>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db));
            else if (eb == 4) TLB_CUDA(launch_pdl(tiled_narrow_kernel<4>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db));
            else TLB_CUDA(launch_pdl(tiled_narrow_kernel<8>, dim3(grid), dim3(kThreads), 0, c.stream, P, sb, db));
            count_launch();
            set_plan("tiled_n");
            *done = true;
            return TLB_OK;
        }
    }
    return TLB_OK;
}

} // namespace

// Exact span of positions for the bounds pre-flight (tensor.hpp:99): Int kind by interval
// arithmetic over the modes (exact on the full domain, outer-mode-restricted on a sub-range),
// Xor kind by the OR-bound with an exact device scan when that bound does not fit.
int bounds_preflight(const tlb_tensor& t, uint64_t i0, uint64_t n, const char* who, cudaStream_t stream, Span* out) {
    const tlb_layout_desc& L = *t.layout;
    Span sp{0, 0};
    if (L.kind == TLB_KIND_INT) {
        __int128 lo = t.origin, hi = t.origin;
        uint64_t prefix = 1;
        for (int r = 0; r < L.n_modes; ++r) {
            int64_t c_lo = 0, c_hi = L.extent[r] - 1;
            if (r + 1 == L.n_modes) {
                c_lo = static_cast<int64_t>(i0 / prefix);
                c_hi = static_cast<int64_t>((i0 + n - 1) / prefix);
            }
            const __int128 a = static_cast<__int128>(c_lo) * L.stride[r], b = static_cast<__int128>(c_hi) * L.stride[r];
            lo += a < b ? a : b;
            hi += a < b ? b : a;
            prefix *= static_cast<uint64_t>(L.extent[r]);
        }
        if (lo < INT64_MIN || hi > INT64_MAX) return fail(TLB_ERR_OVERFLOW, "integer overflow in addition");
        sp.lo = static_cast<int64_t>(lo);
        sp.hi = static_cast<int64_t>(hi);
        // a sub-range narrower than the outermost mode's stride may be over-approximated; verify exactly
        if ((sp.lo < 0 || sp.hi >= t.capacity) && t.accessor == TLB_ACC_BUFFER && n != static_cast<uint64_t>(L.size) &&
            !g_dry_run) {
            long long h[2] = {INT64_MAX, INT64_MIN};
            long long* d = nullptr;
            TLB_CUDA(ws_malloc(reinterpret_cast<void**>(&d), sizeof(h), stream));
            TLB_CUDA(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, stream));
            span_kernel<<<launch_grid(n, kThreads, 8), kThreads, 0, stream>>>(L, t.origin, i0, n, d);
            count_launch();
            TLB_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
            TLB_CUDA(cudaStreamSynchronize(stream));
            cudaFreeAsync(d, stream);
            sp.lo = h[0];
            sp.hi = h[1];
        }
    } else {
        TLB_TRY(position_span(L, t.origin, &sp));
        if ((sp.lo < 0 || sp.hi >= t.capacity) && t.accessor == TLB_ACC_BUFFER && t.origin >= 0 && !g_dry_run) {
            long long h[2] = {INT64_MAX, INT64_MIN};
            long long* d = nullptr;
            TLB_CUDA(ws_malloc(reinterpret_cast<void**>(&d), sizeof(h), stream));
            TLB_CUDA(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, stream));
            span_kernel<<<launch_grid(n, kThreads, 8), kThreads, 0, stream>>>(L, t.origin, i0, n, d);
            count_launch();
            TLB_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
            TLB_CUDA(cudaStreamSynchronize(stream));
            cudaFreeAsync(d, stream);
            sp.lo = h[0];
            sp.hi = h[1];
        }
    }
    if (t.accessor == TLB_ACC_BUFFER && (sp.lo < 0 || sp.hi >= t.capacity))
        return fail(TLB_ERR_BOUNDS, std::string("buffer access out of bounds (") + who + ")");
    *out = sp;
    return TLB_OK;
}

int check_tensor(const tlb_tensor* t, const char* who, bool writable) {
    if (!t || !t->layout) return fail(TLB_ERR_CONTRACT, std::string(who) + ": null tensor");
    if (t->layout->kind == TLB_KIND_BASIS)
        return fail(TLB_ERR_SEMIMODULE, "integer accessor cannot take a coordinate offset");
    if (t->accessor != TLB_ACC_BUFFER && t->accessor != TLB_ACC_COUNTING)
        return fail(TLB_ERR_CONTRACT, std::string(who) + ": unknown accessor");
    if (writable && t->accessor != TLB_ACC_BUFFER) return fail(TLB_ERR_CONTRACT, "only buffer accessors are writable");
    if (t->accessor == TLB_ACC_BUFFER) {
        if (!t->data) return fail(TLB_ERR_CONTRACT, "buffer accessor requires storage");
        if (t->capacity < 0) return fail(TLB_ERR_CONTRACT, std::string(who) + ": negative capacity");
    }
    const int eb = t->elem_bytes;
    if (eb != 1 && eb != 2 && eb != 4 && eb != 8 && eb != 16)
        return fail(TLB_ERR_UNSUPPORTED, std::string(who) + ": element size must be 1, 2, 4, 8 or 16 bytes");
    return TLB_OK;
}

int copy_impl(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end, cudaStream_t stream);

// Non-injective destination whose only aliasing comes from stride-0 (broadcast) modes: every destination cell is written
// once per coordinate of those modes and the LAST writer in ascending i (tensor.hpp:198) is the one whose broadcast
// coordinates are all maximal (i grows with every coordinate). The copy therefore equals the injective copy of the slice
// that fixes those modes at their last coordinate, which the ordinary plans run: nothing else is read. Worked on the
// common refinement (a broadcast mode of the destination may cut across source modes).
thread_local std::string g_lw_plan;
int try_last_writer_slice(const CopyCall& c, bool* done) {
    *done = false;
    const tlb_layout_desc& S = *c.src->layout;
    const tlb_layout_desc& D = *c.dst->layout;
    if (g_copy_path != 0 || S.kind != TLB_KIND_INT || D.kind != TLB_KIND_INT) return TLB_OK;
    if (c.i0 != 0 || c.n != static_cast<uint64_t>(S.size)) return TLB_OK;
    std::vector<JM> modes;
    if (!refine_modes(S, D, &modes)) return TLB_OK;
    std::vector<tlb_mode> sm, dm;
    int64_t shift = 0;
    bool any = false;
    for (const JM& m : modes) {
        if (m.e == 1) continue;
        if (m.ds == 0) {
            int64_t t;
            if (!mul_ok(m.e - 1, m.ss, &t) || __builtin_add_overflow(shift, t, &shift)) return TLB_OK;
            any = true;
            continue;
        }
        sm.push_back({m.e, m.ss, TLB_KIND_INT, 0});
        dm.push_back({m.e, m.ds, TLB_KIND_INT, 0});
    }
    if (!any || sm.size() > TLB_MAX_MODES) return TLB_OK;
    if (sm.empty()) {
        sm.push_back({1, 0, TLB_KIND_INT, 0});
        dm.push_back({1, 0, TLB_KIND_INT, 0});
    }
    tlb_layout_desc ls, ld;
    if (tlb_layout_lower(sm.data(), static_cast<int>(sm.size()), &ls) != TLB_OK) return TLB_OK;
    if (tlb_layout_lower(dm.data(), static_cast<int>(dm.size()), &ld) != TLB_OK) return TLB_OK;
    if (!(ld.flags & TLB_LF_INJECTIVE)) return TLB_OK; // other modes overlap as well: winner election
    tlb_tensor s2 = *c.src, d2 = *c.dst;
    s2.layout = &ls;
    d2.layout = &ld;
    s2.origin += shift;
    const int st = copy_impl(&s2, &d2, 0, static_cast<uint64_t>(ls.size), c.stream);
    if (st == TLB_OK) {
        g_lw_plan = std::string("last_writer+") + tlb_last_plan();
        set_plan(g_lw_plan.c_str());
    }
    *done = true;
    return st;
}

// Ragged extents (a 4000 x 3000 transpose: rows of 3000 cells are not whole 128-byte pieces, 4000 rows not whole tiles).
// The staged plan needs whole tiles, so the call is cut, on the refined modes, into a BODY whose two run modes are rounded
// down to tile multiples and at most two edge strips: the tail of the A run over every b, and the tail of the B run over the
// body's a. The destination is injective and the pieces are disjoint boxes of the coordinate space, so each piece is an
// independent copy and the union is tla::copy's result. Pieces recurse (a 160-row tail is a 128-row body plus 32 rows).
int try_ragged(const CopyCall& c, const Refined& R, bool* done) {
    *done = false;
    if (g_copy_path != 0 || g_ragged_depth >= 3 || knob(K_COPY_RAGGED) == 0 || !R.ok) return TLB_OK;
    const int eb = c.dst->elem_bytes;
    if (eb != 1 && eb != 2 && eb != 4 && eb != 8 && eb != 16) return TLB_OK;
    const std::vector<JM>& modes = R.modes;
    if (modes.size() > TLB_MAX_MODES) return TLB_OK;
    int ia = -1, ib = -1;
    for (size_t r = 0; r < modes.size(); ++r) {
        if (modes[r].ss == 1 && ia < 0) ia = static_cast<int>(r);
        if (modes[r].ds == 1 && ib < 0) ib = static_cast<int>(r);
    }
    if (ia < 0 || ib < 0) return TLB_OK;
    if (c.n < (1ull << std::min(40, knob(K_COPY_RAGGED)))) return TLB_OK;
    if (ia == ib) {
        // one mode contiguous on both sides whose extent is not a whole number of 16-byte vectors (an odd number of bytes):
        // whole vectors on the vec plan, the last cells of the run through the gather
        // ... and a run that STARTS off a 16-byte boundary by the same amount on both sides (a[1:] -> b[1:]): the head cells up to
        // the boundary are gathered as well
        if (eb >= 16) return TLB_OK;
        const int64_t V = 16 / eb, e = modes[ia].e;
        const uintptr_t as = (reinterpret_cast<uintptr_t>(c.src->data) + static_cast<uintptr_t>(R.base_s) * eb) & 15u;
        const uintptr_t ad = (reinterpret_cast<uintptr_t>(c.dst->data) + static_cast<uintptr_t>(R.base_d) * eb) & 15u;
        if (as != ad || as % eb != 0) return TLB_OK;
        const int64_t head = as ? static_cast<int64_t>((16 - as) / eb) : 0;
        if (head >= e) return TLB_OK;
        const int64_t body = (e - head) / V * V;
        if ((body == e && head == 0) || body == 0) return TLB_OK;
        auto part = [&](int64_t a0, int64_t ea) -> int {
            tlb_mode sm[TLB_MAX_MODES], dm[TLB_MAX_MODES];
            for (size_t r = 0; r < modes.size(); ++r) {
                const int64_t ex = static_cast<int>(r) == ia ? ea : modes[r].e;
                sm[r] = {ex, modes[r].ss, TLB_KIND_INT, 0};
                dm[r] = {ex, modes[r].ds, TLB_KIND_INT, 0};
            }
            tlb_layout_desc ls, ld;
            TLB_TRY(tlb_layout_lower(sm, static_cast<int>(modes.size()), &ls));
            TLB_TRY(tlb_layout_lower(dm, static_cast<int>(modes.size()), &ld));
            tlb_tensor s2 = *c.src, d2 = *c.dst;
            s2.layout = &ls;
            d2.layout = &ld;
            s2.origin = R.base_s + a0 * modes[ia].ss;
            d2.origin = R.base_d + a0 * modes[ia].ds;
            ++g_ragged_depth;
            const int st = copy_impl(&s2, &d2, 0, static_cast<uint64_t>(ls.size), c.stream);
            --g_ragged_depth;
            return st;
        };
        const bool was_dry = g_dry_run;
        g_dry_run = true;
        const int probe = part(head, body);
        g_dry_run = was_dry;
        const std::string body_plan = tlb_last_plan();
        if (probe != TLB_OK || body_plan != "vec") return TLB_OK;
        g_ragged_plan = "ragged:vec";
        if (!g_dry_run) {
            TLB_TRY(part(head, body));
            if (head) TLB_TRY(part(0, head));
            if (head + body < e) TLB_TRY(part(head + body, e - head - body));
        }
        set_plan(g_ragged_plan.c_str());
        *done = true;
        return TLB_OK;
    }
    const int64_t La = 128 / eb, eA = modes[ia].e, eB = modes[ib].e;
    // AoS <-> SoA whose long mode is not a whole number of lane pieces: whole pieces on the interleave plan, the last j gathered
    if (eb < 16) {
        auto short_mode = [eb](int64_t e) { return interleave_size(e, eb); };
        const bool deint = modes[ib].ss == eA && short_mode(eA), inter = !deint && modes[ia].ds == eB && short_mode(eB);
        if (deint || inter) {
            const int64_t EC = deint ? eA : eB, eJ = deint ? eB : eA, NJ = (16 / eb) * ((EC % 2) ? 2 : 1), bodyJ = eJ / NJ * NJ;
            if (bodyJ >= NJ && bodyJ != eJ) {
                auto cut = [&](int64_t j0, int64_t ej) { return deint ? std::array<int64_t, 4>{0, eA, j0, ej} : std::array<int64_t, 4>{j0, ej, 0, eB}; };
                auto run = [&](const std::array<int64_t, 4>& q) -> int {
                    tlb_mode sm[TLB_MAX_MODES], dm[TLB_MAX_MODES];
                    for (size_t r = 0; r < modes.size(); ++r) {
                        const int64_t e = static_cast<int>(r) == ia ? q[1] : static_cast<int>(r) == ib ? q[3] : modes[r].e;
                        sm[r] = {e, modes[r].ss, TLB_KIND_INT, 0};
                        dm[r] = {e, modes[r].ds, TLB_KIND_INT, 0};
                    }
                    tlb_layout_desc ls, ld;
                    TLB_TRY(tlb_layout_lower(sm, static_cast<int>(modes.size()), &ls));
                    TLB_TRY(tlb_layout_lower(dm, static_cast<int>(modes.size()), &ld));
                    tlb_tensor s2 = *c.src, d2 = *c.dst;
                    s2.layout = &ls;
                    d2.layout = &ld;
                    s2.origin = R.base_s + q[0] * modes[ia].ss + q[2] * modes[ib].ss;
                    d2.origin = R.base_d + q[0] * modes[ia].ds + q[2] * modes[ib].ds;
                    ++g_ragged_depth;
                    const int st = copy_impl(&s2, &d2, 0, static_cast<uint64_t>(ls.size), c.stream);
                    --g_ragged_depth;
                    return st;
                };
                const bool was_dry = g_dry_run;
                g_dry_run = true;
                const int probe = run(cut(0, bodyJ));
                g_dry_run = was_dry;
                if (probe == TLB_OK && std::string(tlb_last_plan()) == "interleave") {
                    g_ragged_plan = "ragged:interleave";
                    if (!g_dry_run) {
                        TLB_TRY(run(cut(0, bodyJ)));
                        TLB_TRY(run(cut(bodyJ, eJ - bodyJ)));
                    }
                    set_plan(g_ragged_plan.c_str());
                    *done = true;
                    return TLB_OK;
                }
            }
        }
    }
    // small copies: one gather launch beats a handful of launches (1000 x 1000 fp32: 13 us as one gather). The knob is the
    // log2 of the smallest element count that is cut (default 22).
    if (c.n < (1ull << std::min(40, knob(K_COPY_RAGGED)))) return TLB_OK;
    // the tallest tile that fits (the leftover rows recurse into shorter tiles: measured better than starting with short
    // tiles, 300^3 reversal 65 us against 78 us)
    int64_t Lb = 0;
    for (int64_t cand : {256, 128, 64, 32}) {
        if ((cand == 256 && !lb256_enabled()) || (eb == 1 && cand < 128) || cand > eB) continue;
        Lb = cand;
        break;
    }
    const bool narrow = eA < La;   // a short A mode: the narrow-run staged kernel takes it whole, only B is cut
    const bool narrow_b = !narrow && Lb == 0 && eB >= 2 && eB < (eb == 1 ? 128 : 32) && eb <= 8 && eA >= 128;   // a short B mode: only A is cut (128-cell pieces)
    if ((Lb == 0 && !narrow_b) || (narrow && (eA < 2 || eb > 8))) return TLB_OK;
    const int64_t bodyA = narrow ? eA : narrow_b ? eA / 128 * 128 : eA / La * La, bodyB = narrow_b ? eB : eB / Lb * Lb;
    if (bodyA == eA && bodyB == eB) return TLB_OK; // whole tiles already: the staged plan was refused for another reason
    // one piece: A coordinates [a0, a0 + ea), B coordinates [b0, b0 + ebx), every other mode whole
    auto piece = [&](int64_t a0, int64_t ea, int64_t b0, int64_t ebx) -> int {
        tlb_mode sm[TLB_MAX_MODES], dm[TLB_MAX_MODES];
        for (size_t r = 0; r < modes.size(); ++r) {
            const int64_t e = static_cast<int>(r) == ia ? ea : static_cast<int>(r) == ib ? ebx : modes[r].e;
            sm[r] = {e, modes[r].ss, TLB_KIND_INT, 0};
            dm[r] = {e, modes[r].ds, TLB_KIND_INT, 0};
        }
        tlb_layout_desc ls, ld;
        TLB_TRY(tlb_layout_lower(sm, static_cast<int>(modes.size()), &ls));
        TLB_TRY(tlb_layout_lower(dm, static_cast<int>(modes.size()), &ld));
        tlb_tensor s2 = *c.src, d2 = *c.dst;
        s2.layout = &ls;
        d2.layout = &ld;
        s2.origin = R.base_s + a0 * modes[ia].ss + b0 * modes[ib].ss;
        d2.origin = R.base_d + a0 * modes[ia].ds + b0 * modes[ib].ds;
        ++g_ragged_depth;
        const int st = copy_impl(&s2, &d2, 0, static_cast<uint64_t>(ls.size), c.stream);
        --g_ragged_depth;
        return st;
    };
    // the cut pays only if the body takes a staged plan: ask the planner first
    const bool was_dry = g_dry_run;
    g_dry_run = true;
    const int probe = piece(0, bodyA, 0, bodyB);
    g_dry_run = was_dry;
    const std::string body_plan = tlb_last_plan();
    if (probe != TLB_OK || body_plan.compare(0, 5, "tiled") != 0) return TLB_OK;
    g_ragged_plan = "ragged:" + body_plan;
    if (!g_dry_run) {
        TLB_TRY(piece(0, bodyA, 0, bodyB));
        if (bodyA < eA) TLB_TRY(piece(bodyA, eA - bodyA, 0, eB));
        if (bodyB < eB) TLB_TRY(piece(0, bodyA, bodyB, eB - bodyB));
    }
    set_plan(g_ragged_plan.c_str());
    *done = true;
    return TLB_OK;
}

int copy_impl(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end, cudaStream_t stream) {
    TLB_TRY(check_tensor(src, "tlb_copy source", false));
    TLB_TRY(check_tensor(dst, "tlb_copy destination", true));
    const tlb_layout_desc& S = *src->layout;
    const tlb_layout_desc& D = *dst->layout;
    if (S.size != D.size) return fail(TLB_ERR_CONTRACT, "copy requires equal sizes");
    if (src->elem_bytes != dst->elem_bytes) return fail(TLB_ERR_CONTRACT, "tlb_copy: element sizes differ");
    if (src->accessor == TLB_ACC_COUNTING && dst->elem_bytes != 8)
        return fail(TLB_ERR_CONTRACT, "tlb_copy: a counting source produces 8-byte cells");
    const uint64_t size = static_cast<uint64_t>(S.size);
    if (i_end > size) i_end = size;
    if (i_begin >= i_end) {
        set_plan("empty");
        return TLB_OK;
    }
    if (!g_dry_run) TLB_TRY(require_device());
    CopyCall c{src, dst, i_begin, i_end - i_begin, stream};
    TLB_TRY(overflow_preflight(S, src->origin, i_end - 1));
    TLB_TRY(overflow_preflight(D, dst->origin, i_end - 1));
    Span sspan, dspan;
    TLB_TRY(bounds_preflight(*src, c.i0, c.n, "source", stream, &sspan));
    TLB_TRY(bounds_preflight(*dst, c.i0, c.n, "destination", stream, &dspan));
    // Aliasing (tensor.hpp:29: every sliced view shares one storage): when the byte ranges the two tensors touch
    // intersect, the reference's serial order decides the result; the parallel plans below assume disjoint ranges.
    if (src->accessor == TLB_ACC_BUFFER) {
        const uintptr_t eb = static_cast<uintptr_t>(dst->elem_bytes);
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(src->data) + static_cast<uintptr_t>(sspan.lo) * eb;
        const uintptr_t s1 = reinterpret_cast<uintptr_t>(src->data) + (static_cast<uintptr_t>(sspan.hi) + 1) * eb;
        const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst->data) + static_cast<uintptr_t>(dspan.lo) * eb;
        const uintptr_t d1 = reinterpret_cast<uintptr_t>(dst->data) + (static_cast<uintptr_t>(dspan.hi) + 1) * eb;
        if (s0 < d1 && d0 < s1) return launch_aliased(c, dspan, (D.flags & TLB_LF_INJECTIVE) != 0);
    }
    if (!(D.flags & TLB_LF_INJECTIVE)) {
        bool sliced = false;
        const int st = try_last_writer_slice(c, &sliced);
        if (sliced) return st;
        return launch_ordered(c, dspan);
    }
    if (g_copy_path != 1) {
        bool done = false;
        Refined refined;
        g_defer_narrow = true;
        g_narrow_deferred = false;
        const int st_planned = try_planned(c, &done, &refined);
        g_defer_narrow = false;
        TLB_TRY(st_planned);
        if (done) return TLB_OK;
        if (g_narrow_deferred) {   // ragged interleave first; the narrow-run tiles if that cut does not apply
            g_narrow_deferred = false;
            TLB_TRY(try_ragged(c, refined, &done));
            if (done) return TLB_OK;
            Refined again;
            TLB_TRY(try_planned(c, &done, &again));
            if (done) return TLB_OK;
        }
        if (g_copy_path == 2 || g_copy_path == 3)
            return fail(TLB_ERR_UNSUPPORTED, "tlb_copy: the forced tiled path does not apply to these layouts");
        if (refined.ok) {
            TLB_TRY(try_ragged(c, refined, &done));
            if (done) return TLB_OK;
        }
        if (refined.ok && refined.modes.size() <= TLB_MAX_MODES) return launch_gather_joint(c, refined);
    }
    return launch_gather(c);
}

} // namespace tlb


namespace tlb {
namespace {
// Partitioning IS composition: the tensors a thread-value layout partitions are src o TV and dst o TV,
// layouts over the (thread, value) domain. When TV is a bijection onto [0, size) whose leaves are DIGITS of the integral
// coordinate (sorted by stride they nest: d_0 = 1, d_{k+1} = d_k e_k, what blocked / raked products of compact layouts
// give), A o TV is exact leaf by leaf with no carries between leaves, and each TV leaf splits into sub-digits that lie
// inside one leaf of the source and one leaf of the destination (compose, algebra.hpp:235, without the O(|B|)
// verify_distributed loop: the nesting test is the proof). The copy is then the plain layout-driven copy between the
// two compositions, walked in TV's own order, and takes the planner's staged / vectorised plans. Returns false when TV
// is not such a digit permutation, a sub-digit would straddle a leaf, or the result needs more than TLB_MAX_MODES leaves.
bool tv_compose(const tlb_layout_desc& S, const tlb_layout_desc& D, const tlb_layout_desc& TV, tlb_layout_desc* st, tlb_layout_desc* dt) {
    if (S.kind != TLB_KIND_INT || D.kind != TLB_KIND_INT || TV.kind != TLB_KIND_INT) return false;
    if (TV.size != S.size || S.size != D.size || S.size < 1) return false;
    // TV's leaves as digits of i
    int order[TLB_MAX_MODES], m = 0;
    for (int r = 0; r < TV.n_modes; ++r)
        if (TV.extent[r] > 1) {
            if (TV.stride[r] <= 0) return false;
            order[m++] = r;
        }
    std::sort(order, order + m, [&](int a, int b) { return TV.stride[a] < TV.stride[b]; });
    int64_t next = 1;
    for (int k = 0; k < m; ++k) {
        if (TV.stride[order[k]] != next) return false;
        next *= TV.extent[order[k]];
    }
    if (next != S.size) return false;
    // sub-digit (x, q): extent x at index stride q. Inside leaf r of A (prefix product P_r <= q, q % P_r == 0, (q / P_r) x
    // divides E_r, the last leaf unbounded) it contributes stride_r * (q / P_r) per step.
    auto locate = [](const tlb_layout_desc& A, int64_t q, int64_t* avail, int64_t* stride) {
        int64_t P = 1;
        for (int r = 0; r < A.n_modes; ++r) {
            const bool last = r + 1 == A.n_modes;
            if (!last && q >= P * A.extent[r]) {
                P *= A.extent[r];
                continue;
            }
            if (q % P != 0) return false;
            const int64_t sub = q / P;
            if (!last && A.extent[r] % sub != 0) return false;
            *avail = last ? INT64_MAX : A.extent[r] / sub;
            if (A.stride[r] != 0 && (sub > INT64_MAX / std::max<int64_t>(1, std::llabs(A.stride[r])))) return false;
            *stride = A.stride[r] * sub;
            return true;
        }
        return false;
    };
    tlb_mode ms[TLB_MAX_MODES], md[TLB_MAX_MODES];
    int n = 0;
    for (int r = 0; r < TV.n_modes; ++r) {          // TV's own (colex) leaf order = the order of the composed domain
        int64_t e = TV.extent[r], q = TV.stride[r];
        if (e == 1) continue;
        while (e > 1) {
            int64_t as, ad, ss, ds;
            if (!locate(S, q, &as, &ss) || !locate(D, q, &ad, &ds)) return false;
            const int64_t x = std::min(e, std::min(as, ad));
            if (x < 2 || e % x != 0 || n == TLB_MAX_MODES) return false;
            ms[n] = {x, ss, TLB_KIND_INT, 0};
            md[n] = {x, ds, TLB_KIND_INT, 0};
            ++n;
            e /= x;
            q *= x;
        }
    }
    if (n == 0) return false;
    return tlb_layout_lower(ms, n, st) == TLB_OK && tlb_layout_lower(md, n, dt) == TLB_OK;
}
} // namespace
} // namespace tlb

extern "C" {

// tla::max_common_vector (analysis.hpp:18-28) from the common refinement: the reference takes the stride-1 identity prefix
// of coalesce(B o right_inverse(A)), i.e. the longest run of offsets 0 .. K-1 that both layouts reach from the same
// coordinates. In the refinement that is the chain of modes whose source AND destination strides are 1, e_0, e_0 e_1, ...
int tlb_max_common_vector(const tlb_layout_desc* a, const tlb_layout_desc* b, int64_t* k) {
    if (!a || !b || !k) return tlb::fail(TLB_ERR_CONTRACT, "tlb_max_common_vector: null argument");
    if (a->size != b->size) return tlb::fail(TLB_ERR_CONTRACT, "max_common_vector requires equal sizes");
    *k = 1; // "any inadmissible step falls back to the always-correct scalar answer 1"
    if (a->kind != TLB_KIND_INT || b->kind != TLB_KIND_INT) return TLB_OK;
    std::vector<tlb::JM> modes;
    if (!tlb::refine_modes(*a, *b, &modes)) return TLB_OK;
    std::vector<bool> used(modes.size(), false);
    int64_t K = 1;
    for (;;) {
        int hit = -1;
        for (size_t r = 0; r < modes.size(); ++r)
            if (!used[r] && modes[r].e > 1 && modes[r].ss == K && modes[r].ds == K) {
                hit = static_cast<int>(r);
                break;
            }
        if (hit < 0) break;
        used[hit] = true;
        K *= modes[hit].e;
    }
    *k = K;
    return TLB_OK;
}

int tlb_copy(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end, void* stream) {
    return tlb::copy_impl(src, dst, i_begin, i_end, static_cast<cudaStream_t>(stream));
}

int tlb_copy_plan(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end) {
    tlb::g_dry_run = true;
    const int st = tlb::copy_impl(src, dst, i_begin, i_end, nullptr);
    tlb::g_dry_run = false;
    return st;
}

/* ---- thread-value partitioned copy ----------------------------------------------------------------------------- */
int tlb_copy_tv(const tlb_tensor* src, const tlb_tensor* dst, const tlb_layout_desc* tv, void* stream) {
    using namespace tlb;
    if (!tv) return fail(TLB_ERR_CONTRACT, "tlb_copy_tv: null thread-value layout");
    TLB_TRY(check_tensor(src, "tlb_copy_tv source", false));
    TLB_TRY(check_tensor(dst, "tlb_copy_tv destination", true));
    const tlb_layout_desc& S = *src->layout;
    const tlb_layout_desc& D = *dst->layout;
    if (S.size != D.size) return fail(TLB_ERR_CONTRACT, "copy requires equal sizes");
    if (src->elem_bytes != dst->elem_bytes) return fail(TLB_ERR_CONTRACT, "tlb_copy_tv: element sizes differ");
    if (src->accessor != TLB_ACC_BUFFER) return fail(TLB_ERR_UNSUPPORTED, "tlb_copy_tv: the source must be a buffer tensor");
    if (tv->n_top != 2) return fail(TLB_ERR_CONTRACT, "tlb_copy_tv: the thread-value layout must have rank 2 (thread, value)");
    if (tv->kind != TLB_KIND_INT || (tv->flags & TLB_LF_HAS_NEG))
        return fail(TLB_ERR_SEMIMODULE, "tlb_copy_tv: the thread-value layout must have non-negative integer strides");
    // every cell must have ONE writer: the destination injective, and no two (thread, value) pairs on one coordinate
    if (!(D.flags & TLB_LF_INJECTIVE) || !(tv->flags & TLB_LF_INJECTIVE))
        return fail(TLB_ERR_UNSUPPORTED, "tlb_copy_tv: the destination and the thread-value layout must be injective");
    const uint64_t size = static_cast<uint64_t>(S.size);
    if (size == 0 || tv->size == 0) {
        set_plan("empty");
        return TLB_OK;
    }
    TLB_TRY(require_device());
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    TLB_TRY(overflow_preflight(S, src->origin, size - 1));
    TLB_TRY(overflow_preflight(D, dst->origin, size - 1));
    TLB_TRY(overflow_preflight(*tv, 0, static_cast<uint64_t>(tv->size) - 1));
    Span sspan, dspan;
    TLB_TRY(bounds_preflight(*src, 0, size, "source", cs, &sspan));
    TLB_TRY(bounds_preflight(*dst, 0, size, "destination", cs, &dspan));
    {
        const uintptr_t eb = static_cast<uintptr_t>(dst->elem_bytes);
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(src->data) + static_cast<uintptr_t>(sspan.lo) * eb;
        const uintptr_t s1 = reinterpret_cast<uintptr_t>(src->data) + (static_cast<uintptr_t>(sspan.hi) + 1) * eb;
        const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst->data) + static_cast<uintptr_t>(dspan.lo) * eb;
        const uintptr_t d1 = reinterpret_cast<uintptr_t>(dst->data) + (static_cast<uintptr_t>(dspan.hi) + 1) * eb;
        if (s0 < d1 && d0 < s1) return fail(TLB_ERR_UNSUPPORTED, "tlb_copy_tv: source and destination overlap in memory (use tlb_copy)");
    }
    // the partitioned tensors as compositions src o TV / dst o TV: the planner's own plans (vec, tiled, ...) in TV's order
    if (knob(K_COPY_TV_COMPOSE) != 0) {
        tlb_layout_desc st, dt;
        if (tv_compose(S, D, *tv, &st, &dt)) {
            tlb_tensor cs_t = *src, cd_t = *dst;
            cs_t.layout = &st;
            cd_t.layout = &dt;
            const int rc = copy_impl(&cs_t, &cd_t, 0, UINT64_MAX, cs);
            if (rc == TLB_OK) {
                static thread_local char plan_name[64];
                std::snprintf(plan_name, sizeof(plan_name), "tv:%s", tlb_last_plan());
                set_plan(plan_name);
            }
            return rc;
        }
    }
    uint64_t n_threads = 1, n_values = 1;
    for (int r = tv->top_start[0]; r < tv->top_start[1]; ++r) n_threads *= static_cast<uint64_t>(tv->extent[r]);
    for (int r = tv->top_start[1]; r < tv->top_start[2]; ++r) n_values *= static_cast<uint64_t>(tv->extent[r]);
    // Vector width: the value mode starts with a unit-stride leaf of extent >= V, nothing else in TV reaches below V, and
    // both tensors keep V-aligned runs of V coordinates contiguous (low_run: Int and Xor layouts).
    const int eb = dst->elem_bytes;
    int V = 1;
    {
        int lead = tv->top_start[1];
        while (lead < tv->top_start[2] && tv->extent[lead] == 1) ++lead;
        if (eb < 16 && lead < tv->top_start[2] && tv->stride[lead] == 1) {
            V = std::min(low_run(*src, 16 / eb), low_run(*dst, 16 / eb));
            while (V > 1) {
                bool ok = tv->extent[lead] % V == 0 && size % static_cast<uint64_t>(V) == 0;
                for (int r = 0; ok && r < tv->n_modes; ++r)
                    if (r != lead && tv->extent[r] > 1) ok = tv->stride[r] % V == 0;
                if (ok) break;
                V >>= 1;
            }
        }
    }
    const uint64_t total = n_threads * (n_values / static_cast<uint64_t>(V));
    const int grid = launch_grid(total, kThreads, 8);
    const char* sb = static_cast<const char*>(src->data);
    char* db = static_cast<char*>(dst->data);
#define TLB_CTV(VB) TLB_CUDA(launch_pdl(copy_tv_kernel<VB>, dim3(grid), dim3(kThreads), 0, cs, *tv, S, D, sb, db, src->origin, dst->origin, n_threads, n_values, size, V, eb))
    switch (V * eb) {
    case 1: TLB_CTV(1); break;
    case 2: TLB_CTV(2); break;
    case 4: TLB_CTV(4); break;
    case 8: TLB_CTV(8); break;
    default: TLB_CTV(16); break;
    }
#undef TLB_CTV
    count_launch();
    set_plan(V > 1 ? "tv_vec" : "tv");
    return TLB_OK;
}

int tlb_copy_tv_auto(const tlb_layout_desc* src, const tlb_layout_desc* dst, int elem_bytes, int threads, tlb_mode* tv_modes,
                     int32_t* n_modes, int32_t* top_leaves2) {
    using namespace tlb;
    if (!src || !dst || !tv_modes || !n_modes || !top_leaves2) return fail(TLB_ERR_CONTRACT, "tlb_copy_tv_auto: null argument");
    if (src->size != dst->size) return fail(TLB_ERR_CONTRACT, "copy requires equal sizes");
    if (threads < 1 || (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16))
        return fail(TLB_ERR_CONTRACT, "tlb_copy_tv_auto: bad thread count or element size");
    int64_t mcv = 1;
    TLB_TRY(tlb_max_common_vector(src, dst, &mcv));
    int64_t V = 1;
    while (V * 2 <= 16 / elem_bytes && V * 2 <= mcv && mcv % (V * 2) == 0) V *= 2;
    const int64_t T = threads, tile = T * V;
    const int64_t R = (src->size + tile - 1) / tile;
    // raked_product((V):(1), (T):(1)) = (T, V):(V, 1) (algebra.hpp:633) is one tile of T vectors; the tiles follow in the
    // value mode, so thread t owns vector t of every tile: ((T), (V, R)) : ((V), (1, T V))
    tv_modes[0] = {T, V, TLB_KIND_INT, 0};
    tv_modes[1] = {V, 1, TLB_KIND_INT, 0};
    tv_modes[2] = {R, tile, TLB_KIND_INT, 0};
    *n_modes = 3;
    top_leaves2[0] = 1;
    top_leaves2[1] = 2;
    return TLB_OK;
}

int tlb_copy_set_path(int path) {
    const int prev = tlb::g_copy_path;
    if (path >= 0 && path <= 3) tlb::g_copy_path = path;
    return prev;
}

} // extern "C"

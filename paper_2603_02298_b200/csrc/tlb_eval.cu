// Bulk layout evaluation on device (BASELINE config C5): index maps L(i), natural
// coordinates, crd2idx and the right-inverse / composition identities, all bit-exact int64.
//
// Every kernel here is write-bound (8 B or more stored per evaluation, nothing read), so the
// design rule is: one 16-byte coalesced store per thread per step, a grid of a few waves of
// 148 SMs running a grid-stride loop, and a peel that costs a shift/mask per power-of-two
// leaf (magic multiply otherwise) so the integer pipe stays far below the HBM write time.
#include <algorithm>
#include <cstdlib>

#include "tlb_internal.h"

namespace tlb {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void st_cs_v2(int64_t* p, int64_t a, int64_t b) {
    // streaming 16-byte store: the map is written once and not re-read by this kernel
    asm volatile("st.global.cs.v2.s64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// out[k] = L(i0 + k). Pairs of consecutive k share one 16-byte store when `out` is 16-byte aligned.
template <bool kPairs>
__global__ void __launch_bounds__(kThreads) eval_range_kernel(const __grid_constant__ tlb_layout_desc L,
                                                              uint64_t i0, uint64_t n, int64_t* __restrict__ out) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (kPairs) {
        const uint64_t pairs = n >> 1;
        for (uint64_t p = t; p < pairs; p += stride) {
            const uint64_t k = p << 1;
            st_cs_v2(out + k, dev_eval(L, i0 + k), dev_eval(L, i0 + k + 1));
        }
        if (t == 0 && (n & 1)) out[n - 1] = dev_eval(L, i0 + n - 1);
    } else {
        for (uint64_t k = t; k < n; k += stride) out[k] = dev_eval(L, i0 + k);
    }
}

// Grouped evaluation: G consecutive indices that share every coordinate except the low bits of the
// first leaf (extent[0] % G == 0, i0 % G == 0) cost ONE peel: L(i + j) = L(i) + j*d0 for Int strides,
// L(i) ^ clmul(j, mask0) for Xor strides (the leaf coordinate c0 + j equals c0 ^ j when c0 % G == 0
// and clmul is linear over GF(2)). The map is write-bound only if an output costs about one
// instruction, so: the peel runs in 32-bit shifts when every extent is a power of two and the index
// fits 32 bits; the G outputs share their high word whenever the low word does not carry (one IADD
// per output); and each thread stores whole 32-byte sectors with 256-bit stores.
__device__ __forceinline__ void st_cs_v4(int64_t* p, int64_t a, int64_t b, int64_t c, int64_t d) {
    asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// Peel for all-power-of-two extents and i < 2^32: every coordinate is an independent shift+mask.
__device__ __forceinline__ int64_t dev_eval_pow2_u32(const tlb_layout_desc& L, uint32_t i) {
    int64_t acc = 0;
    const int n = L.n_modes;
    const bool is_xor = L.kind == TLB_KIND_XOR;
    uint32_t sh = 0;
    for (int r = 0; r < n; ++r) {
        uint32_t c = sh < 32 ? (i >> sh) : 0u;
        if (r + 1 < n) c &= static_cast<uint32_t>(L.extent[r]) - 1u;
        sh += L.log2e[r];
        if (is_xor) acc ^= dev_clmul(c, static_cast<uint64_t>(L.stride[r]));
        else acc += static_cast<int64_t>(c) * L.stride[r];
    }
    return acc;
}

template <int G, bool kPow2U32, bool kWide>
__global__ void __launch_bounds__(kThreads) eval_group_kernel(const __grid_constant__ tlb_layout_desc L, uint64_t i0,
                                                              uint64_t n_groups, int64_t* __restrict__ out) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool is_xor = L.kind == TLB_KIND_XOR;
    const int64_t d0 = L.stride[0];
    // Int strides: the low words of the G outputs stay below 2^32 past the base's low word?
    const bool small_step = !is_xor && d0 >= 0 && static_cast<uint64_t>(d0) * (G - 1) < (1ull << 32);
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n_groups; g += stride) {
        const uint64_t i = i0 + g * G;
        const int64_t base = kPow2U32 ? dev_eval_pow2_u32(L, static_cast<uint32_t>(i)) : dev_eval(L, i);
        int64_t v[G];
        if (is_xor) {
            v[0] = base;
#pragma unroll
            for (int j = 1; j < G; ++j) {
                // clmul(j, m) = clmul(j with its lowest set bit cleared, m) ^ (m << ctz(j))
                const int low = j & -j;
                int sh = 0;
                while ((1 << sh) != low) ++sh;
                v[j] = v[j - low] ^ static_cast<int64_t>(static_cast<uint64_t>(d0) << sh);
            }
        } else {
            const uint32_t lo = static_cast<uint32_t>(base);
            const uint32_t step = static_cast<uint32_t>(d0);
            const uint32_t last = lo + step * static_cast<uint32_t>(G - 1);
            if (small_step && last >= lo) {
                const uint64_t hi = static_cast<uint64_t>(base) & 0xffffffff00000000ull;
#pragma unroll
                for (int j = 0; j < G; ++j) v[j] = static_cast<int64_t>(hi | (lo + step * static_cast<uint32_t>(j)));
            } else {
#pragma unroll
                for (int j = 0; j < G; ++j) v[j] = base + j * d0;
            }
        }
        int64_t* o = out + g * G;
        if constexpr (kWide && G >= 4) {
#pragma unroll
            for (int j = 0; j < G; j += 4) st_cs_v4(o + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < G; j += 2) st_cs_v2(o + j, v[j], v[j + 1]);
        }
    }
}

// Odometer evaluation: 8 consecutive indices per thread for Int layouts whose LEADING leaf is not a multiple of the group
// sizes above (a leaf of 3, 5, 6 ... cells: every index there cost a full peel, 2 TB/s against 7 TB/s). One peel gives the
// coordinates of leaves 0 and 1 and the offset of the rest; the next index advances c0 by one stride, carries into c1 when
// c0 wraps, and only a wrap of c1 (once per e0 * e1 indices) peels the rest again. Same values as the flat peel of
// oracle_eval (oracle.hpp:58-69), last leaf unbounded.
template <bool kWide>
__global__ void __launch_bounds__(kThreads) eval_odo_kernel(const __grid_constant__ tlb_layout_desc L, uint64_t i0,
                                                            uint64_t n_groups, int64_t* __restrict__ out) {
    constexpr int G = 8;
    pdl_wait();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const int n = L.n_modes;
    const uint64_t e0 = static_cast<uint64_t>(L.extent[0]), e1 = static_cast<uint64_t>(L.extent[1]);
    const int64_t d0 = L.stride[0], d1 = L.stride[1], wrap0 = static_cast<int64_t>(e0) * d0;
    const bool bounded1 = n > 2;   // leaf 1 is the last leaf: unbounded, it never wraps
    // offset of the leaves 2.. at their integral coordinate q (last leaf unbounded)
    auto rest_of = [&](uint64_t q) {
        int64_t acc = 0;
        for (int r = 2; r < n; ++r) {
            uint64_t c;
            if (r + 1 < n) {
                const uint64_t qq = dev_div(L, r, q);
                c = q - qq * static_cast<uint64_t>(L.extent[r]);
                q = qq;
            } else {
                c = q;
            }
            acc += static_cast<int64_t>(c) * L.stride[r];
        }
        return acc;
    };
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n_groups; g += stride) {
        const uint64_t i = i0 + g * G;
        const uint64_t q0 = dev_div(L, 0, i);
        uint64_t c0 = i - q0 * e0, c1 = q0, q1 = 0;
        if (bounded1) {
            q1 = dev_div(L, 1, q0);
            c1 = q0 - q1 * e1;
        }
        int64_t rest = bounded1 ? rest_of(q1) : 0;
        int64_t acc = rest + static_cast<int64_t>(c1) * d1 + static_cast<int64_t>(c0) * d0;
        int64_t v[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            v[j] = acc;
            acc += d0;
            if (++c0 == e0) {
                c0 = 0;
                acc += d1 - wrap0;
                if (++c1 == e1 && bounded1) {
                    c1 = 0;
                    rest = rest_of(++q1);
                    acc = rest;
                }
            }
        }
        int64_t* o = out + g * G;
        if constexpr (kWide) {
            st_cs_v4(o, v[0], v[1], v[2], v[3]);
            st_cs_v4(o + 4, v[4], v[5], v[6], v[7]);
        } else {
#pragma unroll
            for (int j = 0; j < G; ++j) o[j] = v[j];
        }
    }
}

// Warp-coalesced grouped evaluation: a warp owns 32 consecutive groups of G indices (32*G outputs, 256*G bytes).
// Lane l peels group l ONCE; the bases then travel by shuffle so that store j of the warp covers the 128
// consecutive outputs [j*128, j*128+128): lane l writes outputs j*128 + 4l .. +3 (one 32-byte sector per lane,
// 1 KiB contiguous per STG.256 instruction -> 8 full 128-byte lines instead of 32 partial ones). The in-group
// offsets (4l mod G) + k of a lane do not depend on j, so their stride products / carry-less products are
// computed once per thread.
template <int G, bool kPow2U32>
__global__ void __launch_bounds__(kThreads) eval_warp_kernel(const __grid_constant__ tlb_layout_desc L, uint64_t i0,
                                                             uint64_t n_super, int64_t* __restrict__ out) {
    static_assert(G >= 4 && G <= 32 && (G & (G - 1)) == 0, "G in {4,8,16,32}");
    constexpr int kStores = G / 4;        // STG.256 per lane per superblock
    constexpr int kLanesPerGroup = G / 4; // lanes that share one group inside a store
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint64_t warp0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const bool is_xor = L.kind == TLB_KIND_XOR;
    const int64_t d0 = L.stride[0];
    const uint32_t sub = (static_cast<uint32_t>(lane) * 4u) & (G - 1);
    int64_t off[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        off[k] = is_xor ? static_cast<int64_t>(dev_clmul(sub + k, static_cast<uint64_t>(d0))) : static_cast<int64_t>(sub + k) * d0;
    const int src0 = lane / kLanesPerGroup;
    for (uint64_t sb = warp0; sb < n_super; sb += warps) {
        const uint64_t i = i0 + (sb * 32 + lane) * G;
        const int64_t base = kPow2U32 ? dev_eval_pow2_u32(L, static_cast<uint32_t>(i)) : dev_eval(L, i);
        int64_t* o = out + sb * (32 * G) + lane * 4;
#pragma unroll
        for (int j = 0; j < kStores; ++j) {
            const int64_t b = __shfl_sync(0xffffffffu, base, j * (128 / G) + src0);
            if (is_xor) st_cs_v4(o + j * 128, b ^ off[0], b ^ off[1], b ^ off[2], b ^ off[3]);
            else st_cs_v4(o + j * 128, b + off[0], b + off[1], b + off[2], b + off[3]);
        }
    }
}

// out[k*nm + r] = natural coordinate leaf r of i0+k (idx2crd, int_tuple.hpp:129). NM = 2 / 4 leaves: the whole
// coordinate of one index is 16 / 32 contiguous bytes and leaves as ONE vector store (a loop of 8-byte stores writes
// a quarter of every 32-byte sector per instruction: 1.9 TB/s against 6+ TB/s); NM = 0 is the general loop.
template <int NM>
__global__ void __launch_bounds__(kThreads) idx2crd_kernel(const __grid_constant__ tlb_layout_desc S, uint64_t i0,
                                                           uint64_t n, int64_t* __restrict__ out) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const int nm = NM ? NM : S.n_modes;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        uint64_t i = i0 + k;
        int64_t* o = out + k * nm;
        if constexpr (NM == 0) {
            for (int r = 0; r < nm; ++r) {
                if (r + 1 < nm) {
                    const uint64_t q = dev_div(S, r, i);
                    o[r] = static_cast<int64_t>(i - q * static_cast<uint64_t>(S.extent[r]));
                    i = q;
                } else {
                    o[r] = static_cast<int64_t>(i);
                }
            }
        } else {
            int64_t c[NM];
#pragma unroll
            for (int r = 0; r < NM; ++r) {
                if (r + 1 < NM) {
                    const uint64_t q = dev_div(S, r, i);
                    c[r] = static_cast<int64_t>(i - q * static_cast<uint64_t>(S.extent[r]));
                    i = q;
                } else {
                    c[r] = static_cast<int64_t>(i);
                }
            }
            if constexpr (NM == 2) st_cs_v2(o, c[0], c[1]);
            else st_cs_v4(o, c[0], c[1], c[2], c[3]);
        }
    }
}

// out[k] = sum_r crd[k*nm + r] * prod_{q<r} extent[q]  (crd2idx, int_tuple.hpp:148-158). The reference accepts any
// coordinate VALUES (only the tree shape is validated, which the flat [n][n_modes] input fixes by construction) and
// detects wrapping through checked_mul / checked_add (common.hpp:99-109); so does this kernel: a wrapped element
// is not written and *d_status (when given) becomes TLB_ERR_OVERFLOW. The prefix products themselves are proven to
// fit on the host (the lowering rejects shapes whose size overflows).
// NM > 0: the coordinate vectors have NM (even) entries and are read with 16-byte streaming loads (a thread's NM int64
// are contiguous: scalar loads would touch every 32-byte sector NM / 4 times per warp instruction); NM == 0: any length.
template <int NM>
__global__ void __launch_bounds__(kThreads) crd2idx_kernel(const __grid_constant__ tlb_layout_desc S,
                                                           const int64_t* __restrict__ crd, uint64_t n,
                                                           int64_t* __restrict__ out, int* d_status) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const int nm = NM > 0 ? NM : S.n_modes;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        const int64_t* c = crd + k * nm;
        int64_t idx = 0, scale = 1;
        bool ovf = false;
        auto step = [&](int r, int64_t x) {
            const int64_t lo = static_cast<int64_t>(static_cast<uint64_t>(x) * static_cast<uint64_t>(scale));
            ovf |= __mul64hi(x, scale) != (lo >> 63);
            const int64_t sum = static_cast<int64_t>(static_cast<uint64_t>(idx) + static_cast<uint64_t>(lo));
            ovf |= ((idx ^ sum) & (lo ^ sum)) < 0;
            idx = sum;
            scale *= S.extent[r];
        };
        if constexpr (NM > 0) {
            int64_t x[NM];
#pragma unroll
            for (int r = 0; r < NM; r += 2)
                asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0, %1}, [%2];" : "=l"(x[r]), "=l"(x[r + 1]) : "l"(c + r));
#pragma unroll
            for (int r = 0; r < NM; ++r) step(r, x[r]);
        } else {
            for (int r = 0; r < nm; ++r) step(r, c[r]);
        }
        if (ovf) {
            if (d_status) atomicExch(d_status, TLB_ERR_OVERFLOW);
        } else {
            out[k] = idx;
        }
    }
}

__device__ __forceinline__ void block_count(unsigned long long bad, unsigned long long* d_mismatch) {
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    __shared__ unsigned long long warp_bad[kThreads / 32];
    if ((threadIdx.x & 31) == 0) warp_bad[threadIdx.x >> 5] = bad;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < kThreads / 32; ++w) s += warp_bad[w];
        if (s) atomicAdd(d_mismatch, s);
    }
}

// The peel for Int layouts whose extents are all powers of two, on an index below 2^32: masks and shifts in 32 bits (the
// checkers are compute bound: the generic peel spends most of its instructions on 64-bit division by multiplication).
// NL: an upper bound on the leaf count the loop is unrolled for (4: the C5 layouts; the masks, shifts and strides then
// stay in registers across a thread's grid-stride iterations), TLB_MAX_MODES: any count.
template <int NL> __device__ __forceinline__ int64_t dev_eval_p2(const tlb_layout_desc& L, uint32_t i) {
    int64_t acc = 0;
    const int n = L.n_modes;
#pragma unroll
    for (int r = 0; r < NL; ++r) {
        if (r < n) {
            const uint32_t c = (r + 1 < n) ? (i & (static_cast<uint32_t>(L.extent[r]) - 1u)) : i;
            i = (r + 1 < n) ? (i >> L.log2e[r]) : 0u;
            acc += static_cast<int64_t>(c) * L.stride[r];
        }
    }
    return acc;
}
// FAST > 0: every layout is Int with power-of-two extents (each below 2^32), at most FAST leaves, and the index range
// ends below 2^32; an intermediate offset at or above 2^32 (or negative) takes the generic peel.
template <int FAST> __device__ __forceinline__ int64_t dev_eval_sel(const tlb_layout_desc& L, uint64_t i) {
    if constexpr (FAST > 0) {
        if ((i >> 32) == 0) return dev_eval_p2<FAST>(L, static_cast<uint32_t>(i));
    }
    return dev_eval(L, i);
}

// Counts k with L(R(k)) != k.
template <int FAST>
__global__ void __launch_bounds__(kThreads) rinv_check_kernel(const __grid_constant__ tlb_layout_desc L,
                                                              const __grid_constant__ tlb_layout_desc R, uint64_t k0,
                                                              uint64_t n, unsigned long long* d_mismatch) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long bad = 0;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
        const uint64_t k = k0 + j;
        const int64_t rk = dev_eval_sel<FAST>(R, k);
        const int64_t back = rk < 0 ? -1 : dev_eval_sel<FAST>(L, static_cast<uint64_t>(rk));
        bad += (back != static_cast<int64_t>(k));
    }
    block_count(bad, d_mismatch);
}

// Counts i with A(B(i)) != Rr(i).
template <int FAST>
__global__ void __launch_bounds__(kThreads) compose_check_kernel(const __grid_constant__ tlb_layout_desc A,
                                                                 const __grid_constant__ tlb_layout_desc B,
                                                                 const __grid_constant__ tlb_layout_desc Rr,
                                                                 uint64_t i0, uint64_t n,
                                                                 unsigned long long* d_mismatch) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long bad = 0;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
        const uint64_t i = i0 + j;
        const int64_t b = dev_eval_sel<FAST>(B, i);
        const int64_t want = b < 0 ? INT64_MIN : dev_eval_sel<FAST>(A, static_cast<uint64_t>(b));
        bad += (want != dev_eval_sel<FAST>(Rr, i));
    }
    block_count(bad, d_mismatch);
}

struct AxesModes {
    int32_t n_modes;
    int32_t n_axes;
    int64_t extent[TLB_MAX_MODES];
    int64_t scale[TLB_MAX_MODES];
    int32_t axis[TLB_MAX_MODES]; // -1 for Int(0) leaves
};

// Per-axis offsets of a coordinate (Basis) layout (layout_eval_axes, layout.hpp:103). NA = 1..4 axes (the TMA
// coordinate tensors of rank <= 4): accumulators in registers, one vector store per index. NA = 0: any axis count,
// accumulating in the output cells.
template <int NA>
__global__ void __launch_bounds__(kThreads) eval_axes_kernel(const __grid_constant__ AxesModes M, uint64_t i0,
                                                             uint64_t n, int64_t* __restrict__ out) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
        uint64_t i = i0 + k;
        int64_t* o = out + k * M.n_axes;
        int64_t acc[NA ? NA : 1];
        if constexpr (NA == 0) {
            for (int a = 0; a < M.n_axes; ++a) o[a] = 0;
        } else {
#pragma unroll
            for (int a = 0; a < NA; ++a) acc[a] = 0;
        }
        for (int r = 0; r < M.n_modes; ++r) {
            uint64_t c;
            if (r + 1 < M.n_modes) {
                const uint64_t e = static_cast<uint64_t>(M.extent[r]);
                if ((e & (e - 1)) == 0) {
                    c = i & (e - 1);
                    i >>= __ffsll(static_cast<long long>(e)) - 1;
                } else {
                    c = i % e;
                    i /= e;
                }
            } else {
                c = i;
            }
            const int64_t v = static_cast<int64_t>(c) * M.scale[r];
            if constexpr (NA == 0) {
                if (M.axis[r] >= 0) o[M.axis[r]] += v;
            } else {
#pragma unroll
                for (int a = 0; a < NA; ++a) acc[a] += (M.axis[r] == a) ? v : 0;
            }
        }
        if constexpr (NA == 1) o[0] = acc[0];
        else if constexpr (NA == 2) st_cs_v2(o, acc[0], acc[1]);
        else if constexpr (NA == 3) { o[0] = acc[0]; o[1] = acc[1]; o[2] = acc[2]; }
        else if constexpr (NA == 4) st_cs_v4(o, acc[0], acc[1], acc[2], acc[3]);
    }
}

int grid_for(uint64_t work_items) {
    // a few resident waves of 148 SMs x (2048/kThreads) CTAs, never more CTAs than work
    const uint64_t per_wave = static_cast<uint64_t>(sm_count()) * (2048 / kThreads);
    uint64_t blocks = (work_items + kThreads - 1) / kThreads;
    blocks = std::min<uint64_t>(blocks, per_wave * 4);
    return static_cast<int>(std::max<uint64_t>(blocks, 1));
}

// TLB_EVAL_NO_WARP=1 keeps the per-thread grouped kernel only (A/B comparisons of the store pattern).
bool eval_no_warp() { return knob(K_EVAL_NO_WARP) == 1; }

int check_int_or_xor(const tlb_layout_desc* L, const char* who) {
    if (!L) return fail(TLB_ERR_CONTRACT, std::string(who) + ": null layout");
    if (L->kind == TLB_KIND_BASIS) return fail(TLB_ERR_SEMIMODULE, "not an integer stride");
    return TLB_OK;
}

} // namespace
} // namespace tlb

using namespace tlb;

extern "C" {

int tlb_eval_range(const tlb_layout_desc* layout, uint64_t i0, uint64_t n, int64_t* d_out, void* stream) {
    TLB_TRY(check_int_or_xor(layout, "tlb_eval_range"));
    if (n == 0) return TLB_OK;
    if (!d_out) return fail(TLB_ERR_CONTRACT, "tlb_eval_range: null output");
    if (i0 + n < i0 || (i0 + n - 1) >> 63) return fail(TLB_ERR_OVERFLOW, "index range exceeds int64");
    TLB_TRY(require_device());
    TLB_TRY(overflow_preflight(*layout, 0, i0 + n - 1));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool aligned = (reinterpret_cast<uintptr_t>(d_out) & 15) == 0;
    // grouped fast path: the first leaf must absorb a whole group
    int G = 1;
    if (aligned) {
        for (int g = 32; g >= 2; g >>= 1)
            if (i0 % g == 0 && (layout->n_modes == 1 || layout->extent[0] % g == 0) && n >= static_cast<uint64_t>(g) * 1024) {
                G = g;
                break;
            }
        if (G == 1)
            for (int g = 8; g >= 2; g >>= 1)
                if (i0 % g == 0 && (layout->n_modes == 1 || layout->extent[0] % g == 0) && n >= static_cast<uint64_t>(g)) {
                    G = g;
                    break;
                }
    }
    if (G > 1) {
        const uint64_t groups = n / G;
        const bool wide = (reinterpret_cast<uintptr_t>(d_out) & 31) == 0;
        const bool p32 = (layout->flags & TLB_LF_ALL_POW2) && (i0 + n - 1) < (1ull << 32);
        // Warp-coalesced kernel first (whole superblocks of 32 groups), the per-thread kernel on what is left.
        uint64_t groups_done = 0;
        if (wide && G >= 4 && groups >= 32 && !eval_no_warp()) {
            const uint64_t n_super = groups / 32;
            // one superblock per warp: a grid-stride loop over a few waves leaves a ragged last pass (6 or 7
            // superblocks per warp on C5: 7.03 TB/s against 7.34 TB/s with exactly one each)
            const int gw = static_cast<int>(std::min<uint64_t>((n_super + kThreads / 32 - 1) / (kThreads / 32), 1u << 22));
#define TLB_EVAL_W(GG)                                                                                   \
    do {                                                                                                 \
        if (p32) TLB_CUDA(launch_pdl(eval_warp_kernel<GG, true>, dim3(gw), dim3(kThreads), 0, s, *layout, i0, n_super, d_out)); \
        else TLB_CUDA(launch_pdl(eval_warp_kernel<GG, false>, dim3(gw), dim3(kThreads), 0, s, *layout, i0, n_super, d_out));   \
    } while (0)
            switch (G) {
            case 32: TLB_EVAL_W(32); break;
            case 16: TLB_EVAL_W(16); break;
            case 8: TLB_EVAL_W(8); break;
            default: TLB_EVAL_W(4); break;
            }
#undef TLB_EVAL_W
            count_launch();
            TLB_CUDA(cudaGetLastError());
            groups_done = n_super * 32;
            set_plan(G == 32 ? "eval_warp32" : G == 16 ? "eval_warp16" : G == 8 ? "eval_warp8" : "eval_warp4");
        } else {
            set_plan(G == 32 ? "eval_group32" : G == 16 ? "eval_group16" : G == 8 ? "eval_group8" : G == 4 ? "eval_group4" : "eval_group2");
        }
        const uint64_t groups_left = groups - groups_done;
        const uint64_t i0g = i0 + groups_done * G;
        int64_t* outg = d_out + groups_done * G;
        const int grid = grid_for(groups_left);
#define TLB_EVAL_G(GG)                                                                                          \
    do {                                                                                                        \
        if (p32 && wide) eval_group_kernel<GG, true, true><<<grid, kThreads, 0, s>>>(*layout, i0g, groups_left, outg);   \
        else if (p32) eval_group_kernel<GG, true, false><<<grid, kThreads, 0, s>>>(*layout, i0g, groups_left, outg);     \
        else if (wide) eval_group_kernel<GG, false, true><<<grid, kThreads, 0, s>>>(*layout, i0g, groups_left, outg);    \
        else eval_group_kernel<GG, false, false><<<grid, kThreads, 0, s>>>(*layout, i0g, groups_left, outg);             \
    } while (0)
        if (groups_left) switch (G) {
        case 32: TLB_EVAL_G(32); break;
        case 16: TLB_EVAL_G(16); break;
        case 8: TLB_EVAL_G(8); break;
        case 4: TLB_EVAL_G(4); break;
        default: TLB_EVAL_G(2); break;
        }
#undef TLB_EVAL_G
        if (groups_left) {
            count_launch();
            TLB_CUDA(cudaGetLastError());
        }
        const uint64_t done = groups * G;
        if (done < n) {
            eval_range_kernel<false><<<grid_for(n - done), kThreads, 0, s>>>(*layout, i0 + done, n - done, d_out + done);
            count_launch();
            TLB_CUDA(cudaGetLastError());
        }
        return TLB_OK;
    }
    if (layout->kind == TLB_KIND_INT && layout->n_modes >= 2 && n >= 8 && knob(K_EVAL_ODOMETER) != 0) {
        // no group size divides the leading leaf: 8 indices per thread by odometer over leaves 0 and 1
        const uint64_t groups = n / 8;
        const bool wide = (reinterpret_cast<uintptr_t>(d_out) & 31) == 0;
        if (wide) TLB_CUDA(launch_pdl(eval_odo_kernel<true>, dim3(grid_for(groups)), dim3(kThreads), 0, s, *layout, i0, groups, d_out));
        else TLB_CUDA(launch_pdl(eval_odo_kernel<false>, dim3(grid_for(groups)), dim3(kThreads), 0, s, *layout, i0, groups, d_out));
        count_launch();
        if (groups * 8 < n) {
            eval_range_kernel<false><<<grid_for(n - groups * 8), kThreads, 0, s>>>(*layout, i0 + groups * 8, n - groups * 8, d_out + groups * 8);
            count_launch();
            TLB_CUDA(cudaGetLastError());
        }
        set_plan("eval_odo");
        return TLB_OK;
    }
    set_plan("eval_scalar");
    const bool pairs = aligned && n >= 2;
    if (pairs) eval_range_kernel<true><<<grid_for(n >> 1), kThreads, 0, s>>>(*layout, i0, n, d_out);
    else eval_range_kernel<false><<<grid_for(n), kThreads, 0, s>>>(*layout, i0, n, d_out);
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

int tlb_idx2crd_range(const tlb_layout_desc* shape, uint64_t i0, uint64_t n, int64_t* d_out, void* stream) {
    if (!shape) return fail(TLB_ERR_CONTRACT, "tlb_idx2crd_range: null shape");
    if (n == 0) return TLB_OK;
    if (!d_out) return fail(TLB_ERR_CONTRACT, "tlb_idx2crd_range: null output");
    if (i0 + n < i0 || (i0 + n - 1) >> 63) return fail(TLB_ERR_OVERFLOW, "index range exceeds int64");
    TLB_TRY(require_device());
    {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const uintptr_t al = reinterpret_cast<uintptr_t>(d_out);
        // one CTA pass per element block (no ragged grid-stride tail), vector stores when the coordinate is 16 / 32 bytes
        const int grid = static_cast<int>(std::min<uint64_t>((n + kThreads - 1) / kThreads, 1u << 22));
        if (shape->n_modes == 4 && (al & 31) == 0) idx2crd_kernel<4><<<grid, kThreads, 0, st>>>(*shape, i0, n, d_out);
        else if (shape->n_modes == 2 && (al & 15) == 0) idx2crd_kernel<2><<<grid, kThreads, 0, st>>>(*shape, i0, n, d_out);
        else idx2crd_kernel<0><<<grid_for(n), kThreads, 0, st>>>(*shape, i0, n, d_out);
    }
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

int tlb_crd2idx_range_checked(const tlb_layout_desc* shape, const int64_t* d_crd, uint64_t n, int64_t* d_out,
                              int32_t* d_status, void* stream) {
    if (!shape) return fail(TLB_ERR_CONTRACT, "tlb_crd2idx_range: null shape");
    if (n == 0) return TLB_OK;
    if (!d_crd || !d_out) return fail(TLB_ERR_CONTRACT, "tlb_crd2idx_range: null buffer");
    // scale = checked_mul(scale, size(mode)) runs for every mode, the last included (int_tuple.hpp:155): the
    // lowering has already proven that the full product fits (shape->size), so no prefix product can wrap.
    if (shape->size < 1) return fail(TLB_ERR_OVERFLOW, "integer overflow in multiplication");
    TLB_TRY(require_device());
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const bool al16 = (reinterpret_cast<uintptr_t>(d_crd) & 15) == 0;
    if (al16 && shape->n_modes == 2) crd2idx_kernel<2><<<grid_for(n), kThreads, 0, cs>>>(*shape, d_crd, n, d_out, d_status);
    else if (al16 && shape->n_modes == 4) crd2idx_kernel<4><<<grid_for(n), kThreads, 0, cs>>>(*shape, d_crd, n, d_out, d_status);
    else if (al16 && shape->n_modes == 6) crd2idx_kernel<6><<<grid_for(n), kThreads, 0, cs>>>(*shape, d_crd, n, d_out, d_status);
    else if (al16 && shape->n_modes == 8) crd2idx_kernel<8><<<grid_for(n), kThreads, 0, cs>>>(*shape, d_crd, n, d_out, d_status);
    else crd2idx_kernel<0><<<grid_for(n), kThreads, 0, cs>>>(*shape, d_crd, n, d_out, d_status);
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

int tlb_crd2idx_range(const tlb_layout_desc* shape, const int64_t* d_crd, uint64_t n, int64_t* d_out, void* stream) {
    return tlb_crd2idx_range_checked(shape, d_crd, n, d_out, nullptr, stream);
}

namespace {
// Int layout, every extent a power of two below 2^32 (the last leaf's coordinate is unbounded: it is never masked).
bool pow2_fast(const tlb_layout_desc& L) {
    if (L.kind != TLB_KIND_INT || !(L.flags & TLB_LF_ALL_POW2)) return false;
    for (int r = 0; r < L.n_modes; ++r)
        if (L.extent[r] >= (1ll << 32)) return false;
    return true;
}
} // namespace

int tlb_rinv_check_range(const tlb_layout_desc* L, const tlb_layout_desc* R, uint64_t k0, uint64_t n,
                         unsigned long long* d_mismatch, void* stream) {
    TLB_TRY(check_int_or_xor(L, "tlb_rinv_check_range"));
    TLB_TRY(check_int_or_xor(R, "tlb_rinv_check_range"));
    if (n == 0) return TLB_OK;
    if (!d_mismatch) return fail(TLB_ERR_CONTRACT, "tlb_rinv_check_range: null counter");
    if (k0 + n < k0 || (k0 + n - 1) >> 63) return fail(TLB_ERR_OVERFLOW, "index range exceeds int64");
    TLB_TRY(require_device());
    TLB_TRY(overflow_preflight(*R, 0, k0 + n - 1));
    // L is evaluated at R(k), and k may lie in R's extended domain: bound |R(k)| over [0, k0 + n)
    TLB_TRY(overflow_preflight(*L, 0, max_abs_offset(*R, k0 + n - 1)));
    const bool fast = pow2_fast(*L) && pow2_fast(*R) && k0 + n <= (1ull << 32);
    if (fast && L->n_modes <= 4 && R->n_modes <= 4)
        rinv_check_kernel<4><<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*L, *R, k0, n, d_mismatch);
    else if (fast)
        rinv_check_kernel<TLB_MAX_MODES><<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*L, *R, k0, n, d_mismatch);
    else
        rinv_check_kernel<0><<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*L, *R, k0, n, d_mismatch);
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

int tlb_compose_check_range(const tlb_layout_desc* A, const tlb_layout_desc* B, const tlb_layout_desc* R,
                            uint64_t i0, uint64_t n, unsigned long long* d_mismatch, void* stream) {
    TLB_TRY(check_int_or_xor(A, "tlb_compose_check_range"));
    TLB_TRY(check_int_or_xor(B, "tlb_compose_check_range"));
    TLB_TRY(check_int_or_xor(R, "tlb_compose_check_range"));
    if (B->kind != TLB_KIND_INT) return fail(TLB_ERR_SEMIMODULE, "xor strides are not admissible on the right of composition");
    if (n == 0) return TLB_OK;
    if (!d_mismatch) return fail(TLB_ERR_CONTRACT, "tlb_compose_check_range: null counter");
    if (i0 + n < i0 || (i0 + n - 1) >> 63) return fail(TLB_ERR_OVERFLOW, "index range exceeds int64");
    TLB_TRY(require_device());
    TLB_TRY(overflow_preflight(*B, 0, i0 + n - 1));
    TLB_TRY(overflow_preflight(*R, 0, i0 + n - 1));
    TLB_TRY(overflow_preflight(*A, 0, max_abs_offset(*B, i0 + n - 1)));
    const bool fast = pow2_fast(*A) && pow2_fast(*B) && pow2_fast(*R) && i0 + n <= (1ull << 32);
    if (fast && A->n_modes <= 4 && B->n_modes <= 4 && R->n_modes <= 4)
        compose_check_kernel<4><<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*A, *B, *R, i0, n, d_mismatch);
    else if (fast)
        compose_check_kernel<TLB_MAX_MODES><<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*A, *B, *R, i0, n, d_mismatch);
    else
        compose_check_kernel<0><<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*A, *B, *R, i0, n, d_mismatch);
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

int tlb_compose_check(const tlb_layout_desc* A, const tlb_layout_desc* B, const tlb_layout_desc* R, uint64_t* mismatches,
                      void* stream) {
    if (!A || !B || !R || !mismatches) return fail(TLB_ERR_CONTRACT, "tlb_compose_check: null argument");
    *mismatches = 0;
    if (B->size != R->size) return fail(TLB_ERR_CONTRACT, "tlb_compose_check: size(B) != size(R)");
    TLB_TRY(require_device());
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long* d = nullptr;
    unsigned long long h = 0;
    TLB_CUDA(ws_malloc(reinterpret_cast<void**>(&d), sizeof(h), s));
    cudaError_t e = cudaMemsetAsync(d, 0, sizeof(h), s);
    int st = TLB_OK;
    if (e == cudaSuccess) st = tlb_compose_check_range(A, B, R, 0, static_cast<uint64_t>(B->size), d, stream);
    if (e == cudaSuccess && st == TLB_OK) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && st == TLB_OK) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d, s);
    TLB_CUDA(e);
    *mismatches = h;
    return st;
}

int tlb_eval_axes_range(const tlb_mode* modes, int n_modes, int n_axes, uint64_t i0, uint64_t n, int64_t* d_out,
                        void* stream) {
    if (!modes || n_modes < 1 || n_modes > TLB_MAX_MODES) return fail(TLB_ERR_CONTRACT, "tlb_eval_axes_range: bad modes");
    if (n_axes < 1 || n_axes > TLB_MAX_MODES) return fail(TLB_ERR_CONTRACT, "tlb_eval_axes_range: bad axis count");
    AxesModes M{};
    M.n_modes = n_modes;
    M.n_axes = n_axes;
    for (int r = 0; r < n_modes; ++r) {
        if (modes[r].extent < 1) return fail(TLB_ERR_STRUCTURAL, "shape leaves must be positive");
        M.extent[r] = modes[r].extent;
        if (modes[r].kind == TLB_KIND_BASIS) {
            if (modes[r].axis < 0 || modes[r].axis >= n_axes) return fail(TLB_ERR_CONTRACT, "basis axis out of range");
            M.axis[r] = modes[r].axis;
            M.scale[r] = modes[r].stride;
        } else if (modes[r].kind == TLB_KIND_INT && modes[r].stride == 0) {
            M.axis[r] = -1;
        } else {
            return fail(TLB_ERR_SEMIMODULE, "per-axis evaluation requires coordinate strides");
        }
    }
    if (n == 0) return TLB_OK;
    if (!d_out) return fail(TLB_ERR_CONTRACT, "tlb_eval_axes_range: null output");
    if (i0 + n < i0 || (i0 + n - 1) >> 63) return fail(TLB_ERR_OVERFLOW, "index range exceeds int64");
    {
        // checked_mul / checked_add of layout_eval_axes (stride.hpp:152, layout.hpp:92): prove per axis that the sum of
        // the largest leaf contributions over [0, i0 + n) fits in int64 (the last leaf is unbounded)
        unsigned __int128 per_axis[TLB_MAX_MODES] = {};
        uint64_t rest = i0 + n - 1;
        for (int r = 0; r < n_modes; ++r) {
            const uint64_t e = static_cast<uint64_t>(M.extent[r]);
            const uint64_t cmax = (r + 1 < n_modes) ? std::min<uint64_t>(rest, e - 1) : rest;
            rest /= e;
            if (M.axis[r] < 0) continue;
            const uint64_t a = M.scale[r] < 0 ? 0 - static_cast<uint64_t>(M.scale[r]) : static_cast<uint64_t>(M.scale[r]);
            per_axis[M.axis[r]] += static_cast<unsigned __int128>(cmax) * a;
            if (per_axis[M.axis[r]] >> 63) return fail(TLB_ERR_OVERFLOW, "integer overflow in layout evaluation");
        }
    }
    TLB_TRY(require_device());
    {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const uintptr_t al = reinterpret_cast<uintptr_t>(d_out);
        const int grid = static_cast<int>(std::min<uint64_t>((n + kThreads - 1) / kThreads, 1u << 22));
        if (n_axes == 1) eval_axes_kernel<1><<<grid, kThreads, 0, st>>>(M, i0, n, d_out);
        else if (n_axes == 2 && (al & 15) == 0) eval_axes_kernel<2><<<grid, kThreads, 0, st>>>(M, i0, n, d_out);
        else if (n_axes == 3) eval_axes_kernel<3><<<grid, kThreads, 0, st>>>(M, i0, n, d_out);
        else if (n_axes == 4 && (al & 31) == 0) eval_axes_kernel<4><<<grid, kThreads, 0, st>>>(M, i0, n, d_out);
        else eval_axes_kernel<0><<<grid_for(n), kThreads, 0, st>>>(M, i0, n, d_out);
    }
    count_launch();
    TLB_CUDA(cudaGetLastError());
    return TLB_OK;
}

} // extern "C"

// tla::gemm(A, B, C) (tensor.hpp:214-233): contract checks, plan selection, and the
// layout-evaluating SIMT kernels that serve every layout family the tcgen05 path does not
// (NT, NTT, BLIS strides, GETT folded modes, Xor strides) as well as the reference's own
// checked-int64 value type.
//
//   C(m,n) += sum_k A(m,k) * B(n,k)     all tensors rank 2, modes addressed by 1-D coordinates
//
// The SIMT kernels keep the reference's summation order (k ascending, accumulator starts
// from C), so for bf16 they are bit-exact against the sequential fp32 restatement
// (bf16 x bf16 is exact in fp32, hence fma(a, b, acc) == acc + a*b).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "tlb_internal.h"
#include "tlb_gemm.h"

namespace tlb {
namespace {

thread_local int g_gemm_path = 0; // 0 auto, 1 SIMT, 2 tcgen05 cta_group::1, 3 tcgen05 cta_group::2
thread_local const tlb_gemm_tiler* g_tiler = nullptr; // set for the duration of a tlb_gemm_*_tiled call

constexpr int kThreads = 256;

// TLB_GEMM_SPLIT_TAIL=0 keeps every C cell owned by one CTA (bitwise run-to-run reproducible sums).
bool split_tail_enabled() { return knob(K_GEMM_SPLIT_TAIL) != 0; }

struct SimtArgs {
    int64_t a_origin, b_origin, c_origin;
    int64_t a_bs, b_bs, c_bs; // batch strides (elements)
    int64_t M, N, K;
    TileGrid grid;
    uint32_t tile_begin, tile_end; // global tile ids (batch-major)
    int32_t batch_begin, batch_end;
    int32_t ab_f16; // 2-byte operands are fp16 instead of bf16
    int32_t c_16;   // C cells have the operands' 2-byte type
    int32_t swapped; // tile ids refer to the TRANSPOSED problem (the tcgen05 plans run m-contiguous C as C^T): tile_of(n, m)
};

__device__ __forceinline__ int64_t combine(int kind, int64_t a, int64_t b) { return kind == TLB_KIND_XOR ? (a ^ b) : (a + b); }

template <bool kI64>
__global__ void __launch_bounds__(kThreads)
gemm_simt_kernel(const __grid_constant__ tlb_layout_desc LA, const __grid_constant__ tlb_layout_desc LB,
                 const __grid_constant__ tlb_layout_desc LC, const void* __restrict__ A, const void* __restrict__ B,
                 void* C, const __grid_constant__ SimtArgs p, int* d_status) {
    const uint64_t per_batch = static_cast<uint64_t>(p.M) * static_cast<uint64_t>(p.N);
    const uint64_t total = per_batch * static_cast<uint64_t>(p.batch_end - p.batch_begin);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint32_t tpb = tiles_per_batch(p.grid);
    for (uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const int64_t batch = p.batch_begin + static_cast<int64_t>(idx / per_batch);
        const uint64_t e = idx % per_batch;
        const int64_t m = static_cast<int64_t>(e % static_cast<uint64_t>(p.M));
        const int64_t n = static_cast<int64_t>(e / static_cast<uint64_t>(p.M));
        const uint64_t tile = static_cast<uint64_t>(batch) * tpb + (p.swapped ? tile_of(p.grid, n, m) : tile_of(p.grid, m, n));
        if (tile < p.tile_begin || tile >= p.tile_end) continue;
        const int64_t a_m = dev_eval_top(LA, 0, m), b_n = dev_eval_top(LB, 0, n);
        const int64_t cp = dev_position(LC, p.c_origin, combine(LC.kind, dev_eval_top(LC, 0, m), dev_eval_top(LC, 1, n))) +
                           batch * p.c_bs;
        if constexpr (kI64) {
            const int64_t* a = static_cast<const int64_t*>(A) + batch * p.a_bs;
            const int64_t* b = static_cast<const int64_t*>(B) + batch * p.b_bs;
            int64_t* c = static_cast<int64_t*>(C);
            int64_t acc = c[cp];
            bool ovf = false;
            for (int64_t k = 0; k < p.K; ++k) {
                const int64_t x = a[dev_position(LA, p.a_origin, combine(LA.kind, a_m, dev_eval_top(LA, 1, k)))];
                const int64_t y = b[dev_position(LB, p.b_origin, combine(LB.kind, b_n, dev_eval_top(LB, 1, k)))];
                // checked_mul / checked_add (common.hpp:99-109)
                const int64_t lo = static_cast<int64_t>(static_cast<uint64_t>(x) * static_cast<uint64_t>(y));
                const int64_t hi = __mul64hi(x, y);
                if (hi != (lo >> 63)) { ovf = true; break; }
                const int64_t s = static_cast<int64_t>(static_cast<uint64_t>(acc) + static_cast<uint64_t>(lo));
                if (((acc ^ s) & (lo ^ s)) < 0) { ovf = true; break; }
                acc = s;
            }
            if (ovf) {
                if (d_status) atomicExch(d_status, TLB_ERR_OVERFLOW);
            } else {
                c[cp] = acc;
            }
        } else {
            const uint16_t* a = static_cast<const uint16_t*>(A) + batch * p.a_bs;
            const uint16_t* b = static_cast<const uint16_t*>(B) + batch * p.b_bs;
            float* c = static_cast<float*>(C);
            uint16_t* c16 = static_cast<uint16_t*>(C);
            float acc;
            if (p.c_16) acc = p.ab_f16 ? __half2float(__ushort_as_half(c16[cp])) : __uint_as_float(static_cast<uint32_t>(c16[cp]) << 16);
            else acc = c[cp];
            // bf16 x bf16 and fp16 x fp16 products are exact in fp32, so fma(x, y, acc) == acc + x * y
            for (int64_t k = 0; k < p.K; ++k) {
                const uint16_t xb = a[dev_position(LA, p.a_origin, combine(LA.kind, a_m, dev_eval_top(LA, 1, k)))];
                const uint16_t yb = b[dev_position(LB, p.b_origin, combine(LB.kind, b_n, dev_eval_top(LB, 1, k)))];
                const float x = p.ab_f16 ? __half2float(__ushort_as_half(xb)) : __uint_as_float(static_cast<uint32_t>(xb) << 16);
                const float y = p.ab_f16 ? __half2float(__ushort_as_half(yb)) : __uint_as_float(static_cast<uint32_t>(yb) << 16);
                acc = __fmaf_rn(x, y, acc);
            }
            if (p.c_16) c16[cp] = p.ab_f16 ? __half_as_ushort(__float2half_rn(acc)) : __bfloat16_as_ushort(__float2bfloat16_rn(acc));
            else c[cp] = acc;
        }
    }
}

// ---- tiled SIMT plan for 2-byte operands --------------------------------------------------------------------------------
// Every layout family the tcgen05 plans do not take (BLIS strides, Xor strides, strides TMA cannot address, folded modes
// whose tiles straddle leaves): the offset of A(m, k) is f(m) (+|^) g(k) with f and g the evaluations of the two top-level
// modes, so a CTA evaluates the layouts ONCE per row / column / k of its tile (offset tables in shared memory) instead of
// twice per MAC, stages 64 x 16 and 64 x 16 operand tiles as fp32 in shared memory, and every thread accumulates a 4 x 4
// block of C with k ascending: the reference's summation order (tensor.hpp:223-231), hence bit-exact against the
// sequential fp32 restatement (products of bf16 / fp16 pairs are exact in fp32).
constexpr int TS_M = 64, TS_N = 64, TS_K = 16;

__global__ void __launch_bounds__(kThreads)
gemm_simt_tiled_kernel(const __grid_constant__ tlb_layout_desc LA, const __grid_constant__ tlb_layout_desc LB,
                       const __grid_constant__ tlb_layout_desc LC, const uint16_t* __restrict__ A, const uint16_t* __restrict__ B,
                       void* C, const __grid_constant__ SimtArgs p, int a_k_fast, int b_k_fast) {
    __shared__ __align__(16) float sa[TS_K][TS_M + 4];
    __shared__ __align__(16) float sb[TS_K][TS_N + 4];
    __shared__ int64_t off_am[TS_M], off_bn[TS_N], off_ak[TS_K], off_bk[TS_K];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const uint32_t tiles_m = static_cast<uint32_t>((p.M + TS_M - 1) / TS_M);
    const int64_t m0 = static_cast<int64_t>(blockIdx.x % tiles_m) * TS_M, n0 = static_cast<int64_t>(blockIdx.x / tiles_m) * TS_N;
    const int64_t batch = p.batch_begin + blockIdx.y;
    const uint16_t* a = A + batch * p.a_bs;
    const uint16_t* b = B + batch * p.b_bs;
    auto cvt = [&](uint16_t v) { return p.ab_f16 ? __half2float(__ushort_as_half(v)) : __uint_as_float(static_cast<uint32_t>(v) << 16); };
    if (tid < TS_M) off_am[tid] = m0 + tid < p.M ? dev_eval_top(LA, 0, static_cast<uint64_t>(m0 + tid)) : 0;
    else if (tid < TS_M + TS_N) off_bn[tid - TS_M] = n0 + tid - TS_M < p.N ? dev_eval_top(LB, 0, static_cast<uint64_t>(n0 + tid - TS_M)) : 0;
    // this thread's 4 x 4 block of C: positions, tile membership, starting accumulators
    const uint32_t tpb = tiles_per_batch(p.grid);
    int64_t cpos[4][4];
    bool live[4][4];
    float acc[4][4];
    float* c32 = static_cast<float*>(C);
    uint16_t* c16 = static_cast<uint16_t*>(C);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = m0 + ty * 4 + i;
        const int64_t cm = m < p.M ? dev_eval_top(LC, 0, static_cast<uint64_t>(m)) : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t n = n0 + tx * 4 + j;
            live[i][j] = m < p.M && n < p.N;
            acc[i][j] = 0.f;
            if (live[i][j]) {
                const uint64_t tile = static_cast<uint64_t>(batch) * tpb + (p.swapped ? tile_of(p.grid, n, m) : tile_of(p.grid, m, n));
                live[i][j] = tile >= p.tile_begin && tile < p.tile_end;
            }
            if (live[i][j]) {
                cpos[i][j] = dev_position(LC, p.c_origin, combine(LC.kind, cm, dev_eval_top(LC, 1, static_cast<uint64_t>(n)))) + batch * p.c_bs;
                acc[i][j] = p.c_16 ? cvt(c16[cpos[i][j]]) : c32[cpos[i][j]];
            }
        }
    }
    for (int64_t k0 = 0; k0 < p.K; k0 += TS_K) {
        if (tid < TS_K) off_ak[tid] = k0 + tid < p.K ? dev_eval_top(LA, 1, static_cast<uint64_t>(k0 + tid)) : 0;
        else if (tid < 2 * TS_K) off_bk[tid - TS_K] = k0 + tid - TS_K < p.K ? dev_eval_top(LB, 1, static_cast<uint64_t>(k0 + tid - TS_K)) : 0;
        __syncthreads();
#pragma unroll
        for (int u = 0; u < TS_M * TS_K / kThreads; ++u) {
            const int idx = tid + u * kThreads;
            // consecutive threads walk the operand's faster mode (coalescing where the layout allows it)
            const int am = a_k_fast ? idx / TS_K : idx % TS_M, ak = a_k_fast ? idx % TS_K : idx / TS_M;
            const int bn = b_k_fast ? idx / TS_K : idx % TS_N, bk = b_k_fast ? idx % TS_K : idx / TS_N;
            float va = 0.f, vb = 0.f;
            if (m0 + am < p.M && k0 + ak < p.K) va = cvt(a[dev_position(LA, p.a_origin, combine(LA.kind, off_am[am], off_ak[ak]))]);
            if (n0 + bn < p.N && k0 + bk < p.K) vb = cvt(b[dev_position(LB, p.b_origin, combine(LB.kind, off_bn[bn], off_bk[bk]))]);
            sa[ak][am] = va;
            sb[bk][bn] = vb;
        }
        __syncthreads();
        const int kmax = static_cast<int>(min(static_cast<int64_t>(TS_K), p.K - k0)); // no padded k: -0 + 0 would flip a sign bit
        for (int kk = 0; kk < kmax; ++kk) {
            const float4 a4 = *reinterpret_cast<const float4*>(&sa[kk][ty * 4]);
            const float4 b4 = *reinterpret_cast<const float4*>(&sb[kk][tx * 4]);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (live[i][j]) {
                if (p.c_16) c16[cpos[i][j]] = p.ab_f16 ? __half_as_ushort(__float2half_rn(acc[i][j])) : __bfloat16_as_ushort(__float2bfloat16_rn(acc[i][j]));
                else c32[cpos[i][j]] = acc[i][j];
            }
}

// Smallest |stride| among the leaves of a top-level mode (which of an operand's two modes walks memory faster).
int64_t min_abs_stride(const tlb_layout_desc& L, int t) {
    int64_t best = INT64_MAX;
    for (int r = L.top_start[t]; r < L.top_start[t + 1]; ++r)
        if (L.extent[r] > 1) best = std::min<int64_t>(best, std::llabs(L.stride[r]));
    return best;
}

int64_t top_size(const tlb_layout_desc& L, int t) {
    int64_t s = 1;
    for (int r = L.top_start[t]; r < L.top_start[t + 1]; ++r) s *= L.extent[r];
    return s;
}

// A top-level mode as one (extent, stride) pair, if its leaves coalesce to that.
bool single_stride(const tlb_layout_desc& L, int t, int64_t* extent, int64_t* stride) {
    int64_t e = 1, s = 0;
    bool have = false;
    for (int r = L.top_start[t]; r < L.top_start[t + 1]; ++r) {
        if (L.extent[r] == 1) continue;
        if (!have) {
            e = L.extent[r];
            s = L.stride[r];
            have = true;
        } else if (L.stride[r] == s * e) {
            e *= L.extent[r];
        } else {
            return false;
        }
    }
    *extent = e;
    *stride = have ? s : 0;
    return true;
}

struct GemmDims {
    int64_t M, N, K;
};

int check_gemm(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int ab_bytes, int c_bytes, GemmDims* d) {
    TLB_TRY(check_tensor(A, "tlb_gemm A", false));
    TLB_TRY(check_tensor(B, "tlb_gemm B", false));
    TLB_TRY(check_tensor(C, "tlb_gemm C", true));
    if (A->accessor != TLB_ACC_BUFFER || B->accessor != TLB_ACC_BUFFER)
        return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: operands must be buffer tensors");
    if (A->layout->n_top != 2 || B->layout->n_top != 2 || C->layout->n_top != 2)
        return fail(TLB_ERR_CONTRACT, "gemm requires rank-2 tensors");
    d->M = top_size(*A->layout, 0);
    d->N = top_size(*B->layout, 0);
    d->K = top_size(*A->layout, 1);
    if (d->M != top_size(*C->layout, 0) || d->N != top_size(*C->layout, 1) || d->K != top_size(*B->layout, 1))
        return fail(TLB_ERR_CONTRACT, "gemm mode extents do not agree");
    const bool c_ok = C->elem_bytes == c_bytes || (ab_bytes == 2 && C->elem_bytes == 2); // C may share the operands' type
    if (A->elem_bytes != ab_bytes || B->elem_bytes != ab_bytes || !c_ok)
        return fail(TLB_ERR_CONTRACT, "tlb_gemm: element sizes do not match the entry point");
    return TLB_OK;
}

// Batched bounds: every batch must stay inside the buffer.
int gemm_bounds(const tlb_tensor& t, int64_t bs, int b0, int b1, const char* who, cudaStream_t stream) {
    tlb_tensor lo = t, hi = t;
    lo.origin = t.origin + bs * b0;
    hi.origin = t.origin + bs * (b1 - 1);
    Span sp;
    const uint64_t n = static_cast<uint64_t>(t.layout->size);
    TLB_TRY(overflow_preflight(*t.layout, hi.origin, n - 1));
    TLB_TRY(bounds_preflight(lo, 0, n, who, stream, &sp));
    if (b1 - 1 != b0) TLB_TRY(bounds_preflight(hi, 0, n, who, stream, &sp));
    return TLB_OK;
}

// Byte range [lo, hi) that a (batched) operand may touch (conservative: span of the whole offset image).
bool byte_range(const tlb_tensor& t, int64_t bs, int b0, int b1, uintptr_t* lo, uintptr_t* hi) {
    Span sp;
    if (position_span(*t.layout, t.origin, &sp) != TLB_OK) return false;
    const int64_t first = bs * b0, last = bs * (b1 - 1);
    // the bounds pre-flight has passed: every access lies inside [0, capacity) (Xor spans are OR-bounds, possibly loose)
    const int64_t plo = std::max<int64_t>(sp.lo + std::min(first, last), 0);
    const int64_t phi = std::min<int64_t>(sp.hi + std::max(first, last), t.capacity - 1);
    const uintptr_t base = reinterpret_cast<uintptr_t>(t.data);
    *lo = base + static_cast<uintptr_t>(plo) * static_cast<uintptr_t>(t.elem_bytes);
    *hi = base + (static_cast<uintptr_t>(phi) + 1) * static_cast<uintptr_t>(t.elem_bytes);
    return true;
}

// The tcgen05 plan applies to K-major A and B with single-stride C modes and TMA-legal strides. When C is
// m-contiguous (the paper's TN row, (M,N):(1,ldc)) the problem is run transposed, C^T += B * A^T: the roles of
// A and B swap, so the accumulator's TMEM lanes run along n and every epilogue thread holds 32 consecutive m
// -- contiguous in memory -- which the swizzled 128-bit staging stores and the TMA reduction need.
struct UmmaFit {
    bool ok = false;
    bool swapped = false;
    UmmaProblem p;
};

UmmaFit fit_umma(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, const GemmDims& d, int64_t a_bs,
                 int64_t b_bs, int64_t c_bs, int batch_begin, int batch_end) {
    UmmaFit f;
    if (A->layout->kind != TLB_KIND_INT || B->layout->kind != TLB_KIND_INT || C->layout->kind != TLB_KIND_INT) return f;
    int64_t eCm = 0, csm = 0, eCn = 0, csn = 0;
    const bool c_flat = single_stride(*C->layout, 0, &eCm, &csm) && single_stride(*C->layout, 1, &eCn, &csn);
    const bool batched = batch_end - batch_begin > 1 || batch_begin > 0;
    // C with hierarchical modes (a GETT-style folded m or n): the reduce-add epilogue addresses it through
    // a rank-4/5 tensor map when the mode that runs along the accumulator's columns starts with a unit-stride leaf.
    int c_col_top = -1;
    if (!c_flat) {
        const int cb = C->elem_bytes;
        for (int top = 1; top >= 0 && c_col_top < 0; --top) {
            int64_t e[4], st[4];
            const int n = mode_leaves(*C->layout, top, e, st, 4);
            TileDims td;
            if (n > 0 && st[0] == 1 &&
                tile_dims_derive(*C->layout, top, 1 - top, cb == 2 ? 64 : 32, 32, 1, 0, batch_end, c_bs, cb, &td) == TLB_OK &&
                tile_dims_derive(*C->layout, top, 1 - top, 32, 128, 1, 0, batch_end, c_bs, cb, &td) == TLB_OK)
                c_col_top = top;
        }
        if (c_col_top < 0) return f;
        // no register epilogue for folded C: the tensor-map path must apply (16-byte aligned base)
        if ((reinterpret_cast<uintptr_t>(static_cast<char*>(C->data) + C->origin * cb) & 15) != 0) return f;
    }
    // Operand majorness from the layout: K-major when the k mode starts with a unit-stride leaf (the paper's "T"
    // operands), MN-major when the row mode does (the "N" operands of the NT / NTT rows). Modes may
    // be hierarchical (GETT-style folded modes): the operand qualifies when the k-block tiles of
    // zipped_divide(operand, [rows, 64]) are TMA boxes (tile_dims_derive: pure host arithmetic, nothing is encoded here).
    auto operand = [&](const tlb_layout_desc& L, int64_t bs, bool* mn) {
        int64_t e[4], st[4];
        const int nk = mode_leaves(L, 1, e, st, 4);
        if (nk < 0) return false;
        const bool k_unit = nk == 0 || st[0] == 1;
        const int nr = mode_leaves(L, 0, e, st, 4);
        if (nr < 0) return false;
        const bool r_unit = nr == 0 || st[0] == 1;
        if (!k_unit && !r_unit) return false;
        *mn = !k_unit;
        TileDims td;
        if (!*mn) return tile_dims_derive(L, 1, 0, 64, 256, 1, 0, batch_end, bs, 2, &td) == TLB_OK &&
                         tile_dims_derive(L, 1, 0, 64, 128, 1, 0, batch_end, bs, 2, &td) == TLB_OK;
        return tile_dims_derive(L, 0, 1, 64, 64, 0, 1, batch_end, bs, 2, &td) == TLB_OK;
    };
    bool a_mn = false, b_mn = false;
    bool ok = operand(*A->layout, a_bs, &a_mn) && operand(*B->layout, b_bs, &b_mn) &&
              (!c_flat || (csm >= 0 && csn >= 0 && (csm > 0 || d.M == 1) && (csn > 0 || d.N == 1))) &&
              (C->layout->flags & TLB_LF_INJECTIVE) && (!batched || (a_bs > 0 && b_bs > 0));
    const char* a_ptr = static_cast<const char*>(A->data) + A->origin * 2;
    const char* b_ptr = static_cast<const char*>(B->data) + B->origin * 2;
    ok = ok && (reinterpret_cast<uintptr_t>(a_ptr) % 16 == 0) && (reinterpret_cast<uintptr_t>(b_ptr) % 16 == 0);
    if (!ok) return f;
    UmmaProblem& p = f.p;
    std::memset(&p, 0, sizeof(p));
    f.swapped = c_flat ? (csm == 1 && csn != 1) : (c_col_top == 0);
    p.c_fold_tma = c_flat ? 0 : 1;
    p.A = f.swapped ? b_ptr : a_ptr;
    p.B = f.swapped ? a_ptr : b_ptr;
    p.C = reinterpret_cast<float*>(static_cast<char*>(C->data) + C->origin * C->elem_bytes);
    p.c_16 = C->elem_bytes == 2 ? 1 : 0;
    p.la = f.swapped ? B->layout : A->layout;
    p.lb = f.swapped ? A->layout : B->layout;
    p.lc = C->layout;
    p.c_row_top = f.swapped ? 1 : 0;
    p.bn = 256;
    p.a_mn = (f.swapped ? b_mn : a_mn) ? 1 : 0;
    p.b_mn = (f.swapped ? a_mn : b_mn) ? 1 : 0;
    p.cs_m = f.swapped ? csn : csm;
    p.cs_n = f.swapped ? csm : csn;
    p.M = static_cast<int32_t>(f.swapped ? d.N : d.M);
    p.N = static_cast<int32_t>(f.swapped ? d.M : d.N);
    p.K = static_cast<int32_t>(d.K);
    p.batch = batch_end;
    p.a_bs = f.swapped ? b_bs : a_bs;
    p.b_bs = f.swapped ? a_bs : b_bs;
    p.c_bs = c_bs;
    f.ok = true;
    return f;
}

int run_gemm(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, bool i64, int64_t a_bs, int64_t b_bs,
             int64_t c_bs, int batch_begin, int batch_end, uint32_t tile_begin, uint32_t tile_end, int* d_status,
             cudaStream_t stream, uint32_t* count_only = nullptr, bool f16 = false);

// ---- packed plan ------------------------------------------------------------------------------------------------
// Operands or a C that no tensor map can address (BLIS-style general strides on every mode, test_tensor.cpp:187 and
// PAPER.md:1769; Xor strides; leading dimensions that are not multiples of 16 bytes) still run on the tensor cores: the
// layout-driven copy (tlb_copy, any layout pair) PACKS A and B into K-major panels and C into an n-contiguous fp32 (or
// 2-byte) tile buffer, the tcgen05 plan runs on the packed tensors, and the copy scatters C back through its layout.
// This is BLIS's own recipe (pack, then a fixed-layout micro-kernel) with the packing expressed as tla::copy between two
// layouts. C += A B^T is preserved (packed C starts as a copy of C); the workspace lives on the stream
// (cudaMallocAsync / cudaFreeAsync). Copies cost O(MK + NK + MN) against O(MNK) of math: 2048^3 with no unit stride
// anywhere ran at 7 TFLOP/s on the SIMT plan.
thread_local bool g_in_packed = false;
thread_local std::string g_packed_plan;

int lower_rowmajor(int64_t rows, int64_t cols, int64_t ld, tlb_layout_desc* out) {
    const tlb_mode m[2] = {{rows, ld, TLB_KIND_INT, 0}, {cols, 1, TLB_KIND_INT, 0}};
    const int32_t tops[2] = {1, 1};
    return tlb_layout_lower_ranked(m, 2, tops, 2, out);
}

int run_packed(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, const GemmDims& d, bool f16, cudaStream_t stream) {
    const int cb = C->elem_bytes;
    const int64_t Kp = (d.K + 7) / 8 * 8, Np = (d.N + 16 / cb - 1) / (16 / cb) * (16 / cb); // 16-byte rows
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t bytes_a = up(static_cast<size_t>(d.M) * Kp * 2), bytes_b = up(static_cast<size_t>(d.N) * Kp * 2),
                 bytes_c = up(static_cast<size_t>(d.M) * Np * cb);
    tlb_layout_desc la, lb, lc;
    TLB_TRY(lower_rowmajor(d.M, d.K, Kp, &la));
    TLB_TRY(lower_rowmajor(d.N, d.K, Kp, &lb));
    TLB_TRY(lower_rowmajor(d.M, d.N, Np, &lc));
    char* ws = nullptr;
    TLB_CUDA(ws_malloc(reinterpret_cast<void**>(&ws), bytes_a + bytes_b + bytes_c, stream));
    const tlb_tensor pa{&la, ws, 0, d.M * Kp, 2, TLB_ACC_BUFFER}, pb{&lb, ws + bytes_a, 0, d.N * Kp, 2, TLB_ACC_BUFFER},
        pc{&lc, ws + bytes_a + bytes_b, 0, d.M * Np, cb, TLB_ACC_BUFFER};
    int st = tlb_copy(A, &pa, 0, static_cast<uint64_t>(d.M) * d.K, stream);
    if (st == TLB_OK) st = tlb_copy(B, &pb, 0, static_cast<uint64_t>(d.N) * d.K, stream);
    if (st == TLB_OK) st = tlb_copy(C, &pc, 0, static_cast<uint64_t>(d.M) * d.N, stream);
    if (st == TLB_OK) {
        g_in_packed = true;
        st = run_gemm(&pa, &pb, &pc, false, 0, 0, 0, 0, 1, 0, UINT32_MAX, nullptr, stream, nullptr, f16);
        g_in_packed = false;
    }
    if (st == TLB_OK) {
        g_packed_plan = std::string("packed+") + tlb_last_plan();
        st = tlb_copy(&pc, C, 0, static_cast<uint64_t>(d.M) * d.N, stream);
    }
    cudaFreeAsync(ws, stream);
    if (st == TLB_OK) set_plan(g_packed_plan.c_str());
    return st;
}

int run_gemm(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, bool i64, int64_t a_bs, int64_t b_bs,
             int64_t c_bs, int batch_begin, int batch_end, uint32_t tile_begin, uint32_t tile_end, int* d_status,
             cudaStream_t stream, uint32_t* count_only, bool f16) {
    GemmDims d;
    TLB_TRY(check_gemm(A, B, C, i64 ? 8 : 2, i64 ? 8 : 4, &d));
    if (batch_begin < 0 || batch_end < batch_begin) return fail(TLB_ERR_CONTRACT, "tlb_gemm: bad batch range");
    if (batch_end == batch_begin && !count_only) return TLB_OK;
    if (d.M >= (1ll << 31) || d.N >= (1ll << 31) || d.K >= (1ll << 31))
        return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: extents must be below 2^31");
    UmmaFit fit;
    if (!i64 && g_gemm_path != 1) fit = fit_umma(A, B, C, d, a_bs, b_bs, c_bs, batch_begin, batch_end);
    // Tiles are 128 x 256 over (rows, columns) of the problem AS THE PLAN RUNS IT (transposed for m-contiguous C).
    const int64_t rows = fit.ok ? fit.p.M : d.M, cols = fit.ok ? fit.p.N : d.N;
    TileGrid grid{static_cast<uint32_t>((rows + 255) / 256), static_cast<uint32_t>((cols + 255) / 256)};
    const uint64_t tpb = tiles_per_batch(grid);
    if (tpb * static_cast<uint64_t>(std::max(batch_end, 1)) > 0xffffffffull)
        return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: too many tiles");
    if (count_only) {
        *count_only = static_cast<uint32_t>(tpb);
        return TLB_OK;
    }
    TLB_TRY(require_device());
    TLB_TRY(gemm_bounds(*A, a_bs, batch_begin, batch_end, "A", stream));
    TLB_TRY(gemm_bounds(*B, b_bs, batch_begin, batch_end, "B", stream));
    TLB_TRY(gemm_bounds(*C, c_bs, batch_begin, batch_end, "C", stream));
    {
        // Aliasing rule (include/tlb.h): C must not overlap A or B. In the reference the three tensors may share storage
        // (tensor.hpp:29) and the serial m, n, k order then decides what later cells read; no parallel plan keeps that.
        uintptr_t clo, chi, olo, ohi;
        if (byte_range(*C, c_bs, batch_begin, batch_end, &clo, &chi))
            for (const tlb_tensor* o : {A, B})
                if (byte_range(*o, o == A ? a_bs : b_bs, batch_begin, batch_end, &olo, &ohi) && olo < chi && clo < ohi)
                    return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: C overlaps an operand in memory (aliased accumulators are order-dependent)");
    }
    // Global tile range: the caller's range applies inside [batch_begin, batch_end).
    uint64_t t0 = static_cast<uint64_t>(batch_begin) * tpb, t1 = static_cast<uint64_t>(batch_end) * tpb;
    if (tile_begin != 0 || tile_end != UINT32_MAX) {
        t0 = std::max<uint64_t>(t0, tile_begin);
        t1 = std::min<uint64_t>(t1, tile_end);
        if (t0 >= t1) return TLB_OK;
    }

    if (g_tiler) {
        // A caller-chosen tiler [bm, bn, bk]: the CTA (pair) tile of zipped_divide(C, [bm, bn]) and the k-block. The
        // TiledMMA atoms are tcgen05.mma 128 x N x 16 (one CTA) and 256 x N x 16 (cta_group::2), N = 128 or 256, so the
        // tile is one or two atoms high; bk is the 64-element (128-byte) swizzle row.
        if (i64 || !fit.ok) return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm_*_tiled: these layouts run on the SIMT plan, which takes no tiler");
        if (tile_begin != 0 || tile_end != UINT32_MAX) return fail(TLB_ERR_CONTRACT, "tlb_gemm_*_tiled: tile ranges refer to the default tiling");
        const int tm = fit.swapped ? g_tiler->bn : g_tiler->bm, tn = fit.swapped ? g_tiler->bm : g_tiler->bn;
        if (g_tiler->bk != 64 || (tn != 128 && tn != 256) || (tm != 128 && tm != 256 && !(tm == 512 && tn == 256)))
            return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm_*_tiled: supported tilers are [128|256, 128|256, 64] and [512, 256, 64] "
                                             "(rows x columns of C as the plan runs it: transposed for an m-contiguous C)");
    }
    if (!i64 && g_gemm_path != 1) {
        if (fit.ok) {
            UmmaProblem& p = fit.p;
            p.tile_begin = static_cast<uint32_t>(t0);
            p.tile_end = static_cast<uint32_t>(t1);
            const bool even = (t0 % 2 == 0) && (t1 % 2 == 0);
            p.split_tail = split_tail_enabled() ? 1 : 0;
            p.cta_group = g_gemm_path == 2 ? 1 : g_gemm_path == 3 ? 2 : (even ? 2 : 1);
            p.full_range = (t0 == 0 && t1 == tpb * static_cast<uint64_t>(batch_end)) ? 1 : 0;
            p.ab_f16 = f16 ? 1 : 0;
            if (g_tiler) {
                const int tm = fit.swapped ? g_tiler->bn : g_tiler->bm, tn = fit.swapped ? g_tiler->bm : g_tiler->bn;
                p.bn = tn;
                p.cta_group = tm == 128 ? 1 : 2;
                p.force_wide = tm == 512 ? 1 : -1;
                if (!p.full_range) return fail(TLB_ERR_CONTRACT, "tlb_gemm_*_tiled: whole problems only");
            }
            // MN-major operands and a 2-byte C run on both tcgen05 plans (the latter through the TMA reduce-add epilogues only)
            if (!p.c_16 || umma_wide_applies(p) || umma_c16_applies(p)) {
                if (p.cta_group == 2 && !even)
                    return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: cta_group::2 needs a tile range aligned to tile pairs");
                return umma_gemm_launch(p, stream);
            }
            // a 2-byte C the TMA epilogues cannot address runs on the packed or the SIMT plan
            if (g_gemm_path == 2 || g_gemm_path == 3)
                return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: a 2-byte C needs a TMA-addressable layout on the tcgen05 plans (n-contiguous rows, multiples of 16 bytes)");
        } else if (g_gemm_path == 2 || g_gemm_path == 3) {
            return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: the forced tcgen05 path does not apply to these layouts");
        }
    }

    if (!(C->layout->flags & TLB_LF_INJECTIVE))
        return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: C must be injective (aliased accumulators are order-dependent)");
    // ---- packed plan: whole single problems that are large enough for three packing copies and one scatter to pay
    if (!i64 && g_gemm_path == 0 && !g_in_packed && !g_tiler && knob(K_GEMM_PACK) != 0 && batch_begin == 0 && batch_end == 1 &&
        tile_begin == 0 && tile_end == UINT32_MAX && A->accessor == TLB_ACC_BUFFER && B->accessor == TLB_ACC_BUFFER &&
        static_cast<double>(d.M) * static_cast<double>(d.N) * static_cast<double>(d.K) >= std::ldexp(1.0, knob(K_GEMM_PACK_MIN)))
        return run_packed(A, B, C, d, f16, stream);
    // ---- SIMT plan
    SimtArgs p;
    std::memset(&p, 0, sizeof(p));
    p.a_origin = A->origin;
    p.b_origin = B->origin;
    p.c_origin = C->origin;
    p.a_bs = a_bs;
    p.b_bs = b_bs;
    p.c_bs = c_bs;
    p.M = d.M;
    p.N = d.N;
    p.K = d.K;
    p.grid = grid;
    p.tile_begin = static_cast<uint32_t>(t0);
    p.tile_end = static_cast<uint32_t>(t1);
    p.batch_begin = batch_begin;
    p.batch_end = batch_end;
    p.ab_f16 = f16 ? 1 : 0;
    p.c_16 = C->elem_bytes == 2 ? 1 : 0;
    // the grid above was built from the problem as the tcgen05 plans run it; keep the SAME tile ids when this call falls
    // through to SIMT (sharded ranges may mix plans across ranks), i.e. index the grid with (n, m) when it is transposed
    p.swapped = (fit.ok && fit.swapped) ? 1 : 0;
    const uint64_t total = static_cast<uint64_t>(d.M) * d.N * (batch_end - batch_begin);
    const uint64_t blocks = std::min<uint64_t>((total + kThreads - 1) / kThreads, static_cast<uint64_t>(sm_count()) * 32);
    const int gridx = static_cast<int>(std::max<uint64_t>(blocks, 1));
    if (i64)
        gemm_simt_kernel<true><<<gridx, kThreads, 0, stream>>>(*A->layout, *B->layout, *C->layout, A->data, B->data, C->data, p, d_status);
    else {
        const uint64_t tiles = static_cast<uint64_t>((d.M + TS_M - 1) / TS_M) * static_cast<uint64_t>((d.N + TS_N - 1) / TS_N);
        const int nbatch = batch_end - batch_begin;
        if (tiles > 0x7fffffffull || nbatch > 65535) return fail(TLB_ERR_UNSUPPORTED, "tlb_gemm: too many tiles for the SIMT plan");
        gemm_simt_tiled_kernel<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(nbatch)), kThreads, 0, stream>>>(
            *A->layout, *B->layout, *C->layout, static_cast<const uint16_t*>(A->data), static_cast<const uint16_t*>(B->data), C->data, p,
            min_abs_stride(*A->layout, 1) < min_abs_stride(*A->layout, 0) ? 1 : 0,
            min_abs_stride(*B->layout, 1) < min_abs_stride(*B->layout, 0) ? 1 : 0);
    }
    count_launch();
    TLB_CUDA(cudaGetLastError());
    set_plan(i64 ? "simt_i64" : f16 ? "simt_f16" : "simt_bf16");
    return TLB_OK;
}

} // namespace

bool gemm_flat_view(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, GemmFlat* out) {
    GemmDims d;
    if (check_gemm(A, B, C, 2, 4, &d) != TLB_OK) return false;
    if (A->layout->kind != TLB_KIND_INT || B->layout->kind != TLB_KIND_INT || C->layout->kind != TLB_KIND_INT) return false;
    int64_t e;
    GemmFlat f{d.M, d.N, d.K, 0, 0, 0, 0, 0, 0};
    if (!single_stride(*A->layout, 0, &e, &f.a_sm) || !single_stride(*A->layout, 1, &e, &f.a_sk) ||
        !single_stride(*B->layout, 0, &e, &f.b_sn) || !single_stride(*B->layout, 1, &e, &f.b_sk) ||
        !single_stride(*C->layout, 0, &e, &f.c_sm) || !single_stride(*C->layout, 1, &e, &f.c_sn))
        return false;
    *out = f;
    return true;
}

int gemm_bf16_impl(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int64_t a_bs, int64_t b_bs, int64_t c_bs,
                   int batch_begin, int batch_end, uint32_t tile_begin, uint32_t tile_end, cudaStream_t stream) {
    return run_gemm(A, B, C, false, a_bs, b_bs, c_bs, batch_begin, batch_end, tile_begin, tile_end, nullptr, stream);
}

} // namespace tlb

extern "C" {

int tlb_gemm_bf16(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, uint32_t tile_begin, uint32_t tile_end,
                  void* stream) {
    return tlb::run_gemm(A, B, C, false, 0, 0, 0, 0, 1, tile_begin, tile_end, nullptr, static_cast<cudaStream_t>(stream));
}

int tlb_gemm_bf16_batched(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int64_t a_batch_stride,
                          int64_t b_batch_stride, int64_t c_batch_stride, int32_t batch_begin, int32_t batch_end,
                          void* stream) {
    return tlb::run_gemm(A, B, C, false, a_batch_stride, b_batch_stride, c_batch_stride, batch_begin, batch_end, 0,
                         UINT32_MAX, nullptr, static_cast<cudaStream_t>(stream));
}

int tlb_gemm_f16(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, uint32_t tile_begin, uint32_t tile_end,
                 void* stream) {
    return tlb::run_gemm(A, B, C, false, 0, 0, 0, 0, 1, tile_begin, tile_end, nullptr, static_cast<cudaStream_t>(stream),
                         nullptr, true);
}

int tlb_gemm_f16_batched(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int64_t a_batch_stride,
                         int64_t b_batch_stride, int64_t c_batch_stride, int32_t batch_begin, int32_t batch_end,
                         void* stream) {
    return tlb::run_gemm(A, B, C, false, a_batch_stride, b_batch_stride, c_batch_stride, batch_begin, batch_end, 0,
                         UINT32_MAX, nullptr, static_cast<cudaStream_t>(stream), nullptr, true);
}

int tlb_gemm_i64(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int32_t* d_status, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (d_status) return tlb::run_gemm(A, B, C, true, 0, 0, 0, 0, 1, 0, UINT32_MAX, d_status, s);
    // No status word from the caller: the call owns one, waits for the kernel and reports the reference's
    // overflow_error (common.hpp:99-109) as its return value, so a wrap can never pass silently.
    int32_t* d = nullptr;
    int32_t h = 0;
    uint32_t tiles = 0;
    TLB_TRY(tlb::run_gemm(A, B, C, true, 0, 0, 0, 0, 1, 0, UINT32_MAX, nullptr, nullptr, &tiles)); // contracts first, no device needed
    if (tlb::require_device() != TLB_OK) return TLB_ERR_CUDA;
    TLB_CUDA(tlb::ws_malloc(reinterpret_cast<void**>(&d), sizeof(int32_t), s));
    cudaError_t e = cudaMemsetAsync(d, 0, sizeof(int32_t), s);
    int st = e == cudaSuccess ? tlb::run_gemm(A, B, C, true, 0, 0, 0, 0, 1, 0, UINT32_MAX, d, s) : TLB_OK;
    if (e == cudaSuccess && st == TLB_OK) e = cudaMemcpyAsync(&h, d, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && st == TLB_OK) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d, s);
    TLB_CUDA(e);
    if (st != TLB_OK) return st;
    if (h == TLB_ERR_OVERFLOW) return tlb::fail(TLB_ERR_OVERFLOW, "integer overflow in gemm accumulation");
    return TLB_OK;
}

int tlb_gemm_bf16_tiled(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, const tlb_gemm_tiler* tiler,
                        void* stream) {
    if (!tiler) return tlb::fail(TLB_ERR_CONTRACT, "tlb_gemm_bf16_tiled: null tiler");
    tlb::g_tiler = tiler;
    const int st = tlb::run_gemm(A, B, C, false, 0, 0, 0, 0, 1, 0, UINT32_MAX, nullptr, static_cast<cudaStream_t>(stream));
    tlb::g_tiler = nullptr;
    return st;
}

int tlb_gemm_tile_count(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, uint32_t* tiles) {
    if (!tiles) return tlb::fail(TLB_ERR_CONTRACT, "tlb_gemm_tile_count: null output");
    return tlb::run_gemm(A, B, C, false, 0, 0, 0, 0, 1, 0, UINT32_MAX, nullptr, nullptr, tiles);
}

int tlb_gemm_set_path(int path) {
    const int prev = tlb::g_gemm_path;
    if (path >= 0 && path <= 3) tlb::g_gemm_path = path;
    return prev;
}

} // extern "C"

// tcgen05 GEMM for the TN family of tla::gemm (tensor.hpp:214-233):
//   C(m,n) += sum_k A(m,k) * B(n,k),  A (M,K):(lda,1), B (N,K):(ldb,1) bf16, C fp32 any strides.
//
// Partitioning follows the paper's local_tile / TiledMMA picture:
// zipped_divide(C, [128,256]) gives the CTA tiles, zipped_divide(A, [128,64]) / (B, [256,64])
// the k-blocks; the TMA tensor maps are exactly those divided layouts (box = tile mode,
// globalDim/globalStrides = parent layout), the 128-byte swizzle of the staged tiles is
// Swizzle<3,4,3> on byte offsets = the reference layout (128,8):(f1,f144).
//
// Kernel shape (persistent, warp-specialised, 192 threads, 1 CTA per SM):
//   warp 0   TMA producer: ring of kStages {A tile, B tile} stages, full/empty mbarriers
//   warp 1   TMEM allocator + single-thread tcgen05.mma issuer (UMMA 128x256x16 or, with
//            cta_group::2, 256x256x16 across a CTA pair), accumulators in TMEM, double buffered
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 -> registers -> C += acc (coalesced along the
//            contiguous mode of C), overlapped with the next tile's MMAs
// No CUTLASS / CuTe: descriptors are encoded by hand below.
#include <algorithm>
#include <cstring>

#include <cuda.h>

#include "tlb_internal.h"
#include "tlb_gemm.h"

namespace tlb {
namespace {

constexpr int BM = 128;      // rows of C per CTA
constexpr int BN = 256;      // columns of C per CTA (UMMA N)
constexpr int BK = 64;       // k-block: 64 bf16 = one 128-byte swizzle row
constexpr int UMMA_K = 16;
constexpr int kUmmaThreads = 192;
constexpr uint32_t kTmemCols = 512; // two 256-column fp32 accumulators

template <int CG> struct Cfg {
    static constexpr int kStages = CG == 1 ? 4 : 7;
    static constexpr int kBRows = CG == 1 ? BN : BN / 2; // rows of B this CTA stages
    static constexpr uint32_t kABytes = BM * BK * 2;
    static constexpr uint32_t kBBytes = kBRows * BK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

// ---- PTX wrappers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Bounded wait: a pipeline bug must trap, never hang the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    const long long t0 = clock64();
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (clock64() - t0 > 6000000000ll) __trap();
    }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* map, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// cta_group::2 form: the transaction bytes complete on the LEADER CTA's barrier (cluster address).
__device__ __forceinline__ void tma_load_3d_2sm(uint32_t dst, const void* map, uint32_t leader_bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(map), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

template <int CG> __device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t cols) {
    if constexpr (CG == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(cols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(cols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
}
template <int CG> __device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    if constexpr (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
template <int CG>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
    if constexpr (CG == 1) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
            : "memory");
    }
}
// tcgen05.commit: the barrier is arrived on when every previously issued MMA has finished.
template <int CG> __device__ __forceinline__ void umma_commit(uint32_t bar) {
    if constexpr (CG == 1) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    } else {
        const uint16_t mask = 3; // both CTAs of the pair, same barrier offset in each
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
            "h"(mask)
            : "memory");
    }
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor of a K-major bf16 tile staged with the 128-byte swizzle:
// rows of 128 B, 8-row groups 1024 B apart (SBO), sm_100 descriptor version 1, layout type 2.
__device__ __forceinline__ uint64_t make_kmajor_sw128_desc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3fffu);       // start address  [0,14)
    d |= static_cast<uint64_t>(1) << 16;                          // LBO (unused for swizzled K-major) [16,30)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;                  // SBO = 1024 B   [32,46)
    d |= static_cast<uint64_t>(1) << 46;                          // version = 1    [46,48)
    d |= static_cast<uint64_t>(2) << 61;                          // SWIZZLE_128B   [61,64)
    return d;
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, N = 256, M = 128 * CG.
template <int CG> __device__ __forceinline__ constexpr uint32_t make_idesc() {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
           (static_cast<uint32_t>((BM * CG) >> 4) << 24);
}

struct UmmaArgs {
    float* C;
    int64_t cs_m, cs_n, c_bs;
    int32_t M, N, K;
    uint32_t mb, nb;           // 256x256 blocks along m and n
    uint32_t unit_begin, unit_end; // CG=1: 128x256 tile ids; CG=2: 256x256 block ids (all batches)
    int32_t c_vec;             // 1: C rows are n-contiguous and 16-byte aligned (vector epilogue)
};

// unit -> (batch, m_tile (128 rows), n_blk (256 cols)). Blocks are walked in groups of kGroupM
// m-blocks, m fastest inside a group, so that concurrently resident CTAs share A and B panels in L2.
template <int CG>
__device__ __forceinline__ void decode_unit(const UmmaArgs& a, uint32_t unit, uint32_t rank, uint32_t* batch,
                                            uint32_t* m_tile, uint32_t* n_blk) {
    const uint32_t blocks = a.mb * a.nb;
    const uint32_t g = CG == 1 ? unit >> 1 : unit;
    const uint32_t half = CG == 1 ? (unit & 1u) : rank;
    *batch = g / blocks;
    const uint32_t blk = g % blocks;
    const uint32_t per = kGemmGroupM * a.nb;
    const uint32_t grp = blk / per, rem = blk % per;
    const uint32_t gm = min(static_cast<uint32_t>(kGemmGroupM), a.mb - grp * kGemmGroupM);
    *m_tile = (grp * kGemmGroupM + rem % gm) * 2 + half;
    *n_blk = rem / gm;
}

template <int CG>
__global__ void __launch_bounds__(kUmmaThreads, 1)
umma_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ UmmaArgs args) {
    using C = Cfg<CG>;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t bar_base = smem_base + C::kStages * C::kStageBytes;
    auto a_stage = [&](int s) { return smem_base + s * C::kStageBytes; };
    auto b_stage = [&](int s) { return smem_base + s * C::kStageBytes + C::kABytes; };
    auto full_bar = [&](int s) { return bar_base + 8u * s; };
    auto empty_bar = [&](int s) { return bar_base + 8u * (C::kStages + s); };
    auto tfull_bar = [&](int s) { return bar_base + 8u * (2 * C::kStages + s); };
    auto tempty_bar = [&](int s) { return bar_base + 8u * (2 * C::kStages + 2 + s); };
    const uint32_t tmem_slot = bar_base + 8u * (2 * C::kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const uint32_t n_workers = CG == 2 ? gridDim.x / 2 : gridDim.x;
    const uint32_t worker = CG == 2 ? blockIdx.x / 2 : blockIdx.x;
    const int kblocks = (args.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(full_bar(s), CG);       // CG=2: leader's own arrive + the peer's remote arrive
            mbar_init(empty_bar(s), 1);       // one tcgen05.commit
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(tfull_bar(s), 1);       // one tcgen05.commit
            mbar_init(tempty_bar(s), 4 * CG); // one lane of each epilogue warp (of both CTAs)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc<CG>(tmem_slot, kTmemCols);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (uint32_t u = args.unit_begin + worker; u < args.unit_end; u += n_workers) {
                uint32_t batch, m_tile, n_blk;
                decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
                if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
                const int m0 = m_tile * BM;
                const int n0 = n_blk * BN + (CG == 2 ? rank * (BN / 2) : 0);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(empty_bar(stage), phase ^ 1u);
                    if constexpr (CG == 1) {
                        mbar_expect_tx(full_bar(stage), C::kStageBytes);
                        tma_load_3d(a_stage(stage), &map_a, full_bar(stage), kb * BK, m0, batch);
                        tma_load_3d(b_stage(stage), &map_b, full_bar(stage), kb * BK, n0, batch);
                    } else {
                        const uint32_t lbar = map_to_cta(full_bar(stage), 0);
                        if (leader) mbar_expect_tx(full_bar(stage), 2 * C::kStageBytes);
                        else mbar_arrive_cluster(lbar);
                        tma_load_3d_2sm(a_stage(stage), &map_a, lbar, kb * BK, m0, batch);
                        tma_load_3d_2sm(b_stage(stage), &map_b, lbar, kb * BK, n0, batch);
                    }
                    if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one thread; leader CTA only under cta_group::2) =====
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = make_idesc<CG>();
            int stage = 0;
            uint32_t phase = 0, acc = 0, acc_phase = 0;
            for (uint32_t u = args.unit_begin + worker; u < args.unit_end; u += n_workers) {
                uint32_t batch, m_tile, n_blk;
                decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
                if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
                mbar_wait(tempty_bar(acc), acc_phase ^ 1u); // epilogue has drained this accumulator
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(full_bar(stage), phase);
                    tc_fence_after();
                    const uint64_t da = make_kmajor_sw128_desc(a_stage(stage));
                    const uint64_t db = make_kmajor_sw128_desc(b_stage(stage));
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        // advancing K inside the 128-byte swizzle row: +32 B on the start address
                        umma_bf16<CG>(d_tmem, da + static_cast<uint64_t>(k * 2), db + static_cast<uint64_t>(k * 2), idesc,
                                      (kb | k) != 0 ? 1u : 0u);
                    }
                    umma_commit<CG>(empty_bar(stage)); // frees the smem stage once these MMAs retire
                    if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
                }
                umma_commit<CG>(tfull_bar(acc)); // accumulator complete -> epilogue
                acc ^= 1u;
                if (acc == 0) acc_phase ^= 1u;
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> C += acc =====
        const uint32_t quad = warp & 3;            // the TMEM lane quadrant this warp may read
        const uint32_t row = quad * 32 + lane;
        uint32_t acc = 0, acc_phase = 0;
        const uint32_t tempty_leader = CG == 2 ? map_to_cta(tempty_bar(0), 0) : 0u;
        for (uint32_t u = args.unit_begin + worker; u < args.unit_end; u += n_workers) {
            uint32_t batch, m_tile, n_blk;
            decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
            if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
            mbar_wait(tfull_bar(acc), acc_phase);
            tc_fence_after();
            const int64_t m = static_cast<int64_t>(m_tile) * BM + row;
            float* crow = args.C + batch * args.c_bs + m * args.cs_m;
            const bool m_ok = m < args.M;
#pragma unroll 1
            for (int col = 0; col < BN; col += 32) {
                uint32_t v[32];
                __syncwarp(); // lanes of an edge tile diverge below; tcgen05.ld is .sync.aligned
                tmem_ld32(tmem_base + ((quad * 32u) << 16) + acc * BN + col, v);
                tmem_ld_wait();
                const int64_t n0 = static_cast<int64_t>(n_blk) * BN + col;
                if (!m_ok || n0 >= args.N) continue;
                if (args.c_vec && n0 + 32 <= args.N) {
                    float4* p = reinterpret_cast<float4*>(crow + n0);
                    float4 c[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) c[j] = p[j];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        c[j].x += __uint_as_float(v[4 * j + 0]);
                        c[j].y += __uint_as_float(v[4 * j + 1]);
                        c[j].z += __uint_as_float(v[4 * j + 2]);
                        c[j].w += __uint_as_float(v[4 * j + 3]);
                        p[j] = c[j];
                    }
                } else if (n0 + 32 <= args.N) {
                    float c[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) c[j] = crow[(n0 + j) * args.cs_n];
#pragma unroll
                    for (int j = 0; j < 32; ++j) crow[(n0 + j) * args.cs_n] = c[j] + __uint_as_float(v[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (n0 + j < args.N) crow[(n0 + j) * args.cs_n] += __uint_as_float(v[j]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 1) mbar_arrive(tempty_bar(acc));
                else mbar_arrive_cluster(tempty_leader + 8u * acc);
            }
            acc ^= 1u;
            if (acc == 0) acc_phase ^= 1u;
        }
    }

    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, kTmemCols);
    }
}

int encode_operand_map(TmaDesc* out, const void* base, int64_t ld, int64_t batch_stride, int rows, int K, int batch,
                       int box_rows) {
    const uint64_t dims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(rows), static_cast<uint64_t>(batch)};
    const uint64_t strides[2] = {static_cast<uint64_t>(ld) * 2,
                                 static_cast<uint64_t>(batch > 1 ? batch_stride : ld * static_cast<int64_t>(rows)) * 2};
    const uint32_t box[3] = {BK, static_cast<uint32_t>(box_rows), 1};
    return tma_encode(out, 2, true, 3, const_cast<void*>(base), dims, strides, box, TMA_SW_128, 256);
}

template <int CG> int launch(const UmmaProblem& p, cudaStream_t stream) {
    using C = Cfg<CG>;
    static bool attr_set[64] = {false};
    int dev = 0;
    TLB_CUDA(cudaGetDevice(&dev));
    if (dev >= 0 && dev < 64 && !attr_set[dev]) {
        TLB_CUDA(cudaFuncSetAttribute(umma_gemm_kernel<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        attr_set[dev] = true;
    }
    TmaDesc ma, mb;
    TLB_TRY(encode_operand_map(&ma, p.A, p.lda, p.a_bs, p.M, p.K, p.batch, BM));
    TLB_TRY(encode_operand_map(&mb, p.B, p.ldb, p.b_bs, p.N, p.K, p.batch, C::kBRows));
    UmmaArgs a;
    std::memset(&a, 0, sizeof(a));
    a.C = p.C;
    a.cs_m = p.cs_m;
    a.cs_n = p.cs_n;
    a.c_bs = p.c_bs;
    a.M = p.M;
    a.N = p.N;
    a.K = p.K;
    a.mb = (p.M + 255) / 256;
    a.nb = (p.N + 255) / 256;
    a.unit_begin = CG == 1 ? p.tile_begin : p.tile_begin / 2;
    a.unit_end = CG == 1 ? p.tile_end : p.tile_end / 2;
    a.c_vec = (p.cs_n == 1 && p.cs_m % 4 == 0 && p.c_bs % 4 == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0) ? 1 : 0;
    const uint32_t units = a.unit_end - a.unit_begin;
    if (units == 0) return TLB_OK;
    const int sms = sm_count();
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    if (CG == 1) {
        cfg.gridDim = dim3(std::min<uint32_t>(units, static_cast<uint32_t>(sms)));
        cfg.numAttrs = 0;
    } else {
        cfg.gridDim = dim3(2 * std::min<uint32_t>(units, static_cast<uint32_t>(sms / 2)));
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    cfg.blockDim = dim3(kUmmaThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    CUtensorMap tma, tmb;
    std::memcpy(&tma, ma.bytes, 128);
    std::memcpy(&tmb, mb.bytes, 128);
    TLB_CUDA(cudaLaunchKernelEx(&cfg, umma_gemm_kernel<CG>, tma, tmb, a));
    count_launch();
    set_plan(CG == 1 ? "umma_1sm" : "umma_2sm");
    return TLB_OK;
}

} // namespace

int umma_gemm_launch(const UmmaProblem& p, cudaStream_t stream) {
    if (p.cta_group == 2) return launch<2>(p, stream);
    return launch<1>(p, stream);
}

} // namespace tlb

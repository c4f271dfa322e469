// tcgen05 GEMM for the K-major family of tla::gemm (tensor.hpp:214-233):
//   C(m,n) += sum_k A(m,k) * B(n,k),  A (M,K):(lda,1), B (N,K):(ldb,1) bf16, C fp32.
// The dispatcher (tlb_gemm_simt.cu) hands this file a problem whose C is n-contiguous whenever C has a
// contiguous mode at all: the paper's TN row, C = (M,N):(1,ldc), is run transposed (C^T += B * A^T).
//
// Partitioning follows the paper's local_tile / TiledMMA picture:
// zipped_divide(C, [128,256]) gives the CTA tiles, zipped_divide(A, [128,64]) / (B, [256,64]) the k-blocks;
// the TMA tensor maps are exactly those divided layouts (box = tile mode, globalDim / globalStrides = parent
// layout), and the 128-byte swizzle of every staged tile is Swizzle<3,4,3> on byte offsets, i.e. the reference
// layout (128,8):(f1,f144) per 1 KiB (stride.hpp:142).
//
// Kernel shape (persistent, warp-specialised, 320 threads, 1 CTA per SM):
//   warps 0-7  epilogue. Warp w owns TMEM lane quadrant w % 4 and columns [128 * (w / 4), +128):
//              tcgen05.ld 32x32b.x32 -> registers -> 128-byte-swizzled smem chunk (32 n x 128 m fp32) ->
//              cp.reduce.async.bulk.tensor .add: the TMA unit / L2 performs C += chunk, the SM never loads C.
//              (Generic C strides fall back to a register epilogue.) Overlaps the next tile's MMAs.
//   warp 8     TMA producer: ring of kStages {A tile, B tile} stages, full / empty mbarriers
//   warp 9     TMEM allocator + tcgen05.mma issue (one elected lane, warp-uniform control flow so that
//              descriptors live in uniform registers): UMMA 128x256x16, or 256x256x16 across a CTA pair with
//              cta_group::2; fp32 accumulators in TMEM, double buffered (2 x 256 columns)
// Scheduling: static round-robin over tiles; the tiles of the last partial wave are split along K into
// slices that run first and combine through the same reduce-add epilogue (tail-wave balancing).
// No CUTLASS / CuTe: descriptors are encoded by hand below.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <type_traits>

#include <cuda.h>

#include "tlb_internal.h"
#include "tlb_gemm.h"
#include "tlb_umma_ptx.h"

namespace tlb {
namespace {

constexpr int BM = 128;      // rows of C per CTA
// columns of C per CTA / CTA pair (UMMA N) are the template parameter BN: 256 (default plans) or 128 (from a tiler)
constexpr int BK = 64;       // k-block: 64 bf16 = one 128-byte swizzle row
constexpr int UMMA_K = 16;
constexpr int kEpiWarps = 8; // two warps per TMEM lane quadrant, 128 columns each
constexpr int kUmmaThreads = 64 + 32 * kEpiWarps;
// The single-thread MMA issuer is latency critical; it is the last warp of the CTA.
constexpr int kProducerWarp = kEpiWarps;
constexpr int kMmaWarp = kEpiWarps + 1;
constexpr uint32_t kTmemCols = 512; // two 256-column fp32 accumulators

// Epilogue flavours: how C += acc reaches memory.
//   EPI_REGS   any C strides: registers; C loaded / added / stored per element (prefetched a chunk ahead),
//              K-slices of split tiles use red.global.add
//   EPI_TMA    C n-contiguous: 32(n) x 128(m) fp32 chunks staged with the 128-byte swizzle, TMA reduce-add
enum { EPI_REGS = 0, EPI_TMA = 1 };
constexpr uint32_t kEpiChunkBytes = BM * 32 * 4; // 16 KiB

#ifndef TLB_UMMA_STAGES
#define TLB_UMMA_STAGES 6
#endif
#ifndef TLB_UMMA_EPIBUFS
#define TLB_UMMA_EPIBUFS 1
#endif
template <int CG, int EPI, int BN> struct Cfg {
    static constexpr int kEpiBufs = EPI == EPI_REGS ? 0 : (CG == 2 ? TLB_UMMA_EPIBUFS : 1); // staging buffers per column half
    static constexpr int kStages = CG == 1 ? 4 : TLB_UMMA_STAGES; // even: smem stages are released in pairs
    static constexpr int kPairs = kStages / 2;
    static constexpr int kBRows = CG == 1 ? BN : BN / 2; // rows of B this CTA stages
    static constexpr uint32_t kABytes = BM * BK * 2;
    static constexpr uint32_t kBBytes = kBRows * BK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kEpiBytes = 2 * kEpiBufs * kEpiChunkBytes;
    static constexpr uint32_t kSmem = kStages * kStageBytes + kEpiBytes + 1024 /*align*/ + 256 /*barriers*/;
};

using namespace umma;

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, N = 256, M = 128 * CG.
template <int CG, int BN> __device__ __forceinline__ constexpr uint32_t make_idesc() {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
           (static_cast<uint32_t>((BM * CG) >> 4) << 24);
}

struct UmmaArgs {
    float* C;
    int64_t cs_m, cs_n, c_bs;
    int32_t M, N, K;
    uint32_t mb, nb;               // blocks of 256 rows x BN columns along m and n
    uint32_t group_m;              // m-blocks per rasterisation group (L2 reuse of the A panel)
    uint32_t unit_begin, unit_end; // CG=1: 128x256 tile ids; CG=2: 256x256 block ids (all batches)
    uint32_t n_split_units;        // the LAST n_split_units units of the range are split along K ...
    uint32_t split;                // ... into `split` slices each; the slices are scheduled first
    uint32_t work_end;             // unit_begin + n_split_units * split + (units - n_split_units)
    int32_t c_vec;                 // register epilogue: C rows are n-contiguous and 16-byte aligned
    uint32_t backoff_ns;           // nanosleep between barrier probes of the idle roles (0 = spin)
    uint32_t hints;                // L2 cache hints: 1 = operand loads evict_last, 2 = C reductions evict_first
    uint32_t debug;                // TLB_GEMM_DEBUG timing experiments (results are garbage): 1 = no TMA loads after
                                   // the ring is filled once, 2 = epilogue without smem / global traffic,
                                   // 4 = no staging stores, 8 = no TMA store, 16 = plain TMA store instead of reduce-add
    long long* trace;              // optional per-CTA timeline (TLB_GEMM_TRACE=<file>), kTraceSlots int64 per CTA
    uint32_t ab_f16;               // operands are fp16 (A / B format fields of the instruction descriptor = 0)
    uint32_t c_16;                 // C has the operands' 2-byte type (TMA epilogue only): 64-column chunks, rounded once, added at L2
    uint32_t a_mn, b_mn;           // operand is MN-major: staged as 64-row chunks of [64 k][128 B] (the map's dimension 0 is the
                                   // row index), MN-major UMMA descriptors (LBO = 8 KiB between chunks, idesc bits 15 / 16)
    long long* clk;                // optional (TLB_GEMM_CLOCK=1): CTA 0 stamps {clock64, globaltimer} at entry and exit
    // how a tile's (row, k | column, batch) start turns into the coordinates of the layout-derived tensor maps
    int32_t rank_a, rank_b, rank_c;
    TmaCoord ca[5], cb[5], cc[5];
};
constexpr int kTraceSlots = 128;
#define TLB_TRACE(slot)                                                                                    \
    do {                                                                                                   \
        if (args.trace && (slot) < kTraceSlots) args.trace[blockIdx.x * kTraceSlots + (slot)] = clock64(); \
    } while (0)

// Work item w -> (unit, k-block range). The K-slices of the split units come first, whole units after.
__device__ __forceinline__ void decode_work(const UmmaArgs& a, uint32_t w, int kblocks, uint32_t* unit, int* kb0, int* kb1,
                                            bool* partial) {
    const uint32_t r = w - a.unit_begin;
    const uint32_t n_slices = a.n_split_units * a.split;
    if (r >= n_slices) {
        *unit = a.unit_begin + (r - n_slices);
        *kb0 = 0;
        *kb1 = kblocks;
        *partial = false;
        return;
    }
    *unit = a.unit_end - a.n_split_units + r / a.split;
    const uint32_t sl = r % a.split;
    *kb0 = static_cast<int>(static_cast<int64_t>(kblocks) * sl / a.split);
    *kb1 = static_cast<int>(static_cast<int64_t>(kblocks) * (sl + 1) / a.split);
    *partial = a.split > 1;
}

// unit -> (batch, m_tile (128 rows), n_blk (256 cols)). Blocks are walked in groups of kGemmGroupM
// m-blocks, m fastest inside a group, so that concurrently resident CTAs share A and B panels in L2.
template <int CG>
__device__ __forceinline__ void decode_unit(const UmmaArgs& a, uint32_t unit, uint32_t rank, uint32_t* batch,
                                            uint32_t* m_tile, uint32_t* n_blk) {
    const uint32_t blocks = a.mb * a.nb;
    const uint32_t g = CG == 1 ? unit >> 1 : unit;
    const uint32_t half = CG == 1 ? (unit & 1u) : rank;
    *batch = g / blocks;
    const uint32_t blk = g % blocks;
    const uint32_t per = a.group_m * a.nb;
    const uint32_t grp = blk / per, rem = blk % per;
    const uint32_t gm = min(a.group_m, a.mb - grp * a.group_m);
    *m_tile = (grp * a.group_m + rem % gm) * 2 + half;
    *n_blk = rem / gm;
}

template <int CG, int EPI, int BN, bool PLAIN>
__global__ void __launch_bounds__(kUmmaThreads, 1)
umma_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_c, const __grid_constant__ UmmaArgs args) {
    using C = Cfg<CG, EPI, BN>;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t epi_base = smem_base + C::kStages * C::kStageBytes; // 1 KiB aligned (stage sizes are)
    const uint32_t bar_base = epi_base + C::kEpiBytes;
    auto a_stage = [&](int s) { return smem_base + s * C::kStageBytes; };
    auto b_stage = [&](int s) { return smem_base + s * C::kStageBytes + C::kABytes; };
    auto full_bar = [&](int s) { return bar_base + 8u * s; };
    auto empty_bar = [&](int s) { return bar_base + 8u * (C::kStages + s); };
    auto tfull_bar = [&](int s) { return bar_base + 8u * (2 * C::kStages + s); };
    auto tempty_bar = [&](int s) { return bar_base + 8u * (2 * C::kStages + 2 + s); };
    const uint32_t tmem_slot = bar_base + 8u * (2 * C::kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank_a = PLAIN ? 3 : args.rank_a, rank_b = PLAIN ? 3 : args.rank_b, rank_c = PLAIN ? 3 : args.rank_c;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const uint32_t n_workers = CG == 2 ? gridDim.x / 2 : gridDim.x;
    const uint32_t worker = CG == 2 ? blockIdx.x / 2 : blockIdx.x;
    const int kblocks = (args.K + BK - 1) / BK;
    if (threadIdx.x == 0) {
        TLB_TRACE(0);
        if (args.trace) {
            unsigned long long gt;
            uint32_t smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            args.trace[blockIdx.x * kTraceSlots + 2] = static_cast<long long>(gt);
            args.trace[blockIdx.x * kTraceSlots + 3] = smid;
        }
    }

    if (warp == kProducerWarp && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
        if (EPI != EPI_REGS) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_c) : "memory");
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(full_bar(s), 1);  // the (leader's) producer arrive; the TMA bytes complete the phase
            mbar_init(empty_bar(s), 1); // pair s < kPairs: one tcgen05.commit (leader) / one relayed arrive (peer)
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(tfull_bar(s), 1);               // one tcgen05.commit
            mbar_init(tempty_bar(s), kEpiWarps * CG); // one lane of each epilogue warp (of both CTAs)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) tmem_alloc<CG>(tmem_slot, kTmemCols);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));
    // the prologue above may overlap the tail of the previous kernel of the stream (programmatic dependent launch)
    griddep_wait();
    griddep_launch_dependents();
    if (threadIdx.x == 0 && blockIdx.x == 0 && args.clk) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.clk[0] = clock64();
        args.clk[1] = static_cast<long long>(gt);
    }
    if (threadIdx.x == 0) TLB_TRACE(1);

    if (warp == kProducerWarp) {
        // ===== TMA producer (whole warp in the loops, one elected lane issues) =====
        int stage = 0;
        uint32_t phase = 0;
        bool ring_filled = false, ring_wrapped = false;
        const uint32_t peer_empty0 = CG == 2 ? map_to_cta(empty_bar(0), 1) : 0u;
        const uint32_t lbar0 = CG == 2 ? map_to_cta(full_bar(0), 0) : full_bar(0);
        const uint64_t pol_ab = policy_evict_last();
        const bool hint_ab = (args.hints & 1u) != 0;
        for (uint32_t w = args.unit_begin + worker; w < args.work_end; w += n_workers) {
            uint32_t u, batch, m_tile, n_blk;
            int kb0, kb1;
            bool partial;
            decode_work(args, w, kblocks, &u, &kb0, &kb1, &partial);
            decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
            if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
            const int m0 = m_tile * BM;
            const int n0 = n_blk * BN + (CG == 2 ? rank * (BN / 2) : 0);
            const int item = static_cast<int>((w - args.unit_begin) / n_workers);
            if (lane == 0) TLB_TRACE(8 + item * 10 + 0);
            // row / batch coordinates of this tile's operand boxes: once per tile, k refreshed per k-block
            int ta[5], tb[5];
            if (!args.a_mn) tile_coords_t<PLAIN>(args.ca, rank_a, false, m0, 0, batch, ta);
            if (!args.b_mn) tile_coords_t<PLAIN>(args.cb, rank_b, false, n0, 0, batch, tb);
            // one operand tile of this k-block: a single box (K-major) or 64-row chunks of [64 k][64 rows] (MN-major)
            auto load_operand = [&](auto cg2, bool mn, const void* map, const TmaCoord* tcd, int rk, uint32_t dst, uint32_t bar,
                                    int row0, int rows, int kb, int* tk, bool hint) {
                constexpr bool CG2 = decltype(cg2)::value;
                if (!mn) {
                    if (kb == kb0 || (args.debug & 64u)) tile_coords_k<PLAIN>(tcd, rk, kb * BK, tk);
                    else tile_coords_step<PLAIN>(tcd, rk, tk);
                    if (hint) tma_load_tile_hint<CG2>(dst, map, bar, rk, tk, pol_ab);
                    else tma_load_tile<CG2>(dst, map, bar, rk, tk);
                } else {
                    int tc[5];
                    for (int c = 0; c < rows / 64; ++c) {
                        tile_coords_t<PLAIN>(tcd, rk, true, row0 + c * 64, kb * BK, batch, tc);
                        tma_load_tile<CG2>(dst + c * 8192, map, bar, rk, tc);
                    }
                }
            };
            for (int kb = kb0; kb < kb1; ++kb) {
                // Stages are released in pairs (one commit per 8 MMAs). The MMA thread commits on the LEADER's
                // barrier only; the leader's producer relays each release to the peer CTA's barrier.
                if ((stage & 1) == 0) {
                    mbar_wait(empty_bar(stage >> 1), phase ^ 1u, args.backoff_ns);
                    if (CG == 2 && leader && ring_wrapped && lane == 0) mbar_arrive_cluster(peer_empty0 + 8u * (stage >> 1));
                }
                if (elect_one()) {
                    if ((args.debug & 1u) && ring_filled) {
                        if (leader) mbar_arrive(full_bar(stage)); // timing experiment: stale smem, no TMA traffic
                    } else if constexpr (CG == 1) {
                        mbar_expect_tx(full_bar(stage), C::kStageBytes);
                        load_operand(std::false_type{}, args.a_mn != 0, &map_a, args.ca, rank_a, a_stage(stage), full_bar(stage), m0, BM, kb, ta, hint_ab);
                        load_operand(std::false_type{}, args.b_mn != 0, &map_b, args.cb, rank_b, b_stage(stage), full_bar(stage), n0, C::kBRows, kb, tb, hint_ab);
                    } else {
                        // The leader's barrier expects the bytes of BOTH CTAs; the peer's TMA may complete before
                        // this expect_tx is issued (tx-count goes transiently negative, as with multicast).
                        const uint32_t lbar = lbar0 + 8u * stage;
                        if (leader) mbar_expect_tx(full_bar(stage), 2 * C::kStageBytes);
                        load_operand(std::true_type{}, args.a_mn != 0, &map_a, args.ca, rank_a, a_stage(stage), lbar, m0, BM, kb, ta, hint_ab);
                        load_operand(std::true_type{}, args.b_mn != 0, &map_b, args.cb, rank_b, b_stage(stage), lbar, n0, C::kBRows, kb, tb, hint_ab);
                    }
                }
                __syncwarp();
                if (stage == C::kStages - 1) ring_filled = true;
                if (++stage == C::kStages) { stage = 0; phase ^= 1u; ring_wrapped = true; }
            }
            if (lane == 0) TLB_TRACE(8 + item * 10 + 1);
        }
    } else if (warp == kMmaWarp) {
        // ===== MMA issuer (leader CTA only under cta_group::2). Control flow is warp-uniform; one elected
        // lane issues the MMAs and the commits (tcgen05.commit tracks the MMAs of the issuing thread). =====
        if (leader) {
            // A / B format fields (bits 7-9, 10-12): 1 = bf16, 0 = fp16
            // K-major tiles: rows of 128 B, 8-row groups 1024 B apart (SBO), a k-step of 16 advances the start by 32 B; MN-major
            // tiles: 64-row chunks of [64 k][128 B], 8-k groups 1024 B apart (SBO), chunks 8192 B apart (LBO), a k-step of 16
            // advances the start by 2 KiB; idesc bits 15 / 16 select MN-major A / B
            const uint32_t idesc = (args.ab_f16 ? (make_idesc<CG, BN>() & ~((1u << 7) | (1u << 10))) : make_idesc<CG, BN>()) |
                                   (args.a_mn ? (1u << 15) : 0u) | (args.b_mn ? (1u << 16) : 0u);
            const uint32_t mn_lbo = (8192u >> 4) << 16;
            const uint32_t a_lo0 = args.a_mn ? (((a_stage(0) >> 4) & 0x3fffu) | mn_lbo) : desc_lo(a_stage(0));
            const uint32_t b_lo0 = args.b_mn ? (((b_stage(0) >> 4) & 0x3fffu) | mn_lbo) : desc_lo(b_stage(0));
            const uint32_t a_kstep = args.a_mn ? (2048u >> 4) : 2u, b_kstep = args.b_mn ? (2048u >> 4) : 2u;
            int stage = 0;
            uint32_t phase = 0, acc = 0, acc_phase = 0;
            for (uint32_t w = args.unit_begin + worker; w < args.work_end; w += n_workers) {
                uint32_t u, batch, m_tile, n_blk;
                int kb0, kb1;
                bool partial;
                decode_work(args, w, kblocks, &u, &kb0, &kb1, &partial);
                decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
                if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
                const int item = static_cast<int>((w - args.unit_begin) / n_workers);
                mbar_wait(tempty_bar(acc), acc_phase ^ 1u); // the epilogue has drained this accumulator
                tc_fence_after();
                if (lane == 0) TLB_TRACE(8 + item * 10 + 2);
                const uint32_t d_tmem = tmem_base + acc * BN;
                // The issuing thread may run 4-5 MMAs ahead of the tensor pipe (measured queue depth), which hides
                // the barrier probe; commits are the expensive part, so a smem PAIR is released per commit.
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(full_bar(stage), phase);
                    tc_fence_after();
                    if (kb == kb0 && lane == 0) TLB_TRACE(8 + item * 10 + 3);
                    if (elect_one()) {
                        const uint32_t a_lo = a_lo0 + stage * (C::kStageBytes >> 4);
                        const uint32_t b_lo = b_lo0 + stage * (C::kStageBytes >> 4);
#pragma unroll
                        for (int k = 0; k < BK / UMMA_K; ++k)
                            umma_bf16<CG>(d_tmem, make_desc(a_lo + a_kstep * k), make_desc(b_lo + b_kstep * k), idesc,
                                          (kb != kb0 || k != 0) ? 1u : 0u);
                        if (stage & 1) umma_commit_local<CG>(empty_bar(stage >> 1)); // both stages of the pair are consumed
                        if (kb == kb1 - 1) umma_commit<CG>(tfull_bar(acc)); // accumulator complete -> epilogue (both CTAs)
                    }
                    __syncwarp();
                    if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
                }
                if (lane == 0) TLB_TRACE(8 + item * 10 + 4);
                acc ^= 1u;
                if (acc == 0) acc_phase ^= 1u;
            }
        }
    } else {
        // ===== epilogue =====
        const uint32_t quad = warp & 3;                         // the TMEM lane quadrant this warp may read
        const uint32_t half = static_cast<uint32_t>(warp) >> 2; // which 128 columns
        const uint32_t row = quad * 32 + lane;
        uint32_t acc = 0, acc_phase = 0;
        const uint32_t tempty_leader = CG == 2 ? map_to_cta(tempty_bar(0), 0) : 0u;
        constexpr int kChunks = BN / 2 / 32;
        if constexpr (EPI == EPI_TMA) {
            // ---- TMEM -> registers -> swizzled smem chunk -> cp.reduce.async.bulk.tensor (C += chunk)
            const bool issuer = (warp & 3) == 0 && lane == 0; // one thread per column half
            const uint32_t bar_id = 1 + half;
            const uint64_t pol_c = policy_evict_first();
            const bool hint_c = (args.hints & 2u) != 0;
            uint32_t chunk_no = 0;
            for (uint32_t w = args.unit_begin + worker; w < args.work_end; w += n_workers) {
                uint32_t u, batch, m_tile, n_blk;
                int kb0, kb1;
                bool partial;
                decode_work(args, w, kblocks, &u, &kb0, &kb1, &partial);
                decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
                if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
                const int item = static_cast<int>((w - args.unit_begin) / n_workers);
                if (warp == 0 && lane == 0) TLB_TRACE(8 + item * 10 + 5);
                mbar_wait(tfull_bar(acc), acc_phase, args.backoff_ns * 4);
                tc_fence_after();
                if (warp == 0 && lane == 0) TLB_TRACE(8 + item * 10 + 6);
                const int m0 = static_cast<int>(m_tile) * BM;
                const int nbase = static_cast<int>(n_blk) * BN + static_cast<int>(half) * (BN / 2);
                // fp32 C: 32-column chunks (128 B rows); 2-byte C: 64-column chunks, two TMEM loads rounded to nearest even
                const int n_chunks = args.c_16 ? kChunks / 2 : kChunks, cw = args.c_16 ? 64 : 32;
#pragma unroll 1
                for (int ci = 0; ci < n_chunks; ++ci, ++chunk_no) {
                    const uint32_t buf = epi_base + (half * C::kEpiBufs + (chunk_no % C::kEpiBufs)) * kEpiChunkBytes;
                    // the TMA store that last used this buffer must have finished reading it
                    if (issuer) bulk_wait_read<C::kEpiBufs - 1>();
                    named_bar(bar_id, 128);
                    uint32_t v[32];
                    const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * BN + half * (BN / 2) + ci * cw;
                    tmem_ld32(taddr, v);
                    if (args.c_16) {
                        uint32_t w[32];
                        tmem_ld32(taddr + 32, w);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            uint32_t lo, hi;
                            if (args.ab_f16) {
                                asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(__uint_as_float(v[2 * j + 1])), "f"(__uint_as_float(v[2 * j])));
                                asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(__uint_as_float(w[2 * j + 1])), "f"(__uint_as_float(w[2 * j])));
                            } else {
                                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(__uint_as_float(v[2 * j + 1])), "f"(__uint_as_float(v[2 * j])));
                                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(__uint_as_float(w[2 * j + 1])), "f"(__uint_as_float(w[2 * j])));
                            }
                            v[j] = lo;        // v[0..15]: columns 0..31 packed, v[16..31]: columns 32..63
                            w[j] = hi;
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[16 + j] = w[j];
                    } else {
                        tmem_ld_wait();
                    }
                    if (ci == n_chunks - 1) {
                        // every TMEM read of this accumulator is done: hand it back to the MMA warp early
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if constexpr (CG == 1) mbar_arrive(tempty_bar(acc));
                            else mbar_arrive_cluster(tempty_leader + 8u * acc);
                        }
                    }
                    if (!(args.debug & (2u | 4u))) {
                        // chunk as (n fastest, m): row = m (128 B), 16-byte chunk c stored at c ^ (m & 7)
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + row * 128u + ((c ^ (row & 7u)) << 4)),
                                         "r"(v[4 * c + 0]), "r"(v[4 * c + 1]), "r"(v[4 * c + 2]), "r"(v[4 * c + 3])
                                         : "memory");
                    }
                    fence_async_smem();
                    named_bar(bar_id, 128);
                    if (issuer && !(args.debug & (2u | 8u))) {
                        int tc[5];
                        tile_coords_t<PLAIN>(args.cc, rank_c, false, m0, nbase + ci * cw, batch, tc);
                        if ((args.debug & 16u) && rank_c == 3)  // timing experiment: plain store instead of the L2 reduction
                            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(&map_c),
                                         "r"(buf), "r"(tc[0]), "r"(tc[1]), "r"(tc[2]) : "memory");
                        else if (hint_c && rank_c == 3) tma_reduce_add_3d_hint(&map_c, buf, tc[0], tc[1], tc[2], pol_c);
                        else tma_reduce_add_tile(&map_c, buf, rank_c, tc);
                        bulk_commit();
                    }
                }
                if (warp == 0 && lane == 0) TLB_TRACE(8 + item * 10 + 7);
                acc ^= 1u;
                if (acc == 0) acc_phase ^= 1u;
            }
            // the staging buffers must have been read before the CTA (and its smem) goes away; the reductions
            // themselves complete asynchronously and are ordered before the end of the grid
            if (issuer) bulk_wait_read<0>();
        } else {
            // ---- register epilogue: C loaded a chunk ahead, added, stored (any strides)
            for (uint32_t w = args.unit_begin + worker; w < args.work_end; w += n_workers) {
                uint32_t u, batch, m_tile, n_blk;
                int kb0, kb1;
                bool partial;
                decode_work(args, w, kblocks, &u, &kb0, &kb1, &partial);
                decode_unit<CG>(args, u, rank, &batch, &m_tile, &n_blk);
                if (CG == 1 && m_tile * BM >= static_cast<uint32_t>(args.M)) continue;
                const int item = static_cast<int>((w - args.unit_begin) / n_workers);
                const int64_t m = static_cast<int64_t>(m_tile) * BM + row;
                float* crow = args.C + batch * args.c_bs + m * args.cs_m;
                const bool m_ok = m < args.M;
                const int64_t nbase = static_cast<int64_t>(n_blk) * BN + half * (BN / 2);
                const bool vec = args.c_vec && m_ok && nbase + BN / 2 <= args.N;
                const bool no_global = (args.debug & 2u) != 0;
                float cur[32], nxt[32];
                auto load_c = [&](int ci, float (&dst)[32]) {
                    const int64_t n0 = nbase + ci * 32;
                    if (vec) {
                        const float4* p = reinterpret_cast<const float4*>(crow + n0);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float4 t = p[j];
                            dst[4 * j + 0] = t.x; dst[4 * j + 1] = t.y; dst[4 * j + 2] = t.z; dst[4 * j + 3] = t.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) dst[j] = (m_ok && n0 + j < args.N) ? crow[(n0 + j) * args.cs_n] : 0.f;
                    }
                };
                if (!partial && !no_global) load_c(0, cur);
                if (warp == 0 && lane == 0) TLB_TRACE(8 + item * 10 + 5);
                mbar_wait(tfull_bar(acc), acc_phase, args.backoff_ns * 4);
                tc_fence_after();
                if (warp == 0 && lane == 0) TLB_TRACE(8 + item * 10 + 6);
#pragma unroll
                for (int ci = 0; ci < kChunks; ++ci) {
                    if (ci + 1 < kChunks && !partial && !no_global) load_c(ci + 1, nxt);
                    uint32_t v[32];
                    __syncwarp(); // tcgen05.ld is .sync.aligned; lanes of an edge tile may have diverged
                    tmem_ld32(tmem_base + ((quad * 32u) << 16) + acc * BN + half * (BN / 2) + ci * 32, v);
                    tmem_ld_wait();
                    const int64_t n0 = nbase + ci * 32;
                    if (no_global) {
                        if (v[0] == 0x7fc12345u) crow[0] = 1.f; // keep the TMEM load alive
                    } else if (partial) {
                        // K-slice of a split tile: several CTAs add into the same C cells -> reductions at L2
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (m_ok && n0 + j < args.N) red_add_f32(crow + (n0 + j) * args.cs_n, __uint_as_float(v[j]));
                    } else if (vec) {
                        float4* p = reinterpret_cast<float4*>(crow + n0);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            p[j] = make_float4(cur[4 * j + 0] + __uint_as_float(v[4 * j + 0]), cur[4 * j + 1] + __uint_as_float(v[4 * j + 1]),
                                               cur[4 * j + 2] + __uint_as_float(v[4 * j + 2]), cur[4 * j + 3] + __uint_as_float(v[4 * j + 3]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (m_ok && n0 + j < args.N) crow[(n0 + j) * args.cs_n] = cur[j] + __uint_as_float(v[j]);
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) cur[j] = nxt[j];
                }
                tc_fence_before();
                __syncwarp();
                if (warp == 0 && lane == 0) TLB_TRACE(8 + item * 10 + 7);
                if (lane == 0) {
                    if constexpr (CG == 1) mbar_arrive(tempty_bar(acc));
                    else mbar_arrive_cluster(tempty_leader + 8u * acc);
                }
                acc ^= 1u;
                if (acc == 0) acc_phase ^= 1u;
            }
        }
    }

    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, kTmemCols);
    }
    if (threadIdx.x == 0) TLB_TRACE(120);
    if (threadIdx.x == 0 && blockIdx.x == 0 && args.clk) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.clk[2] = clock64();
        args.clk[3] = static_cast<long long>(gt);
    }
}

// TLB_GEMM_CLOCK=1: SM clock actually seen by the kernel (cycles of CTA 0 / globaltimer ns), reported at exit.
// The stamps land in mapped pinned host memory, one 4-word slot per launch (ring of 4096).
constexpr int kClkSlots = 4096;
long long* g_clk_host = nullptr;
long long* g_clk_dev = nullptr;
std::atomic<unsigned> g_clk_next{0};
void clk_fetch() {
    cudaDeviceSynchronize();
    cudaMemcpy(g_clk_host, g_clk_dev, kClkSlots * 4 * sizeof(long long), cudaMemcpyDeviceToHost);
}
void clk_report() {
    if (!g_clk_host) return;
    clk_fetch();
    std::vector<double> mhz, us;
    for (int i = 0; i < kClkSlots; ++i) {
        const long long* c = g_clk_host + 4 * i;
        if (c[3] > c[1] && c[2] > c[0]) {
            mhz.push_back(static_cast<double>(c[2] - c[0]) / static_cast<double>(c[3] - c[1]) * 1e3);
            us.push_back(static_cast<double>(c[3] - c[1]) * 1e-3);
        }
    }
    if (mhz.empty()) return;
    std::sort(mhz.begin(), mhz.end());
    std::sort(us.begin(), us.end());
    std::fprintf(stderr, "[tlb gemm clock] %zu launches: SM clock median %.0f MHz (min %.0f, max %.0f); CTA-0 lifetime median %.1f us\n",
                 mhz.size(), mhz[mhz.size() / 2], mhz.front(), mhz.back(), us[us.size() / 2]);
}
long long* clk_slot() {
    static const bool on = [] {
        if (knob(K_GEMM_CLOCK) != 1) return false;
        // device memory, fetched on demand: stamps in mapped host memory would put a PCIe round trip into every
        // kernel's completion (measured: about +4 us per launch)
        const size_t bytes = kClkSlots * 4 * sizeof(long long);
        g_clk_host = static_cast<long long*>(std::malloc(bytes));
        if (!g_clk_host || cudaMalloc(reinterpret_cast<void**>(&g_clk_dev), bytes) != cudaSuccess) return false;
        if (cudaMemset(g_clk_dev, 0, bytes) != cudaSuccess) return false;
        std::memset(g_clk_host, 0, bytes);
        std::atexit(clk_report);
        return true;
    }();
    if (!on) return nullptr;
    return g_clk_dev + 4 * (g_clk_next.fetch_add(1, std::memory_order_relaxed) % kClkSlots);
}

} // namespace

// Tensor maps of the plans, derived from the operand layouts (tlb_tma.cu: tensormap_for_tile): the k-blocks are the tiles
// of zipped_divide(operand, [box_rows, 64]); K-major operands put k in dimension 0, MN-major ones the rows (staged as
// chunks of 64 rows x 64 k); C tiles are zipped_divide(C, [box_m, box_n]) with the contiguous (column) mode innermost.
int umma_operand_map(const UmmaProblem& p, int which, int box_rows, TmaTileMap* out) {
    const tlb_layout_desc& L = which == 0 ? *p.la : *p.lb;
    const bool mn = which == 0 ? p.a_mn != 0 : p.b_mn != 0;
    const void* base = which == 0 ? p.A : p.B;
    const int64_t bs = which == 0 ? p.a_bs : p.b_bs;
    if (!mn) return tensormap_for_tile(L, 1, 0, BK, box_rows, 1, 0, base, p.batch, bs, 2, 1, TMA_SW_128, 256, out);
    return tensormap_for_tile(L, 0, 1, 64, BK, 0, 1, base, p.batch, bs, 2, 1, TMA_SW_128, 256, out);
}
int umma_c_map(const UmmaProblem& p, int box_n, int box_m, int swizzle, TmaTileMap* out) {
    const int cb = p.c_16 ? 2 : 4;
    return tensormap_for_tile(*p.lc, 1 - p.c_row_top, p.c_row_top, box_n, box_m, 1, 0, p.C, p.batch, p.c_bs, cb,
                              p.c_16 && p.ab_f16 ? 2 : 1, swizzle, 0, out);
}

namespace {

int pick_epilogue(const UmmaProblem& p) {
    if (knob(K_GEMM_EPILOGUE) == 1) return EPI_REGS; // "regs": keep C in registers (profiling / A-B comparisons)
    const bool base_ok = (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && (p.batch <= 1 || (p.c_bs % 4 == 0 && p.c_bs > 0));
    if (p.c_16) return EPI_TMA; // umma_c16_applies has checked the TMA constraints
    if (base_ok && p.cs_n == 1 && p.cs_m % 4 == 0 && p.cs_m >= p.N) return EPI_TMA;
    if (base_ok && p.c_fold_tma) return EPI_TMA; // folded C modes with a unit-stride column leaf (GETT-style C)
    return EPI_REGS;
}

template <int CG, int EPI, int BN> int launch(const UmmaProblem& p, cudaStream_t stream) {
    using C = Cfg<CG, EPI, BN>;
    auto* const kern_plain = umma_gemm_kernel<CG, EPI, BN, true>;
    auto* const kern_any = umma_gemm_kernel<CG, EPI, BN, false>;
    static std::atomic<bool> attr_set[64];   // per device; setting the attribute twice from two threads is harmless
    int dev = 0;
    TLB_CUDA(cudaGetDevice(&dev));
    if (dev >= 0 && dev < 64 && !attr_set[dev].load(std::memory_order_acquire)) {
        TLB_CUDA((cudaFuncSetAttribute(kern_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem)));
        TLB_CUDA((cudaFuncSetAttribute(kern_any, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem)));
        attr_set[dev].store(true, std::memory_order_release);
    }
    TmaTileMap ma, mb, mc;
    TLB_TRY(umma_operand_map(p, 0, BM, &ma));
    TLB_TRY(umma_operand_map(p, 1, C::kBRows, &mb));
    if (EPI != EPI_REGS) TLB_TRY(umma_c_map(p, p.c_16 ? 64 : 32, BM, TMA_SW_128, &mc));
    else mc = ma; // unused by the register epilogue
    TLB_TRY(epilogue_partition_check(BN, 1)); // tcgen05.ld partition derived from the accumulator layout (tlb_gemm_layout.cu)
    UmmaArgs a;
    std::memset(&a, 0, sizeof(a));
    a.C = p.C;
    a.cs_m = p.cs_m;
    a.cs_n = p.cs_n;
    a.c_bs = p.c_bs;
    a.M = p.M;
    a.N = p.N;
    a.K = p.K;
    a.ab_f16 = p.ab_f16 ? 1u : 0u;
    a.a_mn = p.a_mn ? 1u : 0u;
    a.b_mn = p.b_mn ? 1u : 0u;
    a.c_16 = p.c_16 ? 1u : 0u;
    a.mb = (p.M + 255) / 256;
    a.nb = (p.N + BN - 1) / BN;
    a.rank_a = ma.rank;
    a.rank_b = mb.rank;
    a.rank_c = mc.rank;
    for (int d = 0; d < 5; ++d) {
        a.ca[d] = ma.c[d];
        a.cb[d] = mb.c[d];
        a.cc[d] = mc.c[d];
    }
    a.group_m = static_cast<uint32_t>(std::max(1, knob(K_GEMM_GROUP_M)));
    a.unit_begin = CG == 1 ? p.tile_begin : p.tile_begin / 2;
    a.unit_end = CG == 1 ? p.tile_end : p.tile_end / 2;
    if (p.full_range) { // tile ids are 128 x 256 tiles; with a 128-column tiler the units are counted from the blocks
        a.unit_begin = 0;
        a.unit_end = a.mb * a.nb * static_cast<uint32_t>(std::max(p.batch, 1)) * (CG == 1 ? 2u : 1u);
    }
    a.c_vec = (p.cs_n == 1 && p.cs_m % 4 == 0 && p.c_bs % 4 == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0) ? 1 : 0;
    const uint32_t units = a.unit_end - a.unit_begin;
    if (units == 0) return TLB_OK;
    const int sms = sm_count();
    // Tail-wave balancing: with W workers, the units of the last partial wave are split along K into slices
    // that run FIRST (so their epilogues overlap later mainloops); slices of one unit combine through the
    // reduce-add epilogue (TMA reduction, or red.global.add with the register epilogue).
    {
        const uint32_t W = CG == 1 ? static_cast<uint32_t>(sms) : static_cast<uint32_t>(sms / 2);
        const uint32_t tail = units % W;
        const int kblocks = (p.K + BK - 1) / BK;
        uint32_t split = 1;
        // (2-byte C: every K-slice would be one more rounding at L2, so tiles are never split)
        if (p.split_tail && !p.c_16 && tail > 0 && units > W) {
            split = W / tail;
            split = std::min<uint32_t>(split, 4);
            while (split > 1 && kblocks / static_cast<int>(split) < 8) --split;
        }
        a.split = split;
        a.n_split_units = split > 1 ? tail : 0;
        a.work_end = a.unit_begin + (units - a.n_split_units) + a.n_split_units * split;
    }
    a.backoff_ns = static_cast<uint32_t>(knob(K_GEMM_BACKOFF_NS));
    a.debug = static_cast<uint32_t>(knob(K_GEMM_DEBUG));
    a.hints = static_cast<uint32_t>(knob(K_GEMM_HINTS));
    a.clk = clk_slot();
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    const uint32_t work = a.work_end - a.unit_begin;
    if (CG == 1) {
        cfg.gridDim = dim3(std::min<uint32_t>(work, static_cast<uint32_t>(sms)));
        cfg.numAttrs = 0;
        cfg.attrs = attr;
    } else {
        cfg.gridDim = dim3(2 * std::min<uint32_t>(work, static_cast<uint32_t>(sms / 2)));
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    if (umma_pdl_enabled()) {
        attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
        ++cfg.numAttrs;
    }
    cfg.blockDim = dim3(kUmmaThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    CUtensorMap tma, tmb, tmc;
    std::memcpy(&tma, ma.desc, 128);
    std::memcpy(&tmb, mb.desc, 128);
    std::memcpy(&tmc, mc.desc, 128);
    // Debug timeline: TLB_GEMM_TRACE=<file> makes this launch synchronous and dumps per-CTA clock64 stamps.
    static const char* const trace_path = std::getenv("TLB_GEMM_TRACE"); // debug timeline: read once per process
    const size_t trace_bytes = static_cast<size_t>(cfg.gridDim.x) * kTraceSlots * sizeof(long long);
    if (trace_path && trace_path[0]) {
        TLB_CUDA(cudaMalloc(reinterpret_cast<void**>(&a.trace), trace_bytes));
        TLB_CUDA(cudaMemset(a.trace, 0, trace_bytes));
    }
    // plain (unfolded) operands and C: the coordinates of every map are the kernel's loop variables (tile_coords_t)
    const bool plain = tma_map_is_plain(ma, p.a_mn != 0) && tma_map_is_plain(mb, p.b_mn != 0) && (EPI == EPI_REGS || tma_map_is_plain(mc, false));
    TLB_CUDA((cudaLaunchKernelEx(&cfg, plain ? kern_plain : kern_any, tma, tmb, tmc, a)));
    count_launch();
    static const char* const names[2][2][2] = {{{"umma_1sm_regs", "umma_1sm"}, {"umma_2sm_regs", "umma_2sm"}},
                                               {{"umma_1sm_n128_regs", "umma_1sm_n128"}, {"umma_2sm_n128_regs", "umma_2sm_n128"}}};
    set_plan(names[BN == 128 ? 1 : 0][CG - 1][EPI]);
    if (a.trace) {
        std::vector<long long> h(trace_bytes / sizeof(long long));
        TLB_CUDA(cudaStreamSynchronize(stream));
        TLB_CUDA(cudaMemcpy(h.data(), a.trace, trace_bytes, cudaMemcpyDeviceToHost));
        cudaFree(a.trace);
        if (FILE* f = std::fopen(trace_path, "wb")) {
            const long long hdr[4] = {static_cast<long long>(cfg.gridDim.x), kTraceSlots, CG, static_cast<long long>(a.split)};
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::fwrite(h.data(), 1, trace_bytes, f);
            std::fclose(f);
        }
    }
    return TLB_OK;
}

template <int CG> int launch_cg(const UmmaProblem& p, cudaStream_t stream) {
    const bool tma = pick_epilogue(p) == EPI_TMA;
    if (p.bn == 128) return tma ? launch<CG, EPI_TMA, 128>(p, stream) : launch<CG, EPI_REGS, 128>(p, stream);
    return tma ? launch<CG, EPI_TMA, 256>(p, stream) : launch<CG, EPI_REGS, 256>(p, stream);
}

} // namespace

long long* umma_clk_slot() { return clk_slot(); }
// 2-byte C on the 256 x 256 plans: the TMA reduce-add epilogue must be able to address it (n-contiguous rows that are
// multiples of 16 bytes, or folded modes the rank-4/5 map covers).
bool umma_c16_applies(const UmmaProblem& p) {
    const bool base_ok = (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && (p.batch <= 1 || (p.c_bs % 8 == 0 && p.c_bs > 0));
    if (!p.c_16 || !base_ok) return false;
    if (p.c_fold_tma) return true;
    return p.cs_n == 1 && p.cs_m % 8 == 0 && p.cs_m >= p.N;
}
// TLB_GEMM_PDL=0 turns programmatic dependent launch off (A/B comparisons).
bool umma_pdl_enabled() { return knob(K_GEMM_PDL) != 0; }

} // namespace tlb

extern "C" int tlb_gemm_clock_stats(double* median_mhz, double* median_us, uint32_t* launches) {
    using namespace tlb;
    if (!median_mhz || !median_us || !launches) return fail(TLB_ERR_CONTRACT, "tlb_gemm_clock_stats: null output");
    *median_mhz = *median_us = 0.0;
    *launches = 0;
    if (!g_clk_host) return TLB_OK;
    clk_fetch();
    TLB_CUDA(cudaMemset(g_clk_dev, 0, kClkSlots * 4 * sizeof(long long)));
    std::vector<double> mhz, us;
    for (int i = 0; i < kClkSlots; ++i) {
        long long* c = g_clk_host + 4 * i;
        if (c[3] > c[1] && c[2] > c[0]) {
            mhz.push_back(static_cast<double>(c[2] - c[0]) / static_cast<double>(c[3] - c[1]) * 1e3);
            us.push_back(static_cast<double>(c[3] - c[1]) * 1e-3);
        }
    }
    if (mhz.empty()) return TLB_OK;
    std::sort(mhz.begin(), mhz.end());
    std::sort(us.begin(), us.end());
    *median_mhz = mhz[mhz.size() / 2];
    *median_us = us[us.size() / 2];
    *launches = static_cast<uint32_t>(mhz.size());
    return TLB_OK;
}

namespace tlb {

int umma_gemm_launch(const UmmaProblem& p, cudaStream_t stream) {
    if (umma_wide_applies(p)) return umma_wide_launch(p, stream);
    if (p.cta_group == 2) return launch_cg<2>(p, stream);
    return launch_cg<1>(p, stream);
}

} // namespace tlb

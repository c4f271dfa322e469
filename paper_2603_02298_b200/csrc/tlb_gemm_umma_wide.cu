// tcgen05 GEMM, wide plan: a CTA PAIR owns a 512 x 256 tile of C (256 rows per CTA), bf16 or fp16 operands that are
// K-major or MN-major, fp32 accumulators that fill all of TMEM.        C(m,n) += sum_k A(m,k) * B(n,k)      (tensor.hpp:214-233)
//
// Why this shape: on a 1 kW part the kernel is POWER bound (SM clock 1.5 GHz under load, MMA duty cycle < 80 %),
// so the figure of merit is energy per flop, and operand movement is the largest controllable term. A 512 x 256
// pair tile moves (512 + 256) / (512 * 256) operand bytes per MAC against (256 + 256) / (256 * 256) for the
// 256 x 256 tile of tlb_gemm_umma.cu: 25 % less L2 -> SM traffic and shared-memory fill for the same math.
//
// Partitioning in the paper's terms: zipped_divide(C, [512,256]) are the pair tiles,
// zipped_divide(A, [256,64]) / (B, [128,64]) the per-CTA k-blocks (the TMA boxes), and the TiledMMA is the 2-CTA
// UMMA atom 256 x 256 x 16 applied to the two 128-row halves h of each CTA: half h of both CTAs forms one
// cta_group::2 instruction whose accumulator lives in TMEM columns [256 h, 256 h + 256) of each CTA.
//
// Kernel shape (persistent, warp-specialised, 320 threads, 1 CTA per SM, clusters of 2):
//   warp 8     TMA producer: 4-stage ring of {A 256 x 64, B 128 x 64} stages (48 KiB), full / empty mbarriers
//              (MN-major operands arrive as 64-row chunks of [64 k][128 B]); optional L2 prefetch of the tile's C
//              cells (TLB_GEMM_PREFETCH_C=1; off: measured, it evicts operand lines and loses 1.5-7 %)
//   warp 9     MMA issue (leader CTA): per k-block 4 + 4 UMMAs (half 0, half 1), ONE non-multicast commit per
//              stage (a commit every 8 MMAs is free, a multicast commit is not: tools/probes/mma_rate.cu);
//              the leader's producer relays each stage release to the peer CTA
//   warps 0-7  epilogue: warp w drains TMEM lane quadrant w % 4, columns [128 (w / 4), +128) of each half through
//              a PRIVATE 4 KiB staging tile (32 rows x 32 columns, 128-byte swizzle) and its own
//              cp.reduce.async.bulk.tensor (C += chunk at L2): no CTA-wide barriers in the epilogue
// The accumulators are single-buffered, so a tile's epilogue is overlapped per HALF: half 0 is released to the
// epilogue one k-block early, and the next tile's half-0 MMAs of the first kStages-1 k-blocks are issued while
// half 1 is still being drained.
// Scheduling: the last (units mod workers) tiles are cut stream-K style into one k-range per worker, balanced by cost
// (every tile a range touches is one more epilogue), and run FIRST; whole tiles follow round-robin. Partial tiles
// combine through the same reduce-add epilogue. The prologue overlaps the previous kernel's tail (griddepcontrol).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>

#include "tlb_internal.h"
#include "tlb_gemm.h"
#include "tlb_umma_ptx.h"

namespace tlb {
namespace {
using namespace umma;

constexpr int BMH = 128;           // rows per accumulator half
constexpr int BMC = 2 * BMH;       // rows of C per CTA
constexpr int BN = 256;            // columns of C per pair (UMMA N)
constexpr int BK = 64;             // one 128-byte swizzle row of bf16
constexpr int UMMA_K = 16;
#ifndef TLB_WIDE_STAGES
#define TLB_WIDE_STAGES 4
#endif
constexpr int kStages = TLB_WIDE_STAGES;
constexpr int kEpiBufs = kStages == 3 ? 2 : 1; // private staging tiles per epilogue warp
constexpr int kEpiWarps = 8;
constexpr int kThreadsW = 64 + 32 * kEpiWarps;
constexpr int kProducerWarp = kEpiWarps;
constexpr int kMmaWarp = kEpiWarps + 1;
constexpr uint32_t kABytes = BMC * BK * 2;        // 32 KiB
constexpr uint32_t kBBytes = (BN / 2) * BK * 2;   // 16 KiB: this CTA's half of B
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kEpiWarpBytes = 32 * 32 * 4;   // 4 KiB private staging tile per epilogue warp
constexpr uint32_t kSmemW = kStages * kStageBytes + kEpiWarps * kEpiBufs * kEpiWarpBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kMaxWorkers = 80;                   // CTA pairs (74 on a 148-SM part)
constexpr int kMinSeg = 4;                        // stream-K cuts closer than this to a tile boundary snap to it

struct WideArgs {
    int32_t M, N, K;
    uint32_t mbw, nb;         // 512-row pair tiles along m, 256-column blocks along n
    uint32_t group_w;         // pair tiles (along m) per rasterisation group
    uint32_t ab_f16;          // operands are fp16 instead of bf16
    uint32_t c_16;            // C has the operands' 2-byte type: the epilogue rounds to it, 64-column chunks
    uint32_t a_mn, b_mn;      // operand is MN-major: staged as 64-row chunks of [64 k][128 B], MN-major UMMA descriptors
    uint32_t unit_begin;      // first 512 x 256 pair tile of the range (all batches)
    uint32_t dp_units;        // whole tiles, dealt round-robin
    uint32_t sk_units;        // the tiles after them, cut into one k-range per worker
    uint32_t prefetch_c;      // > 0: map_cp is valid; 1: prefetch this tile's C cells into L2 at the tile's start, n > 1: n k-blocks before its end
    uint32_t early_release;   // fp32 C: drain a half to registers and release its TMEM before the reductions (GEMM_EARLY_RELEASE)
    uint32_t hints;           // L2 hints: 1 = operand loads evict_last, 2 = C reductions evict_first
    uint32_t debug;           // TLB_GEMM_DEBUG timing experiments (garbage results): 1 = no TMA loads once the ring is
                              // full, 2 = epilogue without staging / reductions, 4 = plain TMA store instead of reduce-add, 8 = staging only, 32 = all reductions into the first tile
    uint32_t sk_cut[kMaxWorkers + 1]; // k-range [sk_cut[w], sk_cut[w+1]) of the stream-K tiles owned by worker w
    long long* clk;
    long long* cta_times;     // optional (TLB_GEMM_CTA_TIMES=<file>): {globaltimer at entry, at exit} of every CTA
    // how a tile's (row, k | column, batch) start turns into the coordinates of the layout-derived tensor maps
    int32_t rank_a, rank_b, rank_c;
    TmaCoord ca[5], cb[5], cc[5];
};

struct Item {
    uint32_t unit;
    int kb0, kb1;
};

// Work list of one worker, as an iterator every role walks identically: first its k-range of the stream-K tiles (the
// partial wave), cut at tile boundaries, then its whole tiles, round-robin.
struct Sched {
    uint64_t sk_lo, sk_hi;
    uint32_t n_workers, dp_next;
    __device__ void init(const WideArgs& a, uint32_t w, uint32_t W) {
        n_workers = W;
        dp_next = w;
        sk_lo = sk_hi = 0;
        if (a.sk_units) {
            sk_lo = a.sk_cut[w];
            sk_hi = a.sk_cut[w + 1];
        }
    }
    __device__ __forceinline__ bool next(const WideArgs& a, int kblocks, Item* it) {
        if (sk_lo < sk_hi) {
            const uint32_t t = static_cast<uint32_t>(sk_lo / kblocks);
            it->kb0 = static_cast<int>(sk_lo % kblocks);
            it->kb1 = static_cast<int>(min(static_cast<uint64_t>(kblocks), it->kb0 + (sk_hi - sk_lo)));
            it->unit = a.unit_begin + a.dp_units + t;
            sk_lo += static_cast<uint64_t>(it->kb1 - it->kb0);
            return true;
        }
        if (dp_next < a.dp_units) {
            it->unit = a.unit_begin + dp_next;
            it->kb0 = 0;
            it->kb1 = kblocks;
            dp_next += n_workers;
            return true;
        }
        return false;
    }
};

// pair tile id -> (batch, first 128-row tile index (multiple of 4), 256-column block). Pair tiles are walked in groups
// of group_w tiles along m, m fastest inside a group, then n: when ceil(M/256) is even this is exactly the order of the
// 128 x 256 tile ids of tlb_gemm.h (pair tile g = tiles 4g .. 4g+3), which is what lets tile-id ranges select pair tiles.
__device__ __forceinline__ void decode_pair_tile(const WideArgs& a, uint32_t g, uint32_t* batch, uint32_t* m_tile, uint32_t* n_blk) {
    const uint32_t tiles = a.mbw * a.nb;
    *batch = g / tiles;
    const uint32_t t = g % tiles;
    const uint32_t per = a.group_w * a.nb;
    const uint32_t grp = t / per, rem = t % per;
    const uint32_t gw = min(a.group_w, a.mbw - grp * a.group_w);
    *m_tile = (grp * a.group_w + rem % gw) * 4;
    *n_blk = rem / gw;
}

__device__ __forceinline__ void tma_prefetch_3d(const void* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
// Sleeping wait: try_wait suspends the thread in hardware for up to the hint (ns) instead of spinning.
__device__ __forceinline__ bool mbar_try_sleep(uint32_t bar, uint32_t parity, uint32_t hint_ns) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(hint_ns)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const long long t0 = clock64();
    for (;;) {
        if (mbar_try_sleep(bar, parity, 20000u)) return;
        if (clock64() - t0 > 6000000000ll) __trap();
    }
}

constexpr uint32_t kIdescW = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(256 >> 4) << 24);

// PLAIN (tile_coords_t, tlb_umma_ptx.h): all three tensor maps are rank 3 with identity coordinates (unfolded operands, the
// common case): the general rank 3..5 decomposition is compiled out of the producer's and the epilogue's loops.
// MC (clusters of 4 = two CTA pairs on n-adjacent pair tiles, K-major plain operands): the two pairs need the same 512
// rows of A, so every CTA loads only a QUARTER of them (128 rows x 64 k, 16 KiB) and multicasts it to its counterpart in
// the other pair: L2 -> SM requests per CTA and k-block drop from 48 KiB to 32 KiB (the cluster tile is 512 x 512). A
// stage is then written by CTAs of BOTH pairs, so it is released only when both pairs' MMAs have consumed it: the MMA
// thread commits on its leader's `done` barrier, the leader's producer relays that to the `empty` barrier (count 2) of
// all four CTAs.
template <bool PLAIN, bool MC>
__global__ void __launch_bounds__(kThreadsW, 1)
umma_wide_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_cp,
                 const __grid_constant__ WideArgs args) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t epi_base = smem_base + kStages * kStageBytes;
    const uint32_t bar_base = epi_base + kEpiWarps * kEpiBufs * kEpiWarpBytes;
    auto a_stage = [&](int s) { return smem_base + s * kStageBytes; };
    auto b_stage = [&](int s) { return smem_base + s * kStageBytes + kABytes; };
    auto full_bar = [&](int s) { return bar_base + 8u * s; };
    auto empty_bar = [&](int s) { return bar_base + 8u * (kStages + s); };
    auto tfull_bar = [&](int h) { return bar_base + 8u * (2 * kStages + h); };
    auto tempty_bar = [&](int h) { return bar_base + 8u * (2 * kStages + 2 + h); };
    const uint32_t tmem_slot = bar_base + 8u * (2 * kStages + 4);
    auto done_bar = [&](int s) { return bar_base + 8u * (2 * kStages + 5 + s); };   // MC only, pair leaders

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();           // 0..3 with MC, 0..1 otherwise
    const uint32_t pair = MC ? crank >> 1 : 0u;      // which CTA pair of the cluster
    const uint32_t rank = crank & 1u;                // position inside the pair
    const uint32_t lead_cta = pair * 2u;             // cluster rank of this pair's leader
    const bool leader = rank == 0;
    constexpr uint32_t kCluster = MC ? 4u : 2u;
    const uint32_t n_workers = gridDim.x / kCluster, worker = blockIdx.x / kCluster;
    const int kblocks = (args.K + BK - 1) / BK;
    const int rank_a = PLAIN ? 3 : args.rank_a, rank_b = PLAIN ? 3 : args.rank_b, rank_c = PLAIN ? 3 : args.rank_c;
    if (threadIdx.x == 0 && args.cta_times) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.cta_times[2 * blockIdx.x] = static_cast<long long>(gt);
    }

    if (warp == kProducerWarp && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_c) : "memory");
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full_bar(s), 1);  // the leader's producer arrive; the TMA bytes of both CTAs complete the phase
            mbar_init(empty_bar(s), MC ? 2 : 1); // one tcgen05.commit (leader) / one relayed arrive (peer); MC: one relay per pair
            if (MC) mbar_init(done_bar(s), 1);   // this pair's tcgen05.commit
        }
        for (int h = 0; h < 2; ++h) {
            mbar_init(tfull_bar(h), 1);              // one multicast tcgen05.commit
            mbar_init(tempty_bar(h), kEpiWarps * 2); // one lane of every epilogue warp of both CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) tmem_alloc<2>(tmem_slot, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));
    // everything above (barriers, TMEM, cluster handshake) may overlap the tail of the previous kernel of the stream
    griddep_wait();
    griddep_launch_dependents();
    if (threadIdx.x == 0 && blockIdx.x == 0 && args.clk) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.clk[0] = clock64();
        args.clk[1] = static_cast<long long>(gt);
    }

    Sched sched;
    sched.init(args, worker, n_workers);

    if (warp == kProducerWarp) {
        // ===== TMA producer (whole warp in the loops, one elected lane issues) =====
        int stage = 0;
        uint32_t phase = 0;
        bool ring_wrapped = false;
        const uint32_t peer_empty0 = map_to_cta(empty_bar(0), lead_cta + 1);
        const uint32_t lbar0 = map_to_cta(full_bar(0), lead_cta);
        uint32_t all_empty0[4] = {0, 0, 0, 0};
        if constexpr (MC)
            for (uint32_t c = 0; c < 4; ++c) all_empty0[c] = map_to_cta(empty_bar(0), c);
        const uint16_t a_mask = static_cast<uint16_t>((1u << crank) | (1u << (crank ^ 2u))); // this CTA and its counterpart
        const uint64_t pol_ab = policy_evict_last();
        Item it;
        while (sched.next(args, kblocks, &it)) {
            uint32_t batch, m_tile, n_blk;
            decode_pair_tile(args, it.unit, &batch, &m_tile, &n_blk);
            if constexpr (MC) n_blk = n_blk * 2 + pair;   // units are 512 x 512 cluster tiles
            const int m0 = static_cast<int>(m_tile) * BMH + static_cast<int>(rank) * BMC;
            const int n0 = static_cast<int>(n_blk) * BN;
            if (args.prefetch_c == 1 && lane < 2) {
                // this CTA's 256 x 256 cells of C -> L2 (two 128-row boxes), long before the reductions need them
                tma_prefetch_3d(&map_cp, n0, m0 + lane * BMH, static_cast<int>(batch));
            }
            // row / batch coordinates of this tile's K-major operand boxes: once per tile, k refreshed per k-block
            const int nb0 = n0 + static_cast<int>(rank) * (BN / 2);
            int tca[5], tcb[5];
            if (!args.a_mn) tile_coords_t<PLAIN>(args.ca, rank_a, false, m0, 0, batch, tca);
            if (!args.b_mn) tile_coords_t<PLAIN>(args.cb, rank_b, false, nb0, 0, batch, tcb);
            const int kb_pf = args.prefetch_c > 1 ? max(it.kb0, it.kb1 - static_cast<int>(args.prefetch_c)) : -1;
            for (int kb = it.kb0; kb < it.kb1; ++kb) {
                // late prefetch: the tile's C cells reach L2 shortly before the reduce-add epilogue needs them (the L2
                // then adds in place instead of fetching each line from DRAM under the atomics)
                if (kb == kb_pf && lane < 2) tma_prefetch_3d(&map_cp, n0, m0 + lane * BMH, static_cast<int>(batch));
                if constexpr (MC) {
                    if (leader && ring_wrapped) {
                        mbar_wait(done_bar(stage), phase ^ 1u, 64);   // this pair's MMAs have consumed the stage ...
                        if (elect_one()) {
#pragma unroll
                            for (uint32_t c = 0; c < 4; ++c) mbar_arrive_cluster(all_empty0[c] + 8u * stage); // ... tell all four CTAs
                        }
                        __syncwarp();
                    }
                }
                mbar_wait(empty_bar(stage), phase ^ 1u, 64);
                if (elect_one()) {
                    if (!MC && leader && ring_wrapped) mbar_arrive_cluster(peer_empty0 + 8u * stage); // relay the release
                    if ((args.debug & 1u) && ring_wrapped) {
                        if (leader) mbar_arrive(full_bar(stage)); // timing experiment: stale smem, no TMA traffic
                    } else {
                        const uint32_t lbar = lbar0 + 8u * stage;
                        if (leader) mbar_expect_tx(full_bar(stage), 2 * kStageBytes);
                        int tc[5];
                        if constexpr (MC) {
                            // this CTA's quarter of the cluster's A rows -> the same half slot of this CTA and of its counterpart
                            tma_load_3d_2sm_mc(a_stage(stage) + pair * (BMH * BK * 2), &map_a, lbar, kb * BK, m0 + static_cast<int>(pair) * BMH,
                                               static_cast<int>(batch), a_mask);
                        } else if (!args.a_mn) {
                            // K-major A: one box of 256 rows x 64 k (rows of 128 B)
                            if (kb == it.kb0 || (args.debug & 64u)) tile_coords_k<PLAIN>(args.ca, rank_a, kb * BK, tca);
                            else tile_coords_step<PLAIN>(args.ca, rank_a, tca);
                            if (args.hints & 1u) tma_load_tile_hint<true>(a_stage(stage), &map_a, lbar, rank_a, tca, pol_ab);
                            else tma_load_tile<true>(a_stage(stage), &map_a, lbar, rank_a, tca);
                        } else {
                            // MN-major A: four chunks of 64 rows, each [64 k][64 m] (the map's dimension 0 is m)
#pragma unroll
                            for (int c = 0; c < BMC / 64; ++c) {
                                tile_coords_t<PLAIN>(args.ca, rank_a, true, m0 + c * 64, kb * BK, batch, tc);
                                tma_load_tile<true>(a_stage(stage) + c * 8192, &map_a, lbar, rank_a, tc);
                            }
                        }
                        if (!args.b_mn) {
                            if (kb == it.kb0 || (args.debug & 64u)) tile_coords_k<PLAIN>(args.cb, rank_b, kb * BK, tcb);
                            else tile_coords_step<PLAIN>(args.cb, rank_b, tcb);
                            if (args.hints & 1u) tma_load_tile_hint<true>(b_stage(stage), &map_b, lbar, rank_b, tcb, pol_ab);
                            else tma_load_tile<true>(b_stage(stage), &map_b, lbar, rank_b, tcb);
                        } else {
#pragma unroll
                            for (int c = 0; c < BN / 2 / 64; ++c) {
                                tile_coords_t<PLAIN>(args.cb, rank_b, true, nb0 + c * 64, kb * BK, batch, tc);
                                tma_load_tile<true>(b_stage(stage) + c * 8192, &map_b, lbar, rank_b, tc);
                            }
                        }
                    }
                }
                __syncwarp();
                if (++stage == kStages) { stage = 0; phase ^= 1u; ring_wrapped = true; }
            }
        }
    } else if (warp == kMmaWarp) {
        // ===== MMA issuer (leader CTA). Warp-uniform control flow, one elected lane issues. =====
        if (leader) {
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            const uint16_t pair_mask = static_cast<uint16_t>(3u << lead_cta); // both CTAs of THIS pair
            // 4 UMMAs of k-block `kb` in ring slot s into accumulator half h
            // Descriptors: K-major tiles are rows of 128 B with 8-row groups 1024 B apart (SBO), a k-step of 16 advances
            // the start by 32 B; MN-major tiles are 64-row chunks of [64 k][128 B]: 8-k groups 1024 B apart (SBO), chunks
            // 8192 B apart (LBO), a k-step of 16 advances the start by 2 KiB. idesc bits 15 / 16 select MN-major A / B.
            const uint32_t idesc = (args.ab_f16 ? (kIdescW & ~((1u << 7) | (1u << 10))) : kIdescW) | (args.a_mn ? (1u << 15) : 0u) |
                                   (args.b_mn ? (1u << 16) : 0u);
            const uint32_t a_lbo = args.a_mn ? ((8192u >> 4) << 16) : (1u << 16), b_lbo = args.b_mn ? ((8192u >> 4) << 16) : (1u << 16);
            const uint32_t a_kstep = args.a_mn ? (2048u >> 4) : 2u, b_kstep = args.b_mn ? (2048u >> 4) : 2u;
            const uint32_t a_base = ((a_stage(0) >> 4) & 0x3fffu), b_base = ((b_stage(0) >> 4) & 0x3fffu);
            auto issue_half = [&](int s, int h, bool first_kb) {
                const uint32_t a_lo = (a_base + s * (kStageBytes >> 4) + h * ((BMH * BK * 2) >> 4)) | a_lbo;
                const uint32_t b_lo = (b_base + s * (kStageBytes >> 4)) | b_lbo;
                const uint32_t d_tmem = tmem_base + h * BN;
#pragma unroll
                for (int k = 0; k < BK / UMMA_K; ++k)
                    umma_bf16<2>(d_tmem, make_desc(a_lo + a_kstep * k), make_desc(b_lo + b_kstep * k), idesc, (first_kb && k == 0) ? 0u : 1u);
            };
            Item it;
            while (sched.next(args, kblocks, &it)) {
                const int n = it.kb1 - it.kb0;
                const int pre = min(n, kStages - 1);
                // --- head: half-0 MMAs of the first `pre` k-blocks run while the epilogue still drains half 1
                mbar_wait(tempty_bar(0), acc_phase ^ 1u);
                tc_fence_after();
                {
                    int s = stage;
                    uint32_t ph = phase;
                    for (int j = 0; j < pre; ++j) {
                        mbar_wait(full_bar(s), ph);
                        tc_fence_after();
                        if (elect_one()) {
                            issue_half(s, 0, j == 0);
                            if (j == n - 1) umma_commit<2>(tfull_bar(0), pair_mask);
                        }
                        __syncwarp();
                        if (++s == kStages) { s = 0; ph ^= 1u; }
                    }
                }
                mbar_wait(tempty_bar(1), acc_phase ^ 1u);
                tc_fence_after();
                for (int j = 0; j < pre; ++j) {
                    if (elect_one()) {
                        issue_half(stage, 1, j == 0);
                        umma_commit_local<2>(MC ? done_bar(stage) : empty_bar(stage)); // both halves of this stage are consumed
                        if (j == n - 1) umma_commit<2>(tfull_bar(1), pair_mask);
                    }
                    __syncwarp();
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
                // --- steady state
                for (int j = pre; j < n; ++j) {
                    mbar_wait(full_bar(stage), phase);
                    tc_fence_after();
                    if (elect_one()) {
                        issue_half(stage, 0, false);
                        if (j == n - 1) umma_commit<2>(tfull_bar(0), pair_mask); // half 0 complete: its epilogue starts a k-block early
                        issue_half(stage, 1, false);
                        umma_commit_local<2>(MC ? done_bar(stage) : empty_bar(stage));
                        if (j == n - 1) umma_commit<2>(tfull_bar(1), pair_mask);
                    }
                    __syncwarp();
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
                acc_phase ^= 1u;
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> private swizzled 4 KiB tile -> cp.reduce.async.bulk.tensor (C += tile)
        const uint32_t quad = warp & 3;                         // TMEM lane quadrant this warp may read
        const uint32_t colh = static_cast<uint32_t>(warp) >> 2; // which 128 columns of a half
        const uint32_t buf0 = epi_base + static_cast<uint32_t>(warp) * kEpiBufs * kEpiWarpBytes;
        uint32_t chunk_no = 0;
        const uint32_t tempty_leader = map_to_cta(tempty_bar(0), lead_cta);
        const uint64_t pol_c = policy_evict_first();
        const uint32_t row = lane;
        uint32_t acc_phase = 0;
        Item it;
        while (sched.next(args, kblocks, &it)) {
            uint32_t batch, m_tile, n_blk;
            decode_pair_tile(args, it.unit, &batch, &m_tile, &n_blk);
            if constexpr (MC) n_blk = n_blk * 2 + pair;
            int m0 = static_cast<int>(m_tile) * BMH + static_cast<int>(rank) * BMC + static_cast<int>(quad) * 32;
            int n0 = static_cast<int>(n_blk) * BN + static_cast<int>(colh) * (BN / 2);
            if (args.debug & 32u) {  // timing experiment: every CTA reduces into the first tile (L2-resident, no DRAM traffic)
                m0 = static_cast<int>(rank) * BMC + static_cast<int>(quad) * 32;
                n0 = static_cast<int>(colh) * (BN / 2);
            }
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                mbar_wait_sleep(tfull_bar(h), acc_phase);
                tc_fence_after();
                if (args.c_16) {
                    // C in the operands' 2-byte type: two 32-column TMEM loads make one staged row of 64 cells (128 B),
                    // rounded to nearest even from the fp32 accumulator; the TMA reduction adds in that type at L2.
#pragma unroll 1
                    for (int ci = 0; ci < 2; ++ci, ++chunk_no) {
                        const uint32_t buf = buf0 + (chunk_no % kEpiBufs) * kEpiWarpBytes;
                        uint32_t v[32], w[32];
                        const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + h * BN + colh * (BN / 2) + ci * 64;
                        tmem_ld32(taddr, v);
                        tmem_ld32(taddr + 32, w);
                        if (lane == 0) bulk_wait_read<kEpiBufs - 1>();
                        tmem_ld_wait();
                        if (ci == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(tempty_leader + 8u * h);
                        } else {
                            __syncwarp();
                        }
                        uint32_t pk[32];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (args.ab_f16) {
                                asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(pk[j]) : "f"(__uint_as_float(v[2 * j + 1])), "f"(__uint_as_float(v[2 * j])));
                                asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(pk[16 + j]) : "f"(__uint_as_float(w[2 * j + 1])), "f"(__uint_as_float(w[2 * j])));
                            } else {
                                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk[j]) : "f"(__uint_as_float(v[2 * j + 1])), "f"(__uint_as_float(v[2 * j])));
                                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk[16 + j]) : "f"(__uint_as_float(w[2 * j + 1])), "f"(__uint_as_float(w[2 * j])));
                            }
                        }
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + row * 128u + ((c ^ (row & 7u)) << 4)),
                                         "r"(pk[4 * c + 0]), "r"(pk[4 * c + 1]), "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3])
                                         : "memory");
                        fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            int tc[5];
                            tile_coords_t<PLAIN>(args.cc, rank_c, false, m0 + h * BMH, n0 + ci * 64, batch, tc);
                            tma_reduce_add_tile(&map_c, buf, rank_c, tc);
                            bulk_commit();
                        }
                    }
                    continue;
                }
                if (args.early_release) {
                    // The warp's whole share of this half (32 lanes x 128 columns) goes to REGISTERS first (4 x 32 fp32 per
                    // thread: the epilogue warps have the budget, 1 CTA per SM), the half is handed back to the MMA warp
                    // at once, and only then do the four chunks trickle through the staging tile at the pace of the L2
                    // reductions. TMEM is free ~0.5 k cycles after the half completes instead of after three reductions.
                    uint32_t v[4][32];
                    const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + h * BN + colh * (BN / 2);
#pragma unroll
                    for (int ci = 0; ci < 4; ++ci) tmem_ld32(taddr + ci * 32, v[ci]);
                    tmem_ld_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader + 8u * h);
#pragma unroll
                    for (int ci = 0; ci < 4; ++ci, ++chunk_no) {
                        const uint32_t buf = buf0 + (chunk_no % kEpiBufs) * kEpiWarpBytes;
                        if (lane == 0) bulk_wait_read<kEpiBufs - 1>(); // the reduction that last used this staging tile has read it
                        __syncwarp();
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + row * 128u + ((c ^ (row & 7u)) << 4)),
                                         "r"(v[ci][4 * c + 0]), "r"(v[ci][4 * c + 1]), "r"(v[ci][4 * c + 2]), "r"(v[ci][4 * c + 3])
                                         : "memory");
                        fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            int tc[5];
                            tile_coords_t<PLAIN>(args.cc, rank_c, false, m0 + h * BMH, n0 + ci * 32, batch, tc);
                            if ((args.hints & 2u) && rank_c == 3) tma_reduce_add_3d_hint(&map_c, buf, tc[0], tc[1], tc[2], pol_c);
                            else tma_reduce_add_tile(&map_c, buf, rank_c, tc);
                            bulk_commit();
                        }
                    }
                    continue;
                }
#pragma unroll 1
                for (int ci = 0; ci < 4; ++ci, ++chunk_no) {
                    const uint32_t buf = buf0 + (chunk_no % kEpiBufs) * kEpiWarpBytes;
                    uint32_t v[32];
                    long long* et = (args.cta_times && blockIdx.x == 0 && warp == 0 && lane == 0 && chunk_no < 12) ? args.cta_times + 320 + chunk_no * 5 : nullptr;
                    if (et) et[0] = clock64();
                    tmem_ld32(tmem_base + ((quad * 32u) << 16) + h * BN + colh * (BN / 2) + ci * 32, v);
                    // the reduction that last used this warp's staging tile must have read it
                    if (lane == 0) bulk_wait_read<kEpiBufs - 1>();
                    if (et) et[1] = clock64();
                    tmem_ld_wait();
                    if (et) et[2] = clock64();
                    if (ci == 3) {
                        // every TMEM read of this half is done: hand it back to the MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(tempty_leader + 8u * h);
                    } else {
                        __syncwarp();
                    }
                    if (!(args.debug & 2u)) {
                        // staging tile: row = m (128 B = 32 n), 16-byte chunk c stored at c ^ (m & 7)
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + row * 128u + ((c ^ (row & 7u)) << 4)),
                                         "r"(v[4 * c + 0]), "r"(v[4 * c + 1]), "r"(v[4 * c + 2]), "r"(v[4 * c + 3])
                                         : "memory");
                        fence_async_smem();
                        __syncwarp();
                        if (et) et[3] = clock64();
                        if (lane == 0 && !(args.debug & 8u)) {
                            int tc[5];
                            tile_coords_t<PLAIN>(args.cc, rank_c, false, m0 + h * BMH, n0 + ci * 32, batch, tc);
                            if ((args.debug & 4u) && rank_c == 3)  // timing experiment: plain store instead of the L2 reduction
                                asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(&map_c),
                                             "r"(buf), "r"(tc[0]), "r"(tc[1]), "r"(tc[2]) : "memory");
                            else if ((args.hints & 2u) && rank_c == 3)
                                tma_reduce_add_3d_hint(&map_c, buf, tc[0], tc[1], tc[2], pol_c);
                            else
                                tma_reduce_add_tile(&map_c, buf, rank_c, tc);
                            bulk_commit();
                            if (et) et[4] = clock64();
                        }
                    }
                }
            }
            acc_phase ^= 1u;
        }
        if (lane == 0) bulk_wait_read<0>();
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<2>(tmem_base, 512);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0 && args.clk) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.clk[2] = clock64();
        args.clk[3] = static_cast<long long>(gt);
    }
    if (threadIdx.x == 0 && args.cta_times) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.cta_times[2 * blockIdx.x + 1] = static_cast<long long>(gt);
    }
}

// TLB_GEMM_CTA_TIMES=<file>: per-CTA entry / exit times of the last 64 launches (debug; dumped at process exit).
constexpr int kCtaRing = 64, kCtaSlots = 2 * 160 + 64; // + 64: epilogue step stamps of CTA 0 / warp 0 (debug)
long long* g_cta_host = nullptr;
long long* g_cta_dev = nullptr;
std::atomic<unsigned> g_cta_next{0};
void cta_times_dump() {
    const char* path = std::getenv("TLB_GEMM_CTA_TIMES");
    if (!g_cta_host || !path) return;
    cudaDeviceSynchronize();
    cudaMemcpy(g_cta_host, g_cta_dev, static_cast<size_t>(kCtaRing) * kCtaSlots * sizeof(long long), cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(path, "wb")) {
        const long long hdr[4] = {kCtaRing, kCtaSlots, static_cast<long long>(g_cta_next.load()), 0};
        std::fwrite(hdr, sizeof(hdr), 1, f);
        std::fwrite(g_cta_host, sizeof(long long), static_cast<size_t>(kCtaRing) * kCtaSlots, f);
        std::fclose(f);
    }
}
long long* cta_times_slot() {
    static const bool on = [] {
        const char* e = std::getenv("TLB_GEMM_CTA_TIMES");
        if (!(e && e[0])) return false;
        const size_t bytes = static_cast<size_t>(kCtaRing) * kCtaSlots * sizeof(long long);
        // device memory, copied back at exit: stamps written to mapped host memory would add a PCIe round trip to
        // every kernel's completion (measured: +4 us per launch)
        g_cta_host = static_cast<long long*>(std::malloc(bytes));
        if (!g_cta_host || cudaMalloc(reinterpret_cast<void**>(&g_cta_dev), bytes) != cudaSuccess) return false;
        if (cudaMemset(g_cta_dev, 0, bytes) != cudaSuccess) return false;
        std::atexit(cta_times_dump);
        return true;
    }();
    if (!on) return nullptr;
    return g_cta_dev + static_cast<size_t>(g_cta_next.fetch_add(1, std::memory_order_relaxed) % kCtaRing) * kCtaSlots;
}

} // namespace

// Cuts of the stream-K k-block space [0, sk_units * kblocks) into one range per worker, balanced by COST: a range
// pays `epi` k-block equivalents for every tile it touches (each touched tile is one more reduce-add epilogue, about
// 7 us against 0.65 us per k-block), so workers whose range straddles a tile boundary get fewer k-blocks. Cuts closer
// than kMinSeg to a tile boundary snap to it.
void stream_k_cuts(uint32_t sk_units, uint32_t kblocks, uint32_t W, uint32_t epi, uint32_t* cut) {
    const uint64_t total = static_cast<uint64_t>(sk_units) * kblocks;
    auto snap = [&](uint64_t x) {
        const uint32_t r = static_cast<uint32_t>(x % kblocks);
        if (r < static_cast<uint32_t>(kMinSeg)) return x - r;
        if (kblocks - r < static_cast<uint32_t>(kMinSeg)) return x + (kblocks - r);
        return x;
    };
    auto assign = [&](uint64_t T) {
        uint64_t pos = 0;
        cut[0] = 0;
        for (uint32_t w = 0; w < W; ++w) {
            int64_t budget = static_cast<int64_t>(T);
            uint64_t q = pos;
            while (q < total) {
                budget -= epi; // the tile this range is about to touch
                if (budget < kMinSeg) break;
                const uint64_t to_boundary = kblocks - q % kblocks;
                const uint64_t step = std::min<uint64_t>(to_boundary, static_cast<uint64_t>(budget));
                q += step;
                budget -= static_cast<int64_t>(step);
                if (step < to_boundary) break;
            }
            q = std::min<uint64_t>(snap(q), total);
            if (q < pos) q = pos;
            pos = q;
            cut[w + 1] = static_cast<uint32_t>(pos);
        }
        return pos >= total;
    };
    uint64_t lo = total / W, hi = total / W + 4ull * epi + kblocks + 8;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (assign(mid)) hi = mid;
        else lo = mid + 1;
    }
    assign(lo);
    cut[W] = static_cast<uint32_t>(total);
}

bool umma_wide_applies(const UmmaProblem& p) {
    const int wide_knob = p.force_wide ? (p.force_wide > 0 ? 1 : 0) : knob(K_GEMM_WIDE);
    if (wide_knob == 0 || p.bn != 256) return false;
    if (p.cta_group != 2) return false;
    // A range of 128 x 256 tile ids selects whole pair tiles when ceil(M/256) is even (pair tile g = tiles 4g .. 4g+3);
    // the full range of a problem does for any M (the last pair tile is clipped by the TMA bounds).
    const uint32_t mb = static_cast<uint32_t>((p.M + 255) / 256);
    if (!p.full_range && (mb % 2 != 0 || p.tile_begin % 4 != 0 || p.tile_end % 4 != 0)) return false;
    // small problems keep the 256 x 256 plan (finer tiles, overlapped epilogue; measured better up to 2048^3, worse from
    // 3072^3) unless the wide plan is forced (TLB_GEMM_WIDE=1)
    {
        const uint64_t nb = static_cast<uint64_t>((p.N + 255) / 256);
        const uint64_t pair_tiles = p.full_range ? static_cast<uint64_t>((p.M + 511) / 512) * nb * static_cast<uint64_t>(std::max(p.batch, 1))
                                                 : (p.tile_end - p.tile_begin) / 4;
        if (wide_knob != 1 && pair_tiles < 48) return false;
        // short k-loops: a 512 x 256 tile flushes 256 KiB per CTA after only K / 64 k-blocks and cannot hide it (TMEM is
        // full), the 256 x 256 plan overlaps its flush with the next tile. Measured crossover (round 2, 4096^2 and 8192^2
        // outputs): K = 2048 the 256 x 256 plan is 13 % ahead, K = 3072 0-3 %, K = 4096 a tie, from K = 5120 the wide plan
        // leads (6144^3 +4 %, 3072^2 x 8192 +7 %).
        // (a 2-byte C flushes half the bytes: the wide plan already leads at K = 2048, 1285 vs 1268 TFLOP/s)
        if (wide_knob != 1 && (p.K + BK - 1) / BK < (p.c_16 ? 32 : 64)) return false;
    }
    const bool base_ok = (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && (p.batch <= 1 || (p.c_bs % 4 == 0 && p.c_bs > 0));
    if (p.c_fold_tma) return base_ok && (!p.c_16 || p.batch <= 1 || p.c_bs % 8 == 0);
    return base_ok && p.cs_n == 1 && p.cs_m % (p.c_16 ? 8 : 4) == 0 && p.cs_m >= p.N &&   // TMA reduce-add epilogue only
           (!p.c_16 || p.batch <= 1 || p.c_bs % 8 == 0);
}


// One launch over `units` pair tiles starting at a.unit_begin: partial-wave cut, grid, cluster and PDL attributes.
static int launch_units(const UmmaProblem& p, WideArgs& a, uint32_t units, uint32_t W, int kblocks, bool plain, bool mc, const CUtensorMap& tma,
                 const CUtensorMap& tmb, const CUtensorMap& tmc, const CUtensorMap& tmcp, cudaStream_t stream) {
    // Tail balancing: the (units mod W) tiles of the partial wave become one k-range per worker (run first). With
    // split_tail off (TLB_GEMM_SPLIT_TAIL=0) every tile is summed by one CTA pair in k order: bitwise reproducible.
    // Partial tiles cost an extra epilogue (C traffic is the expensive part), so the partial wave is only cut when whole
    // tiles would leave more than TLB_GEMM_SK_PCT % (default 4) of the CTA pairs idle in the last wave.
    // (2-byte C: every partial tile would be one more rounding step at L2, so the partial wave is not cut unless
    // TLB_GEMM_C16_SK=1 asks for it: 4096^3 1449 -> 1486 TFLOP/s)
    const bool c16_sk = knob(K_GEMM_C16_SK) == 1;
    a.sk_units = (p.split_tail && (!p.c_16 || c16_sk) && kblocks >= 2 * kMinSeg) ? units % W : 0;
    if (a.sk_units && units > W) {
        const int pct = knob(K_GEMM_SK_PCT);
        const uint32_t waves = (units + W - 1) / W;
        const double idle = 1.0 - static_cast<double>(units) / (static_cast<double>(waves) * W);
        if (idle * 100.0 <= pct) a.sk_units = 0;
    }
    a.dp_units = units - a.sk_units;
    if (a.sk_units && (W > static_cast<uint32_t>(kMaxWorkers) || static_cast<uint64_t>(a.sk_units) * kblocks > 0xffffffffull)) {
        a.sk_units = 0;
        a.dp_units = units;
    }
    if (a.sk_units) {
        const uint32_t epi = static_cast<uint32_t>(std::max(0, knob(K_GEMM_EPI_KB)));
        stream_k_cuts(a.sk_units, static_cast<uint32_t>(kblocks), W, epi, a.sk_cut);
    }
    const uint32_t workers = a.sk_units ? W : std::min(units, W);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    cfg.gridDim = dim3((mc ? 4 : 2) * workers);
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mc ? 4 : 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = umma_pdl_enabled() ? 2 : 1;
    cfg.blockDim = dim3(kThreadsW);
    cfg.dynamicSmemBytes = kSmemW;
    cfg.stream = stream;
    if (mc) TLB_CUDA(cudaLaunchKernelEx(&cfg, umma_wide_kernel<true, true>, tma, tmb, tmc, tmcp, a));
    else if (plain) TLB_CUDA(cudaLaunchKernelEx(&cfg, umma_wide_kernel<true, false>, tma, tmb, tmc, tmcp, a));
    else TLB_CUDA(cudaLaunchKernelEx(&cfg, umma_wide_kernel<false, false>, tma, tmb, tmc, tmcp, a));
    count_launch();
    return TLB_OK;
}

static std::atomic<int> g_clusters4[64]; // co-resident clusters of 4 of the multicast kernel, per device

int umma_wide_launch(const UmmaProblem& p, cudaStream_t stream) {
    static std::atomic<bool> attr_set[64];
    int dev = 0;
    TLB_CUDA(cudaGetDevice(&dev));
    if (dev >= 0 && dev < 64 && !attr_set[dev].load(std::memory_order_acquire)) {
        TLB_CUDA((cudaFuncSetAttribute(umma_wide_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemW)));
        TLB_CUDA((cudaFuncSetAttribute(umma_wide_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemW)));
        TLB_CUDA((cudaFuncSetAttribute(umma_wide_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemW)));
        // how many clusters of 4 fit (GPCs whose SM count is not a multiple of 4 leave SMs over: 132 of 148 on B200)
        cudaLaunchConfig_t qc = {};
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = 4;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.gridDim = dim3(4 * 64);
        qc.blockDim = dim3(kThreadsW);
        qc.dynamicSmemBytes = kSmemW;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int n4 = 0;
        if (cudaOccupancyMaxActiveClusters(&n4, umma_wide_kernel<true, true>, &qc) != cudaSuccess) n4 = 0;
        (void)cudaGetLastError();
        g_clusters4[dev].store(n4, std::memory_order_relaxed);
        attr_set[dev].store(true, std::memory_order_release);
    }
    // tensor maps = the divided layouts: zipped_divide(A, [256, 64]), zipped_divide(B, [128, 64]) (64 x 64 chunks for
    // MN-major operands), zipped_divide(C, [32, 32 | 64])
    // Multicast plan (clusters of 4, A quarters shared between two n-adjacent pair tiles): K-major unfolded operands, whole
    // problems, an even number of 256-column blocks. GEMM_MCAST: 0 never, 1 when it applies, -1 auto (see below).
    const uint32_t nb_all = static_cast<uint32_t>((p.N + 255) / 256);
    const int n4 = (dev >= 0 && dev < 64) ? g_clusters4[dev].load(std::memory_order_relaxed) : 0;
    const int mc_knob = knob(K_GEMM_MCAST);
    bool use_mc = mc_knob != 0 && n4 > 0 && !p.a_mn && !p.b_mn && p.full_range && nb_all % 2 == 0 && nb_all >= 2;
    if (use_mc && mc_knob < 0) use_mc = static_cast<uint64_t>((p.M + 511) / 512) * (nb_all / 2) * static_cast<uint64_t>(std::max(p.batch, 1)) >= static_cast<uint64_t>(n4);
    TmaTileMap ma, mb, mc, mcp;
    TLB_TRY(umma_operand_map(p, 0, use_mc ? BMH : BMC, &ma));
    TLB_TRY(umma_operand_map(p, 1, BN / 2, &mb));
    TLB_TRY(umma_c_map(p, p.c_16 ? 64 : 32, 32, TMA_SW_128, &mc));
    TLB_TRY(epilogue_partition_check(BN, 2)); // tcgen05.ld partition derived from the accumulator layout (tlb_gemm_layout.cu)
    WideArgs a;
    std::memset(&a, 0, sizeof(a));
    // C prefetch into L2 is off by default: measured, it evicts operand lines and costs 1.5 % (8192^3) to 7 % (4096^3).
    a.prefetch_c = static_cast<uint32_t>(std::max(0, knob(K_GEMM_PREFETCH_C)));
    if (a.prefetch_c && (p.c_16 || umma_c_map(p, 256, BMH, TMA_SW_NONE, &mcp) != TLB_OK || mcp.rank != 3)) a.prefetch_c = 0;
    if (!a.prefetch_c) mcp = mc;
    a.M = p.M;
    a.N = p.N;
    a.K = p.K;
    a.mbw = static_cast<uint32_t>((p.M + 511) / 512);
    a.nb = nb_all;
    a.ab_f16 = p.ab_f16 ? 1u : 0u;
    a.c_16 = p.c_16 ? 1u : 0u;
    a.a_mn = p.a_mn ? 1u : 0u;
    a.b_mn = p.b_mn ? 1u : 0u;
    a.rank_a = ma.rank;
    a.rank_b = mb.rank;
    a.rank_c = mc.rank;
    for (int d = 0; d < 5; ++d) {
        a.ca[d] = ma.c[d];
        a.cb[d] = mb.c[d];
        a.cc[d] = mc.c[d];
    }
    a.group_w = std::max(1u, static_cast<uint32_t>(std::max(1, knob(K_GEMM_GROUP_M))) / 2);
    a.debug = static_cast<uint32_t>(knob(K_GEMM_DEBUG));
    a.hints = static_cast<uint32_t>(knob(K_GEMM_HINTS));
    a.early_release = knob(K_GEMM_EARLY_RELEASE) != 0 ? 1u : 0u;
    const uint32_t unit_begin = p.full_range ? 0u : p.tile_begin / 4;
    const uint32_t units_all = p.full_range ? a.mbw * a.nb * static_cast<uint32_t>(std::max(p.batch, 1)) : p.tile_end / 4 - unit_begin;
    if (units_all == 0) return TLB_OK;
    uint32_t W = static_cast<uint32_t>(sm_count() / 2);
    if (const int cap = knob(K_GEMM_WORKERS); cap > 0) W = std::max(1u, std::min(W, static_cast<uint32_t>(cap)));
    const int kblocks = (p.K + BK - 1) / BK;
    a.clk = umma_clk_slot();
    a.cta_times = cta_times_slot();
    CUtensorMap tma, tmb, tmc, tmcp;
    std::memcpy(&tma, ma.desc, 128);
    std::memcpy(&tmb, mb.desc, 128);
    std::memcpy(&tmc, mc.desc, 128);
    std::memcpy(&tmcp, mcp.desc, 128);
    // plain (unfolded) operands and C: the coordinates of every map are the kernel's loop variables
    const bool plain = tma_map_is_plain(ma, p.a_mn != 0) && tma_map_is_plain(mb, p.b_mn != 0) && tma_map_is_plain(mc, false);
    if (use_mc && !plain) { // folded operands keep the pair plan (the A map goes back to 256-row boxes)
        use_mc = false;
        TLB_TRY(umma_operand_map(p, 0, BMC, &ma));
        std::memcpy(&tma, ma.desc, 128);
        a.rank_a = ma.rank;
        for (int d = 0; d < 5; ++d) a.ca[d] = ma.c[d];
    }
    if (use_mc) {
        a.nb = nb_all / 2;   // units are 512 x 512 cluster tiles; pair p of a cluster takes column block 2 n + p
        W = static_cast<uint32_t>(n4);
        if (const int cap = knob(K_GEMM_WORKERS); cap > 0) W = std::max(1u, std::min(W, static_cast<uint32_t>(cap)));
    }
    const uint32_t units_total = use_mc ? a.mbw * a.nb * static_cast<uint32_t>(std::max(p.batch, 1)) : units_all;

    // One launch covers at most ~GEMM_CHUNK_WAVES waves of pair tiles. The workers of a persistent launch are only
    // synchronised at its start: every tile boundary adds a little jitter, after some tens of tiles the CTAs that share an
    // operand panel no longer read it at the same time, the panel is fetched from DRAM once per straggler instead of once,
    // and on a power-capped part the extra DRAM traffic is paid in SM clock. Measured on 8192^3 batches (ncu, one launch):
    // 1.39 GB of DRAM traffic per batch in a 1-batch launch, 2.35 GB at 8 batches, 3.99 GB at 64 (L2 hit rate 74 % -> 45 %);
    // the same 64 batches run 1200 TFLOP/s as one launch and 1400 as one launch per batch. Cutting the range into
    // launches re-aligns the workers every few waves (programmatic dependent launch hides the launch gaps), and every
    // launch balances its own partial wave.
    std::vector<uint32_t> cuts{0u};
    {
        const uint32_t waves = static_cast<uint32_t>(std::max(0, knob(K_GEMM_CHUNK_WAVES)));
        const uint32_t per_batch = a.mbw * a.nb;
        if (waves > 0 && units_total > (waves + waves / 2) * W) {
            // boundaries at whole batches when a batch holds at least a wave, else anywhere; single problems at whole
            // rasterisation groups
            uint32_t align = 1;
            if (p.full_range && std::max(p.batch, 1) > 1) align = per_batch >= W ? per_batch : 1u;
            else if (p.full_range) align = a.group_w * a.nb;
            const uint32_t target = waves * W;
            const uint32_t step = align >= target ? align : std::max(1u, target / align) * align;
            for (uint32_t u = step; u + step / 2 < units_total; u += step) cuts.push_back(u);
        }
        cuts.push_back(units_total);
    }
    for (size_t ci = 0; ci + 1 < cuts.size(); ++ci) {
        a.unit_begin = unit_begin + cuts[ci];
        const uint32_t units = cuts[ci + 1] - cuts[ci];
        TLB_TRY(launch_units(p, a, units, W, kblocks, plain, use_mc, tma, tmb, tmc, tmcp, stream));
    }
    set_plan(use_mc ? "umma_2sm_wide_mc" : "umma_2sm_wide");
    return TLB_OK;
}

} // namespace tlb

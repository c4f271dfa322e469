// PTX wrappers shared by the tcgen05 GEMM kernels (tlb_gemm_umma.cu, tlb_gemm_umma_wide.cu): mbarriers, TMA loads and
// reductions, tcgen05 alloc / mma / commit / ld, and the hand-encoded shared-memory matrix descriptor. No CUTLASS / CuTe.
#pragma once

#include <cstdint>

#include <cuda.h>

#include "tlb_gemm.h"

namespace tlb {
namespace umma {

// ---- PTX wrappers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}
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
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a pipeline bug must trap, never hang the GPU. The first probe is free of bookkeeping; roles
// that idle for microseconds (epilogue, producer) back off with nanosleep between probes.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, uint32_t backoff_ns = 0) {
    if (mbar_try(bar, parity)) return;
    const long long t0 = clock64();
    for (;;) {
        if (backoff_ns) __nanosleep(backoff_ns);
        if (mbar_try(bar, parity)) return;
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
// cta_group::2 + multicast: the box lands at the same offset in every CTA of `mask` and each destination's bytes complete
// on the barrier at leader_bar's offset in THAT destination's pair leader (measured: tools/probes/mcast_probe.cu).
__device__ __forceinline__ void tma_load_3d_2sm_mc(uint32_t dst, const void* map, uint32_t leader_bar, int c0, int c1, int c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}
// L2 eviction-priority policies for the per-tensor cache hints.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const void* map, uint32_t bar, int c0, int c1, int c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm_hint(uint32_t dst, const void* map, uint32_t leader_bar, int c0, int c1, int c2,
                                                     uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(map), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d_hint(const void* map, uint32_t src, int c0, int c1, int c2, uint64_t pol) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(map),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
                 : "memory");
}
// C += staged chunk, performed by the TMA unit / L2 (fp32 add, element type from the tensor map).
__device__ __forceinline__ void tma_reduce_add_3d(const void* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Programmatic dependent launch: the next kernel of the stream may be scheduled (and run its prologue) while this one
// drains; griddep_wait() blocks until the PREVIOUS kernel of the stream has completed and its writes are visible, so
// it must precede every global-memory access of the kernel.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
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
// tcgen05.commit: the barrier is arrived on when every MMA previously issued by this thread has finished.
template <int CG> __device__ __forceinline__ void umma_commit(uint32_t bar, uint16_t mask = 3) {
    if constexpr (CG == 1) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    } else {
        // mask: both CTAs of the pair (cluster ranks; 3 for the first pair of a cluster), same barrier offset in each
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
            "h"(mask)
            : "memory");
    }
}
// Non-multicast commit on a barrier of the issuing CTA. Measured (tools/probes/mma_rate.cu): a multicast commit
// every 4 or 8 MMAs stretches the 128-cycle MMA to 139.5 cycles, a local commit every 8 MMAs costs nothing.
template <int CG> __device__ __forceinline__ void umma_commit_local(uint32_t bar) {
    if constexpr (CG == 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    else asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
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
__device__ __forceinline__ void red_add_f32(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Shared-memory matrix descriptor of a K-major bf16 tile staged with the 128-byte swizzle: rows of 128 B,
// 8-row groups 1024 B apart (SBO), sm_100 descriptor version 1, layout type 2 (SWIZZLE_128B). Only the low
// word depends on the tile address; advancing K by 16 elements inside the swizzle row adds 32 B (+2).
// ---- tiles of layout-derived tensor maps (TmaTileMap, tlb_gemm.h) --------------------------------------------------
// TMA coordinates of the tile that starts at (row0, k0, batch) of its operand: per dimension one division and one
// remainder, both by multiply-shift with host-built magic numbers (TmaCoord, tlb_gemm.h): branch free, no hardware-free
// division in the producer's k-loop.
__device__ __forceinline__ void tile_coords(const TmaCoord* tc, int rank, uint32_t row0, uint32_t k0, uint32_t batch, int* c) {
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        if (d < rank) {
            const uint32_t v = tc[d].src == 0u ? row0 : (tc[d].src == 1u ? k0 : batch);
            const uint32_t q = static_cast<uint32_t>((static_cast<uint64_t>(v) * tc[d].div_m) >> tc[d].div_s);
            const uint32_t t = static_cast<uint32_t>((static_cast<uint64_t>(q) * tc[d].mod_m) >> tc[d].mod_s);
            c[d] = static_cast<int>(q - t * tc[d].mod);
        } else {
            c[d] = 0;
        }
    }
}
// PLAIN: the map is rank 3 with identity coordinates ((k | row, row | k, batch) and (column, row, batch): unfolded
// operands, tma_map_is_plain): the tile coordinates are the kernel's own loop variables. With the general decomposition
// in its k-loop the TMA producer (one thread, ~150 dependent uniform-datapath instructions and constant loads per
// k-block) paces the kernel instead of the tensor pipe: 4096^3 1350 -> 1205 TFLOP/s even with multiply-shift division.
template <bool PLAIN>
__device__ __forceinline__ void tile_coords_t(const TmaCoord* tc, int rank, bool dim0_is_row, uint32_t row0, uint32_t k0, uint32_t batch, int* c) {
    if constexpr (PLAIN) {
        c[0] = static_cast<int>(dim0_is_row ? row0 : k0);
        c[1] = static_cast<int>(dim0_is_row ? k0 : row0);
        c[2] = static_cast<int>(batch);
        c[3] = c[4] = 0;
    } else {
        tile_coords(tc, rank, row0, k0, batch, c);
    }
}
// Inside a tile's k-loop only the dimensions fed by k move: the row / batch dimensions are computed once per tile
// (tile_coords_t with k0 = 0) and this refreshes the others.
template <bool PLAIN>
__device__ __forceinline__ void tile_coords_k(const TmaCoord* tc, int rank, uint32_t k0, int* c) {
    if constexpr (PLAIN) {
        c[0] = static_cast<int>(k0);
    } else {
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            if (d < rank && tc[d].src == 1u) {
                const uint32_t q = static_cast<uint32_t>((static_cast<uint64_t>(k0) * tc[d].div_m) >> tc[d].div_s);
                const uint32_t t = static_cast<uint32_t>((static_cast<uint64_t>(q) * tc[d].mod_m) >> tc[d].mod_s);
                c[d] = static_cast<int>(q - t * tc[d].mod);
            }
        }
    }
}
// One k-block further: every k-fed dimension advances by its kinc; a dimension that reaches its extent wraps and carries
// one into the next k-fed dimension (their divisors are the running products of the extents before them, so the carry is
// exactly one). Valid when the tile starts at a multiple of 64 in k and the divisors divide 64 or are multiples of it,
// which tile_dims_derive guarantees for 64-element k boxes. Adds and compares only.
template <bool PLAIN>
__device__ __forceinline__ void tile_coords_step(const TmaCoord* tc, int rank, int* c) {
    if constexpr (PLAIN) {
        c[0] += 64;
    } else {
        uint32_t carry = 0;
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            if (d < rank && tc[d].src == 1u) {
                uint32_t v = static_cast<uint32_t>(c[d]) + tc[d].kinc + carry;
                carry = 0;
                if (tc[d].mod && v >= tc[d].mod) {
                    v -= tc[d].mod;
                    carry = 1;
                }
                c[d] = static_cast<int>(v);
            }
        }
    }
}
// cp.async.bulk.tensor of rank 3..5; CG2: cta_group::2 form (transaction bytes complete on the leader's barrier).
template <bool CG2>
__device__ __forceinline__ void tma_load_tile(uint32_t dst, const void* map, uint32_t bar, int rank, const int* c) {
    if (rank == 3) {
        if constexpr (CG2) tma_load_3d_2sm(dst, map, bar, c[0], c[1], c[2]);
        else tma_load_3d(dst, map, bar, c[0], c[1], c[2]);
    } else if (rank == 4) {
        if constexpr (CG2)
            asm volatile("cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
                         "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
                         "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
    } else {
        if constexpr (CG2)
            asm volatile("cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
                         "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
                         "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
    }
}
template <bool CG2>
__device__ __forceinline__ void tma_load_tile_hint(uint32_t dst, const void* map, uint32_t bar, int rank, const int* c, uint64_t pol) {
    if (rank == 3) {
        if constexpr (CG2) tma_load_3d_2sm_hint(dst, map, bar, c[0], c[1], c[2], pol);
        else tma_load_3d_hint(dst, map, bar, c[0], c[1], c[2], pol);
    } else {
        tma_load_tile<CG2>(dst, map, bar, rank, c); // folded modes: no hinted form
    }
}
// C += staged chunk through a rank 3..5 map.
__device__ __forceinline__ void tma_reduce_add_tile(const void* map, uint32_t src, int rank, const int* c) {
    if (rank == 3) {
        tma_reduce_add_3d(map, src, c[0], c[1], c[2]);
    } else if (rank == 4) {
        asm volatile("cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
                     "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
    } else {
        asm volatile("cp.reduce.async.bulk.tensor.5d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map),
                     "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
    }
}

constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
__device__ __forceinline__ uint32_t desc_lo(uint32_t smem_addr) { return ((smem_addr >> 4) & 0x3fffu) | (1u << 16); }
__device__ __forceinline__ uint64_t make_desc(uint32_t lo) { return (static_cast<uint64_t>(kDescHi) << 32) | lo; }
} // namespace umma
} // namespace tlb

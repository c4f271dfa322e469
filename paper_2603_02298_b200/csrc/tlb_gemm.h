// Shared between the GEMM dispatcher (tlb_gemm_simt.cu) and the tcgen05 kernel (tlb_gemm_umma.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace tlb {

// Output tiles are 128 (m) x 256 (n). Tile id t: the pair (2g, 2g+1) are the two m-halves of
// 256x256 block g; blocks are walked in groups of kGemmGroupM m-blocks, m fastest inside a
// group, then n, then the next group (L2-friendly rasterisation). Batches are outermost.
constexpr int kGemmGroupM = 8;

struct TileGrid {
    uint32_t mb, nb; // 256x256 blocks along m and n
};
__host__ __device__ inline uint32_t tiles_per_batch(const TileGrid& g) { return g.mb * g.nb * 2u; }
// (m, n) -> tile id inside one batch (the inverse of decode_unit in tlb_gemm_umma.cu)
__host__ __device__ inline uint32_t tile_of(const TileGrid& g, int64_t m, int64_t n) {
    const uint32_t m_tile = static_cast<uint32_t>(m >> 7), m_blk = m_tile >> 1, half = m_tile & 1u;
    const uint32_t n_blk = static_cast<uint32_t>(n >> 8);
    const uint32_t grp = m_blk / kGemmGroupM;
    const uint32_t left = g.mb - grp * kGemmGroupM;
    const uint32_t gm = left < static_cast<uint32_t>(kGemmGroupM) ? left : static_cast<uint32_t>(kGemmGroupM);
    const uint32_t blk = grp * kGemmGroupM * g.nb + n_blk * gm + (m_blk - grp * kGemmGroupM);
    return blk * 2u + half;
}

struct UmmaProblem {
    const void* A;   // bf16, (M,K):(lda,1), or (M,K):(1,lda) when a_mn
    const void* B;   // bf16, (N,K):(ldb,1), or (N,K):(1,ldb) when b_mn
    float* C;        // fp32, (M,N):(cs_m,cs_n)
    int64_t lda, ldb, cs_m, cs_n;
    int32_t M, N, K;
    int32_t batch;
    int64_t a_bs, b_bs, c_bs;      // batch strides (elements)
    uint32_t tile_begin, tile_end; // global tile ids (batch-major), [begin, end)
    int32_t cta_group;             // 1 or 2
    int32_t split_tail;            // 1: split the units of the last partial wave along K (red.add epilogue)
    int32_t a_mn, b_mn;            // operand is MN-major (its m / n mode is the contiguous one): wide plan only
    int32_t full_range;            // [tile_begin, tile_end) is every tile of every batch
    int32_t ab_f16;                // operands are IEEE fp16 instead of bf16 (instruction-descriptor formats 0 / 1)
    int32_t c_16;                  // C has the operands' 2-byte type (C points at 2-byte cells): wide plan only
};
int umma_gemm_launch(const UmmaProblem& p, cudaStream_t stream);
// Wide plan (tlb_gemm_umma_wide.cu): 512 x 256 pair tiles, chosen when the tile range is a whole number of them.
bool umma_pdl_enabled();      // programmatic dependent launch (TLB_GEMM_PDL=0 turns it off)
long long* umma_clk_slot();   // TLB_GEMM_CLOCK=1: where CTA 0 stamps {clock64, globaltimer}; nullptr when off
bool umma_wide_applies(const UmmaProblem& p);
int umma_wide_launch(const UmmaProblem& p, cudaStream_t stream);

} // namespace tlb

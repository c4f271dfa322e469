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

// ---- tensor maps derived from divided layouts (tlb_tma.cu) --------------------------------------------------
// A GEMM operand is a rank-2 layout (rows, k) (+ a batch stride). The k-blocks a CTA loads are the tiles of
// zipped_divide(operand, [box_rows, box_k]) (algebra.hpp:595): the PARENT layout's leaves become the TMA dimensions
// (globalDim / globalStrides), the TILE mode's leaves become the box (boxDim). Modes may be hierarchical (GETT-style
// folded modes): every leaf is its own TMA dimension, and the element index where a tile starts in
// that dimension follows from the tile's 1-D coordinate in its mode by one division and one remainder.
// The kernels evaluate it per k-block, so both steps are multiply-shift (Granlund-Montgomery magic numbers for dividends
// below 2^31, built on the host): a hardware-free division costs ~100 cycles and five dimensions of them in the TMA
// producer's loop made the producer, not the tensor pipe, the pace of the kernel (measured: 4096^3 1350 -> 1160 TFLOP/s).
struct TmaCoord {
    uint32_t src;          // which tile coordinate feeds this dimension: 0 = row index, 1 = k (or column) index, 2 = batch
    uint32_t div_m, div_s; // q = (value * div_m) >> div_s                 == value / div
    uint32_t mod, mod_m, mod_s; // coordinate = q - ((q * mod_m) >> mod_s) * mod  == q % mod; mod == 0: no remainder
    uint32_t kinc;         // k-fed dimensions: what one k-block (64 elements of k) adds to the coordinate, before carries
                           // (tile_coords_step: the producer's k-loop advances coordinates instead of recomputing them)
};
inline void magic_u31(uint32_t d, uint32_t* m, uint32_t* s) { // floor(v / d) == (uint64(v) * m) >> s for every v < 2^31
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    *s = 31 + l;
    *m = static_cast<uint32_t>(((1ull << *s) + d - 1) / d);
}
inline TmaCoord tma_coord(uint32_t src, uint32_t div, uint32_t mod) {
    TmaCoord c = {src, 0u, 0u, mod, 0u, 0u, 0u};
    magic_u31(div ? div : 1u, &c.div_m, &c.div_s);
    if (mod) magic_u31(mod, &c.mod_m, &c.mod_s);
    const uint32_t d = div ? div : 1u;
    if (src == 1u && d <= 64u && 64u % d == 0u) c.kinc = mod ? (64u / d) % mod : 64u / d;
    return c;
}
struct TmaTileMap {
    alignas(64) unsigned char desc[128];
    int32_t rank;      // 3..5 (padded to 3 with unit dimensions)
    TmaCoord c[5];
};
// A rank-3 map whose coordinates are the tile's own (inner, outer, batch) start, undivided: dimension 0 fed by the k (or
// column) index for K-major operands and C, by the row index for MN-major operands.
inline bool tma_map_is_plain(const TmaTileMap& m, bool dim0_is_row) {
    if (m.rank != 3) return false;
    const uint32_t want[3] = {dim0_is_row ? 0u : 1u, dim0_is_row ? 1u : 0u, 2u};
    for (int d = 0; d < 3; ++d)
        if (m.c[d].src != want[d] || m.c[d].div_s != 31u || m.c[d].div_m != (1u << 31) || m.c[d].mod != 0u) return false;
    return true;
}
// Leaves of top-level mode `top` of `L`, coalesced in colex order (extent-1 leaves dropped). Returns the leaf count.
int mode_leaves(const tlb_layout_desc& L, int top, int64_t* extent, int64_t* stride, int cap);
struct TileDims {      // the derivation alone (pure host arithmetic, no driver call): what tlb_tensormap_describe reports
    int32_t rank;
    uint64_t dims[5], strides[5]; // extents and strides (elements), dimension 0 first
    uint32_t box[5];
    TmaCoord c[5];
};
int tile_dims_derive(const tlb_layout_desc& L, int inner_top, int outer_top, int64_t box_inner, int64_t box_outer,
                     int inner_src, int outer_src, int batch, int64_t batch_stride, int elem_bytes, TileDims* out);
// inner_top: the top-level mode whose first leaf has stride 1 (it becomes TMA dimension 0 and the inner box extent);
// outer_top: the other mode. box_inner / box_outer: tile extents along them (elements of the modes' 1-D coordinates).
// Fails with TLB_ERR_UNSUPPORTED (nothing written) when the layout is not TMA-addressable that way: no unit-stride
// leaf, a stride that is not a multiple of 16 bytes, a tile that straddles leaf boundaries, more than 5 dimensions.
int tensormap_for_tile(const tlb_layout_desc& L, int inner_top, int outer_top, int64_t box_inner, int64_t box_outer,
                       int inner_src, int outer_src, const void* base, int batch, int64_t batch_stride, int elem_bytes,
                       int is_float, int swizzle, int l2_promotion, TmaTileMap* out);

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
    // The layouts the tensor maps are derived from, as the plan runs them (A / B swapped when C is m-contiguous):
    // top-level mode 0 = rows (m or n), mode 1 = k; for C: mode c_row_top = rows of the plan, the other = columns.
    const tlb_layout_desc* la;
    const tlb_layout_desc* lb;
    const tlb_layout_desc* lc;
    int32_t c_row_top;
    int32_t bn;                    // UMMA N of the 128 x bn / 256 x bn plans (256 default, 128 from a tiler)
    int32_t c_fold_tma;            // C has folded (hierarchical) modes that the reduce-add tensor map can address
    int32_t force_wide;            // a tiler asked for the 512 x 256 plan / forbade it: 1 / -1 (0: planner decides)
};
int umma_operand_map(const UmmaProblem& p, int which /* 0 A, 1 B */, int box_rows, TmaTileMap* out);
int umma_c_map(const UmmaProblem& p, int box_n, int box_m, int swizzle, TmaTileMap* out);
// The tcgen05.ld partition of a 128-lane x bn-column accumulator (x halves), derived from the accumulator layout and the
// instruction's offset layout (locate_offsets, analysis.hpp:40-56) and checked against the kernels' compile-time shape.
int epilogue_partition_check(int bn, int halves);
int umma_gemm_launch(const UmmaProblem& p, cudaStream_t stream);
// Wide plan (tlb_gemm_umma_wide.cu): 512 x 256 pair tiles, chosen when the tile range is a whole number of them.
bool umma_pdl_enabled();      // programmatic dependent launch (TLB_GEMM_PDL=0 turns it off)
long long* umma_clk_slot();   // TLB_GEMM_CLOCK=1: where CTA 0 stamps {clock64, globaltimer}; nullptr when off
bool umma_wide_applies(const UmmaProblem& p);
bool umma_c16_applies(const UmmaProblem& p);   // 2-byte C on the 256 x 256 plans (TMA reduce-add epilogue)
int umma_wide_launch(const UmmaProblem& p, cudaStream_t stream);

} // namespace tlb

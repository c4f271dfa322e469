// Layout-driven planning of the tcgen05 GEMM epilogue: which TMEM offsets does a tcgen05.ld touch, and where do they sit
// in the accumulator's logical coordinates? That is tla::locate_offsets (analysis.hpp:40-56):
//
//     R = left_inverse(A) o T,   admissible iff  A(R(i)) == T(i)  for every instruction index i,
//
// with A the data layout (logical coordinate -> TMEM offset) and T the instruction layout (instruction coordinate -> TMEM
// offset). The host half below computes R for the leaf-in-leaf case (every instruction leaf lands inside one coalesced
// leaf of A: strided accumulators, which is what TMEM tiles are); the O(size(T)) admissibility loop runs on the device
// (tlb_compose_check_range). zipped_divide(A, R) is then the partition of the accumulator by the instruction, and the
// kernels' compile-time epilogue shape is checked against it instead of being trusted.
#include <algorithm>
#include <mutex>
#include <vector>

#include "tlb_internal.h"
#include "tlb_gemm.h"

namespace tlb {
namespace {

struct ALeaf {
    int64_t extent, stride, prefix; // prefix: product of the extents before this leaf in A's colex order
};

// R(i) = left_inverse(A)(T(i)), one leaf of R per leaf of T.
int locate_host(const tlb_layout_desc& A, const tlb_layout_desc& T, tlb_mode* r, int* n) {
    if (A.kind != TLB_KIND_INT || T.kind != TLB_KIND_INT) return fail(TLB_ERR_SEMIMODULE, "locate_offsets requires integer strides");
    std::vector<ALeaf> leaves;
    int64_t prefix = 1;
    for (int k = 0; k < A.n_modes; ++k) {
        if (A.extent[k] > 1) {
            // left_inverse needs an injective layout with positive strides (algebra.hpp:543-552)
            if (A.stride[k] <= 0) return fail(TLB_ERR_ADMISSIBILITY, "offsets cannot be located: layout is not left-invertible");
            leaves.push_back({A.extent[k], A.stride[k], prefix});
        }
        prefix *= A.extent[k];
    }
    std::sort(leaves.begin(), leaves.end(), [](const ALeaf& x, const ALeaf& y) { return x.stride < y.stride; });
    std::vector<ALeaf> co; // coalesced: consecutive in offset space AND in coordinate space
    for (const ALeaf& l : leaves) {
        if (!co.empty() && co.back().stride * co.back().extent == l.stride && co.back().prefix * co.back().extent == l.prefix)
            co.back().extent *= l.extent;
        else
            co.push_back(l);
    }
    for (size_t k = 0; k + 1 < co.size(); ++k)
        if (co[k].stride * co[k].extent > co[k + 1].stride)
            return fail(TLB_ERR_ADMISSIBILITY, "offsets cannot be located: layout is not left-invertible");
    *n = T.n_modes;
    for (int j = 0; j < T.n_modes; ++j) {
        r[j].extent = T.extent[j];
        r[j].kind = TLB_KIND_INT;
        r[j].axis = 0;
        r[j].stride = 0;
        const int64_t d = T.stride[j];
        if (T.extent[j] == 1 || d == 0) continue;
        if (d < 0) return fail(TLB_ERR_ADMISSIBILITY, "offsets cannot be located: negative instruction stride");
        const ALeaf* hit = nullptr;
        for (const ALeaf& l : co)
            if (l.stride <= d && d % l.stride == 0) hit = &l; // the largest stride that divides d
        if (!hit) return fail(TLB_ERR_ADMISSIBILITY, "offsets cannot be located: stride " + std::to_string(d) + " is not in the image of the layout");
        r[j].stride = (d / hit->stride) * hit->prefix;
    }
    // every located coordinate must lie inside A's domain (the device loop evaluates A on the extended domain, where the
    // last leaf is unbounded, so an out-of-domain coordinate could read back the right offset by accident)
    __int128 top = 0;
    for (int j = 0; j < T.n_modes; ++j) top += static_cast<__int128>(r[j].extent - 1) * r[j].stride;
    if (top >= A.size) return fail(TLB_ERR_ADMISSIBILITY, "offsets cannot be located: coordinate outside the layout's domain");
    return TLB_OK;
}

} // namespace

// Partition of a TMEM accumulator tile by tcgen05.ld.32x32b.x32, derived (not assumed):
//   A = (128, columns):(65536, 1)      logical (lane, column) -> TMEM address (lane in bits 31:16; the paper models the lane
//                                      stride as 16384, the hardware uses 65536)
//   T = (32, 32):(1, 65536)            the offsets one warp's instruction touches: 32 columns x 32 lanes
//   R = locate_offsets(A, T) = (32, 32):(128, 1): instruction columns step the logical coordinate by 128 (one column),
//       instruction lanes by 1 (one lane) -> the instruction covers a 32-lane x 32-column block of the tile, so
//       zipped_divide(A, R) has 128 / 32 = 4 lane blocks (the warp quadrants: warp w may only address lanes 32 (w % 4) ..)
//       and columns / 32 column blocks, dealt to the 8 epilogue warps as (w % 4, w / 4).
// The kernels hard-wire: 32 lanes x 32 columns per load, quadrant = warp % 4, columns / 64 loads per warp per tile.
int epilogue_partition_check(int bn, int halves) {
    static std::mutex mu;
    static bool done[3][3] = {};
    const int bi = bn == 256 ? 2 : bn == 128 ? 1 : 0;
    if (bi == 0 || halves < 1 || halves > 2) return fail(TLB_ERR_UNSUPPORTED, "epilogue partition: unsupported accumulator shape");
    {
        std::lock_guard<std::mutex> lock(mu);
        if (done[bi][halves]) return TLB_OK;
    }
    const int columns = bn * halves;
    tlb_mode am[2] = {{128, 65536, TLB_KIND_INT, 0}, {columns, 1, TLB_KIND_INT, 0}};
    tlb_mode tm[2] = {{32, 1, TLB_KIND_INT, 0}, {32, 65536, TLB_KIND_INT, 0}};
    tlb_layout_desc A, T;
    TLB_TRY(tlb_layout_lower(am, 2, &A));
    TLB_TRY(tlb_layout_lower(tm, 2, &T));
    tlb_mode r[TLB_MAX_MODES];
    int n = 0;
    TLB_TRY(locate_host(A, T, r, &n));
    const bool shape_ok = n == 2 && r[0].extent == 32 && r[0].stride == 128 && r[1].extent == 32 && r[1].stride == 1;
    // blocks of the partition: lanes 128 / 32 quadrants, columns / 32 chunks; 8 epilogue warps = 4 quadrants x 2
    const int quadrants = 128 / static_cast<int>(r[1].extent), chunks = columns / static_cast<int>(r[0].extent);
    const int per_warp = chunks / 2;
    if (!shape_ok || quadrants != 4 || per_warp * 2 != chunks || per_warp != (bn / 2 / 32) * halves)
        return fail(TLB_ERR_UNSUPPORTED, "epilogue partition derived from the accumulator layout does not match the kernel's tcgen05.ld shape");
    std::lock_guard<std::mutex> lock(mu);
    done[bi][halves] = true;
    return TLB_OK;
}

} // namespace tlb

using namespace tlb;

extern "C" int tlb_locate_offsets(const tlb_layout_desc* A, const tlb_layout_desc* T, tlb_mode* r_modes, int32_t* n_modes,
                                  void* stream) {
    if (!A || !T || !r_modes || !n_modes) return fail(TLB_ERR_CONTRACT, "tlb_locate_offsets: null argument");
    int n = 0;
    TLB_TRY(locate_host(*A, *T, r_modes, &n));
    *n_modes = n;
    // the admissibility loop A(R(i)) == T(i), i < size(T), on the device
    tlb_layout_desc R;
    TLB_TRY(tlb_layout_lower(r_modes, n, &R));
    TLB_TRY(require_device());
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long* d_bad = nullptr;
    unsigned long long h_bad = 0;
    TLB_CUDA(ws_malloc(reinterpret_cast<void**>(&d_bad), sizeof(unsigned long long), s));
    cudaError_t e = cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s);
    int st = TLB_OK;
    if (e == cudaSuccess) st = tlb_compose_check_range(A, &R, T, 0, static_cast<uint64_t>(T->size), d_bad, stream);
    if (e == cudaSuccess && st == TLB_OK) e = cudaMemcpyAsync(&h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && st == TLB_OK) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d_bad, s);
    TLB_CUDA(e);
    if (st != TLB_OK) return st == TLB_ERR_OVERFLOW ? fail(TLB_ERR_ADMISSIBILITY, "offsets cannot be located: coordinate outside the layout's domain") : st;
    if (h_bad) return fail(TLB_ERR_ADMISSIBILITY, std::to_string(h_bad) + " instruction offset(s) are not in the image of the layout");
    return TLB_OK;
}

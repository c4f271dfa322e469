// Scratch probe: where does the complete_tx of a MULTICAST cp.async.bulk.tensor with .cta_group::2 land?
// Cluster of 4 = two CTA pairs (0,1) and (2,3). Test 1: only CTA 0 issues one multicast load to CTAs {0, 2}, naming its own
// barrier. H1 (per destination, redirected to the destination's pair leader): the barriers of CTA 0 and CTA 2 each see
// 16 KiB. H2 (all bytes on the named barrier): CTA 0 sees 32 KiB, CTA 2 nothing. Test 2: CTA 1 issues to {1, 3} naming
// the barrier of ITS LEADER (CTA 0): H1 -> barriers of CTA 0 and CTA 2 see 16 KiB each. Test 3: the pattern the GEMM would
// use (every CTA multicasts its quarter of A to {r, r^2}, plus a private B box), data verified.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
__device__ bool wait_bounded(uint32_t bar, uint32_t parity, long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles)
        if (try_wait(bar, parity)) return true;
    return false;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void load_mc(uint32_t dst, const void* map, uint32_t bar, int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void load_2sm(uint32_t dst, const void* map, uint32_t bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(map),
                 "r"(c0), "r"(c1), "r"(bar)
                 : "memory");
}

// rows of 64 bf16 (128 B); box = 128 rows x 64 = 16 KiB. Row r holds the value r in every element (as uint16).
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(32) probe(const __grid_constant__ CUtensorMap map, int* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gen = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t bar = base + 3 * 16384; // barriers after three 16 KiB slots
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8 * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();
    const long long kWait = 20000000ll;
    // ---- test 1: CTA 0 multicasts to {0, 2}, naming its own barrier 0
    if (lane == 0) {
        if (rank == 0 || rank == 2) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(16384) : "memory");
    }
    cluster_sync();
    if (lane == 0 && rank == 0) load_mc(base, &map, bar, 0, 0, 0x5);
    if (lane == 0 && (rank == 0 || rank == 2)) out[rank] = wait_bounded(bar, 0, kWait) ? 1 : 0; // H1: both 1; H2: both 0 (CTA 0 over-counts)
    cluster_sync();
    // ---- test 2: CTA 1 multicasts to {1, 3}, naming the barrier 1 of ITS LEADER (CTA 0)
    if (lane == 0 && (rank == 0 || rank == 2)) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar + 8), "r"(16384) : "memory");
    cluster_sync();
    if (lane == 0 && rank == 1) load_mc(base, &map, mapa(bar + 8, 0), 0, 128, 0xA);
    if (lane == 0 && (rank == 0 || rank == 2)) out[4 + rank] = wait_bounded(bar + 8, 0, kWait) ? 1 : 0;
    cluster_sync();
    // ---- test 3: GEMM pattern. CTA r loads A quarter (rows 512 + 128 * quarter index) into slot (r >> 1) of CTAs {r, r ^ 2},
    // and a private box into slot 2; pair leaders expect 2 * (2 * 16 KiB + 16 KiB) = 96 KiB on barrier 2.
    if (lane == 0 && (rank & 1) == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar + 16), "r"(6 * 16384) : "memory");
    cluster_sync();
    if (lane == 0) {
        const uint32_t lbar = mapa(bar + 16, rank & ~1u);
        const int a_row = 512 + static_cast<int>(rank & 1) * 256 + static_cast<int>(rank >> 1) * 128;
        load_mc(base + (rank >> 1) * 16384, &map, lbar, 0, a_row, static_cast<uint16_t>((1u << rank) | (1u << (rank ^ 2u))));
        load_2sm(base + 2 * 16384, &map, lbar, 0, 2048 + static_cast<int>(rank) * 128);
    }
    bool ok3 = true;
    if ((rank & 1) == 0) {
        if (lane == 0) out[8 + rank] = wait_bounded(bar + 16, 0, kWait) ? 1 : 0;
    }
    __syncwarp();
    cluster_sync(); // the leaders have seen every byte of their pair (or timed out)
    // verify: slot q of CTA r holds rows 512 + (r & 1) * 256 + q * 128 ..; slot 2 rows 2048 + r * 128 (128B swizzle keeps a row's value)
    for (int q = 0; q < 3; ++q) {
        const int row0 = q < 2 ? 512 + static_cast<int>(rank & 1) * 256 + q * 128 : 2048 + static_cast<int>(rank) * 128;
        for (int r = lane; r < 128; r += 32) {
            const uint16_t v = *reinterpret_cast<const uint16_t*>(gen + q * 16384 + r * 128);
            if (v != static_cast<uint16_t>(row0 + r)) ok3 = false;
        }
    }
    ok3 = __all_sync(0xffffffffu, ok3);
    if (lane == 0) out[12 + rank] = ok3 ? 1 : 0;
}

int main() {
    const int rows = 4096, cols = 64;
    uint16_t* h = new uint16_t[rows * cols];
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) h[r * cols + c] = static_cast<uint16_t>(r);
    uint16_t* d;
    cudaMalloc(&d, rows * cols * 2);
    cudaMemcpy(d, h, rows * cols * 2, cudaMemcpyHostToDevice);
    int* out;
    cudaMalloc(&out, 64 * sizeof(int));
    cudaMemset(out, 0xff, 64 * sizeof(int));
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                            const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    CUtensorMap map;
    const cuuint64_t gd[2] = {cols, rows};
    const cuuint64_t gs[1] = {cols * 2};
    const cuuint32_t bx[2] = {cols, 128};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = reinterpret_cast<Fn>(fp)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", int(r));
    const size_t smem = 3 * 16384 + 1024 + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    probe<<<4, 32, smem>>>(map, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    int ho[64];
    cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("test1 (CTA0 -> {0,2}, own barrier): leader0 %d leader2 %d   [H1: 1 1, H2: 0 0]\n", ho[0], ho[2]);
    printf("test2 (CTA1 -> {1,3}, leader's barrier): leader0 %d leader2 %d   [H1: 1 1]\n", ho[4], ho[6]);
    printf("test3 (GEMM pattern): leader0 %d leader2 %d, data ok per CTA: %d %d %d %d\n", ho[8], ho[10], ho[12], ho[13], ho[14], ho[15]);
    return 0;
}

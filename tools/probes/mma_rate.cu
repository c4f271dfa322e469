// Scratch probe: raw tcgen05.mma issue/retire rate (cycles per instruction) for kind::f16 bf16, K = 16, with
// operands resident in shared memory (zeros), no TMA traffic and no epilogue. Answers: what is the tensor-pipe floor of
// one 128xNx16 (cta_group::1) or 256xNx16 (cta_group::2) instruction on this part?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
__device__ __forceinline__ uint64_t make_desc(uint32_t addr) { return (static_cast<uint64_t>(kDescHi) << 32) | ((addr >> 4) & 0x3fffu) | (1u << 16); }

template <int CG> __device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (CG == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_mc(uint32_t bar) {
    const uint16_t mask = 3;
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar), "h"(mask) : "memory");
}
template <int CG> __device__ __forceinline__ void commit(uint32_t bar) {
    if constexpr (CG == 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    else asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

template <int CG>
__global__ void __launch_bounds__(128, 1) rate_kernel(int N, int iters, int per_commit, int stages, long long* out, int st_warps = 0, int st_gap = 0) {
    __shared__ volatile int stop_flag;
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bars[2];
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    for (uint32_t i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    uint32_t rank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) stop_flag = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp >= 1 && warp <= st_warps) {
        // background shared-memory store traffic (conflict-free 512 B per warp instruction) next to the MMAs
        const uint32_t dst = base + 160 * 1024 + (warp - 1) * 8192 + (threadIdx.x & 31) * 16;
        long long n = 0;
        const long long t0 = clock64();
        while (!stop_flag) {
#pragma unroll
            for (int u = 0; u < 16; ++u)
                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(dst + u * 512), "r"(u) : "memory");
            n += 16;
            if (st_gap) __nanosleep(st_gap);
        }
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) { out[300 + blockIdx.x * 4 + warp] = n * 512; out[300 + blockIdx.x * 4] = t1 - t0; }
    }
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>((128 * CG) >> 4) << 24);
        const uint32_t stage_bytes = 16384 + (N / CG) * 128;
        const long long t0 = clock64();
        int n = 0, st = 0;
        for (int i = 0; i < iters; ++i) {
            const uint32_t a = base + st * stage_bytes, b = a + 16384;
#pragma unroll
            for (int k = 0; k < 4; ++k) mma<CG>(tmem, make_desc(a + 32 * k), make_desc(b + 32 * k), idesc, (i | k) ? 1u : 0u);
            n += 4;
            if (per_commit > 0 && n % per_commit == 0) commit<CG>(smem_u32(&bars[1]));
            if (per_commit < 0 && n % (-per_commit) == 0) { if constexpr (CG == 2) commit_mc(smem_u32(&bars[1])); }
            if (++st == stages) st = 0;
        }
        commit<CG>(smem_u32(&bars[0]));
        const long long t1 = clock64();
        uint32_t ok = 0;
        while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bars[0])) : "memory");
        const long long t2 = clock64();
        out[blockIdx.x * 2 + 0] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
        stop_flag = 1;
    }
    if (threadIdx.x == 0 && rank != 0) {
        // peer CTA: keep its store warps running for about as long as the leader's MMAs
        const long long t0 = clock64();
        while (clock64() - t0 < 128ll * 4 * iters) {}
        stop_flag = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    if (threadIdx.x < 32) {
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

template <int CG> void run(int N, int iters, int per_commit, int stages, int ctas, int st_warps = 0, int st_gap = 0) {
    long long* d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    cudaMemset(d, 0, 1024 * sizeof(long long));
    const int smem = 201 * 1024;
    cudaFuncSetAttribute(rate_kernel<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem; cfg.attrs = attr; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, rate_kernel<CG>, N, iters, per_commit, stages, d, st_warps, st_gap);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (st_warps) {
        double bytes = 0;
        for (int w = 1; w <= st_warps; ++w) bytes += (double)h[300 + w];
        printf("   + %d store warps (gap %d ns): %.1f B/clk of st.shared in CTA 0\n", st_warps, st_gap, bytes / (double)h[300]);
    }
    printf("cta_group::%d M=%d N=%3d ctas=%3d commit/%d stages=%d: issue %.1f cyc/mma, retire %.1f cyc/mma  (%s)\n", CG, 128 * CG, N, ctas,
           per_commit, stages, (double)h[0] / (iters * 4.0), (double)h[1] / (iters * 4.0), cudaGetErrorString(e));
    cudaFree(d);
}


// Issue-queue depth: time stamps after each of the first 24 MMA issues (idle pipe at start).
__global__ void __launch_bounds__(128, 1) depth_kernel(long long* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    for (uint32_t i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(256 >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
        long long t[25];
        const uint64_t da = make_desc(base), db = make_desc(base + 16384);
        t[0] = clock64();
#pragma unroll
        for (int i = 0; i < 24; ++i) {
            mma<1>(tmem, da, db, idesc, 1u);
            t[i + 1] = clock64();
        }
        commit<1>(smem_u32(&bar));
        uint32_t ok = 0;
        while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        const long long te = clock64();
        for (int i = 0; i < 25; ++i) out[i] = t[i] - t[0];
        out[25] = te - t[0];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}
void run_depth() {
    long long* d;
    cudaMalloc(&d, 32 * sizeof(long long));
    cudaFuncSetAttribute(depth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 101 * 1024);
    for (int rep = 0; rep < 2; ++rep) depth_kernel<<<1, 128, 101 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("issue time stamps (cycles after the first issue), 24 MMAs 128x256x16, then all retired at %lld (%s):\n  ", h[25], cudaGetErrorString(e));
    for (int i = 1; i <= 24; ++i) printf("%lld ", h[i]);
    printf("\n");
    cudaFree(d);
}

int main() {
    run_depth();
    const int iters = 4096;
    run<2>(256, iters, 0, 4, 148);
    run<2>(256, iters, -4, 4, 148);
    return 0;
}

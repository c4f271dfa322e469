// Scratch probe: idle gap between back-to-back launches of a persistent-style kernel (148 CTAs, ~50 us each) as a
// function of cluster size, dynamic shared memory and parameter size.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
struct Big { unsigned char bytes[640]; };
template <int PARAM>
__global__ void __launch_bounds__(320, 1) k(unsigned long long* t, int launch, long long spin, const __grid_constant__ Big big) {
    extern __shared__ unsigned char smem[];
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    if (threadIdx.x == 0) {
        if (PARAM && big.bytes[5] == 77) smem[0] = 1;
        const long long c0 = clock64();
        while (clock64() - c0 < spin) {}
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        atomicMin(&t[2 * launch], g0);
        atomicMax(&t[2 * launch + 1], g1);
    }
}
// variant: TMEM allocation of all 512 columns by one warp (cta_group::2 when clustered), released before exit
template <int CG>
__global__ void __launch_bounds__(320, 1) ktmem(unsigned long long* t, int launch, long long spin) {
    __shared__ unsigned slot;
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&slot));
    if (threadIdx.x < 32) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const long long c0 = clock64();
        while (clock64() - c0 < spin) {}
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    if (threadIdx.x < 32) {
        const unsigned ta = slot;
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(ta) : "memory");
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(ta) : "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        atomicMin(&t[2 * launch], g0);
        atomicMax(&t[2 * launch + 1], g1);
    }
}
template <int CG> void run_tmem(const char* name) {
    const int N = 20;
    unsigned long long* d;
    cudaMalloc(&d, 2 * N * sizeof(unsigned long long));
    unsigned long long h[2 * N];
    for (int i = 0; i < N; ++i) { h[2 * i] = ~0ull; h[2 * i + 1] = 0; }
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int i = 0; i < N; ++i) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = 0; cfg.attrs = attr; cfg.numAttrs = CG > 1 ? 1 : 0;
        cudaLaunchKernelEx(&cfg, ktmem<CG>, d, i, 80000ll);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double gap = 0, dur = 0;
    for (int i = 5; i < N; ++i) { gap += (double)(h[2 * i] - h[2 * i - 1]); dur += (double)(h[2 * i + 1] - h[2 * i]); }
    printf("%-44s cluster %d: kernel %.1f us, gap to next launch %.2f us (%s)\n", name, CG, dur / (N - 5) / 1e3, gap / (N - 5) / 1e3, cudaGetErrorString(e));
    cudaFree(d);
}
template <int PARAM> void run(int cluster, int smem, const char* name) {
    const int N = 20;
    unsigned long long* d;
    cudaMalloc(&d, 2 * N * sizeof(unsigned long long));
    unsigned long long h[2 * N];
    for (int i = 0; i < N; ++i) { h[2 * i] = ~0ull; h[2 * i + 1] = 0; }
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k<PARAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    Big big; memset(&big, 0, sizeof(big));
    for (int i = 0; i < N; ++i) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cluster; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem; cfg.attrs = attr; cfg.numAttrs = cluster > 1 ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k<PARAM>, d, i, 80000ll, big);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double gap = 0, dur = 0;
    for (int i = 5; i < N; ++i) { gap += (double)(h[2 * i] - h[2 * i - 1]); dur += (double)(h[2 * i + 1] - h[2 * i]); }
    printf("%-44s cluster %d smem %6d: kernel %.1f us, gap to next launch %.2f us (%s)\n", name, cluster, smem, dur / (N - 5) / 1e3, gap / (N - 5) / 1e3, cudaGetErrorString(e));
    cudaFree(d);
}
int main() {
    run<0>(1, 0, "plain");
    run<0>(1, 230000, "230 KB smem");
    run<0>(2, 0, "cluster 2");
    run<0>(2, 230000, "cluster 2, 230 KB smem");
    run<1>(2, 230000, "cluster 2, 230 KB smem, 640 B param read");
    run_tmem<1>("TMEM 512 columns alloc/dealloc");
    run_tmem<2>("TMEM 512 columns alloc/dealloc");
    return 0;
}

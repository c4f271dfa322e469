// Host-buffer entry points: the call a user of the reference makes (tla::copy / tla::gemm on
// host-resident cells), served by the device path. Buffers are staged through a per-thread device
// buffer; the destination is read back before returning.
// There is no CPU compute here: without a device these return TLB_ERR_CUDA.
#include <cstring>

#include "tlb_internal.h"

namespace tlb {
namespace {

// Per-thread staging context: one stream and one grow-only device buffer, created on first use and kept for the
// life of the thread. (A stream and three cudaMallocAsync allocations per call cost 1-15 ms per call: the default
// pool hands its memory back at every synchronise, and a fresh stream pays the driver's per-stream setup.)
struct HostCtx {
    cudaStream_t s = nullptr;
    int device = -1;
    char* buf = nullptr;
    size_t cap = 0, used = 0;
    // No destructor on purpose: at thread / process exit the CUDA runtime may already be shutting down, and the
    // driver reclaims the stream and the buffer with the context.
    int begin(size_t total_bytes) {
        int dev = 0;
        TLB_CUDA(cudaGetDevice(&dev));
        if (dev != device) {
            if (buf) cudaFree(buf);
            if (s) cudaStreamDestroy(s);
            buf = nullptr;
            s = nullptr;
            cap = 0;
            device = dev;
        }
        if (!s) TLB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        if (total_bytes > cap) {
            if (buf) {
                TLB_CUDA(cudaStreamSynchronize(s));
                TLB_CUDA(cudaFree(buf));
                buf = nullptr;
                cap = 0;
            }
            TLB_CUDA(cudaMalloc(reinterpret_cast<void**>(&buf), total_bytes));
            cap = total_bytes;
        }
        used = 0;
        return TLB_OK;
    }
    void* take(size_t bytes) {
        void* p = buf + used;
        used += (bytes + 255) & ~static_cast<size_t>(255);
        return p;
    }
};
thread_local HostCtx g_host;

size_t staged_bytes(const tlb_tensor& t) {
    if (t.accessor != TLB_ACC_BUFFER) return 0;
    const size_t bytes = static_cast<size_t>(t.capacity) * t.elem_bytes;
    return ((bytes ? bytes : 16) + 255) & ~static_cast<size_t>(255);
}

int stage_in(const tlb_tensor& host, bool upload, HostCtx& ctx, tlb_tensor* dev) {
    *dev = host;
    if (host.accessor != TLB_ACC_BUFFER) return TLB_OK;
    const size_t bytes = static_cast<size_t>(host.capacity) * host.elem_bytes;
    void* p = ctx.take(bytes ? bytes : 16);
    if (upload && bytes) TLB_CUDA(cudaMemcpyAsync(p, host.data, bytes, cudaMemcpyHostToDevice, ctx.s));
    dev->data = p;
    return TLB_OK;
}

// True when every cell of the buffer is overwritten by a store through this layout, so the
// old contents need not be uploaded.
bool covers_buffer(const tlb_tensor& t) {
    const tlb_layout_desc& L = *t.layout;
    return L.kind == TLB_KIND_INT && (L.flags & TLB_LF_INJECTIVE) && t.origin + L.min_offset == 0 &&
           t.origin + L.max_offset == t.capacity - 1 && L.size == t.capacity;
}

} // namespace
} // namespace tlb

using namespace tlb;

extern "C" {

int tlb_copy_host(const tlb_tensor* src, const tlb_tensor* dst) {
    TLB_TRY(check_tensor(src, "tlb_copy_host source", false));
    TLB_TRY(check_tensor(dst, "tlb_copy_host destination", true));
    TLB_TRY(require_device());
    HostCtx& ctx = g_host;
    TLB_TRY(ctx.begin(staged_bytes(*src) + staged_bytes(*dst)));
    tlb_tensor ds, dd;
    TLB_TRY(stage_in(*src, true, ctx, &ds));
    TLB_TRY(stage_in(*dst, !covers_buffer(*dst), ctx, &dd));
    TLB_TRY(copy_impl(&ds, &dd, 0, UINT64_MAX, ctx.s));
    TLB_CUDA(cudaMemcpyAsync(dst->data, dd.data, static_cast<size_t>(dst->capacity) * dst->elem_bytes,
                             cudaMemcpyDeviceToHost, ctx.s));
    TLB_CUDA(cudaStreamSynchronize(ctx.s));
    return TLB_OK;
}

int tlb_gemm_bf16_host(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C) {
    TLB_TRY(check_tensor(A, "tlb_gemm_bf16_host A", false));
    TLB_TRY(check_tensor(B, "tlb_gemm_bf16_host B", false));
    TLB_TRY(check_tensor(C, "tlb_gemm_bf16_host C", true));
    TLB_TRY(require_device());
    HostCtx& ctx = g_host;
    TLB_TRY(ctx.begin(staged_bytes(*A) + staged_bytes(*B) + staged_bytes(*C)));
    tlb_tensor da, db, dc;
    TLB_TRY(stage_in(*A, true, ctx, &da));
    TLB_TRY(stage_in(*B, true, ctx, &db));
    TLB_TRY(stage_in(*C, true, ctx, &dc)); // C += ...: the accumulator starts from C
    TLB_TRY(gemm_bf16_impl(&da, &db, &dc, 0, 0, 0, 0, 1, 0, UINT32_MAX, ctx.s));
    TLB_CUDA(cudaMemcpyAsync(C->data, dc.data, static_cast<size_t>(C->capacity) * C->elem_bytes, cudaMemcpyDeviceToHost,
                             ctx.s));
    TLB_CUDA(cudaStreamSynchronize(ctx.s));
    return TLB_OK;
}

} // extern "C"

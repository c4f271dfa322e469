// Host-buffer entry points: the call a user of the reference makes (tla::copy / tla::gemm on
// host-resident cells), served by the device path. Buffers are staged through device memory
// that lives for the duration of the call; the destination is read back before returning.
// There is no CPU compute here: without a device these return TLB_ERR_CUDA.
#include <cstring>

#include "tlb_internal.h"

namespace tlb {
namespace {

struct DeviceBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DeviceBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() {
        if (s) cudaStreamDestroy(s);
    }
};

int stage_in(const tlb_tensor& host, bool upload, cudaStream_t s, DeviceBuf* buf, tlb_tensor* dev) {
    *dev = host;
    if (host.accessor != TLB_ACC_BUFFER) return TLB_OK;
    const size_t bytes = static_cast<size_t>(host.capacity) * host.elem_bytes;
    buf->s = s;
    TLB_CUDA(cudaMallocAsync(&buf->p, bytes ? bytes : 16, s));
    if (upload && bytes) TLB_CUDA(cudaMemcpyAsync(buf->p, host.data, bytes, cudaMemcpyHostToDevice, s));
    dev->data = buf->p;
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
    StreamGuard sg;
    TLB_CUDA(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
    DeviceBuf bs, bd;
    tlb_tensor ds, dd;
    TLB_TRY(stage_in(*src, true, sg.s, &bs, &ds));
    TLB_TRY(stage_in(*dst, !covers_buffer(*dst), sg.s, &bd, &dd));
    TLB_TRY(copy_impl(&ds, &dd, 0, UINT64_MAX, sg.s));
    TLB_CUDA(cudaMemcpyAsync(dst->data, dd.data, static_cast<size_t>(dst->capacity) * dst->elem_bytes,
                             cudaMemcpyDeviceToHost, sg.s));
    TLB_CUDA(cudaStreamSynchronize(sg.s));
    return TLB_OK;
}

int tlb_gemm_bf16_host(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C) {
    TLB_TRY(check_tensor(A, "tlb_gemm_bf16_host A", false));
    TLB_TRY(check_tensor(B, "tlb_gemm_bf16_host B", false));
    TLB_TRY(check_tensor(C, "tlb_gemm_bf16_host C", true));
    TLB_TRY(require_device());
    StreamGuard sg;
    TLB_CUDA(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
    DeviceBuf ba, bb, bc;
    tlb_tensor da, db, dc;
    TLB_TRY(stage_in(*A, true, sg.s, &ba, &da));
    TLB_TRY(stage_in(*B, true, sg.s, &bb, &db));
    TLB_TRY(stage_in(*C, true, sg.s, &bc, &dc)); // C += ...: the accumulator starts from C
    TLB_TRY(gemm_bf16_impl(&da, &db, &dc, 0, 0, 0, 0, 1, 0, UINT32_MAX, sg.s));
    TLB_CUDA(cudaMemcpyAsync(C->data, dc.data, static_cast<size_t>(C->capacity) * C->elem_bytes, cudaMemcpyDeviceToHost,
                             sg.s));
    TLB_CUDA(cudaStreamSynchronize(sg.s));
    return TLB_OK;
}

} // extern "C"

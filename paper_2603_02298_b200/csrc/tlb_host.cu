// Host-buffer entry points: the call a user of the reference makes (tla::copy / tla::gemm on
// host-resident cells), served by the device path. Buffers are staged through a per-thread device
// buffer; the destination is read back before returning.
// There is no CPU compute here: without a device these return TLB_ERR_CUDA.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tlb_internal.h"

namespace tlb {
namespace {

// Per-thread staging context: one stream and one grow-only device buffer, created on first use and kept for the
// life of the thread. (A stream and three cudaMallocAsync allocations per call cost 1-15 ms per call: the default
// pool hands its memory back at every synchronise, and a fresh stream pays the driver's per-stream setup.)
constexpr int kMaxPanels = 16;
struct HostCtx {
    cudaStream_t s = nullptr;
    int device = -1;
    char* buf = nullptr;
    size_t cap = 0, used = 0;
    // No destructor on purpose: at thread / process exit the CUDA runtime may already be shutting down, and the
    // driver reclaims the stream and the buffer with the context.
    cudaStream_t s2 = nullptr;       // second stream of the pipelined GEMM: compute + download, while `s` uploads
    cudaEvent_t ev[kMaxPanels + 1] = {};
    int begin(size_t total_bytes) {
        int dev = 0;
        TLB_CUDA(cudaGetDevice(&dev));
        if (dev != device) {
            if (buf) cudaFree(buf);
            if (s) cudaStreamDestroy(s);
            if (s2) cudaStreamDestroy(s2);
            for (cudaEvent_t& e : ev)
                if (e) cudaEventDestroy(e), e = nullptr;
            buf = nullptr;
            s = nullptr;
            s2 = nullptr;
            cap = 0;
            device = dev;
        }
        if (!s) {
            TLB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            TLB_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
            for (cudaEvent_t& e : ev) TLB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
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

// Pipelined host GEMM: C2-sized problems are PCIe bound (128 MB up, 64 MB down against 0.1 ms of math), so the
// download of finished panels of C should run under the upload of the next ones. Applies to flat row-major-style
// problems: K-major A and B and a C with one contiguous mode. The operand that is NOT sliced goes up first, then
// panels of 512 rows of the other operand and of C; each panel's GEMM and download run on the second stream.
// Returns false (nothing enqueued) when the problem does not have that shape.
bool gemm_host_pipelined(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, HostCtx& ctx, int* status) {
    *status = TLB_OK;
    if (knob(K_HOST_PIPELINE) == 0) return false;
    GemmFlat f;
    if (C->elem_bytes != 4 || !gemm_flat_view(A, B, C, &f)) return false;
    if (f.a_sk != 1 || f.b_sk != 1 || f.a_sm < f.K || f.b_sn < f.K) return false;
    const bool c_m_contig = f.c_sm == 1 && f.c_sn >= f.M;         // C (M,N):(1,ldc): slice along n (B and C panels)
    const bool c_n_contig = f.c_sn == 1 && f.c_sm >= f.N;         // C (M,N):(ldc,1): slice along m (A and C panels)
    if (!c_m_contig && !c_n_contig) return false;
    const bool slice_n = c_m_contig;
    // measured on C2: 3.03 ms with 1024-row panels (the default), 3.09 with 512, 3.22 with 2048, 3.76 unpipelined
    const int64_t panel = std::max(512, knob(K_HOST_PANEL) / 512 * 512);
    const int64_t rows = slice_n ? f.N : f.M;
    if ((rows + panel - 1) / panel < 2 || (rows + panel - 1) / panel > kMaxPanels - 3) return false;
    // Panel boundaries: full panels, then the last one tapers (1/2, 1/4, 1/4 of a panel, never below 256 rows). What is
    // left after the last upload is that panel's GEMM and download, so the tail should be small: 4 MiB instead of 16 MiB
    // of C on the C2 shape (HOST_TAPER=0 keeps uniform panels).
    int64_t cut[kMaxPanels + 1];
    int n_panels = 0;
    cut[0] = 0;
    {
        int64_t r = 0;
        while (rows - r > panel) cut[++n_panels] = (r += panel);
        const int64_t last = rows - r;
        if (knob(K_HOST_TAPER) != 0 && last >= 1024 && last % 4 == 0) {
            cut[++n_panels] = (r += last / 2);
            cut[++n_panels] = (r += last / 4);
        }
        cut[++n_panels] = rows;
    }
    // the whole buffers are mirrored at the same offsets on the device; a panel is the same layout with fewer rows
    const tlb_tensor& whole_h = slice_n ? *A : *B;                 // uploaded first, in full
    const tlb_tensor& sliced_h = slice_n ? *B : *A;
    const int64_t ld_s = slice_n ? f.b_sn : f.a_sm, ld_c = slice_n ? f.c_sn : f.c_sm;
    auto fail_with = [&](int st) {
        *status = st;
        return true;
    };
#define TLB_P(call)                                               \
    do {                                                          \
        const int st_ = (call);                                   \
        if (st_ != TLB_OK) return fail_with(st_);                 \
    } while (0)
#define TLB_PC(call)                                              \
    do {                                                          \
        if ((call) != cudaSuccess) return fail_with(fail(TLB_ERR_CUDA, cudaGetErrorString(cudaGetLastError()))); \
    } while (0)
    // every contract and bounds failure must surface before the first byte of C can change: check the whole tensors
    {
        Span sp;
        TLB_P(bounds_preflight(*A, 0, static_cast<uint64_t>(A->layout->size), "A", nullptr, &sp));
        TLB_P(bounds_preflight(*B, 0, static_cast<uint64_t>(B->layout->size), "B", nullptr, &sp));
        TLB_P(bounds_preflight(*C, 0, static_cast<uint64_t>(C->layout->size), "C", nullptr, &sp));
        if (!(C->layout->flags & TLB_LF_INJECTIVE)) return false;
    }
    TLB_P(ctx.begin(staged_bytes(*A) + staged_bytes(*B) + staged_bytes(*C)));
    char* d_whole = static_cast<char*>(ctx.take(static_cast<size_t>(whole_h.capacity) * 2));
    char* d_sliced = static_cast<char*>(ctx.take(static_cast<size_t>(sliced_h.capacity) * 2));
    char* d_c = static_cast<char*>(ctx.take(static_cast<size_t>(C->capacity) * 4));
    TLB_PC(cudaMemcpyAsync(d_whole, whole_h.data, static_cast<size_t>(whole_h.capacity) * 2, cudaMemcpyHostToDevice, ctx.s));
    tlb_tensor dw = whole_h;
    dw.data = d_whole;
    for (int p = 0; p < n_panels; ++p) {
        const int64_t r0 = cut[p], nr = cut[p + 1] - r0;
        // element ranges of the panel inside the two sliced buffers (rows r0 .. r0 + nr, padding included)
        const int64_t s_off = sliced_h.origin + r0 * ld_s, s_len = (nr - 1) * ld_s + f.K;
        const int64_t c_off = C->origin + r0 * ld_c, c_len = (nr - 1) * ld_c + (slice_n ? f.M : f.N);
        TLB_PC(cudaMemcpyAsync(d_sliced + s_off * 2, static_cast<const char*>(sliced_h.data) + s_off * 2, static_cast<size_t>(s_len) * 2,
                               cudaMemcpyHostToDevice, ctx.s));
        TLB_PC(cudaMemcpyAsync(d_c + c_off * 4, static_cast<const char*>(C->data) + c_off * 4, static_cast<size_t>(c_len) * 4,
                               cudaMemcpyHostToDevice, ctx.s));
        TLB_PC(cudaEventRecord(ctx.ev[p], ctx.s));
        TLB_PC(cudaStreamWaitEvent(ctx.s2, ctx.ev[p], 0));
        // panel layouts: (nr, K):(ld, 1) for the sliced operand; C panel keeps C's two strides
        tlb_mode ms[2] = {{nr, ld_s, TLB_KIND_INT, 0}, {f.K, 1, TLB_KIND_INT, 0}};
        tlb_mode mc[2] = {{slice_n ? f.M : nr, f.c_sm, TLB_KIND_INT, 0}, {slice_n ? nr : f.N, f.c_sn, TLB_KIND_INT, 0}};
        const int32_t tops[2] = {1, 1};
        tlb_layout_desc ls, lc;
        TLB_P(tlb_layout_lower_ranked(ms, 2, tops, 2, &ls));
        TLB_P(tlb_layout_lower_ranked(mc, 2, tops, 2, &lc));
        tlb_tensor ts = sliced_h, tc = *C;
        ts.layout = &ls;
        ts.data = d_sliced;
        ts.origin = s_off;
        tc.layout = &lc;
        tc.data = d_c;
        tc.origin = c_off;
        TLB_P(gemm_bf16_impl(slice_n ? &dw : &ts, slice_n ? &ts : &dw, &tc, 0, 0, 0, 0, 1, 0, UINT32_MAX, ctx.s2));
        TLB_PC(cudaMemcpyAsync(static_cast<char*>(C->data) + c_off * 4, d_c + c_off * 4, static_cast<size_t>(c_len) * 4,
                               cudaMemcpyDeviceToHost, ctx.s2));
    }
    TLB_PC(cudaStreamSynchronize(ctx.s2));
    TLB_PC(cudaStreamSynchronize(ctx.s));
#undef TLB_P
#undef TLB_PC
    return true;
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
    // Views of ONE host storage (tensor.hpp:29): when the two host buffers overlap they are staged as one device
    // image, so that tlb_copy sees the same aliasing the reference would and resolves it to the serial result.
    if (src->accessor == TLB_ACC_BUFFER && src->elem_bytes == dst->elem_bytes) {
        const char* s0 = static_cast<const char*>(src->data);
        const char* s1 = s0 + static_cast<size_t>(src->capacity) * src->elem_bytes;
        char* d0 = static_cast<char*>(dst->data);
        char* d1 = d0 + static_cast<size_t>(dst->capacity) * dst->elem_bytes;
        if (s0 < d1 && d0 < s1) {
            const char* lo = std::min<const char*>(s0, d0);
            const char* hi = std::max<const char*>(s1, d1);
            const size_t bytes = static_cast<size_t>(hi - lo);
            TLB_TRY(ctx.begin((bytes + 255) & ~static_cast<size_t>(255)));
            char* img = static_cast<char*>(ctx.take(bytes));
            TLB_CUDA(cudaMemcpyAsync(img, lo, bytes, cudaMemcpyHostToDevice, ctx.s));
            tlb_tensor ds = *src, dd = *dst;
            ds.data = img + (s0 - lo);
            dd.data = img + (d0 - lo);
            TLB_TRY(copy_impl(&ds, &dd, 0, UINT64_MAX, ctx.s));
            TLB_CUDA(cudaMemcpyAsync(d0, dd.data, static_cast<size_t>(d1 - d0), cudaMemcpyDeviceToHost, ctx.s));
            TLB_CUDA(cudaStreamSynchronize(ctx.s));
            return TLB_OK;
        }
    }
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

// eval_int over a range into HOST memory: the map is produced in 2^24-element pieces on stream s2 into a two-piece device
// ring while the previous piece drains over PCIe on stream s (the download is the bottleneck: 8 B per evaluation).
int tlb_eval_range_host(const tlb_layout_desc* layout, uint64_t i0, uint64_t n, int64_t* h_out) {
    if (!layout) return fail(TLB_ERR_CONTRACT, "tlb_eval_range_host: null layout");
    if (n == 0) return TLB_OK;
    if (!h_out) return fail(TLB_ERR_CONTRACT, "tlb_eval_range_host: null output");
    TLB_TRY(require_device());
    HostCtx& ctx = g_host;
    const uint64_t piece = std::min<uint64_t>(n, 1ull << 24);
    TLB_TRY(ctx.begin(2 * piece * sizeof(int64_t)));
    int64_t* ring[2] = {static_cast<int64_t*>(ctx.take(piece * sizeof(int64_t))), static_cast<int64_t*>(ctx.take(piece * sizeof(int64_t)))};
    int k = 0;
    for (uint64_t done = 0; done < n; done += piece, ++k) {
        const uint64_t cnt = std::min(piece, n - done);
        const int slot = k & 1;
        // the download that last used this slot (piece k - 2) must be finished before it is overwritten
        if (k >= 2) TLB_CUDA(cudaStreamWaitEvent(ctx.s2, ctx.ev[2 + slot], 0));
        TLB_TRY(tlb_eval_range(layout, i0 + done, cnt, ring[slot], ctx.s2));
        TLB_CUDA(cudaEventRecord(ctx.ev[slot], ctx.s2));
        TLB_CUDA(cudaStreamWaitEvent(ctx.s, ctx.ev[slot], 0));
        TLB_CUDA(cudaMemcpyAsync(h_out + done, ring[slot], cnt * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.s));
        TLB_CUDA(cudaEventRecord(ctx.ev[2 + slot], ctx.s));
    }
    TLB_CUDA(cudaStreamSynchronize(ctx.s));
    TLB_CUDA(cudaStreamSynchronize(ctx.s2));
    return TLB_OK;
}

int tlb_gemm_bf16_host(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C) {
    TLB_TRY(check_tensor(A, "tlb_gemm_bf16_host A", false));
    TLB_TRY(check_tensor(B, "tlb_gemm_bf16_host B", false));
    TLB_TRY(check_tensor(C, "tlb_gemm_bf16_host C", true));
    TLB_TRY(require_device());
    HostCtx& ctx = g_host;
    int pst = TLB_OK;
    if (gemm_host_pipelined(A, B, C, ctx, &pst)) return pst;
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

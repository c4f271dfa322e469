// Host lowering: flat leaves of a tla::Layout -> tlb_layout_desc (device evaluator
// parameters), plus the host-side pre-flight proofs (bounds, overflow, injectivity) that
// stand in for the reference's per-access checks (tensor.hpp:99, common.hpp:99-109).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tlb_internal.h"

namespace tlb {

namespace {
thread_local std::string g_error;
thread_local const char* g_plan = "";
std::atomic<uint64_t> g_launches{0};
} // namespace

int fail(int status, const std::string& msg) {
    g_error = msg;
    return status;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_error = std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what;
    (void)cudaGetLastError(); // clear the sticky-less error state
    return TLB_ERR_CUDA;
}

void set_plan(const char* name) { g_plan = name; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
struct KnobDef {
    const char* name;
    int def;
};
// index = KnobId
const KnobDef kKnobDefs[K_COUNT] = {
    {"GEMM_WIDE", -1}, {"GEMM_SPLIT_TAIL", 1}, {"GEMM_EPILOGUE", 0}, {"GEMM_GROUP_M", 8}, {"GEMM_BACKOFF_NS", 100},
    {"GEMM_DEBUG", 0}, {"GEMM_HINTS", 0}, {"GEMM_PDL", 1}, {"GEMM_PREFETCH_C", 0}, {"GEMM_WORKERS", 0},
    {"GEMM_C16_SK", 0}, {"GEMM_SK_PCT", 4}, {"GEMM_EPI_KB", 10}, {"GEMM_CLOCK", 0}, {"PDL", 1},
    {"COPY_TMA", 0}, {"COPY_LB256", 1}, {"COPY_PERSIST", 1}, {"EVAL_NO_WARP", 0}, {"HOST_PIPELINE", 1}, {"HOST_PANEL", 1024},
    {"COPY_TMA_STAGES", 3}, {"COPY_TMA_CTAS", 2}, {"GEMM_CHUNK_WAVES", 8}, {"GEMM_MCAST", 0}, {"GEMM_EARLY_RELEASE", 1}, {"GEMM_PACK", 1}, {"GEMM_PACK_MIN", 27},
    {"COPY_TV_COMPOSE", 1}, {"COPY_GATHER_RUN", 1}, {"COPY_RAGGED", 22}, {"COPY_INTERLEAVE", 1}, {"COPY_CELL_TILES", 1}, {"EVAL_ODOMETER", 1}, {"COPY_TILES_PER_CTA", 1}, {"COPY_ODD_TILES", 1}, {"HOST_TAPER", 1},
};
std::atomic<int> g_knobs[K_COUNT];
std::once_flag g_knobs_once;

int parse_knob(int id, const char* v) {
    if (!v || !v[0]) return kKnobDefs[id].def;
    if (id == K_GEMM_EPILOGUE) return v[0] == 'r' ? 1 : std::atoi(v);
    return std::atoi(v);
}
void load_knobs() {
    for (int i = 0; i < K_COUNT; ++i) {
        const std::string env = std::string("TLB_") + kKnobDefs[i].name;
        g_knobs[i].store(parse_knob(i, std::getenv(env.c_str())), std::memory_order_relaxed);
    }
}
} // namespace

int knob(KnobId id) {
    std::call_once(g_knobs_once, load_knobs);
    return g_knobs[id].load(std::memory_order_relaxed);
}

int require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n < 1) {
        (void)cudaGetLastError();
        return fail(TLB_ERR_CUDA, "no CUDA device: libtlb has no CPU fallback");
    }
    return TLB_OK;
}

namespace {
std::mutex g_ws_mu;
cudaMemPool_t g_ws_pools[64] = {};
} // namespace

cudaError_t ws_trim(size_t keep_bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaSuccess;
    std::lock_guard<std::mutex> lock(g_ws_mu);
    return g_ws_pools[dev] ? cudaMemPoolTrimTo(g_ws_pools[dev], keep_bytes) : cudaSuccess;
}

cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t stream) {
    std::mutex& mu = g_ws_mu;
    cudaMemPool_t* pools = g_ws_pools;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, stream);
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&pools[dev], &props);
            if (e != cudaSuccess) {
                pools[dev] = nullptr;
                (void)cudaGetLastError();
                return cudaMallocAsync(p, bytes, stream);
            }
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cached[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

namespace {

bool mul_ovf(int64_t a, int64_t b, int64_t* r) { return __builtin_mul_overflow(a, b, r); }
bool add_ovf(int64_t a, int64_t b, int64_t* r) { return __builtin_add_overflow(a, b, r); }

int ilog2_floor(uint64_t x) { return 63 - __builtin_clzll(x); }

// Division by d for every dividend 0 <= i < 2^63 (tla::Int is int64, coordinates are
// non-negative): with l = ceil(log2 d), m = floor(2^(63+l)/d) + 1 satisfies
// 2^(63+l) < m*d <= 2^(63+l) + 2^l, hence floor(i/d) = umulhi64(i, m) >> (l-1)
// (Granlund-Montgomery, N = 63). m < 2^64 because d > 2^(l-1) for non powers of two.
void make_magic(int64_t d, uint64_t* magic, uint8_t* shift, uint8_t* log2e) {
    uint64_t u = static_cast<uint64_t>(d);
    if ((u & (u - 1)) == 0) {
        *log2e = static_cast<uint8_t>(ilog2_floor(u));
        *magic = 0;
        *shift = 0;
        return;
    }
    *log2e = 0xff;
    int l = ilog2_floor(u) + 1;
    unsigned __int128 num = static_cast<unsigned __int128>(1) << (63 + l);
    *magic = static_cast<uint64_t>(num / u) + 1;
    *shift = static_cast<uint8_t>(l - 1);
}

} // namespace

void joint_set_mode(JointDesc* J, int r, int64_t extent, int64_t ss, int64_t ds) {
    J->extent[r] = extent;
    J->ss[r] = ss;
    J->ds[r] = ds;
    make_magic(extent, &J->magic[r], &J->shift[r], &J->log2e[r]);
}

namespace {

int lower_impl(const tlb_mode* modes, int n_modes, const int32_t* top_leaves, int n_top,
               tlb_layout_desc* out) {
    if (!modes || !out) return fail(TLB_ERR_CONTRACT, "tlb_layout_lower: null argument");
    if (n_modes < 1) return fail(TLB_ERR_STRUCTURAL, "empty tuples are not permitted");
    if (n_modes > TLB_MAX_MODES)
        return fail(TLB_ERR_UNSUPPORTED, "layout has more than TLB_MAX_MODES flat leaves; coalesce it first");
    std::memset(out, 0, sizeof(*out));
    out->n_modes = n_modes;
    // stride_kind (stride.hpp:158): Int(0) leaves are neutral, mixed non-zero kinds rejected.
    int kind = TLB_KIND_INT;
    bool seen = false;
    int64_t size = 1;
    int flags = TLB_LF_ALL_POW2;
    for (int r = 0; r < n_modes; ++r) {
        const tlb_mode& m = modes[r];
        if (m.extent < 1) return fail(TLB_ERR_STRUCTURAL, "shape leaves must be positive");
        if (m.kind < 0 || m.kind > 2) return fail(TLB_ERR_STRUCTURAL, "unknown stride kind");
        if (m.kind == TLB_KIND_XOR && m.stride < 0) return fail(TLB_ERR_STRUCTURAL, "xor mask must be non-negative");
        if (m.kind == TLB_KIND_BASIS && m.axis < 0) return fail(TLB_ERR_STRUCTURAL, "basis axis must be non-negative");
        bool zero = (m.kind == TLB_KIND_INT && m.stride == 0);
        if (!zero) {
            if (!seen) { kind = m.kind; seen = true; }
            else if (m.kind != kind) return fail(TLB_ERR_SEMIMODULE, "stride mixes semimodule kinds");
        }
        if (mul_ovf(size, m.extent, &size)) return fail(TLB_ERR_OVERFLOW, "integer overflow in multiplication");
        out->extent[r] = m.extent;
        out->stride[r] = m.stride;
        make_magic(m.extent, &out->magic[r], &out->shift[r], &out->log2e[r]);
        if (out->log2e[r] == 0xff) flags &= ~TLB_LF_ALL_POW2;
        if (m.kind == TLB_KIND_INT && m.stride < 0) flags |= TLB_LF_HAS_NEG;
    }
    out->kind = kind;
    out->size = size;
    if (top_leaves) {
        if (n_top < 1 || n_top > TLB_MAX_MODES) return fail(TLB_ERR_STRUCTURAL, "bad top-level rank");
        int acc = 0;
        for (int t = 0; t < n_top; ++t) {
            if (top_leaves[t] < 1) return fail(TLB_ERR_STRUCTURAL, "empty tuples are not permitted");
            out->top_start[t] = acc;
            acc += top_leaves[t];
        }
        if (acc != n_modes) return fail(TLB_ERR_STRUCTURAL, "top-level leaf counts do not sum to the leaf count");
        out->top_start[n_top] = n_modes;
        out->n_top = n_top;
    } else {
        out->n_top = 1;
        out->top_start[0] = 0;
        out->top_start[1] = n_modes;
    }
    // Offset span over the domain, cosize (layout.hpp:277).
    out->cosize = -1;
    if (kind == TLB_KIND_INT) {
        int64_t lo = 0, hi = 0;
        bool ovf = false;
        for (int r = 0; r < n_modes; ++r) {
            int64_t t;
            if (mul_ovf(out->extent[r] - 1, out->stride[r], &t)) { ovf = true; break; }
            if (t >= 0) { if (add_ovf(hi, t, &hi)) { ovf = true; break; } }
            else { if (add_ovf(lo, t, &lo)) { ovf = true; break; } }
        }
        if (ovf) {
            out->min_offset = INT64_MIN;
            out->max_offset = INT64_MAX;
        } else {
            out->min_offset = lo;
            out->max_offset = hi;
            if (!(flags & TLB_LF_HAS_NEG) && hi != INT64_MAX) out->cosize = hi + 1;
        }
    } else if (kind == TLB_KIND_XOR) {
        uint64_t orb = 0;
        for (int r = 0; r < n_modes; ++r) {
            if (out->extent[r] <= 1 || out->stride[r] == 0) continue;
            int top = ilog2_floor(static_cast<uint64_t>(out->extent[r] - 1));
            uint64_t m = static_cast<uint64_t>(out->stride[r]);
            if (top >= 62 || (m << top) >= (1ull << 62)) { orb = ~0ull >> 1; break; }
            for (int b = 0; b <= top; ++b) orb |= m << b;
        }
        out->min_offset = 0;
        out->max_offset = static_cast<int64_t>(orb);
    }
    out->flags = flags;
    if (provably_injective(*out)) out->flags |= TLB_LF_INJECTIVE;
    return TLB_OK;
}

} // namespace

// Sufficient test for injectivity on [0,size). Int kind: sort the non-trivial leaves by
// |stride| and require |d_(k+1)| >= e_k*|d_k| (the same chain the reference's left_inverse
// demands, algebra.hpp:543-552, extended to signed strides). Xor kind with power-of-two
// extents: full column rank of the bit matrix over GF(2) (linear_form, analysis.hpp:103).
bool provably_injective(const tlb_layout_desc& L) {
    if (L.kind == TLB_KIND_INT) {
        std::vector<std::pair<uint64_t, int64_t>> ms; // |stride|, extent
        for (int r = 0; r < L.n_modes; ++r) {
            if (L.extent[r] == 1) continue;
            if (L.stride[r] == 0) return false;
            uint64_t a = L.stride[r] < 0 ? 0 - static_cast<uint64_t>(L.stride[r]) : static_cast<uint64_t>(L.stride[r]);
            ms.emplace_back(a, L.extent[r]);
        }
        std::sort(ms.begin(), ms.end());
        for (size_t k = 0; k + 1 < ms.size(); ++k) {
            unsigned __int128 need = static_cast<unsigned __int128>(ms[k].first) * static_cast<uint64_t>(ms[k].second);
            if (static_cast<unsigned __int128>(ms[k + 1].first) < need) return false;
        }
        return true;
    }
    if (L.kind == TLB_KIND_XOR) {
        std::vector<uint64_t> cols;
        for (int r = 0; r < L.n_modes; ++r) {
            if (L.extent[r] == 1) continue;
            if (L.log2e[r] == 0xff) return false;
            uint64_t m = static_cast<uint64_t>(L.stride[r]);
            if (m == 0) return false;
            for (int b = 0; b < L.log2e[r]; ++b) {
                if (b + ilog2_floor(m) >= 62) return false;
                cols.push_back(m << b);
            }
        }
        // Gaussian elimination over GF(2).
        std::vector<uint64_t> basis;
        for (uint64_t c : cols) {
            for (uint64_t b : basis) c = std::min(c, c ^ b);
            if (c == 0) return false;
            basis.push_back(c);
            std::sort(basis.rbegin(), basis.rend());
        }
        return true;
    }
    return false;
}

int position_span(const tlb_layout_desc& L, int64_t origin, Span* out) {
    if (L.kind == TLB_KIND_INT) {
        if (L.min_offset == INT64_MIN && L.max_offset == INT64_MAX)
            return fail(TLB_ERR_OVERFLOW, "integer overflow in multiplication");
        if (add_ovf(origin, L.min_offset, &out->lo) || add_ovf(origin, L.max_offset, &out->hi))
            return fail(TLB_ERR_OVERFLOW, "integer overflow in addition");
        return TLB_OK;
    }
    if (L.kind == TLB_KIND_XOR) {
        // origin ^ off where off ranges over the span of the masks: the bits outside the
        // OR-bound never change, the bits inside take (at most) every value.
        uint64_t orb = static_cast<uint64_t>(L.max_offset);
        if (origin < 0) { out->lo = origin; out->hi = origin; return TLB_OK; } // bounds check will reject
        uint64_t o = static_cast<uint64_t>(origin);
        out->lo = static_cast<int64_t>(o & ~orb);
        out->hi = static_cast<int64_t>(o | orb);
        return TLB_OK;
    }
    return fail(TLB_ERR_SEMIMODULE, "integer accessor cannot take a coordinate offset");
}

// Upper bound of |L(i)| over 0 <= i <= max_index (extended domain: the last leaf is unbounded), saturating at 2^63 - 1.
uint64_t max_abs_offset(const tlb_layout_desc& L, uint64_t max_index) {
    unsigned __int128 total = 0;
    uint64_t rest = max_index, orb = 0;
    for (int r = 0; r < L.n_modes; ++r) {
        const uint64_t e = static_cast<uint64_t>(L.extent[r]);
        const uint64_t cmax = (r + 1 < L.n_modes) ? std::min<uint64_t>(rest, e - 1) : rest;
        rest /= e;
        if (L.kind == TLB_KIND_XOR) {
            const uint64_t m = static_cast<uint64_t>(L.stride[r]);
            if (cmax == 0 || m == 0) continue;
            const int top = ilog2_floor(cmax);
            if (top >= 62 || (m << top) >= (1ull << 62)) return INT64_MAX;
            for (int b = 0; b <= top; ++b) orb |= m << b;
        } else {
            const uint64_t a = L.stride[r] < 0 ? 0 - static_cast<uint64_t>(L.stride[r]) : static_cast<uint64_t>(L.stride[r]);
            total += static_cast<unsigned __int128>(cmax) * a;
            if (total >> 63) return INT64_MAX;
        }
    }
    return L.kind == TLB_KIND_XOR ? orb : static_cast<uint64_t>(total);
}

int overflow_preflight(const tlb_layout_desc& L, int64_t origin, uint64_t max_index) {
    // Largest coordinate each leaf sees for i <= max_index; the last leaf is unbounded.
    unsigned __int128 total = origin < 0 ? static_cast<unsigned __int128>(0 - static_cast<uint64_t>(origin))
                                         : static_cast<unsigned __int128>(origin);
    uint64_t rest = max_index;
    for (int r = 0; r < L.n_modes; ++r) {
        uint64_t e = static_cast<uint64_t>(L.extent[r]);
        uint64_t cmax = (r + 1 < L.n_modes) ? std::min<uint64_t>(rest, e - 1) : rest;
        rest /= e;
        if (L.kind == TLB_KIND_XOR) {
            uint64_t m = static_cast<uint64_t>(L.stride[r]);
            if (cmax == 0 || m == 0) continue;
            int top = ilog2_floor(cmax);
            if (top >= 62 || (m << top) >= (1ull << 62)) return fail(TLB_ERR_OVERFLOW, "xor mask overflow");
        } else {
            uint64_t a = L.stride[r] < 0 ? 0 - static_cast<uint64_t>(L.stride[r]) : static_cast<uint64_t>(L.stride[r]);
            total += static_cast<unsigned __int128>(cmax) * a;
            if (total >> 63) return fail(TLB_ERR_OVERFLOW, "integer overflow in layout evaluation");
        }
    }
    return TLB_OK;
}

} // namespace tlb

extern "C" {

int tlb_abi_version(void) { return TLB_ABI_VERSION; }
const char* tlb_last_error(void) { return tlb::g_error.c_str(); }
uint64_t tlb_launch_count(void) { return tlb::g_launches.load(std::memory_order_relaxed); }
const char* tlb_last_plan(void) { return tlb::g_plan; }

int tlb_workspace_trim(uint64_t keep_bytes) {
    if (tlb::require_device() != TLB_OK) return TLB_ERR_CUDA;
    TLB_CUDA(tlb::ws_trim(static_cast<size_t>(keep_bytes)));
    return TLB_OK;
}

int tlb_config_set(const char* name, const char* value) {
    if (!name) return tlb::fail(TLB_ERR_CONTRACT, "tlb_config_set: null name");
    (void)tlb::knob(tlb::K_PDL); // make sure the environment has been read first
    const char* n = std::strncmp(name, "TLB_", 4) == 0 ? name + 4 : name;
    for (int i = 0; i < tlb::K_COUNT; ++i)
        if (std::strcmp(n, tlb::kKnobDefs[i].name) == 0) {
            tlb::g_knobs[i].store(tlb::parse_knob(i, value), std::memory_order_relaxed);
            return TLB_OK;
        }
    return tlb::fail(TLB_ERR_CONTRACT, std::string("tlb_config_set: unknown knob ") + name);
}

int tlb_layout_lower(const tlb_mode* modes, int n_modes, tlb_layout_desc* out) {
    return tlb::lower_impl(modes, n_modes, nullptr, 0, out);
}

int tlb_layout_lower_ranked(const tlb_mode* modes, int n_modes, const int32_t* top_leaves, int n_top,
                            tlb_layout_desc* out) {
    if (!top_leaves) return tlb::fail(TLB_ERR_CONTRACT, "tlb_layout_lower_ranked: null top_leaves");
    return tlb::lower_impl(modes, n_modes, top_leaves, n_top, out);
}

} // extern "C"

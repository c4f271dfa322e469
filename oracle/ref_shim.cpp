// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C shims over the UNMODIFIED reference headers (/root/reference/proj/include/tla),
// compiled where they lie into oracle/_ref/libtla_ref.so by oracle/Makefile.
// Nothing here re-implements an algorithm: every entry point calls the
// reference's own function and only marshals text / raw arrays across a C ABI
// so that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can
// run the real reference (tla::copy tensor.hpp:195, tla::gemm tensor.hpp:214,
// tla::eval_int layout.hpp:74, oracle::oracle_eval_int oracle.hpp:71, and the
// algebra in algebra.hpp) on the same inputs as the CUDA path.
//
// The product library (paper_2603_02298_b200/libtlb.so) never links or loads this.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "tla/tla.hpp"

using namespace tla;

namespace {

// Status codes shared with include/tlb.h (tlb_status).
enum : int {
    ST_OK = 0,
    ST_CONTRACT = 1,
    ST_BOUNDS = 2,
    ST_STRUCTURAL = 3,
    ST_SEMIMODULE = 4,
    ST_OVERFLOW = 5,
    ST_CUDA = 6,
    ST_UNSUPPORTED = 7,
    ST_INDEX = 8,
    ST_STRIDE_DIV = 9,
    ST_SHAPE_DIV = 10,
    ST_NON_DISTRIBUTIVE = 11,
    ST_NOT_COMPLEMENTABLE = 12,
    ST_NOT_LEFT_INVERTIBLE = 13,
    ST_ADMISSIBILITY = 14,
    ST_RESOURCE = 15,
    ST_PARSE = 16,
    ST_OTHER = 17,
};

thread_local std::string g_last_error;

int guarded(const std::function<void()>& fn) {
    g_last_error.clear();
    try {
        fn();
        return ST_OK;
    } catch (const contract_error& e) { g_last_error = e.what(); return ST_CONTRACT;
    } catch (const bounds_error& e) { g_last_error = e.what(); return ST_BOUNDS;
    } catch (const structural_error& e) { g_last_error = e.what(); return ST_STRUCTURAL;
    } catch (const semimodule_error& e) { g_last_error = e.what(); return ST_SEMIMODULE;
    } catch (const overflow_error& e) { g_last_error = e.what(); return ST_OVERFLOW;
    } catch (const index_error& e) { g_last_error = e.what(); return ST_INDEX;
    } catch (const stride_divisibility_error& e) { g_last_error = e.what(); return ST_STRIDE_DIV;
    } catch (const shape_divisibility_error& e) { g_last_error = e.what(); return ST_SHAPE_DIV;
    } catch (const non_distributive_error& e) { g_last_error = e.what(); return ST_NON_DISTRIBUTIVE;
    } catch (const not_complementable_error& e) { g_last_error = e.what(); return ST_NOT_COMPLEMENTABLE;
    } catch (const not_left_invertible_error& e) { g_last_error = e.what(); return ST_NOT_LEFT_INVERTIBLE;
    } catch (const admissibility_error& e) { g_last_error = e.what(); return ST_ADMISSIBILITY;
    } catch (const resource_error& e) { g_last_error = e.what(); return ST_RESOURCE;
    } catch (const parse_error& e) { g_last_error = e.what(); return ST_PARSE;
    } catch (const std::exception& e) { g_last_error = e.what(); return ST_OTHER; }
}

void put(char* out, std::size_t cap, const std::string& s) {
    if (!out || cap == 0) return;
    std::size_t n = std::min(cap - 1, s.size());
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
}

std::shared_ptr<std::vector<Int>> wrap(const Int* p, Int n) {
    return std::make_shared<std::vector<Int>>(p, p + n);
}

SliceCoord parse_slice(const std::string& s, std::size_t& pos) {
    while (pos < s.size() && s[pos] == ' ') ++pos;
    if (pos < s.size() && s[pos] == '(') {
        ++pos;
        std::vector<SliceCoord> kids;
        kids.push_back(parse_slice(s, pos));
        while (pos < s.size() && s[pos] == ' ') ++pos;
        while (pos < s.size() && s[pos] == ',') {
            ++pos;
            kids.push_back(parse_slice(s, pos));
            while (pos < s.size() && s[pos] == ' ') ++pos;
        }
        ++pos;
        return SliceCoord(std::move(kids));
    }
    if (pos < s.size() && s[pos] == '_') {
        ++pos;
        return keep();
    }
    Int v = 0;
    while (pos < s.size() && s[pos] >= '0' && s[pos] <= '9') v = v * 10 + (s[pos++] - '0');
    return fix(v);
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }

// Unary / binary algebra by name; arguments and results are layout text.
// `c` carries the optional integer argument (complement target) or flag text.
int ref_op_str(const char* op, const char* a, const char* b, const char* c, char* out,
               std::size_t cap) {
    std::string o(op ? op : ""), sa(a ? a : ""), sb(b ? b : ""), sc(c ? c : "");
    return guarded([&] {
        std::string r;
        if (o == "parse") r = format_layout(parse_layout(sa));
        else if (o == "coalesce") r = format_layout(coalesce(parse_layout(sa)));
        else if (o == "coalesce_bymode") r = format_layout(coalesce_bymode(parse_layout(sa), parse_int_tuple(sb)));
        else if (o == "flatten") r = format_layout(flatten(parse_layout(sa)));
        else if (o == "size") r = std::to_string(size(parse_layout(sa)));
        else if (o == "cosize") r = std::to_string(cosize(parse_layout(sa)));
        else if (o == "rank") r = std::to_string(rank(parse_layout(sa)));
        else if (o == "depth") r = std::to_string(depth(parse_layout(sa)));
        else if (o == "compose") r = format_layout(compose(parse_layout(sa), parse_layout(sb)));
        else if (o == "compose_bymode") r = format_layout(compose_bymode(parse_layout(sa), parse_tiler(sb)));
        else if (o == "complement") {
            bool relaxed = sc == "relaxed";
            if (sb.empty()) r = format_layout(complement(parse_layout(sa), relaxed));
            else r = format_layout(complement(parse_layout(sa), Int(std::stoll(sb)), relaxed));
        }
        else if (o == "right_inverse") r = format_layout(right_inverse(parse_layout(sa)));
        else if (o == "left_inverse") r = format_layout(left_inverse(parse_layout(sa)));
        else if (o == "logical_divide") r = format_layout(logical_divide(parse_layout(sa), parse_layout(sb)));
        else if (o == "zipped_divide") r = format_layout(zipped_divide(parse_layout(sa), parse_tiler(sb)));
        else if (o == "logical_product") r = format_layout(logical_product(parse_layout(sa), parse_layout(sb)));
        else if (o == "blocked_product") r = format_layout(blocked_product(parse_layout(sa), parse_layout(sb)));
        else if (o == "raked_product") r = format_layout(raked_product(parse_layout(sa), parse_layout(sb)));
        else if (o == "max_common_vector") r = std::to_string(max_common_vector(parse_layout(sa), parse_layout(sb)));
        else if (o == "common_sublayout") r = format_layout(common_sublayout(parse_layout(sa), parse_layout(sb)));
        else if (o == "locate_offsets") r = format_layout(locate_offsets(parse_layout(sa), parse_layout(sb)));
        else if (o == "identity_layout") r = format_layout(identity_layout(parse_int_tuple(sa)));
        else if (o == "coordinate_identity") r = format_layout(coordinate_identity(parse_int_tuple(sa)));
        else if (o == "idx2crd") r = format_int_tuple(idx2crd(Int(std::stoll(sa)), parse_int_tuple(sb)));
        else if (o == "crd2idx") r = std::to_string(crd2idx(parse_int_tuple(sa), parse_int_tuple(sb)));
        else if (o == "eval_coord") {
            StrideElem v = layout_eval(parse_layout(sa), parse_int_tuple(sb));
            r = format_stride_elem(v);
        }
        else if (o == "eval_axes") {
            std::vector<Int> v = layout_eval_axes(parse_layout(sa), parse_int_tuple(sb));
            for (std::size_t i = 0; i < v.size(); ++i) r += (i ? "," : "") + std::to_string(v[i]);
        }
        else if (o == "slice") {
            // a = layout, b = slice coordinate text, c = counting base
            std::size_t pos = 0;
            Tensor t(Accessor::counting(sc.empty() ? 0 : Int(std::stoll(sc))), parse_layout(sa));
            Tensor s = slice(t, parse_slice(sb, pos));
            r = std::to_string(s.accessor().position()) + "|" + format_layout(s.layout());
        }
        else throw contract_error("ref_op_str: unknown op " + o);
        put(out, cap, r);
    });
}

// out[k] = L(i0 + k) for k < n. which: 0 = tla::eval_int (layout.hpp:74),
// 1 = oracle::oracle_eval_int (oracle.hpp:71). Xor layouts return the mask.
int ref_eval_range(const char* layout, std::int64_t i0, std::int64_t n, std::int64_t* out, int which) {
    return guarded([&] {
        Layout l = parse_layout(layout);
        for (Int k = 0; k < n; ++k) {
            StrideElem v = which ? oracle::oracle_eval(l, i0 + k) : layout_eval(l, i0 + k);
            out[k] = v.is_zero() ? 0 : (v.is_xor() ? v.mask() : v.value());
        }
    });
}

// Multi-threaded variant of ref_eval_range for the CPU baseline (pure function).
int ref_eval_range_mt(const char* layout, std::int64_t i0, std::int64_t n, std::int64_t* out, int which,
                      int threads) {
    return guarded([&] {
        Layout l = parse_layout(layout);
        if (threads < 1) threads = 1;
        std::vector<std::thread> pool;
        std::vector<int> status(static_cast<std::size_t>(threads), 0);
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    Int lo = n * t / threads, hi = n * (t + 1) / threads;
                    for (Int k = lo; k < hi; ++k) {
                        StrideElem v = which ? oracle::oracle_eval(l, i0 + k) : layout_eval(l, i0 + k);
                        out[k] = v.is_zero() ? 0 : (v.is_xor() ? v.mask() : v.value());
                    }
                } catch (...) { status[static_cast<std::size_t>(t)] = 1; }
            });
        }
        for (auto& th : pool) th.join();
        for (int s : status) if (s) throw overflow_error("evaluation failed in worker");
    });
}

// Natural coordinates: out[k*nleaves + r] for i0+k (idx2crd int_tuple.hpp:129, flattened).
int ref_idx2crd_range(const char* shape, std::int64_t i0, std::int64_t n, std::int64_t* out) {
    return guarded([&] {
        Shape s = parse_int_tuple(shape);
        std::size_t w = flat_leaves(s).size();
        for (Int k = 0; k < n; ++k) {
            std::vector<Int> c = flat_leaves(idx2crd(i0 + k, s));
            for (std::size_t r = 0; r < w; ++r) out[static_cast<std::size_t>(k) * w + r] = c[r];
        }
    });
}

// tla::copy verbatim (tensor.hpp:195) over Int cells. The caller widens each
// element's bit pattern into one Int cell. Buffers are copied into the
// reference's shared storage and the destination is copied back.
// src_cells == NULL means a counting accessor with base src_origin.
int ref_copy(const char* src_layout, const std::int64_t* src_cells, std::int64_t src_len,
             std::int64_t src_origin, const char* dst_layout, std::int64_t* dst_cells,
             std::int64_t dst_len, std::int64_t dst_origin) {
    std::shared_ptr<std::vector<Int>> ds;
    int st = guarded([&] {
        Layout ls = parse_layout(src_layout);
        Layout ld = parse_layout(dst_layout);
        Accessor sa = src_cells ? Accessor::buffer(wrap(src_cells, src_len), src_origin)
                                : Accessor::counting(src_origin);
        ds = wrap(dst_cells, dst_len);
        Tensor src(sa, ls);
        Tensor dst(Accessor::buffer(ds, dst_origin), ld);
        copy(src, dst);
    });
    // The reference writes partially before a mid-copy bounds_error; reflect that.
    if (ds) std::memcpy(dst_cells, ds->data(), static_cast<std::size_t>(dst_len) * sizeof(Int));
    return st;
}

// tla::copy verbatim where source and destination are views of ONE shared storage (tensor.hpp:29): the serial
// ascending-i order decides what overlapping cells end up holding.
int ref_copy_shared(const char* src_layout, std::int64_t src_origin, const char* dst_layout, std::int64_t dst_origin,
                    std::int64_t* cells, std::int64_t len) {
    std::shared_ptr<std::vector<Int>> st_;
    int st = guarded([&] {
        st_ = wrap(cells, len);
        Tensor src(Accessor::buffer(st_, src_origin), parse_layout(src_layout));
        Tensor dst(Accessor::buffer(st_, dst_origin), parse_layout(dst_layout));
        copy(src, dst);
    });
    if (st_) std::memcpy(cells, st_->data(), static_cast<std::size_t>(len) * sizeof(Int));
    return st;
}

// layout_eval_axes (layout.hpp:103) over a range: out[k*n_axes + a], axes the reference's vector does not reach are 0.
int ref_eval_axes_range(const char* layout, std::int64_t i0, std::int64_t n, int n_axes, std::int64_t* out) {
    return guarded([&] {
        Layout l = parse_layout(layout);
        for (Int k = 0; k < n; ++k) {
            std::vector<Int> v = layout_eval_axes(l, Coord(i0 + k));
            if (static_cast<int>(v.size()) > n_axes) throw contract_error("ref_eval_axes_range: more axes than n_axes");
            for (int a = 0; a < n_axes; ++a)
                out[static_cast<std::size_t>(k) * n_axes + a] = a < static_cast<int>(v.size()) ? v[static_cast<std::size_t>(a)] : 0;
        }
    });
}

// The loop body of tla::copy (dst.store(i, src(i)), tensor.hpp:198) run by
// `threads` std::threads over disjoint i-ranges, operating in place on the
// caller's arrays. Only meaningful for injective destinations. Used as the
// N-core CPU baseline; returns elements copied through *n_out.
int ref_copy_mt(const char* src_layout, const std::int64_t* src_cells, std::int64_t src_len,
                const char* dst_layout, std::int64_t* dst_cells, std::int64_t dst_len,
                std::int64_t i_begin, std::int64_t i_end, int threads) {
    return guarded([&] {
        Layout ls = parse_layout(src_layout);
        Layout ld = parse_layout(dst_layout);
        if (size(ls) != size(ld)) throw contract_error("copy requires equal sizes");
        auto ss = wrap(src_cells, src_len);
        auto ds = wrap(dst_cells, dst_len);
        Tensor src(Accessor::buffer(ss), ls);
        Tensor dst(Accessor::buffer(ds), ld);
        if (threads < 1) threads = 1;
        std::vector<std::thread> pool;
        std::vector<int> status(static_cast<std::size_t>(threads), 0);
        Int n = i_end - i_begin;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    Int lo = i_begin + n * t / threads, hi = i_begin + n * (t + 1) / threads;
                    for (Int i = lo; i < hi; ++i) dst.store(i, src(i));
                } catch (...) { status[static_cast<std::size_t>(t)] = 1; }
            });
        }
        for (auto& th : pool) th.join();
        for (int s : status) if (s) throw bounds_error("copy failed in worker");
        std::memcpy(dst_cells, ds->data(), static_cast<std::size_t>(dst_len) * sizeof(Int));
    });
}

// CPU baseline of the copy configs (bench.py): storage is allocated and filled here, and ONLY the copy is timed.
// threads <= 1: tla::copy verbatim (tensor.hpp:195-199) on one core. threads > 1: the same loop body
// dst.store(i, src(i)) over disjoint i-ranges on std::threads (race free for injective destinations).
// *seconds = wall time of the copy alone, *checksum = sum of the destination cells (defeats dead-code elimination and
// lets the caller check that the two variants agree).
int ref_copy_bench(const char* src_layout, const char* dst_layout, int threads, double* seconds, std::uint64_t* checksum) {
    return guarded([&] {
        Layout ls = parse_layout(src_layout);
        Layout ld = parse_layout(dst_layout);
        auto ss = std::make_shared<std::vector<Int>>(static_cast<std::size_t>(cosize(ls)));
        for (std::size_t i = 0; i < ss->size(); ++i) (*ss)[i] = static_cast<Int>(3 * i + 1);   // acceptance.cpp:289 fill
        auto ds = std::make_shared<std::vector<Int>>(static_cast<std::size_t>(cosize(ld)), Int(-1));
        Tensor src(Accessor::buffer(ss), ls);
        Tensor dst(Accessor::buffer(ds), ld);
        const auto t0 = std::chrono::steady_clock::now();
        if (threads <= 1) {
            copy(src, dst);
        } else {
            if (size(ls) != size(ld)) throw contract_error("copy requires equal sizes");
            const Int n = size(ls);
            std::vector<std::thread> pool;
            std::vector<int> status(static_cast<std::size_t>(threads), 0);
            for (int t = 0; t < threads; ++t) {
                pool.emplace_back([&, t] {
                    try {
                        Int lo = n * t / threads, hi = n * (t + 1) / threads;
                        for (Int i = lo; i < hi; ++i) dst.store(i, src(i));
                    } catch (...) { status[static_cast<std::size_t>(t)] = 1; }
                });
            }
            for (auto& th : pool) th.join();
            for (int s2 : status) if (s2) throw bounds_error("copy failed in worker");
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::uint64_t sum = 0;
        for (Int v : *ds) sum += static_cast<std::uint64_t>(v);
        *checksum = sum;
    });
}

// tla::gemm verbatim (tensor.hpp:214) over Int cells.
int ref_gemm(const char* la, const std::int64_t* a_cells, std::int64_t a_len, const char* lb,
             const std::int64_t* b_cells, std::int64_t b_len, const char* lc, std::int64_t* c_cells,
             std::int64_t c_len) {
    std::shared_ptr<std::vector<Int>> cs;
    int st = guarded([&] {
        Tensor ta(Accessor::buffer(wrap(a_cells, a_len)), parse_layout(la));
        Tensor tb(Accessor::buffer(wrap(b_cells, b_len)), parse_layout(lb));
        cs = wrap(c_cells, c_len);
        Tensor tc(Accessor::buffer(cs), parse_layout(lc));
        gemm(ta, tb, tc);
    });
    if (cs) std::memcpy(c_cells, cs->data(), static_cast<std::size_t>(c_len) * sizeof(Int));
    return st;
}

} // extern "C"

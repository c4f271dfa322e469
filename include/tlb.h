/* tlb.h — C ABI of the B200-native (sm_100a) hot path that sits underneath the
 * `tla` layout algebra of arXiv 2603.02298.
 *
 * The reference (/root/reference/proj/include/tla) has no FFI: everything is
 * inline C++ called directly. The drop-in boundary is therefore the set of C++
 * signatures in namespace tla (kept source-compatible by
 * paper_2603_02298_b200/include/tla/) plus THIS C ABI, the
 * new layer those signatures dispatch to when a tensor lives in device memory.
 * Each entry point names the reference function it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only. Device pointers are BORROWED: never freed,
 *    never retained after the call returns (the reference shares storage by
 *    shared_ptr, tensor.hpp:29; ownership stays with the caller here too).
 *  - Every call returns a tlb_status. The text of the last failure on the
 *    calling thread is available from tlb_last_error(). Status values map
 *    one-to-one onto the reference's exception types (common.hpp:13-97).
 *  - All pre-flight checks (sizes, bounds of the whole offset image, overflow
 *    range proofs) run on the host BEFORE any launch, so a failing call writes
 *    nothing. (The reference writes partially before a mid-copy bounds_error;
 *    documented difference.)
 *  - `stream` is a cudaStream_t passed as void*. Calls are asynchronous with
 *    respect to the host unless stated otherwise. Callable from any host thread:
 *    planner knobs, last error and last plan are per thread; the only shared state
 *    is a launch counter (atomic) and a mutex-guarded cache of encoded TMA tensor
 *    maps keyed by (device, pointer, shape, strides, box).
 *  - Aliasing. tlb_copy: source and destination may overlap in memory (the
 *    reference's views share one storage, tensor.hpp:29); overlap is detected from
 *    the two position spans and resolved to the reference's serial ascending-i
 *    result (plan "aliased" / "serial"). tlb_gemm_*: C must not overlap A or B
 *    (TLB_ERR_UNSUPPORTED); A and B may alias each other.
 *  - There is no CPU fallback. Without a CUDA device every compute entry point
 *    returns TLB_ERR_CUDA.
 */
#ifndef TLB_H_
#define TLB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLB_ABI_VERSION 1
#define TLB_MAX_MODES 16

typedef enum tlb_status {
    TLB_OK = 0,
    TLB_ERR_CONTRACT = 1,    /* tla::contract_error   (tensor.hpp:93,197,216,222) */
    TLB_ERR_BOUNDS = 2,      /* tla::bounds_error     (tensor.hpp:101)            */
    TLB_ERR_STRUCTURAL = 3,  /* tla::structural_error (layout.hpp:57)             */
    TLB_ERR_SEMIMODULE = 4,  /* tla::semimodule_error (tensor.hpp:59)             */
    TLB_ERR_OVERFLOW = 5,    /* tla::overflow_error   (common.hpp:101,107)        */
    TLB_ERR_CUDA = 6,        /* CUDA runtime / driver failure, or no device       */
    TLB_ERR_UNSUPPORTED = 7, /* valid request this build has no kernel for        */
    TLB_ERR_INDEX = 8,       /* tla::index_error                                  */
    TLB_ERR_ADMISSIBILITY = 9 /* tla::admissibility_error (analysis.hpp:45,54)    */
} tlb_status;

/* Stride semimodule of a leaf (stride.hpp:16). */
typedef enum tlb_kind { TLB_KIND_INT = 0, TLB_KIND_BASIS = 1, TLB_KIND_XOR = 2 } tlb_kind;

/* One flat leaf of a layout, as produced by tla::flat_modes (layout.hpp:111):
 * Int: stride; Xor: mask (f<mask>); Basis: scale on `axis` (a*e<axis>). */
typedef struct tlb_mode {
    int64_t extent;
    int64_t stride;
    int32_t kind; /* tlb_kind */
    int32_t axis; /* Basis only */
} tlb_mode;

/* Device-ready layout: the lowering of a host-computed tla::Layout into flat
 * evaluator parameters. POD, passed by value into kernels. Filled by
 * tlb_layout_lower(); treat as opaque apart from the documented fields. */
typedef struct tlb_layout_desc {
    int32_t n_modes;            /* flat leaves, extent-1 leaves kept (they matter for the
                                   extended domain: the LAST leaf is unbounded)          */
    int32_t kind;               /* tlb_kind of the whole layout (stride_kind, stride.hpp:158) */
    int32_t n_top;              /* top-level modes (rank); 1 for a flat request          */
    int32_t flags;              /* TLB_LF_*                                             */
    int64_t size;               /* product of extents (size, int_tuple.hpp:67)          */
    int64_t cosize;             /* 1 + max offset; Int kind, non-negative strides; else -1 (cosize, layout.hpp:277) */
    int64_t min_offset;         /* min over the domain [0,size) (negative strides allowed) */
    int64_t max_offset;         /* max over the domain [0,size); Xor: OR-bound of all masks */
    int32_t top_start[TLB_MAX_MODES + 1]; /* leaf index where top-level mode t starts; [n_top] = n_modes */
    int64_t extent[TLB_MAX_MODES];
    int64_t stride[TLB_MAX_MODES];
    uint64_t magic[TLB_MAX_MODES]; /* fast division by extent for 0 <= i < 2^63, see tlb_lower.cpp */
    uint8_t shift[TLB_MAX_MODES];
    uint8_t log2e[TLB_MAX_MODES];  /* log2(extent) when a power of two, else 0xff          */
} tlb_layout_desc;

#define TLB_LF_ALL_POW2 1  /* every extent is a power of two                     */
#define TLB_LF_HAS_NEG 2   /* some Int stride is negative                        */
#define TLB_LF_INJECTIVE 4 /* proven injective on [0,size) by the sorted-stride test */

/* A tensor = accessor o layout (tensor.hpp:111). */
typedef enum tlb_accessor {
    TLB_ACC_BUFFER = 0,  /* Accessor::buffer   (tensor.hpp:29): data + origin, bounds-checked against capacity */
    TLB_ACC_COUNTING = 1 /* Accessor::counting (tensor.hpp:22): deref returns the position; read-only, 8-byte  */
} tlb_accessor;

typedef struct tlb_tensor {
    const tlb_layout_desc* layout;
    void* data;        /* device pointer to element 0 of the buffer (BORROWED); NULL for counting */
    int64_t origin;    /* accessor position before the layout offset is applied (elements)       */
    int64_t capacity;  /* buffer length in elements (bounds: 0 <= pos < capacity)                */
    int32_t elem_bytes;/* 1, 2, 4, 8 or 16                                                        */
    int32_t accessor;  /* tlb_accessor                                                            */
} tlb_tensor;

/* ---- library ---------------------------------------------------------- */
int tlb_abi_version(void);
const char* tlb_last_error(void);
/* Number of kernels this library has launched on the calling process (for bench.py's gpu_launches). */
uint64_t tlb_launch_count(void);
/* Name of the plan the last tlb_copy / tlb_gemm_* / tlb_eval_range call on this thread selected ("vec", "tiled", "tiled_tma",
 * "gather", "ordered", "aliased", "umma_2sm_wide", "eval_warp32", ...). */
const char* tlb_last_plan(void);

/* Tuning / debugging knobs (GEMM_WIDE, GEMM_SPLIT_TAIL, GEMM_CHUNK_WAVES, GEMM_MCAST, GEMM_EARLY_RELEASE, GEMM_PACK,
 * GEMM_PACK_MIN, COPY_TMA, COPY_TMA_STAGES, COPY_TMA_CTAS, PDL, HOST_PANEL, ...: the table is in csrc/tlb_lower.cpp).
 * The environment variables TLB_<NAME> are read once, at the first call into the library;
 * afterwards a knob changes only through this call (value NULL or "" restores the default). `name` is the variable
 * name with or without the TLB_ prefix, e.g. tlb_config_set("GEMM_WIDE", "1"). Unknown names: TLB_ERR_CONTRACT.
 * Launch paths read knobs with one atomic load (no getenv). */
int tlb_config_set(const char* name, const char* value);

/* Workspaces (winner arrays of the "ordered" copy plan, packed GEMM panels, status words) come from a stream-ordered
 * memory pool the library owns per device; freed blocks stay in the pool so that a call repeated in a loop does not go
 * back to the driver. This releases the pool's unused memory down to keep_bytes (cudaMemPoolTrimTo) on the current device. */
int tlb_workspace_trim(uint64_t keep_bytes);

/* ---- (1) lowering: host layout -> device evaluator parameters --------- */
/* Replaces the per-element call chain Tensor::operator() -> layout_eval -> eval_rec ->
 * idx2crd/eval_leaf (tensor.hpp:119, layout.hpp:49-74) with a one-time flattening
 * (flat_modes, layout.hpp:111; oracle::detail::collect, oracle.hpp:22). */
int tlb_layout_lower(const tlb_mode* modes, int n_modes, tlb_layout_desc* out);
/* Same, keeping the top-level mode boundaries: top_leaves[t] = number of flat leaves in
 * top-level mode t (sum = n_modes). Needed by gemm (rank-2, modes addressed by 1-D coordinates). */
int tlb_layout_lower_ranked(const tlb_mode* modes, int n_modes, const int32_t* top_leaves, int n_top,
                            tlb_layout_desc* out);

/* ---- (2) bulk layout evaluation (config C5) --------------------------- */
/* d_out[k] = L(i0 + k), k < n: tla::eval_int (layout.hpp:74) / oracle::oracle_eval_int
 * (oracle.hpp:71) over a range, extended domain allowed (last leaf unbounded). int64 out.
 * Xor layouts write the mask value. Basis layouts -> TLB_ERR_SEMIMODULE (use tlb_eval_axes_range). */
int tlb_eval_range(const tlb_layout_desc* layout, uint64_t i0, uint64_t n, int64_t* d_out, void* stream);
/* d_out[k*n_modes + r] = r-th natural-coordinate leaf of i0 + k: tla::idx2crd (int_tuple.hpp:129). */
int tlb_idx2crd_range(const tlb_layout_desc* shape, uint64_t i0, uint64_t n, int64_t* d_out, void* stream);
/* d_out[k] = crd2idx(d_crd[k*n_modes ..], shape): tla::crd2idx (int_tuple.hpp:148) on natural coordinates. */
int tlb_crd2idx_range(const tlb_layout_desc* shape, const int64_t* d_crd, uint64_t n, int64_t* d_out, void* stream);
/* Same with the reference's checked arithmetic made visible: like tla::crd2idx, any coordinate VALUES are accepted (the
 * reference validates only the tree shape, which the flat [n][n_modes] input fixes) and a checked_mul / checked_add
 * wrap (int_tuple.hpp:154) sets *d_status = TLB_ERR_OVERFLOW (int32 on device, caller zeroes) and leaves d_out[k]
 * unwritten. tlb_crd2idx_range is this call with d_status = NULL (wrapped elements are skipped silently). */
int tlb_crd2idx_range_checked(const tlb_layout_desc* shape, const int64_t* d_crd, uint64_t n, int64_t* d_out,
                              int32_t* d_status, void* stream);
/* Counts k in [k0, k0+n) with L(R(k)) != k into *d_mismatch (uint64, device, accumulated with atomicAdd;
 * caller zeroes it): the defining property of tla::right_inverse (algebra.hpp:474) checked in bulk. */
int tlb_rinv_check_range(const tlb_layout_desc* L, const tlb_layout_desc* R, uint64_t k0, uint64_t n,
                         unsigned long long* d_mismatch, void* stream);
/* Counts i in [i0, i0+n) with A(B(i)) != R(i): the pointwise definition of tla::compose that
 * detail::verify_distributed (algebra.hpp:211) re-checks on the host in O(size(B)). */
int tlb_compose_check_range(const tlb_layout_desc* A, const tlb_layout_desc* B, const tlb_layout_desc* R,
                            uint64_t i0, uint64_t n, unsigned long long* d_mismatch, void* stream);
/* The whole check in one synchronous call: *mismatches = #{ i < size(B) : A(B(i)) != R(i) }. This is what lets
 * tla::compose skip its O(size(B)) host loop (detail::verify_distributed, algebra.hpp:211-228: about 18 s for the
 * 8192 x 8192 transpose map of config C1): include/tla/device.hpp's compose_device() runs the reference's own
 * per-leaf composition and verifies the result here in milliseconds. */
int tlb_compose_check(const tlb_layout_desc* A, const tlb_layout_desc* B, const tlb_layout_desc* R, uint64_t* mismatches,
                      void* stream);
/* Per-axis evaluation of a Basis (coordinate) layout: d_out[k*n_axes + a] (layout_eval_axes, layout.hpp:103). */
int tlb_eval_axes_range(const tlb_mode* modes, int n_modes, int n_axes, uint64_t i0, uint64_t n,
                        int64_t* d_out, void* stream);

/* ---- (3) layout-driven copy (configs C1, C3) -------------------------- */
/* tla::copy(src, dst) (tensor.hpp:195-199): for i in [i_begin, i_end) ascending,
 * dst(i) = src(i). Pass i_begin = 0, i_end = UINT64_MAX for the whole domain. Last-writer-wins
 * order is preserved for non-injective destinations. Sizes must agree (contract_error).
 * The planner works on the common refinement of the two layouts and picks (tlb_last_plan()):
 *   "vec"           one refined mode contiguous on both sides: <= 16-byte vectors
 *   "tiled"         transposes / permutes: 128-byte swizzle-staged tiles (Swizzle<3,4,3>), 128-bit accesses both ways;
 *                   "tiled_u" with cell-sized accesses for unaligned bases / leading dimensions, "tiled_s" along the
 *                   smallest-stride modes of layouts WITHOUT a unit stride, "tiled_tma" the TMA-fed persistent variant
 *   "interleave"    AoS <-> SoA (a short mode of 2 .. 26, 28, 30 or 32 cells for 2- / 4-byte cells, the common extents for 1- / 8-byte cells, against a long one): register permutation, whole
 *                   sectors on both sides, no shared memory
 *   "tiled_n"       a whole short mode as one of the runs (a 4M x 24 transpose, 9-field AoS): cell-granular staged tiles with
 *                   run-time extents
 *   "ragged:P"      run extents that are not whole tiles, from 2^22 elements: a whole-tile body on staged plan P plus edge
 *                   strips (disjoint boxes of an injective destination, each an independent copy)
 *   "gather_vec"    anything else whose low run (max_common_vector, also for Xor layouts) is >= 2 cells: one evaluation
 *                   of both layouts per <= 16-byte vector;  "gather_run": per 32 / 64-byte run both layouts keep, 256-bit
 *                   accesses;  "gather": one cell per thread
 *   "last_writer+P" non-injective destination whose aliasing is only stride-0 (broadcast) modes: the injective copy
 *                   (plan P) of the slice at their last coordinates;  "ordered": overlapping strides, winner election
 *   "aliased" / "serial"  source and destination overlap in memory (see Aliasing above). */
int tlb_copy(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end, void* stream);
/* Runs the contract checks and the planner of tlb_copy without a device and without launching anything;
 * the plan it would pick is then available from tlb_last_plan(). Pointers are only inspected for
 * alignment. (Xor-kind bounds that need the exact device scan are assumed to pass.) */
int tlb_copy_plan(const tlb_tensor* src, const tlb_tensor* dst, uint64_t i_begin, uint64_t i_end);
/* tla::max_common_vector(a, b) (analysis.hpp:18-28): the number of leading offsets 0 .. K-1 both layouts reach from the
 * same integral coordinates, i.e. how many elements can move as one vector. Host only. Computed from the common
 * refinement the copy planner works on (it is what bounds the "vec" plan's vector width); layouts the reference cannot
 * right-invert give the scalar answer 1, as there. */
int tlb_max_common_vector(const tlb_layout_desc* a, const tlb_layout_desc* b, int64_t* k);
/* Thread-value partitioned copy: the caller chooses WHICH thread moves WHICH elements with a layout, the way the paper
 * partitions work (local_partition; the thread-value maps of proj/demo/partition_demo.cpp:26-40, built
 * with blocked_product / raked_product, algebra.hpp:629-635). `tv` is a rank-2 layout (thread, value) -> integral
 * coordinate of src and dst (from tlb_layout_lower_ranked): logical thread t copies dst(tv(t, v)) = src(tv(t, v)) for every
 * value v; coordinates at or beyond size(src) are skipped, so a TV layout may over-cover a ragged tensor. tv and dst must
 * be injective (one writer per cell), strides non-negative integers. Runs of the value mode that tv, src and dst all keep
 * contiguous and aligned move as <= 16-byte vectors. Plans "tv_vec" / "tv".
 * Partitioning is composition: when tv is a bijection onto [0, size) whose leaves are digits of the integral coordinate
 * (sorted by stride they nest; what blocked_product / raked_product of compact layouts give) and every digit falls inside
 * one leaf of src and of dst, the partitioned tensors src o tv and dst o tv are layouts (compose, algebra.hpp:235; the
 * nesting test replaces its O(|B|) verify_distributed loop) and the call IS tlb_copy between them, walked in tv's order:
 * plans "tv:vec", "tv:tiled", ... at the planner's speed (C1 through the derived TV layout: 0.87 -> 6.0 TB/s). Other TV
 * layouts keep the per-thread kernel; knob COPY_TV_COMPOSE=0 forces it. */
int tlb_copy_tv(const tlb_tensor* src, const tlb_tensor* dst, const tlb_layout_desc* tv, void* stream);
/* The thread-value layout the library derives for (src, dst) itself: V = the widest power-of-two vector that
 * tla::max_common_vector(src, dst) (analysis.hpp:18-28) and 16 bytes allow, one tile = raked_product((V):(1), (T):(1)) =
 * (T, V):(V, 1) (algebra.hpp:633), tiles repeated in the value mode: ((T), (V, R)):((V), (1, T V)). Writes 3 flat modes and
 * top_leaves2 = {1, 2} for tlb_layout_lower_ranked. Host only. */
int tlb_copy_tv_auto(const tlb_layout_desc* src, const tlb_layout_desc* dst, int elem_bytes, int threads, tlb_mode* tv_modes,
                     int32_t* n_modes, int32_t* top_leaves2);
/* Planner knobs for tlb_copy on the calling thread: force one path (testing / profiling).
 * 0 = auto, 1 = gather only, 2 = tiled (LDG-fed), 3 = tiled TMA-fed. Returns the previous value. */
int tlb_copy_set_path(int path);

/* ---- (4) TMA tensor maps derived from divided layouts ------------------ */
/* Builds the CUtensorMap (128 opaque bytes, 64-byte aligned) for loading one tile of
 * zipped_divide(parent, tiler) (algebra.hpp:595): `parent` is the full Int-kind layout,
 * `tile` the tile mode of the divide (its flat leaves select boxDim / elementStrides),
 * both from tlb_layout_lower. swizzle: 0 none, 1 32B, 2 64B, 3 128B (= Swizzle<3,4,3> on byte
 * offsets = the reference layout (128,8):(f1,f144) per 1 KiB, stride.hpp:142). */
int tlb_tensormap_from_divided(const tlb_layout_desc* parent, const tlb_layout_desc* tile, int elem_bytes,
                               int swizzle, void* d_base, void* out_tensormap_128B);

/* The TMA dimensions the builder derives (host only): rank, and per dimension its extent, stride (elements) and
 * box extent, innermost first. Arrays have 5 entries. A tile's TMA coordinate in dimension d is the element
 * index where the tile starts in that dimension. */
int tlb_tensormap_describe(const tlb_layout_desc* parent, const tlb_layout_desc* tile, int32_t* rank, uint64_t* dims5,
                           uint64_t* strides5, uint32_t* box5);
/* Validation aid: fetches ONE box at `coords` through the tensor map into shared memory and writes its
 * box_bytes bytes to d_out de-swizzled (dimension 0 fastest). swizzle must be the mode the map was built with. */
int tlb_tensormap_fetch_tile(const void* tensormap_128B, int rank, const int32_t* coords, uint32_t box_bytes, int swizzle,
                             void* d_out, void* stream);

/* ---- (5) tiled GEMM (configs C2, C4) ----------------------------------- */
/* tla::gemm(A, B, C) (tensor.hpp:214-233): C(m,n) += sum_k A(m,k) * B(n,k), all rank 2.
 * bf16 x bf16 -> fp32, accumulator starts from C. tile_begin/tile_end select a range of the
 * 128 x 256 output tiles (ids from tlb_gemm_tile_count; pairs (2g, 2g+1) form 256 x 256 blocks and, when
 * ceil(rows / 256) is even, quadruples (4g .. 4g+3) form 512 x 256 pair tiles, walked in an L2-friendly order;
 * pass 0 and UINT32_MAX for all) so 1/2/4/8 GPUs can shard one problem by tile-coordinate ranges. Ranges
 * aligned to 4 tiles keep the wide (512 x 256) tcgen05 plan, ranges aligned to 2 the 256 x 256 plan. The ids
 * refer to the tiling of the plan the library selects, which runs the problem transposed when C is
 * m-contiguous; every range partition of [0, count) covers C exactly once.
 * Every operand family of PAPER.md:1766-1771 runs on tcgen05 (TMA -> swizzled smem -> UMMA -> TMEM -> TMA reduce-add):
 * K-major "T" and MN-major "N" operands (TN, NT, NTT rows) with an M- or N-contiguous C directly; hierarchical modes
 * (GETT-folded operands and C, CONV as a GEMM over the im2col LAYOUT of the input) through rank-4/5 tensor maps derived
 * from the divided layouts; layouts no tensor map can address (BLIS strides on every mode, Xor strides, rows that are not
 * multiples of 16 bytes) through the PACKED plan: tlb_copy packs A, B and C into TMA-addressable panels on a stream-ordered
 * workspace, the tcgen05 plan runs on them, tlb_copy scatters C back ("packed+<plan>"; whole single problems of at least
 * 2^GEMM_PACK_MIN MACs). Small problems of that kind, tile ranges of them and the int64 value type run on the
 * layout-evaluating SIMT kernel.
 * Long tile ranges are cut into several launches of about GEMM_CHUNK_WAVES waves (tlb_launch_count counts them): the
 * workers of one persistent launch drift apart and stop sharing operand panels in L2.
 * Partial tiles of the last wave are summed by several CTA pairs through L2 reductions, so fp32 sums are not
 * bitwise reproducible from run to run unless TLB_GEMM_SPLIT_TAIL=0 is set in the environment.
 * A.elem_bytes = B.elem_bytes = 2; C.elem_bytes = 4 (fp32 C) or 2 (C in the operands' type: fp32 accumulation, one
 * rounding to bf16 / fp16, added to C in that type; tcgen05 wide plan or SIMT). */
int tlb_gemm_bf16(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, uint32_t tile_begin,
                  uint32_t tile_end, void* stream);
/* The same GEMM partitioned by a caller-chosen tiler (local_tile(C, [bm, bn], (i, j)) is the tile of C a CTA
 * or CTA pair owns, local_tile(A, [bm, bk], (i, k)) / local_tile(B, [bn, bk], (j, k)) its k-blocks). Every tensor map of the
 * call is the tile mode of the corresponding zipped_divide (tlb_tensormap_from_divided's derivation), and the TiledMMA is
 * the tcgen05.mma atom 128 x N x 16 (one CTA) or 256 x N x 16 (cta_group::2) with N = 128 or 256. Supported tilers, as rows
 * x columns of C the way the plan runs it (an m-contiguous C runs transposed, so bm and bn swap roles):
 * [128, 128|256, 64], [256, 128|256, 64] and [512, 256, 64]. Anything else, and layouts only the SIMT plan serves:
 * TLB_ERR_UNSUPPORTED. Whole problems only; tlb_last_plan() names the kernel ("umma_1sm_n128", "umma_2sm", ...). */
typedef struct tlb_gemm_tiler {
    int32_t bm, bn, bk;
} tlb_gemm_tiler;
int tlb_gemm_bf16_tiled(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, const tlb_gemm_tiler* tiler,
                        void* stream);
/* tla::locate_offsets(A, T) (analysis.hpp:40-56): R = left_inverse(A) o T maps instruction coordinates to logical
 * coordinates of the data layout A; admissible iff A(R(i)) == T(i) for every i < size(T). The host computes R for
 * instruction leaves that each land inside one coalesced leaf of A (strided tiles: what TMEM accumulators are), the
 * O(size(T)) admissibility loop runs on the device. Writes one flat mode of R per leaf of T into r_modes (room for
 * TLB_MAX_MODES) and their count into *n_modes. TLB_ERR_ADMISSIBILITY when some offset of T is not in the image of A.
 * Synchronous. The GEMM kernels' tcgen05.ld partition of their accumulators is derived through this call's host half. */
int tlb_locate_offsets(const tlb_layout_desc* A, const tlb_layout_desc* T, tlb_mode* r_modes, int32_t* n_modes, void* stream);
/* Hits / misses of the tensor-map cache since the library was loaded (diagnostics; either pointer may be NULL). */
int tlb_tensormap_cache_stats(uint64_t* hits, uint64_t* misses);

/* Number of output tiles of one problem under the plan tlb_gemm_bf16 would choose (host-only, no device
 * needed): shard [0, *tiles) across GPUs and pass each range as tile_begin / tile_end. */
int tlb_gemm_tile_count(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, uint32_t* tiles);
/* Batched: `batch` problems, operand b at data + b * batch_stride (elements); batches
 * [batch_begin, batch_end) are executed (tile-range sharding at batch granularity, config C4). */
int tlb_gemm_bf16_batched(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int64_t a_batch_stride,
                          int64_t b_batch_stride, int64_t c_batch_stride, int32_t batch_begin,
                          int32_t batch_end, void* stream);
/* Same contracts with IEEE fp16 operands (fp16 x fp16 products are exact in fp32 as well; tcgen05 kind::f16 takes
 * either format through the instruction descriptor). */
int tlb_gemm_f16(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, uint32_t tile_begin, uint32_t tile_end,
                 void* stream);
int tlb_gemm_f16_batched(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int64_t a_batch_stride,
                         int64_t b_batch_stride, int64_t c_batch_stride, int32_t batch_begin, int32_t batch_end,
                         void* stream);
/* The reference's own value type: int64 cells, wrapping detected as overflow_error
 * (checked_add/checked_mul, common.hpp:99-109). With d_status (int32 on device, caller zeroes) the call is
 * asynchronous and a wrap sets *d_status = TLB_ERR_OVERFLOW (the wrapped cell keeps its old value). With
 * d_status == NULL the call owns the status word, waits for the kernel and RETURNS TLB_ERR_OVERFLOW, so a wrap can
 * never pass silently (this is what tla::gemm in include/tla/device.hpp uses). All elem_bytes = 8. Any layouts. */
int tlb_gemm_i64(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C, int32_t* d_status, void* stream);
/* Planner knob for tlb_gemm_bf16: 0 auto, 1 SIMT only, 2 tcgen05 cta_group::1, 3 tcgen05 cta_group::2. */
int tlb_gemm_set_path(int path);
/* Diagnostics: SM clock the tcgen05 GEMM kernels actually ran at (cycles of CTA 0 / globaltimer), recorded per launch
 * when TLB_GEMM_CLOCK=1 is in the environment at the first GEMM launch. Synchronises the device, returns the medians
 * over the recorded launches (ring of 4096) and clears the record. *launches = 0 when recording is off. */
int tlb_gemm_clock_stats(double* median_mhz, double* median_us, uint32_t* launches);

/* ---- host-buffer convenience (the reference-facing call, used for e2e) -- */
/* Same contracts with HOST pointers in the tlb_tensor.data fields: stages through device memory
 * the library keeps per calling thread (grown on demand, with a private stream pair), copies in, runs, copies
 * the destination back, synchronises. */
int tlb_copy_host(const tlb_tensor* src, const tlb_tensor* dst);
/* tla::eval_int (layout.hpp:74) over [i0, i0 + n) into a HOST array: evaluated on the device in pieces whose download
 * overlaps the next piece's evaluation. Synchronous. */
int tlb_eval_range_host(const tlb_layout_desc* layout, uint64_t i0, uint64_t n, int64_t* h_out);
int tlb_gemm_bf16_host(const tlb_tensor* A, const tlb_tensor* B, const tlb_tensor* C);

#ifdef __cplusplus
}
#endif
#endif /* TLB_H_ */

// common.cuh -- device helpers and the internal kernel interface of librig.
// sm_100a only.  Compiled with --fmad=false: every fused multiply-add in the
// library is an explicit __fma_rn, so no accidental contraction changes a bit
// of the ordering contract (DESIGN.md §3 R4) or of the compensated cutsize.
#pragma once
#include <cuda_runtime.h>
#include <cstdio>

#include <climits>
#include <cstdint>

namespace rig {

// Bounds checks of the debug build (-DRIG_DEBUG_CHECKS, tools/build_variant.sh):
// compute-sanitizer is closed on this GPU pool, so the kernels check their own
// shared and global indices there and trap on a violation.
#ifdef RIG_DEBUG_CHECKS
#define RIG_CHECK(c)                                                                                  \
    do {                                                                                              \
        if (!(c)) {                                                                                   \
            printf("RIG_CHECK failed: %s at %s:%d (block %d thread %d)\n", #c, __FILE__, __LINE__,    \
                   (int)blockIdx.x, (int)threadIdx.x);                                                \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define RIG_CHECK(c) \
    do {             \
    } while (0)
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarp = 32;

// Device error bits, read back at the first synchronisation.
enum : int {
    kErrZeroRow = 1,
    kErrNonFinite = 2,
    kErrNonCanonical = 4,
};

// Rows whose A-row length is <= kMergeMaxLen and whose product count is
// <= kMergeMaxF take the thread-per-row k-way merge path (k_spgemm.cu).
constexpr int kMergeMaxLen = 8;
constexpr int64_t kMergeMaxF = 4096;
// Rows off the merge path are binned by ceil(log2(2 f_i)) in [6, 12]
// (bins 0..6: the mid-row kernels); beyond that the huge bin kNumSymBins.
constexpr int kSymBinMinLog = 6, kSymBinMaxLog = 12;
constexpr int kNumSymBins = kSymBinMaxLog - kSymBinMinLog + 1;  // 7

struct Csr {
    int64_t nrows, ncols, nnz;
    const int64_t *rp;
    const int32_t *ci;
    const double *v;  // scaled values a_hat when scale_rows
};

// CSC of A_hat with one sentinel per column: column k occupies
// [cp[k] + k, cp[k+1] + k) (rows ascending) and ri[cp[k+1] + k] = INT_MAX.
struct Csc {
    const int64_t *cp;  // [ncols+1] entry counts prefix (without sentinels)
    const int32_t *ri;  // [nnz + ncols], ri[-1] and vt[-1] readable (see plan_build)
    const double *vt;   // [nnz + ncols] bit-identical to the CSR value of (i,k)
};
__device__ __forceinline__ int64_t csc_begin(const Csc &T, int k) { return T.cp[k] + k; }
// CSC positions (entries + one sentinel per column + the leading pad) fit int32
inline bool csc_fits_i32(const Csr &A) { return A.nnz + A.ncols + 2 <= (int64_t)INT32_MAX; }

// Counters written by the device and read back by the host at a sync.
constexpr int kSymBins = kNumSymBins + 1;  // + huge
struct DevCounters {
    int err;
    int holes;          // numeric pass dropped an entry (|c| <= tol or exact 0)
    int pad0;
    int max_len;        // longest A row (in the shard) on the merge path
    int64_t products;   // sum f_i over the shard
    int64_t n_mid;      // rows not on the merge path
    int64_t nnz_rows;      // sum of A-row lengths over the shard
    int64_t max_f;         // largest f_i off the merge path
    int64_t mid_slots;     // sum (f_i - len_i) off the merge path: temporary entries
    int64_t sym_count[8];
    int64_t list_count[2]; // mid / huge list lengths (device side)
    int64_t defer_count[4];// rows deferred by the mid, big-far-list, wide-window and global-far-list passes
    // shape statistics (scan_u32_shape, on the column counts and row pointers)
    int64_t max_col;       // longest column of A
    int64_t p_full;        // sum over columns of len^2 = products of the full matrix (>= the shard's)
    int64_t max_row;       // longest row of A in the shard
    int64_t shard_nnz;     // entries of A in the shard's rows
    int64_t min_row_c;     // kMinRowBias - (shortest A row in the shard); 0: no row
};
constexpr int64_t kMinRowBias = int64_t(1) << 40;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Device-side guard of the general transpose (see launch_sym_transpose): a
// kernel given `guard` runs only if *guard != 0 (the pattern-symmetric fast
// path failed); guard == nullptr: always runs.
__device__ __forceinline__ bool guard_skip(const int *guard) {
    return guard != nullptr && *reinterpret_cast<const volatile int *>(guard) == 0;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ double shfl_d(double v, int src) {
    return __shfl_sync(kFull, v, src);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Inclusive warp scan.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int l = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(kFull, v, o);
        if (l >= o) v += u;
    }
    return v;
}

// Launch bookkeeping (rig_launch_count).
void note_launch(int n = 1);
int num_sms();

// ---------------------------------------------------------------- kernels
// k_prep.cu
void launch_validate(const Csr &A, int *err, cudaStream_t s);
void launch_part_check(const int32_t *part, int64_t n, int32_t K, int *bad, cudaStream_t s);
void launch_col_hist(const Csr &A, unsigned *cnt, unsigned *rank /*nullable*/, cudaStream_t s,
                     const int *guard = nullptr);
// k_transpose.cu: bucketed a1 + a2 (see there for the CSC layout with sentinels)
int64_t transpose_buckets(int64_t nnz, int64_t ncols);
constexpr size_t kTransposeRecBytes = 16;
// bcur: u64[transpose_buckets] (initialised here); gcur: u32[ncols] zeroed; big: int[1 + transpose_buckets]
// with big[0] zeroed (list of buckets too large for the warp sort).
void launch_transpose(const Csr &A, int scale, const int64_t *cp, double *ahat, unsigned long long *bcur,
                      void *rec, unsigned *gcur, int *big, int32_t *ri, double *vt, int *err, cudaStream_t s,
                      const int *guard = nullptr);
// Pattern-symmetric fast path of a1 + a2 (square A): when every entry (i,k)
// has its mirror (k,i), column k's rows are row k's columns, so col_ptr =
// row_ptr and the CSC is a gather (each value a_jk found in row j) -- no
// histogram, no buckets, no sort.  Row norms first (nrm, y = RN(1/nrm)); an
// entry without its mirror sets *fail and the guarded general path (given
// `fail` as its guard) rebuilds everything.  With `shape`, the shape
// statistics (DevCounters) are taken from the row pointers instead of the
// column counts, by a kernel that runs only if the gather succeeded.
void launch_sym_transpose(const Csr &A, int scale, double *nrm, double *y, double *ahat, int64_t *cp, int32_t *ri,
                          double *vt, int *fail, int *err, DevCounters *shape, int64_t rb, int64_t re, cudaStream_t s);
void launch_analyze(const Csr &A, const int64_t *cp, int64_t rb, int64_t re, int64_t *f, DevCounters *ctr,
                    cudaStream_t s);
// Ordered row lists (k_prep.cu): list 0 = mid rows (bin8 < kNumSymBins),
// list 1 = huge rows; lists[b * cap ...] in ascending row order; counts[b]
// written when non-null.  cnt: u32[bins_count_elems(nloc)], off: int64[that + 1],
// scan_tmp: scan_tmp_bytes(that).
constexpr uint8_t kBinNone = 0xff;  // bin8 of a merge-path row
size_t bins_count_elems(int64_t nloc);
void launch_bins(const uint8_t *bin8, int64_t rb, int64_t nloc, unsigned *cnt, int64_t *off, void *scan_tmp,
                 int32_t *lists, int64_t cap, int64_t *counts, cudaStream_t s);

// k_sparsify.cu (f1): dense-column cutoffs on the CSC of A_hat (columns with
// cnt > T; list: int[ncols], count zeroed), the A~ row filter (pass 0: nk[i]
// kept per row; pass 1: write at rp2), and exact integer weights.
void launch_sparsify_cutoffs(const unsigned *cnt, int64_t m, int64_t T, const Csc &Tc, int32_t *list, int *count,
                             unsigned long long *ckey, int32_t *crow, cudaStream_t s);
void launch_sparsify_filter(int pass, const Csr &A, const unsigned *cnt, int64_t T, const unsigned long long *ckey,
                            const int32_t *crow, int64_t *nk, const int64_t *rp2, int32_t *ci2, double *v2,
                            cudaStream_t s);
void launch_int_weights(const double *w, int64_t n, int64_t alpha, int64_t *wgt, cudaStream_t s);

// k_scan.cu: out[0..n] = exclusive prefix of in[0..n-1] (out[n] = total).
enum class ScanOp { Identity, UbOffDiag };
void scan_i64(const int64_t *in, int64_t n, int64_t *out, ScanOp op, void *tmp, size_t tmp_bytes,
              cudaStream_t s);
void scan_u32(const unsigned *in, int64_t n, int64_t *out, void *tmp, size_t tmp_bytes, cudaStream_t s,
              const int *guard = nullptr);
// scan_u32 of the column counts that also takes the shape statistics
// (DevCounters max_col, p_full, max_row, shard_nnz of rows [rb, re)) into
// ctr, copies ctr to host_copy and records `ready` before the second kernel.
void scan_u32_shape(const unsigned *in, int64_t n, int64_t *out, void *tmp, DevCounters *ctr, const int64_t *rp,
                    int64_t rb, int64_t re, void *host_copy, cudaEvent_t ready, cudaStream_t s,
                    const int *guard = nullptr);
size_t scan_tmp_bytes(int64_t n);

// k_spgemm.cu
struct SymArgs {
    Csr A;
    Csc T;
    int64_t rb, re;
    int64_t *nnzc;  // [re-rb] merge rows: structural nnz(C_i) incl. the diagonal
    int64_t *fnm;   // [re-rb] rows off the merge path: f_i - len_i (temporary slots), else 0
    int2 *qs;       // [nnz] or null: per A entry of a merge row its CSC run (start csc_begin(k),
                    // length nnz(col k)); x = -1 at the first entry of a row of <= kMergeMaxLen
                    // entries off the merge path
};
struct NumArgs {
    Csr A;
    Csc T;
    int64_t rb, re;
    const int64_t *gptr;  // [re-rb+1] upper-bound (structural) offsets
    int32_t *gcol;
    double *gw;
    double *diag;  // may be null
    double tol;
    int *holes;
    // fused a7 (optional, part == nullptr: off): every kept edge (i,j) with
    // j > i and part[i] != part[j] is added to a per-thread sum (CutSum in the
    // merge kernels, Neumaier in the others); each CTA writes its sum to
    // cutp[blockIdx.x] (deterministic order).
    const int32_t *part;
    int32_t K;
    double *cutp;
    int *bad_part;
    int *cut_used;  // this launch's number of written partials (= gridDim.x)
    int stage_cap;  // merge path: staged graph entries per warp (set by the launcher)
    const int2 *qs;  // SymArgs::qs (null: run starts gathered from the col_ptr)
};

// Neumaier-compensated running sum (compiled with --fmad=false).
struct Comp {
    double s = 0.0, c = 0.0;
    __device__ __forceinline__ void add(double x) {
        const double t = s + x;
        if (fabs(s) >= fabs(x))
            c += (s - t) + x;
        else
            c += (x - t) + s;
        s = t;
    }
    __device__ __forceinline__ double value() const { return s + c; }
};

// Per-lane cut sum inside the fused numeric kernels.  The terms are positive
// weights |c_ij| (no cancellation), a few to a few hundred per lane: plain
// summation has relative error <= (terms) * eps, far inside the 1e-12
// cutsize tolerance; the per-lane / per-row sums are then combined in fixed
// trees and Neumaier-compensated segments (deterministic).
struct CutSum {
    double s = 0.0;
    __device__ __forceinline__ void add(double x) { s += x; }
    __device__ __forceinline__ double value() const { return s; }
};

// Sum of one double per thread over the CTA in a fixed tree order; thread 0
// gets the result.  All threads must call it.
template <int NT>
__device__ __forceinline__ double block_tree_sum(double v) {
    __shared__ double red[NT];
    red[threadIdx.x] = v;
    __syncthreads();
#pragma unroll
    for (int h = NT / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// Merge-path output staging (entries per warp), see stage_cap_for().
constexpr int kMinStageCap = 256, kMaxStageCap = 1536;
// Staging capacity from the mean products per row (P / rows): a 32-row tile
// writes about 32 * nnz(C_i) <= 32 * f_i entries; stencil-like rows have
// f_i ~ 2 nnz(C_i), so 0.6 * 32 * P/rows leaves headroom.  Tiles that do not
// fit fall back to direct global stores (correct, slower).
inline int stage_cap_for(int64_t products, int64_t rows) {
    const double mean = rows > 0 ? (double)products / (double)rows : 0.0;
    int64_t cap = (int64_t)(0.6 * 32.0 * mean) + 32;
    cap = (cap + 31) / 32 * 32;
    if (cap < kMinStageCap) cap = kMinStageCap;
    if (cap > kMaxStageCap) cap = kMaxStageCap;
    return (int)cap;
}

// Pair kernel output stage: 16-row tiles, same estimate as stage_cap_for().
#ifndef RIG_PAIR_STAGE_F
#define RIG_PAIR_STAGE_F 0.6  // measured 0.45-0.75: 0.45 is 1.6 % faster on config 3 (more L1 for the run gathers) but overflows the stage on config 4 (random rows keep most products)
#endif
inline int pair_stage_cap_for(int64_t products, int64_t rows) {
    const double mean = rows > 0 ? (double)products / (double)rows : 0.0;
    int64_t cap = (int64_t)(RIG_PAIR_STAGE_F * 16.0 * mean) + 32;
    cap = (cap + 31) / 32 * 32;
    if (cap < 128) cap = 128;
    if (cap > kMaxStageCap) cap = kMaxStageCap;
    return (int)cap;
}

// Cut slots reserved per numeric launch in the fused-cut partials array.
constexpr int kCutSlotsPerLaunch = 4096;
constexpr int kCutLaunches = 8;  // merge, mid small, mid big, huge (+ spare slots)
// a3 + a4(merge rows) fused: products, merge-row nnzC, bins for the others
// bin8[r]: symbolic bin of row r, or kBinNone on the merge path;
// ctr->sym_count / n_mid: bin totals.
void launch_analyze_sym(const SymArgs &a, uint8_t *bin8, DevCounters *ctr, bool warp_width, cudaStream_t s);
// maxlen: longest A row on the merge path in the shard (DevCounters::max_len)
void launch_sym_merge(const SymArgs &a, int maxlen, cudaStream_t s);
void launch_num_merge(const NumArgs &a, int maxlen, cudaStream_t s);

// Rows off the merge path (k_midrow.cu, k_spgemm.cu huge path): each row is
// written with its exact kept entries to a temporary at toff[r] and
// cnt[r] = kept + 1 (the graph scan subtracts the diagonal slot); k_copy_rows
// places it after the scan and takes its share of the fused cut.
struct MidArgs {
    Csr A;
    Csc T;
    int64_t rb;
    const int32_t *list;    // rows (global ids) to process
    const int64_t *count;   // device: number of rows in list
    const int64_t *toff;    // [nloc] temporary offsets
    int32_t *tcol;
    double *tw;
    int64_t *cnt;           // [nloc] out
    int32_t *defer_list;    // rows whose far list overflowed this kernel's capacity
    int64_t *defer_count;
    double *diag;           // may be null
    double tol;
    int dbg;  // experiment switches (RIG_DEBUG_MASK); 0 in normal operation
    void *fscratch;          // far lists of launch_num_mid_gfar (mid_gfar_scratch_bytes)
    int64_t fscratch_bytes;
    const int64_t *fnm;      // [nloc] f_i - len_i (gfar pass: rows far beyond its capacity skip it)
};
// Fused a7 partials of one launch (part == nullptr: off): each CTA writes the
// Neumaier sum of its cut edges to cutp[blockIdx.x], *used = gridDim.x.
struct CutOut {
    const int32_t *part;
    int32_t K;
    double *cutp;
    int *bad;
    int *used;
};
int debug_mask();  // RIG_DEBUG_MASK environment variable (performance experiments only)
#ifndef RIG_MID_CAP
#define RIG_MID_CAP 256
#endif
constexpr int kMidSmallCap = RIG_MID_CAP, kMidBigCap = 2048;  // far-list capacities of the mid kernels
void launch_num_mid(const MidArgs &a, int fcap, cudaStream_t s);
// second pass over the rows launch_num_mid deferred: window |j - i| < 2048
void launch_num_mid_wide(const MidArgs &a, cudaStream_t s);
// pass over the rows launch_num_mid deferred with a 768-item far list
void launch_num_mid_big(const MidArgs &a, cudaStream_t s);
// pass with a 4096-item far list in global scratch (MidArgs::fscratch)
void launch_num_mid_gfar(const MidArgs &a, cudaStream_t s);
size_t mid_gfar_scratch_bytes();
constexpr int kMidBigFarCapHost = 768;  // = kMidBigFarCap (k_midrow.cu): rows with f_i beyond it may reach the gfar pass
void launch_copy_rows(const int32_t *list, const int64_t *count, int64_t rb, const int64_t *toff, const int64_t *gptr,
                      const int32_t *tcol, const double *tw, int32_t *gcol, double *gw, const CutOut &cut,
                      cudaStream_t s);
// huge rows: CTA per row, dense accumulator + bitmap in global scratch
size_t huge_scratch_bytes(int64_t nrows, int slots, bool numeric);
size_t huge_bitmap_bytes(int64_t nrows, int slots);  // zeroed prefix of the scratch
int huge_slots(int64_t nrows, int64_t n_huge, bool heavy);  // heavy: the shard has huge rows
int huge_slots_rw(int64_t nrows, int64_t n_reach, int64_t per_sm);  // row-window mixed path
void launch_num_huge(const MidArgs &a, int slots, void *scratch, cudaStream_t s);

// k_rowwin.cu: every row of the shard in one kernel, placed straight into the
// graph by a decoupled look-back over the rows' kept counts (no temporary).
struct RowArgs {
    Csr A;
    Csc T;            // CSC offsets must fit int32 (nnz + ncols < 2^31)
    int64_t rb, nloc;
    int32_t *gcol;
    double *gw;
    int64_t cap;      // capacity of gcol / gw; rows beyond it are not written (*overflow |= 1)
    int64_t *row_ptr; // [nloc + 1] local graph row pointers (out)
    unsigned long long *chain;   // [nloc] look-back status words, zeroed
    unsigned long long *ticket;  // row ticket counter, zeroed
    double *diag;     // may be null
    double tol;
    const int32_t *part;  // null: no cut
    int32_t K;
    double *cutrow;   // [nloc] per-row cut sums (when part)
    int *bad_part;
    int *overflow;    // bit 0: capacity too small; bit 1: far list beyond gcap (host bug)
    void *gscratch;   // per-warp far-list slices (rowwin_scratch_bytes(gcap)), may be null if gcap == 0
    int gcap;
    int32_t *stage_col;  // [rowwin_stage_entries()] per-warp staging slots
    double *stage_w;
    // temp mode (mixed path's mid rows; list != null): rows list[0..*count_dev)
    // written exactly to tcol/tw at toff[r], cnt[r] = kept + 1; no look-back
    const int32_t *list;
    const int64_t *count_dev;
    const int64_t *toff;
    int32_t *tcol;
    double *tw;
    int64_t *cnt;
    // temp mode: rows with f_i = fnm[r] + len_i > fskip are not processed but
    // appended to fskip_list (k_row_cta takes them)
    const int64_t *fnm;
    int64_t fskip;
    int32_t *fskip_list;
    int64_t *fskip_count;
    int dbg;          // RIG_DEBUG_MASK experiments (0 in normal operation)
};
int rowwin_grid();
size_t rowwin_scratch_bytes(int gcap);
size_t rowwin_stage_entries();
int rowwin_max_gcap();
int64_t rowwin_max_rows();
void launch_row_win(const RowArgs &a, cudaStream_t s);
// k_rowcta.cu: CTA per row (shared-memory expand / stable radix sort / fold)
// for long rows of scattered columns, temp mode like the mid-row kernels.
struct RcArgs {
    Csr A;
    Csc T;
    int64_t rb;
    const int32_t *list0;  // rows (global ids); list0 then list1
    const int64_t *count0;
    const int32_t *list1;  // may be null
    const int64_t *count1;
    int32_t *rest;         // rows with f_i > fmax (for the huge-row chain)
    int64_t *rest_count;
    unsigned long long *ticket;  // zeroed
    unsigned long long *ticket2; // zeroed, or null: one round (else the rows with f_i > bigf go first)
    int64_t bigf;
    const int64_t *fnm;    // [nloc] f_i - len_i
    const int64_t *toff;
    int32_t *tcol;
    double *tw;
    int64_t *cnt;
    double *diag;
    double tol;
    int fmax;              // items per row held in shared memory
    // RANGE launch (skey != null): rows with fmax < f_i <= scap go through
    // key ranges, staged in per-CTA slices of global scratch
    int32_t *skey;         // [grid][2][scap]
    double *sval;          // [grid][4][scap]
    int64_t scap;
};
size_t rowcta_smem_bytes(int fmax, bool range);
size_t rowcta_scratch_bytes(int64_t scap, int grid);
int rowcta_grid(int fmax, bool range);
int rowcta_range_fmax();  // fmax of the RANGE launch (warps x items per warp range)
void launch_row_cta(const RcArgs &a, cudaStream_t s);

// per-row cut sums -> 256 partials (fixed segments) and *used = 256
void launch_rowcut_partials(const double *cutrow, int64_t n, double *partials, int *used, cudaStream_t s);

// k_probe.cu: gather-only probe of the numeric pass (measurement): sink
// [gather_probe_warps()] doubles
int gather_probe_warps();
void launch_gather_probe(const Csr &A, const Csc &T, int64_t rb, int64_t re, double *sink, cudaStream_t s);

// k_post.cu
void launch_count_kept(const int64_t *gptr_ub, int64_t nloc, const int32_t *gcol, int64_t *kept, cudaStream_t s);
void launch_compact_move(const int64_t *gptr_ub, const int64_t *gptr, int64_t nloc, const int32_t *gcol_in,
                         const double *gw_in, int32_t *gcol, double *gw, cudaStream_t s);
void launch_cutsize(const int64_t *grp, const int32_t *gcol, const double *gw, int64_t nloc, int64_t rb,
                    int64_t n_global, const int32_t *part, int32_t K, double *partials, int nblocks,
                    double *cut, cudaStream_t s);
int cutsize_blocks();
// final fixed-order reduction of cut partials (NaN if *bad)
void launch_cut_final(const double *partials, const int *used, int nseg, int stride, const int *bad, double *cut,
                      cudaStream_t s);
void launch_split(const int64_t *fprefix, int64_t n, int32_t parts, int64_t *split, cudaStream_t s);
// f2: fixed-point limbs of the inter-block inner products (acc [4*K*K]) and
// part weights (wsum [K]), both accumulated (caller-zeroed); *bad set on an
// out-of-range part id or a weight outside [0, 2^63)
void launch_partition_ip(const int64_t *grp, const int32_t *gcol, const double *gw, int64_t nloc, int64_t rb,
                         int64_t n_global, const int32_t *part, int32_t K, const int64_t *arp, unsigned long long *acc,
                         unsigned long long *wsum, int *bad, cudaStream_t s);

// k_coarsen.cu (f4)
void launch_hem_round(const int64_t *rp, const int32_t *col, const int64_t *wgt, int64_t n, int32_t *match,
                      int32_t *cand, cudaStream_t s);
void launch_leader_flags(const int32_t *match, int64_t n, int64_t *flag, cudaStream_t s);
void launch_coarse_map(const int64_t *rp, const int32_t *match, const int64_t *vwgt, int64_t n, const int64_t *cid,
                       int32_t *cmap, int32_t *lead, int64_t *cvwgt, int64_t *citems, unsigned long long *maxit,
                       cudaStream_t s);
void launch_coarse_copy(const int64_t *toff, const int64_t *crp, int64_t nc, const int32_t *tcol, const int64_t *tw,
                        int32_t *ccol, int64_t *cw, cudaStream_t s);
void launch_coarse_rows(int pass, const int64_t *rp, const int32_t *col, const int64_t *wgt, const int32_t *match,
                        const int32_t *cmap, const int32_t *lead, int64_t nc, int64_t *ccnt, const int64_t *crp,
                        int32_t *ccol, int64_t *cw, uint64_t *gscratch, int64_t gcap, int big_warps,
                        cudaStream_t s);

// ---- decoupled look-back over per-item status words (row-window rows):
// count | kAgg (count published), prefix | kPre
constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62, kValMask = (1ull << 62) - 1;
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Exclusive prefix of row idx's count; idx's own status is already published
// (kAgg, or kPre for idx 0).  All lanes call it; lane 0 publishes idx's
// inclusive prefix.  Every lower ticket is held by a running warp, which
// publishes its count without waiting on anything: the walk ends.
__device__ __forceinline__ int64_t lookback(unsigned long long *chain, int64_t idx, int64_t c) {
    const int l = lane_id();
    if (idx == 0) return 0;
    int64_t excl = 0;
    int64_t base = idx - 1;
    while (true) {
        const int64_t j = base - l;
        unsigned long long v = j >= 0 ? ld_relaxed(&chain[j]) : kPre;
        unsigned zm = __ballot_sync(kFull, (v >> 62) == 0);
        unsigned pm = __ballot_sync(kFull, (v & kPre) != 0);
        // wait for the nearest unpublished predecessor that is needed (one
        // lane polls one word with backoff: no polling storm on the
        // frontier's cache lines), then look at the window again
        while (true) {
            const int fp = pm ? __ffs(pm) - 1 : 31;
            const unsigned need = fp == 31 ? kFull : ((2u << fp) - 1u);
            const unsigned wz = zm & need;
            if (!wz) break;
            const int t = __ffs(wz) - 1;
            if (l == t) {
                unsigned ns = 64;
                do {
                    __nanosleep(ns);
                    ns = ns < 2048 ? ns * 2 : 2048;
                    v = ld_relaxed(&chain[j]);
                } while ((v >> 62) == 0);
            }
            __syncwarp();
            zm = __ballot_sync(kFull, (v >> 62) == 0);
            pm = __ballot_sync(kFull, (v & kPre) != 0);
        }
        const int fp = pm ? __ffs(pm) - 1 : 31;
        const unsigned need = fp == 31 ? kFull : ((2u << fp) - 1u);
        const int64_t add = ((need >> l) & 1u) ? (int64_t)(v & kValMask) : 0;
        excl += warp_sum(add);
        if (pm) break;
        base -= 32;
    }
    if (l == 0) st_relaxed(&chain[idx], kPre | (unsigned long long)(excl + c));
    return excl;
}

}  // namespace rig

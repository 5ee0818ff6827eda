// rig_api.cu -- the C ABI declared in include/rig.h: argument checks, device
// memory, pass orchestration, error reporting.  Every step of the path runs
// in the kernels of k_*.cu; this file only sequences them and reads back the
// few counters that size allocations.
//
// Host-overhead budget: a build makes one workspace
// allocation per phase (stream-ordered pool, cached per thread), a few
// memsets, one or two host syncs (counters read into pinned host memory) and
// 10-20 kernel launches depending on the path (merge / row-window / mixed).
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/rig.h"
#include "common.cuh"

namespace rig {

static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int debug_mask() {
    static int m = -1;
    if (m < 0) {
        const char *e = getenv("RIG_DEBUG_MASK");
        m = e ? atoi(e) : 0;
    }
    return m;
}

int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

// ---------------------------------------------------------------- profiling
enum Pass {
    P_VALIDATE = 0,
    P_COLPTR,    // column histogram (+ ranks) + scan
    P_SCATTER,   // a1 scale + a2 scatter
    P_COLSORT,   // a2 per-column order
    P_ANALYZE,   // a3 + a4 for merge-path rows
    P_SYMBOLIC,  // a4 for the other rows (+ numeric binning)
    P_UBSCAN,    // graph row pointers
    P_NUMERIC,   // a5 + a6 (+ fused a7 partials)
    P_COMPACT,   // a6 holes path
    P_CUTSIZE,   // a7 (standalone kernel or fused final reduction)
    P_SPLIT,
    P_KERNEL,  // the dominant numeric kernel alone (merge kernel, or the mid-row kernel)
    P_SPARSIFY,  // f1: dense-column cutoffs, A~ filter, transpose of A~
};
static const char *kPassNames[RIG_NPASS] = {"validate", "colptr",   "scale_scatter", "colsort",
                                            "analyze",  "symbolic", "ub_scan",       "numeric",
                                            "compact",  "cutsize",  "split",         "numeric_kernel",
                                            "sparsify"};
static std::mutex g_prof_mu;
static std::atomic<uint32_t> g_prof_mask{0};
struct ProfRec {
    int pass;
    cudaEvent_t a, b;
};
static std::vector<ProfRec> g_recs;
static std::vector<std::pair<int, cudaEvent_t>> g_pool;  // (device, event)

static cudaEvent_t ev_get() {
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        for (size_t k = 0; k < g_pool.size(); ++k)
            if (g_pool[k].first == dev) {
                cudaEvent_t e = g_pool[k].second;
                g_pool.erase(g_pool.begin() + (long)k);
                return e;
            }
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// CUDA event pair around one pass on the stream it runs on (when enabled).
struct Prof {
    int pass;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    Prof(int p, cudaStream_t st) : pass(p), s(st) {
        if (p >= 0 && (g_prof_mask.load(std::memory_order_relaxed) & (1u << p))) {
            a = ev_get();
            cudaEventRecord(a, s);
        }
    }
    ~Prof() {
        if (!a) return;
        cudaEvent_t b = ev_get();
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_recs.push_back({pass, a, b});
    }
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

static thread_local std::string t_last_error;
static thread_local std::string t_last_path;

#define CK(call)                                                                                \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            throw Error(e_ == cudaErrorMemoryAllocation ? RIG_ERR_NOMEM : RIG_ERR_CUDA,         \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                    \
    } while (0)

// RIG_SYNC_CHECK=1 (debugging): synchronise at every check so a fault is
// attributed to the pass that caused it.
// Smallest nnz for the pattern-symmetric transpose attempt (2^24; the
// RIG_SYM_MIN_NNZ environment variable overrides it: tests, tuning).
static int64_t sym_min_nnz() {
    static int64_t v = -1;
    if (v < 0) {
        const char *e = getenv("RIG_SYM_MIN_NNZ");
        v = e ? atoll(e) : (int64_t(1) << 24);
    }
    return v;
}

// The row-window path (k_rowwin.cu) is taken when no row of the shard is on
// the merge path and the longest row has at most kRowWinMaxF products;
// RIG_ROWWIN=0 turns it off (tests compare both paths).
constexpr int64_t kRowWinMaxF = 1024;
// the same decision from the shape statistics alone uses the looser bound
// f_i <= max_row * max_col (config 5: 23 * ~50 against its true max 636)
constexpr int64_t kRowWinEarlyBound = 2048;
// mixed path: rows with f_i > kRowCtaMinF go from the row-window kernel to the
// CTA-per-row kernel, which holds up to kRowCtaMaxF products in shared memory
// (RIG_CTA_MINF / RIG_CTA_MAXF override them: experiments)
static int64_t env_i64(const char *name, int64_t dflt) {
    const char *e = getenv(name);
    return e ? atoll(e) : dflt;
}
// Measured on configs 4 and 6: 256 / 1280 best.  Longer rows (after the
// wide-window pass) take a second launch (k_row_cta<RANGE>, larger arrays):
// rows beyond its arrays go through key ranges, staged in per-CTA slices of
// global scratch of up to kLongScratchMB in all; the rows it cannot take
// (beyond a slice, or a crowded key sub-bucket) fall to the global-far-list
// and CTA-accumulator kernels, whose scratch is then allocated.
static const int64_t kRowCtaMinF = env_i64("RIG_CTA_MINF", 256), kRowCtaMaxF = env_i64("RIG_CTA_MAXF", 1280),
                     kLongScratchMB = env_i64("RIG_LONG_SCRATCH_MB", 1024);
// longest rows first in the CTA-per-row launches (two rounds over the list):
// the shared-memory launch (0: one round) and the key-range launch
// (measured on configs 4 and 6: 4096 best of 2048-16384 for the latter)
static const int64_t kRowCtaBigF0 = env_i64("RIG_CTA_BIGF0", 0), kRowCtaBigF1 = env_i64("RIG_CTA_BIGF1", 4096);
// huge-kernel slots per SM on the row-window mixed path (each slot is O(n)
// memory); measured 1, 2, 4, 8: 4 is as fast as 8 with half the memory
static const int64_t kHugePerSmRw = env_i64("RIG_HUGE_PER_SM_RW", 4);
static bool rowwin_enabled_env();
// the row-window kernel (row-window and mixed paths) needs int32 CSC offsets
// and row ids below 2^25 (its shared far list packs the unit under the key)
static bool rowwin_ok(const Csr &A) {
    return rowwin_enabled_env() && csc_fits_i32(A) && A.nrows <= rowwin_max_rows();
}
static bool rowwin_enabled_env() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("RIG_ROWWIN");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

static bool sync_check() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("RIG_SYNC_CHECK");
        v = (e && atoi(e)) ? 1 : 0;
    }
    return v == 1;
}

static void check_launch(const char *what) {
    cudaError_t e = sync_check() ? cudaDeviceSynchronize() : cudaSuccess;
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(RIG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static void ensure_pool() {
    static bool done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !done[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        done[dev] = true;
    }
}

// Pinned host staging for the counters read back at syncs (per thread).
struct HostStage {
    DevCounters ctr, shape;
    int64_t v[4];
    int holes;
};
static HostStage *host_stage() {
    static thread_local HostStage *hs = nullptr;
    if (!hs) {
        void *p = nullptr;
        if (cudaMallocHost(&p, sizeof(HostStage)) != cudaSuccess) throw Error(RIG_ERR_NOMEM, "cudaMallocHost");
        hs = static_cast<HostStage *>(p);
    }
    return hs;
}

static cudaEvent_t shape_event() {  // per thread, reused
    static thread_local cudaEvent_t ev = nullptr;
    if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    return ev;
}

// Bump layout over one allocation: add() records 256-byte aligned offsets.
struct Layout {
    size_t bytes = 0;
    size_t add(size_t n) {
        const size_t off = bytes;
        bytes += (n + 255) & ~(size_t)255;
        return off;
    }
};

// Stream-ordered allocations owned by one call / plan.
struct Arena {
    cudaStream_t s;
    std::vector<void *> ptrs;
    explicit Arena(cudaStream_t st) : s(st) {}
    unsigned char *raw(size_t bytes) {
        void *p = nullptr;
        CK(cudaMallocAsync(&p, bytes ? bytes : 256, s));
        ptrs.push_back(p);
        return static_cast<unsigned char *>(p);
    }
    template <typename T>
    T *get(int64_t count) {
        return reinterpret_cast<T *>(raw((size_t)(count > 0 ? count : 1) * sizeof(T)));
    }
    ~Arena() {
        for (void *p : ptrs)
            if (p) cudaFreeAsync(p, s);
    }
};

// Grow-only per-thread workspace cache for the simple API's internal buffers
// (phase A, phase B, numeric temporaries): consecutive builds on the same
// device and stream reuse them in stream order, so the hot loop makes no
// allocator calls besides the returned graph.  rig_trim() releases them.
struct WsCache {
    int dev = -1;
    void *p[3] = {nullptr, nullptr, nullptr};
    size_t n[3] = {0, 0, 0};
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};
};
static thread_local WsCache t_ws;

static void ws_trim() {
    for (int k = 0; k < 3; ++k) {
        if (t_ws.p[k]) cudaFreeAsync(t_ws.p[k], t_ws.s[k]);
        t_ws.p[k] = nullptr;
        t_ws.n[k] = 0;
    }
}

static unsigned char *ws_get(int slot, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (t_ws.dev != dev) {
        if (t_ws.dev >= 0) {  // another device: release on that device
            int cur = dev;
            cudaSetDevice(t_ws.dev);
            ws_trim();
            cudaSetDevice(cur);
        }
        t_ws.dev = dev;
    }
    if (t_ws.p[slot] && t_ws.n[slot] >= bytes && t_ws.s[slot] == s) return static_cast<unsigned char *>(t_ws.p[slot]);
    if (t_ws.p[slot]) CK(cudaFreeAsync(t_ws.p[slot], t_ws.s[slot]));
    t_ws.p[slot] = nullptr;
    const size_t want = bytes + bytes / 8 + 4096;  // headroom for slightly larger inputs
    CK(cudaMallocAsync(&t_ws.p[slot], want, s));
    t_ws.n[slot] = want;
    t_ws.s[slot] = s;
    return static_cast<unsigned char *>(t_ws.p[slot]);
}

// Library-owned graphs: row_ptr and the (col, w, diag) block are two
// allocations; rig_graph_free looks the block up by row_ptr.
static std::mutex g_own_mu;
static std::unordered_map<void *, void *> g_owned;

static int err_to_code(int err) {
    if (err & kErrNonCanonical) return RIG_ERR_NONCANONICAL;
    if (err & kErrNonFinite) return RIG_ERR_NONFINITE;
    if (err & kErrZeroRow) return RIG_ERR_ZERO_ROW;
    return RIG_OK;
}

static const char *err_msg(int code) {
    switch (code) {
        case RIG_ERR_NONCANONICAL: return "input CSR is not canonical";
        case RIG_ERR_NONFINITE: return "non-finite value or row norm";
        case RIG_ERR_ZERO_ROW: return "scale_rows with an empty or all-zero row";
        default: return "error";
    }
}

static void check_csr(const rig_csr_t *A) {
    if (!A) throw Error(RIG_ERR_INVALID, "A is NULL");
    if (A->nrows < 0 || A->ncols < 0 || A->nnz < 0) throw Error(RIG_ERR_INVALID, "negative size");
    if (A->nrows > INT32_MAX || A->ncols > INT32_MAX) throw Error(RIG_ERR_INVALID, "nrows/ncols exceed int32");
    if (!A->row_ptr) throw Error(RIG_ERR_INVALID, "row_ptr is NULL");
    if (A->nnz > 0 && (!A->col_idx || !A->val)) throw Error(RIG_ERR_INVALID, "col_idx/val is NULL");
}

}  // namespace rig

using namespace rig;

// f1: T = ceil(sqrt(n)), the smallest t with t * t >= n (PAPER.md:572-574,
// DESIGN.md reading R20)
static int64_t dense_threshold(int64_t n) {
    if (n <= 0) return 0;
    int64_t t = (int64_t)std::sqrt((double)n);
    while (t * t < n) ++t;
    while (t > 0 && (t - 1) * (t - 1) >= n) --t;
    return t;
}

// ---------------------------------------------------------------- the plan
struct rig_plan {
    cudaStream_t s;
    Arena arena;
    Csr A{};  // scaled view
    Csc T{};
    int scale = 0;
    double tol = 0;
    uint32_t flags = 0;
    int64_t rb = 0, re = 0, nloc = 0;
    DevCounters *ctr = nullptr;  // device
    DevCounters h{};             // host copy (after sync 1)
    int64_t *nnzc = nullptr;     // [nloc] merge rows: structural nnz(C_i); others: kept + 1 (numeric)
    int2 *qs = nullptr;          // merge rows' CSC runs (SymArgs::qs)
    // rows off the merge path (h.n_mid > 0): exact rows in the temporary
    int32_t *lists = nullptr;    // [2 * n_mid]: mid rows, huge rows (ascending)
    int32_t *defer = nullptr;    // [2 * n_mid]: deferred by the small / big mid kernel
    int64_t *toff = nullptr;     // [nloc + 1]
    int32_t *tcol = nullptr;
    double *tw = nullptr;
    void *huge_scratch = nullptr;
    void *gfar = nullptr;  // far-list scratch of launch_num_mid_gfar
    int64_t *fnm = nullptr;  // [nloc] f_i - len_i off the merge path
    int huge_slots_n = 0;
    int64_t nnz_upper = 0;  // >= graph nnz: sum (f_i - len_i)
    bool cached = false;    // simple API: internal buffers from the per-thread cache
    bool early = false;     // all rows on the merge path, decided before the transpose ran:
                            // no synchronisation until the end (errors are read there)
    bool rowwin = false;    // no row on the merge path: one row-window kernel places every
                            // row straight into the graph (k_rowwin.cu, no temporary)
    int rw_gcap = 0;        // its global far-list capacity (0: shared lists only)
    bool mid_rowwin = false;  // mixed path: mid rows through k_row_win (temp mode) instead of the mid passes
    void *mid_rw_scratch = nullptr;  // its global far lists + ticket
    void *long_scratch = nullptr;    // k_row_cta<RANGE> slices (mid_rowwin, max f_i > kRowCtaMaxF)
    int64_t long_scap = 0;
    int long_grid = 0;
    explicit rig_plan(cudaStream_t st) : s(st), arena(st) {}
};

// Steps a0-a4 for rows [rb, re): validation, column pointers, scaling +
// transpose, products / paths / merge-row structure (analyze), and the
// ordered lists and temporary of the rows off the merge path.  One host
// synchronisation (sync 1: errors, products, list sizes).
static void plan_build(rig_plan *p, const rig_csr_t *Ain, bool allow_early = false) {
    cudaStream_t s = p->s;
    const int64_t n = Ain->nrows, m = Ain->ncols, nnz = Ain->nnz, nloc = p->nloc;
    Csr A0{n, m, nnz, Ain->row_ptr, Ain->col_idx, Ain->val};
    // ---- phase-A workspace (one allocation, one memset of the zeroed head)
    Layout L;
    const size_t o_ctr = L.add(sizeof(DevCounters));
    const size_t o_cnt = L.add(sizeof(unsigned) * (size_t)m);
    const size_t o_st1 = L.add(scan_tmp_bytes(m));
    const size_t o_bcur = L.add(sizeof(unsigned long long) * (size_t)transpose_buckets(nnz, m));
    const size_t o_gcur = L.add(sizeof(unsigned) * (size_t)m);
    const size_t o_big = L.add(sizeof(int) * (size_t)(1 + transpose_buckets(nnz, m)));
    const bool sparsify = (p->flags & RIG_FLAG_SPARSIFY) != 0;
    const size_t o_ndense = sparsify ? L.add(sizeof(int)) : 0;
    // pattern-symmetric fast transpose (stencils, FEM meshes), tried on square
    // inputs from 2^24 entries: below that its dependent gathers leave it
    // latency-bound and the bucket transpose is faster (measured: config 2,
    // 5M entries, 0.21 vs 0.18 ms; config 3, 56M entries, 1.30 vs 1.88 ms).
    // A missing mirror entry hands over to the guarded general path.
    const bool try_sym = n == m && nnz > 0 && nnz >= sym_min_nnz() && !sparsify;
    const size_t o_symfail = try_sym ? L.add(sizeof(int)) : 0;
    const size_t zero_bytes = L.bytes;
    const size_t o_nrm = try_sym && p->scale ? L.add(2 * sizeof(double) * (size_t)n) : 0;
    const size_t o_cp = L.add(sizeof(int64_t) * (size_t)(m + 1));
    const size_t o_rec = L.add(kTransposeRecBytes * (size_t)nnz);
    const size_t o_ahat = p->scale ? L.add(sizeof(double) * (size_t)nnz) : 0;
    // + one sentinel per column, + one leading pad entry: a descending merge
    // lane's last advance may read the entry before its run (never used)
    // two readable pad entries lead the arrays: the merge lanes' look-ahead
    // reads up to two entries before a run (never used)
    const size_t o_ri = L.add(sizeof(int32_t) * (size_t)(nnz + m + 3));
    const size_t o_vt = L.add(sizeof(double) * (size_t)(nnz + m + 2));
    const size_t o_nnzc = L.add(sizeof(int64_t) * (size_t)nloc);
    const size_t o_fnm = L.add(sizeof(int64_t) * (size_t)nloc);
    const size_t o_bin8 = L.add((size_t)nloc);
    const bool use_qs = csc_fits_i32(A0);  // run starts fit int32
    const size_t o_qs = use_qs ? L.add(sizeof(int2) * (size_t)nnz) : 0;
    // f1 (RIG_FLAG_SPARSIFY): dense-column list and cutoffs, A~ in CSR
    size_t o_dlist = 0, o_ckey = 0, o_crow = 0, o_nk = 0, o_rp2 = 0, o_ci2 = 0, o_v2 = 0, o_st3 = 0;
    if (sparsify) {
        o_dlist = L.add(sizeof(int32_t) * (size_t)m);
        o_ckey = L.add(sizeof(unsigned long long) * (size_t)m);
        o_crow = L.add(sizeof(int32_t) * (size_t)m);
        o_nk = L.add(sizeof(int64_t) * (size_t)n);
        o_rp2 = L.add(sizeof(int64_t) * (size_t)(n + 1));
        o_ci2 = L.add(sizeof(int32_t) * (size_t)nnz);
        o_v2 = L.add(sizeof(double) * (size_t)nnz);
        o_st3 = L.add(scan_tmp_bytes(n));
    }
    unsigned char *ws = p->cached ? ws_get(0, L.bytes, s) : p->arena.raw(L.bytes);
    CK(cudaMemsetAsync(ws, 0, zero_bytes, s));
    p->ctr = reinterpret_cast<DevCounters *>(ws + o_ctr);
    unsigned *cnt = reinterpret_cast<unsigned *>(ws + o_cnt);
    int64_t *cp = reinterpret_cast<int64_t *>(ws + o_cp);
    double *ahat = p->scale ? reinterpret_cast<double *>(ws + o_ahat) : nullptr;
    int32_t *ri = reinterpret_cast<int32_t *>(ws + o_ri) + 2;
    double *vt = reinterpret_cast<double *>(ws + o_vt) + 2;
    p->nnzc = reinterpret_cast<int64_t *>(ws + o_nnzc);
    int64_t *fnm = reinterpret_cast<int64_t *>(ws + o_fnm);
    p->fnm = fnm;
    uint8_t *bin8 = reinterpret_cast<uint8_t *>(ws + o_bin8);
    HostStage *hs = host_stage();

    // a0: validation must finish before anything indexes with the input
    if (p->flags & RIG_FLAG_VALIDATE) {
        Prof pf(P_VALIDATE, s);
        launch_validate(A0, &p->ctr->err, s);
        check_launch("validate");
        CK(cudaMemcpyAsync(&hs->ctr.err, &p->ctr->err, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int err = hs->ctr.err;
        if (err) throw Error(err_to_code(err), err_msg(err_to_code(err)));
    }
    // a2: column counts -> col_ptr; shape statistics read back while the
    // transpose and the analysis run (simple API)
    cudaEvent_t ev_shape = nullptr;
    const bool want_shape = allow_early && nloc > 0 && !sparsify;
    int *symfail = try_sym ? reinterpret_cast<int *>(ws + o_symfail) : nullptr;  // guard of the general path
    if (try_sym) {  // a1 + a2 as a gather when the pattern is symmetric
        Prof pf(P_SCATTER, s);
        double *nrm = p->scale ? reinterpret_cast<double *>(ws + o_nrm) : nullptr;
        launch_sym_transpose(A0, p->scale, nrm, nrm ? nrm + n : nullptr, ahat, cp, ri, vt, symfail, &p->ctr->err,
                             want_shape ? p->ctr : nullptr, p->rb, p->re, s);
    }
    {
        Prof pf(P_COLPTR, s);
        if (nnz > 0) launch_col_hist(A0, cnt, nullptr, s, symfail);
        if (want_shape) {
            ev_shape = shape_event();
            scan_u32_shape(cnt, m, cp, ws + o_st1, p->ctr, A0.rp, p->rb, p->re, &hs->shape, ev_shape, s, symfail);
        } else {
            scan_u32(cnt, m, cp, ws + o_st1, 0, s, symfail);
        }
    }
    // a1 + a2: scale rows (optional), bucketed transpose into the CSC (skipped
    // on the device when the symmetric gather succeeded)
    {
        Prof pf(P_SCATTER, s);
        launch_transpose(A0, p->scale, cp, ahat, reinterpret_cast<unsigned long long *>(ws + o_bcur), ws + o_rec,
                         reinterpret_cast<unsigned *>(ws + o_gcur), reinterpret_cast<int *>(ws + o_big), ri, vt,
                         &p->ctr->err, s, symfail);
    }
    check_launch("prep");
    p->A = Csr{n, m, nnz, Ain->row_ptr, Ain->col_idx, p->scale ? ahat : Ain->val};
    p->T = Csc{cp, ri, vt};
    if (sparsify && nnz > 0) {
        // f1: A~ from A_hat: cutoffs of the dense columns
        // on the CSC just built, the CSR filter, then column access to A~
        // (its values are already scaled: transposed as they are)
        Prof pf(P_SPARSIFY, s);
        const int64_t Tn = dense_threshold(n);
        auto *ckey = reinterpret_cast<unsigned long long *>(ws + o_ckey);
        auto *crow = reinterpret_cast<int32_t *>(ws + o_crow);
        auto *nk = reinterpret_cast<int64_t *>(ws + o_nk);
        auto *rp2 = reinterpret_cast<int64_t *>(ws + o_rp2);
        auto *ci2 = reinterpret_cast<int32_t *>(ws + o_ci2);
        auto *v2 = reinterpret_cast<double *>(ws + o_v2);
        launch_sparsify_cutoffs(cnt, m, Tn, p->T, reinterpret_cast<int32_t *>(ws + o_dlist),
                                reinterpret_cast<int *>(ws + o_ndense), ckey, crow, s);
        launch_sparsify_filter(0, p->A, cnt, Tn, ckey, crow, nk, nullptr, nullptr, nullptr, s);
        scan_i64(nk, n, rp2, ScanOp::Identity, ws + o_st3, 0, s);
        check_launch("sparsify");
        int64_t nnz2 = 0;
        CK(cudaMemcpyAsync(&hs->v[0], rp2 + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&hs->ctr.err, &p->ctr->err, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        nnz2 = hs->v[0];
        if (hs->ctr.err) throw Error(err_to_code(hs->ctr.err), err_msg(err_to_code(hs->ctr.err)));
        if (nnz2 < nnz) {
            launch_sparsify_filter(1, p->A, cnt, Tn, ckey, crow, nullptr, rp2, ci2, v2, s);
            CK(cudaMemsetAsync(ws + o_cnt, 0, zero_bytes - o_cnt, s));
            const Csr A2{n, m, nnz2, rp2, ci2, v2};
            if (nnz2 > 0) launch_col_hist(A2, cnt, nullptr, s);
            scan_u32(cnt, m, cp, ws + o_st1, 0, s);
            launch_transpose(A2, 0, cp, nullptr, reinterpret_cast<unsigned long long *>(ws + o_bcur), ws + o_rec,
                             reinterpret_cast<unsigned *>(ws + o_gcur), reinterpret_cast<int *>(ws + o_big), ri, vt,
                             &p->ctr->err, s);
            check_launch("sparsify transpose");
            p->A = A2;
        }
    }
    // a3 + a4 (merge rows): products, merge-row nnzC, paths of the others
    p->qs = use_qs ? reinterpret_cast<int2 *>(ws + o_qs) : nullptr;
    // analysis merge width per warp when row lengths vary widely (some rows
    // off the merge path: power-law shards), per lane otherwise (k_spgemm.cu)
    bool an_warp_width = false;
    if (ev_shape && rowwin_ok(p->A)) {
        // row-window path decided from the shape statistics alone (read back
        // while the transpose runs): every row longer than the merge path
        // takes, and f_i <= max_row * max_col small enough.  No analysis and
        // no synchronisation until the end (errors are read there).
        CK(cudaEventSynchronize(ev_shape));
        const DevCounters &sh = hs->shape;
        const int64_t min_row = sh.min_row_c ? kMinRowBias - sh.min_row_c : 0;
        const int64_t fbound = sh.max_row * sh.max_col;
        an_warp_width = sh.max_row > kMergeMaxLen;
        if (nloc > 0 && min_row > kMergeMaxLen && fbound <= kRowWinEarlyBound) {
            p->early = true;
            p->rowwin = true;
            p->h = DevCounters{};
            const int64_t pb = std::min<int64_t>(sh.p_full, sh.shard_nnz * sh.max_col);
            p->h.products = pb;  // an upper bound here
            p->h.max_f = fbound;
            p->h.n_mid = nloc;
            p->nnz_upper = pb - sh.shard_nnz;
            p->rw_gcap = (int)std::max<int64_t>(fbound, 1);
            return;
        }
    }
    SymArgs sa{p->A, p->T, p->rb, p->re, p->nnzc, fnm, p->qs};
    if (nloc > 0) {
        Prof pf(P_ANALYZE, s);
        launch_analyze_sym(sa, bin8, p->ctr, an_warp_width, s);
    }
    check_launch("analyze");
    if (ev_shape) {
        CK(cudaEventSynchronize(ev_shape));
        const DevCounters &sh = hs->shape;
        if (sh.max_row <= kMergeMaxLen && sh.max_col * kMergeMaxLen <= kMergeMaxF) {
            // every row of the shard is a merge row: size the output from the
            // bound sum_k len_k^2 - nnz(shard) >= sum_i (f_i - len_i); the
            // exact counters (and any error flag) are read at the final sync
            p->early = true;
            p->h = DevCounters{};
            p->h.max_len = (int)sh.max_row;
            // a shard's products are at most min(sum_k len_k^2, shard_nnz *
            // max_col) (f_i <= len_i * max_col): the bound scales with the shard
            const int64_t pb = std::min<int64_t>(sh.p_full, sh.shard_nnz * sh.max_col);
            p->h.products = pb;  // an upper bound here (sizes the merge kernel's stage)
            p->nnz_upper = pb - sh.shard_nnz;
            return;
        }
    }
    // sync 1: errors, products, path sizes
    CK(cudaMemcpyAsync(&hs->ctr, p->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    p->h = hs->ctr;
    if (p->h.err) throw Error(err_to_code(p->h.err), err_msg(err_to_code(p->h.err)));
    p->nnz_upper = p->h.products - p->h.nnz_rows;
    const int64_t n_mid = p->h.n_mid;
    if (n_mid == 0) return;
    if (n_mid == nloc && rowwin_ok(p->A) && p->h.max_f <= kRowWinMaxF) {
        p->rowwin = true;  // every row in one kernel, placed by look-back
        p->rw_gcap = (int)std::max<int64_t>(p->h.max_f, 1);  // global far lists: rows beyond the shared list
        return;
    }
    // ---- rows off the merge path: ordered lists, temporary layout
    Prof pf(P_SYMBOLIC, s);
    // the huge path takes the huge bin and every row the mid kernel defers (far
    // list beyond its capacity, or far keys crowding one sort bucket); with
    // short rows only the latter can happen, so a few slots suffice
    const size_t nbc = bins_count_elems(nloc);
    Layout LB;
    const size_t o_toff = LB.add(sizeof(int64_t) * (size_t)(nloc + 1));
    const size_t o_st2 = LB.add(scan_tmp_bytes(nloc));
    const size_t o_lists = LB.add(sizeof(int32_t) * 2 * (size_t)n_mid);
    const size_t o_defer = LB.add(sizeof(int32_t) * 5 * (size_t)n_mid);
    const size_t o_bcnt = LB.add(sizeof(unsigned) * nbc);
    const size_t o_boff = LB.add(sizeof(int64_t) * (nbc + 1));
    const size_t o_bst = LB.add(scan_tmp_bytes((int64_t)nbc));
    const size_t o_tcol = LB.add(sizeof(int32_t) * (size_t)p->h.mid_slots);
    const size_t o_tw = LB.add(sizeof(double) * (size_t)p->h.mid_slots);
    // far lists of the global-far-list pass (rows that can outgrow the 768-item list)
    // mid rows (f_i <= 2^kSymBinMaxLog / 2) through k_row_win in temp mode:
    // global far lists of that capacity, + a zeroed ticket
    p->mid_rowwin = rowwin_ok(p->A);
    const bool need_gfar = p->h.max_f > kMidBigFarCapHost;
    const size_t o_gfar = need_gfar && !p->mid_rowwin ? LB.add(mid_gfar_scratch_bytes()) : 0;
    constexpr int kMidMaxF = 1 << (kSymBinMaxLog - 1);
    p->rw_gcap = (int)std::min<int64_t>(std::max<int64_t>(p->h.max_f, 1), kMidMaxF);
    const size_t o_mrw = p->mid_rowwin ? LB.add(256 + rowwin_scratch_bytes(p->rw_gcap)) : 0;
    size_t o_huge = 0, o_long = 0;
    if (p->mid_rowwin) {
        // the global-far-list and huge kernels get their scratch only if rows
        // reach them (plan_numeric, after the range launch)
        if (p->h.max_f > kRowCtaMaxF) {
            p->long_grid = rowcta_grid(rowcta_range_fmax(), true);
            const int64_t per_item = (int64_t)rowcta_scratch_bytes(1, p->long_grid);
            p->long_scap = std::min<int64_t>(p->h.max_f, (kLongScratchMB << 20) / per_item);
            if (p->long_scap > rowcta_range_fmax()) o_long = LB.add(rowcta_scratch_bytes(p->long_scap, p->long_grid));
            else p->long_scap = 0;
        }
    } else {
        p->huge_slots_n = huge_slots(n, p->h.max_f > kMidSmallCap ? n_mid : std::min<int64_t>(n_mid, 8),
                                     p->h.sym_count[kNumSymBins] > 0);
        o_huge = LB.add(huge_scratch_bytes(n, p->huge_slots_n, true));
    }
    unsigned char *wb = p->cached ? ws_get(1, LB.bytes, s) : p->arena.raw(LB.bytes);
    p->toff = reinterpret_cast<int64_t *>(wb + o_toff);
    p->lists = reinterpret_cast<int32_t *>(wb + o_lists);
    p->defer = reinterpret_cast<int32_t *>(wb + o_defer);
    p->gfar = need_gfar && !p->mid_rowwin ? wb + o_gfar : nullptr;
    p->mid_rw_scratch = p->mid_rowwin ? wb + o_mrw : nullptr;
    p->long_scratch = p->long_scap ? wb + o_long : nullptr;
    p->tcol = reinterpret_cast<int32_t *>(wb + o_tcol);
    p->tw = reinterpret_cast<double *>(wb + o_tw);
    if (!p->mid_rowwin) {
        p->huge_scratch = wb + o_huge;
        CK(cudaMemsetAsync(p->huge_scratch, 0, huge_bitmap_bytes(n, p->huge_slots_n), s));
    }
    scan_i64(fnm, nloc, p->toff, ScanOp::Identity, wb + o_st2, 0, s);
    launch_bins(bin8, p->rb, nloc, reinterpret_cast<unsigned *>(wb + o_bcnt), reinterpret_cast<int64_t *>(wb + o_boff),
                wb + o_bst, p->lists, n_mid, p->ctr->list_count, s);
    check_launch("lists");
}

struct CutReq {
    const int32_t *part = nullptr;
    int32_t K = 0;
    double *cut_dev = nullptr;
};

// a5 + a6 (+ fused a7) into caller arrays of capacity >= p->nnz_upper:
// rows off the merge path into the temporary (exact counts), the scan of all
// rows' counts into the graph row pointers, merge rows in place, the others
// copied into place.  Returns the graph nnz.  Synchronises once (twice if a
// merge row dropped an entry by value: compaction).
// Row-window path: chain + ticket zeroed, the kernel, the fused cut from the
// per-row sums; one synchronisation (overflow flag and nnz).  A capacity
// below the graph nnz leaves the rows beyond it unwritten and throws
// NeedCapacity (build_owned retries with the exact size).
struct NeedCapacity {
    int64_t nnz;
};
static int64_t rowwin_numeric(rig_plan *p, int32_t *gcol, double *gw, int64_t cap, double *dg, int64_t *row_ptr_out,
                              unsigned char *wn, int *flag_d, int *used, double *cutp, const CutReq *cut) {
    cudaStream_t s = p->s;
    Layout L;
    const size_t o_chain = L.add(sizeof(unsigned long long) * (size_t)(p->nloc + 1));
    const size_t zero_bytes = L.bytes;
    const size_t o_cutrow = cut ? L.add(sizeof(double) * (size_t)p->nloc) : 0;
    const size_t o_g = L.add(rowwin_scratch_bytes(p->rw_gcap));
    const size_t o_sc = L.add(sizeof(int32_t) * rowwin_stage_entries());
    const size_t o_sw = L.add(sizeof(double) * rowwin_stage_entries());
    unsigned char *wr = p->cached ? ws_get(1, L.bytes, s) : p->arena.raw(L.bytes);
    CK(cudaMemsetAsync(wr, 0, zero_bytes, s));
    auto *chain = reinterpret_cast<unsigned long long *>(wr + o_chain);
    RowArgs ra{};
    ra.A = p->A;
    ra.T = p->T;
    ra.rb = p->rb;
    ra.nloc = p->nloc;
    ra.gcol = gcol;
    ra.gw = gw;
    ra.cap = cap;
    ra.row_ptr = row_ptr_out;
    ra.chain = chain;
    ra.ticket = chain + p->nloc;
    ra.diag = dg;
    ra.tol = p->tol;
    ra.part = cut ? cut->part : nullptr;
    ra.K = cut ? cut->K : 0;
    ra.cutrow = cut ? reinterpret_cast<double *>(wr + o_cutrow) : nullptr;
    ra.bad_part = used + kCutLaunches;
    ra.overflow = flag_d;
    ra.gscratch = wr + o_g;
    ra.gcap = p->rw_gcap;
    ra.stage_col = reinterpret_cast<int32_t *>(wr + o_sc);
    ra.stage_w = reinterpret_cast<double *>(wr + o_sw);
    ra.dbg = debug_mask();
    {
        Prof pf(P_NUMERIC, s);
        Prof pk(P_KERNEL, s);
        launch_row_win(ra, s);
        check_launch("row-window numeric");
    }
    if (cut) {
        Prof pf(P_CUTSIZE, s);
        launch_rowcut_partials(ra.cutrow, p->nloc, cutp, used, s);
        launch_cut_final(cutp, used, 1, kCutSlotsPerLaunch, ra.bad_part, cut->cut_dev, s);
        check_launch("cut_final");
    }
    HostStage *hs = host_stage();
    CK(cudaMemcpyAsync(&hs->holes, flag_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs->v[0], row_ptr_out + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (p->early) CK(cudaMemcpyAsync(&hs->ctr.err, &p->ctr->err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (p->early && hs->ctr.err) throw Error(err_to_code(hs->ctr.err), err_msg(err_to_code(hs->ctr.err)));
    if (hs->holes & 2) throw Error(RIG_ERR_CUDA, "row-window far list capacity exceeded");
    if (hs->holes & 1) throw NeedCapacity{hs->v[0]};
    return hs->v[0];
}

static int64_t plan_numeric(rig_plan *p, int32_t *gcol, double *gw, double *diag, int64_t *row_ptr_out,
                            Arena &tmp_arena, const CutReq *cut, int64_t cap = INT64_MAX) {
    cudaStream_t s = p->s;
    // zeroed: holes flag, fused-cut used counts + bad flag
    Layout L;
    const size_t o_holes = L.add(sizeof(int));
    const size_t o_used = L.add(sizeof(int) * (kCutLaunches + 1));
    const size_t zero_bytes = L.bytes;
    const size_t o_cutp = cut ? L.add(sizeof(double) * (size_t)kCutLaunches * kCutSlotsPerLaunch) : 0;
    const size_t o_st = L.add(scan_tmp_bytes(p->nloc));
    unsigned char *wn = p->cached ? ws_get(2, L.bytes, s) : tmp_arena.raw(L.bytes);
    CK(cudaMemsetAsync(wn, 0, zero_bytes, s));
    int *holes_d = reinterpret_cast<int *>(wn + o_holes);
    int *used = reinterpret_cast<int *>(wn + o_used);
    int *badp = used + kCutLaunches;
    double *cutp = cut ? reinterpret_cast<double *>(wn + o_cutp) : nullptr;
    double *dg = (p->flags & RIG_FLAG_DIAG) ? diag : nullptr;
    const int64_t n_mid = p->h.n_mid;
    // a7's partition ids range-checked once (the fused kernels gather part[j]
    // unchecked); an id outside [0, K) makes the cut NaN (launch_cut_final)
    if (cut) launch_part_check(cut->part, p->A.nrows, cut->K, badp, s);
    if (p->rowwin) {
        t_last_path = "rowwin";
        return rowwin_numeric(p, gcol, gw, cap, dg, row_ptr_out, wn, holes_d, used, cutp, cut);
    }
    t_last_path = n_mid > 0 ? "mixed" : "merge";
    {
        Prof pf(P_NUMERIC, s);
        if (n_mid > 0) {
            MidArgs ma{p->A,     p->T,     p->rb,  p->lists, p->ctr->list_count, p->toff, p->tcol, p->tw,
                       p->nnzc,  p->defer, p->ctr->defer_count, dg, p->tol, debug_mask()};
            if (p->mid_rowwin) {
                // mid rows (f_i <= 2048): k_row_win in temp mode, nothing deferred;
                // huge rows: wide window -> global far list -> CTA per row
                // header: row-window ticket, CTA ticket, long-row count, rest count
                auto *ticket = reinterpret_cast<unsigned long long *>(p->mid_rw_scratch);
                CK(cudaMemsetAsync(ticket, 0, 256, s));
                int64_t *long_count = reinterpret_cast<int64_t *>(ticket + 2);
                int64_t *rest_count = reinterpret_cast<int64_t *>(ticket + 3);
                int32_t *long_list = p->defer;           // rows left by the row-window kernel
                int32_t *rest_list = p->defer + n_mid;   // rows beyond the CTA kernel's shared arrays
                RowArgs ra{};
                ra.A = p->A;
                ra.T = p->T;
                ra.rb = p->rb;
                ra.nloc = p->nloc;
                ra.ticket = ticket;
                ra.diag = dg;
                ra.tol = p->tol;
                ra.gscratch = static_cast<unsigned char *>(p->mid_rw_scratch) + 256;
                ra.gcap = p->rw_gcap;
                ra.overflow = holes_d + 0;  // bit 1 only (capacity bug); read with the holes flag
                ra.list = p->lists;
                ra.count_dev = p->ctr->list_count;
                ra.toff = p->toff;
                ra.tcol = p->tcol;
                ra.tw = p->tw;
                ra.cnt = p->nnzc;
                ra.dbg = debug_mask();
                ra.fnm = p->fnm;
                ra.fskip = kRowCtaMinF;
                ra.fskip_list = long_list;
                ra.fskip_count = long_count;
                {
                    Prof pk(P_KERNEL, s);
                    launch_row_win(ra, s);
                }
                check_launch("mid rows (row-window, temp mode)");
                // long rows of scattered columns (f_i > kRowCtaMinF, mid and huge
                // bins): CTA per row in shared memory; beyond its arrays, the chain
                RcArgs rc{};
                rc.A = p->A;
                rc.T = p->T;
                rc.rb = p->rb;
                rc.list0 = long_list;
                rc.count0 = long_count;
                rc.list1 = p->lists + n_mid;
                rc.count1 = p->ctr->list_count + 1;
                rc.rest = rest_list;
                rc.rest_count = rest_count;
                rc.ticket = ticket + 1;
                rc.fnm = p->fnm;
                rc.toff = p->toff;
                rc.tcol = p->tcol;
                rc.tw = p->tw;
                rc.cnt = p->nnzc;
                rc.diag = dg;
                rc.tol = p->tol;
                rc.fmax = (int)std::min<int64_t>(std::max<int64_t>(p->h.max_f, 1), kRowCtaMaxF);
                rc.ticket2 = kRowCtaBigF0 > 0 ? ticket + 7 : nullptr;  // longest rows first
                rc.bigf = kRowCtaBigF0;
                launch_row_cta(rc, s);
                check_launch("long rows (CTA per row)");
                // the rest: a wide-window pass (|j - i| < 2048: banded / FEM
                // rows) ...
                MidArgs wd = ma;
                wd.defer_list = p->defer + 2 * n_mid;
                wd.defer_count = p->ctr->defer_count + 2;
                wd.list = rest_list;
                wd.count = rest_count;
                launch_num_mid_wide(wd, s);
                check_launch("long rows (wide window)");
                // ... then key ranges through the CTA kernel's larger arrays
                int32_t *last_list = p->defer + 2 * n_mid;
                int64_t *last_count = p->ctr->defer_count + 2;
                if (p->long_scratch) {
                    RcArgs rl = rc;
                    rl.list0 = last_list;
                    rl.count0 = last_count;
                    rl.list1 = nullptr;
                    rl.count1 = nullptr;
                    last_list = p->defer + 4 * n_mid;
                    last_count = reinterpret_cast<int64_t *>(ticket + 5);
                    rl.rest = last_list;
                    rl.rest_count = last_count;
                    rl.ticket = ticket + 4;
                    rl.ticket2 = ticket + 6;  // rows beyond kRowCtaBigF1 products first
                    rl.bigf = kRowCtaBigF1;
                    rl.fmax = rowcta_range_fmax();
                    rl.skey = static_cast<int32_t *>(p->long_scratch);
                    rl.sval = reinterpret_cast<double *>(rl.skey + (size_t)2 * p->long_scap * p->long_grid);
                    rl.scap = p->long_scap;
                    launch_row_cta(rl, s);
                    check_launch("long rows (CTA per row, key ranges)");
                }
                // rows left (beyond the scratch slices or a crowded key bucket):
                // global far lists, then the CTA accumulator kernel, with their
                // scratch allocated now
                HostStage *hs = host_stage();
                CK(cudaMemcpyAsync(&hs->v[1], last_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                const int64_t n_last = hs->v[1];
                if (n_last > 0) {
                    const int64_t n = p->A.nrows;
                    MidArgs hu = ma;
                    hu.list = last_list;
                    hu.count = last_count;
                    if (p->h.max_f > kMidBigFarCapHost) {
                        MidArgs gf = ma;
                        gf.list = last_list;
                        gf.count = last_count;
                        gf.defer_list = p->defer + 3 * n_mid;
                        gf.defer_count = p->ctr->defer_count + 3;
                        gf.fscratch = tmp_arena.raw(mid_gfar_scratch_bytes());
                        gf.fscratch_bytes = (int64_t)mid_gfar_scratch_bytes();
                        gf.fnm = p->fnm;
                        launch_num_mid_gfar(gf, s);
                        check_launch("long rows (global far lists)");
                        hu.list = p->defer + 3 * n_mid;
                        hu.count = p->ctr->defer_count + 3;
                    }
                    p->huge_slots_n = huge_slots_rw(n, n_last, kHugePerSmRw);
                    p->huge_scratch = tmp_arena.raw(huge_scratch_bytes(n, p->huge_slots_n, true));
                    CK(cudaMemsetAsync(p->huge_scratch, 0, huge_bitmap_bytes(n, p->huge_slots_n), s));
                    launch_num_huge(hu, p->huge_slots_n, p->huge_scratch, s);
                    check_launch("huge rows");
                }
            } else {
            {
                Prof pk(P_KERNEL, s);
                launch_num_mid(ma, kMidSmallCap, s);
            }
            check_launch("mid rows");
            if (p->huge_scratch) {
                MidArgs hu = ma;
                // rows whose far list overflowed: a pass with a 1024-item far
                // list (long rows of random columns); then the rows beyond the
                // mid bins and what that pass deferred: a wide-window pass
                // (|j - i| < 2048: banded / FEM rows); the huge kernel takes
                // what remains
                MidArgs bg = ma;
                bg.list = p->defer;
                bg.count = p->ctr->defer_count;
                bg.defer_list = p->defer + n_mid;
                bg.defer_count = p->ctr->defer_count + 1;
                launch_num_mid_big(bg, s);
                check_launch("deferred rows (long far lists)");
                MidArgs wd = ma;
                wd.defer_list = p->defer + 2 * n_mid;
                wd.defer_count = p->ctr->defer_count + 2;
                wd.list = p->lists + n_mid;  // f_i beyond the mid bins
                wd.count = p->ctr->list_count + 1;
                launch_num_mid_wide(wd, s);
                wd.list = p->defer + n_mid;
                wd.count = p->ctr->defer_count + 1;
                launch_num_mid_wide(wd, s);
                check_launch("huge and deferred rows (wide window)");
                hu.list = p->defer + 2 * n_mid;
                hu.count = p->ctr->defer_count + 2;
                if (p->gfar) {  // far lists up to 4096 items in global scratch
                    MidArgs gf = ma;
                    gf.list = p->defer + 2 * n_mid;
                    gf.count = p->ctr->defer_count + 2;
                    gf.defer_list = p->defer + 3 * n_mid;
                    gf.defer_count = p->ctr->defer_count + 3;
                    gf.fscratch = p->gfar;
                    gf.fscratch_bytes = (int64_t)mid_gfar_scratch_bytes();
                    gf.fnm = p->fnm;
                    launch_num_mid_gfar(gf, s);
                    check_launch("deferred rows (global far lists)");
                    hu.list = p->defer + 3 * n_mid;
                    hu.count = p->ctr->defer_count + 3;
                }
                launch_num_huge(hu, p->huge_slots_n, p->huge_scratch, s);
                check_launch("deferred rows");
            }
            }
        }
        {
            Prof pfs(P_UBSCAN, s);
            scan_i64(p->nnzc, p->nloc, row_ptr_out, ScanOp::UbOffDiag, wn + o_st, 0, s);
        }
        NumArgs na{p->A,
                   p->T,
                   p->rb,
                   p->re,
                   row_ptr_out,
                   gcol,
                   gw,
                   dg,
                   p->tol,
                   holes_d,
                   cut ? cut->part : nullptr,
                   cut ? cut->K : 0,
                   cutp,
                   badp,
                   used,
                   p->qs ? pair_stage_cap_for(p->h.products, p->nloc) : stage_cap_for(p->h.products, p->nloc),
                   p->qs};
        check_launch("graph row pointers");
        if (p->nloc > 0) {
            Prof pk(n_mid > 0 ? -1 : P_KERNEL, s);
            launch_num_merge(na, p->h.max_len, s);
        }
        check_launch("merge rows");
        if (n_mid > 0) {  // cut-partial segments: 0 merge rows, 1 mid rows, 2 huge rows
            auto co = [&](int g) {
                CutOut c{nullptr, 0, nullptr, nullptr, nullptr};
                if (cut) c = CutOut{cut->part, cut->K, cutp + (int64_t)g * kCutSlotsPerLaunch, badp, used + g};
                return c;
            };
            launch_copy_rows(p->lists, p->ctr->list_count, p->rb, p->toff, row_ptr_out, p->tcol, p->tw, gcol, gw,
                             co(1), s);
            if (p->huge_scratch || p->h.sym_count[kNumSymBins] > 0)  // the huge bin's rows
                launch_copy_rows(p->lists + n_mid, p->ctr->list_count + 1, p->rb, p->toff, row_ptr_out, p->tcol, p->tw,
                                 gcol, gw, co(2), s);
        }
        check_launch("numeric");
    }
    if (cut) {
        Prof pf(P_CUTSIZE, s);
        launch_cut_final(cutp, used, kCutLaunches, kCutSlotsPerLaunch, badp, cut->cut_dev, s);
        check_launch("cut_final");
    }
    HostStage *hs = host_stage();
    CK(cudaMemcpyAsync(&hs->holes, holes_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs->v[0], row_ptr_out + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (p->early) CK(cudaMemcpyAsync(&hs->ctr.err, &p->ctr->err, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (p->early && hs->ctr.err) throw Error(err_to_code(hs->ctr.err), err_msg(err_to_code(hs->ctr.err)));
    const int holes = hs->holes;
    const int64_t ub = hs->v[0];
    if (!holes) return ub;
    // holes (merge-row entries dropped by value): count kept entries per row,
    // scan, move into a temporary, copy back
    Prof pf_c(P_COMPACT, s);
    Layout LC;
    const size_t o_copy = LC.add(sizeof(int64_t) * (size_t)(p->nloc + 1));
    const size_t o_kept = LC.add(sizeof(int64_t) * (size_t)p->nloc);
    const size_t o_st2 = LC.add(scan_tmp_bytes(p->nloc));
    const size_t o_c2 = LC.add(sizeof(int32_t) * (size_t)ub);
    const size_t o_w2 = LC.add(sizeof(double) * (size_t)ub);
    unsigned char *wc = tmp_arena.raw(LC.bytes);
    int64_t *ubp = reinterpret_cast<int64_t *>(wc + o_copy);  // structural offsets
    CK(cudaMemcpyAsync(ubp, row_ptr_out, sizeof(int64_t) * (size_t)(p->nloc + 1), cudaMemcpyDeviceToDevice, s));
    int64_t *kept = reinterpret_cast<int64_t *>(wc + o_kept);
    int32_t *c2 = reinterpret_cast<int32_t *>(wc + o_c2);
    double *w2 = reinterpret_cast<double *>(wc + o_w2);
    launch_count_kept(ubp, p->nloc, gcol, kept, s);
    scan_i64(kept, p->nloc, row_ptr_out, ScanOp::Identity, wc + o_st2, 0, s);
    CK(cudaMemcpyAsync(&hs->v[1], row_ptr_out + p->nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    launch_compact_move(ubp, row_ptr_out, p->nloc, gcol, gw, c2, w2, s);
    check_launch("compact");
    CK(cudaStreamSynchronize(s));
    const int64_t g = hs->v[1];
    if (g > 0) {
        CK(cudaMemcpyAsync(gcol, c2, sizeof(int32_t) * (size_t)g, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(gw, w2, sizeof(double) * (size_t)g, cudaMemcpyDeviceToDevice, s));
    }
    return g;
}

static rig_plan *new_plan(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t rb,
                          int64_t re, cudaStream_t s) {
    check_csr(A);
    if (!(drop_tol >= 0.0) || std::isnan(drop_tol)) throw Error(RIG_ERR_INVALID, "drop_tol must be >= 0");
    if (rb < 0 || re > A->nrows || rb > re) throw Error(RIG_ERR_INVALID, "bad row range");
    ensure_pool();
    rig_plan *p = new rig_plan(s);
    p->scale = scale_rows ? 1 : 0;
    p->tol = drop_tol;
    p->flags = flags;
    p->rb = rb;
    p->re = re;
    p->nloc = re - rb;
    return p;
}

static rig_plan *make_plan(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t rb,
                           int64_t re, cudaStream_t s) {
    rig_plan *p = new_plan(A, scale_rows, drop_tol, flags, rb, re, s);
    try {
        plan_build(p, A);
    } catch (...) {
        delete p;
        throw;
    }
    return p;
}

#define ABI_BEGIN try {
#define ABI_END                                 \
    }                                           \
    catch (const Error &e) {                    \
        t_last_error = e.what();                \
        return e.code;                          \
    }                                           \
    catch (const std::exception &e) {           \
        t_last_error = e.what();                \
        return RIG_ERR_INVALID;                 \
    }                                           \
    catch (...) {                               \
        t_last_error = "unknown error";         \
        return RIG_ERR_INVALID;                 \
    }

static void free_owned(rig_graph_t *g, cudaStream_t s) {
    void *block = nullptr;
    bool found = false;
    {
        std::lock_guard<std::mutex> lk(g_own_mu);
        auto it = g_owned.find(g->row_ptr);
        if (it != g_owned.end()) {
            block = it->second;
            g_owned.erase(it);
            found = true;
        }
    }
    if (!found) throw Error(RIG_ERR_INVALID, "graph was not allocated by rig_build*");
    CK(cudaFreeAsync(g->row_ptr, s));
    if (block) CK(cudaFreeAsync(block, s));
    std::memset(g, 0, sizeof(*g));
}

// Library-owned output.  The (col, w, diag) block is sized from the bound
// sum (f_i - len_i) >= graph nnz (known at the first sync), so the numeric
// passes follow without another host round trip.
static void build_owned(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t rb, int64_t re,
                        rig_graph_t *out, cudaStream_t s, const CutReq *cut) {
    if (!out) throw Error(RIG_ERR_INVALID, "out is NULL");
    std::memset(out, 0, sizeof(*out));
    rig_plan *p = new_plan(A, scale_rows, drop_tol, flags, rb, re, s);
    p->cached = true;
    Arena tmp(s);
    int64_t *rp = nullptr;
    unsigned char *block = nullptr;
    int32_t *col = nullptr;
    double *w = nullptr, *diag = nullptr;
    try {
        CK(cudaMallocAsync((void **)&rp, sizeof(int64_t) * (size_t)(p->nloc + 1), s));
        plan_build(p, A, true);
        // capacity: the bound sum (f_i - len_i); on the row-window path a
        // fraction of it (stencil / banded rows keep ~half their products as
        // distinct keys), retried at the exact size if the rows outgrow it
        int64_t cap = std::max<int64_t>(p->nnz_upper, 1);
        if (p->rowwin) cap = std::min<int64_t>(cap, (int64_t)(0.6 * (double)p->nnz_upper) + 4096);
        int64_t g = 0;
        for (int attempt = 0;; ++attempt) {
            Layout L;
            const size_t o_col = L.add(sizeof(int32_t) * (size_t)cap);
            const size_t o_w = L.add(sizeof(double) * (size_t)cap);
            const size_t o_diag =
                (flags & RIG_FLAG_DIAG) ? L.add(sizeof(double) * (size_t)std::max<int64_t>(p->nloc, 1)) : 0;
            CK(cudaMallocAsync((void **)&block, L.bytes, s));
            col = reinterpret_cast<int32_t *>(block + o_col);
            w = reinterpret_cast<double *>(block + o_w);
            diag = (flags & RIG_FLAG_DIAG) ? reinterpret_cast<double *>(block + o_diag) : nullptr;
            try {
                g = plan_numeric(p, col, w, diag, rp, tmp, cut, cap);
                break;
            } catch (const NeedCapacity &nc) {
                if (attempt > 0) throw Error(RIG_ERR_CUDA, "graph capacity retry failed");
                CK(cudaFreeAsync(block, s));
                block = nullptr;
                cap = std::max<int64_t>(nc.nnz, 1);
            }
        }
        out->n = p->nloc;
        out->nnz = g;
        out->row_ptr = rp;
        out->col_idx = col;
        out->w = w;
        out->diag = diag;
        std::lock_guard<std::mutex> lk(g_own_mu);
        g_owned[rp] = block;
    } catch (...) {
        if (rp) cudaFreeAsync(rp, s);
        if (block) cudaFreeAsync(block, s);
        delete p;
        throw;
    }
    delete p;
}

extern "C" {

const char *rig_last_error(void) { return t_last_error.c_str(); }

int rig_profile_enable(int on) {
    // on: 0 = off, 1 = every pass, otherwise a bit mask (bit p = pass p) | 2^31
    const uint32_t u = (uint32_t)on;
    g_prof_mask.store(u == 1u ? 0xffffffffu : (u & 0x7fffffffu));
    return RIG_OK;
}

int rig_profile_read(double *ms, int64_t *count) {
    ABI_BEGIN
    std::vector<ProfRec> recs;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        recs.swap(g_recs);
    }
    for (int k = 0; k < RIG_NPASS; ++k) {
        if (ms) ms[k] = 0.0;
        if (count) count[k] = 0;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    for (auto &r : recs) {
        CK(cudaEventSynchronize(r.b));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, r.a, r.b));
        if (ms) ms[r.pass] += (double)t;
        if (count) count[r.pass] += 1;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_pool.push_back({dev, r.a});
        g_pool.push_back({dev, r.b});
    }
    return RIG_OK;
    ABI_END
}

const char *rig_pass_name(int pass) { return (pass >= 0 && pass < RIG_NPASS) ? kPassNames[pass] : "?"; }

int rig_trim(void) {
    ABI_BEGIN
    ws_trim();
    return RIG_OK;
    ABI_END
}
uint64_t rig_launch_count(void) { return g_launches.load(); }
const char *rig_version(void) { return "librig 0.3 (sm_100a)"; }
const char *rig_last_path(void) { return t_last_path.c_str(); }

int rig_mem_stats(uint64_t *used_now, uint64_t *used_high, int reset) {
    ABI_BEGIN
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    unsigned long long cur = 0, high = 0;  // cuuint64_t
    CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &cur));
    CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high));
    if (used_now) *used_now = (uint64_t)cur;
    if (used_high) *used_high = (uint64_t)high;
    if (reset) {
        unsigned long long zero = 0;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero));
    }
    return RIG_OK;
    ABI_END
}

int rig_gather_probe(const rig_csr_t *A, int scale_rows, double *checksum_host, rig_stream_t stream) {
    ABI_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    rig_plan *p = make_plan(A, scale_rows, 0.0, 0, 0, A->nrows, s);
    try {
        Arena ar(s);
        const int nw = gather_probe_warps();
        double *sink = ar.get<double>(nw);
        launch_gather_probe(p->A, p->T, 0, A->nrows, sink, s);
        check_launch("gather probe");
        std::vector<double> h((size_t)nw);
        CK(cudaMemcpyAsync(h.data(), sink, sizeof(double) * (size_t)nw, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double t = 0.0;
        for (double v : h) t += v;
        if (checksum_host) *checksum_host = t;
    } catch (...) {
        delete p;
        throw;
    }
    delete p;
    return RIG_OK;
    ABI_END
}

int rig_build(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, rig_graph_t *out,
              rig_stream_t stream) {
    ABI_BEGIN
    check_csr(A);
    build_owned(A, scale_rows, drop_tol, flags, 0, A->nrows, out, (cudaStream_t)stream, nullptr);
    return RIG_OK;
    ABI_END
}

int rig_build_rows(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t row_begin,
                   int64_t row_end, rig_graph_t *out, rig_stream_t stream) {
    ABI_BEGIN
    build_owned(A, scale_rows, drop_tol, flags, row_begin, row_end, out, (cudaStream_t)stream, nullptr);
    return RIG_OK;
    ABI_END
}

int rig_build_cut(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t row_begin,
                  int64_t row_end, const int32_t *part, int32_t K, rig_graph_t *out, double *cut_dev,
                  rig_stream_t stream) {
    ABI_BEGIN
    check_csr(A);
    if (!part || !cut_dev) throw Error(RIG_ERR_INVALID, "part/cut_dev is NULL");
    if (K < 1) throw Error(RIG_ERR_INVALID, "K < 1");
    CutReq cr;
    cr.part = part;
    cr.K = K;
    cr.cut_dev = cut_dev;
    build_owned(A, scale_rows, drop_tol, flags, row_begin, row_end, out, (cudaStream_t)stream, &cr);
    return RIG_OK;
    ABI_END
}

int rig_graph_free(rig_graph_t *g, rig_stream_t stream) {
    ABI_BEGIN
    if (!g) throw Error(RIG_ERR_INVALID, "g is NULL");
    if (!g->row_ptr) {
        std::memset(g, 0, sizeof(*g));
        return RIG_OK;
    }
    free_owned(g, (cudaStream_t)stream);
    return RIG_OK;
    ABI_END
}

int rig_plan_create(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t row_begin,
                    int64_t row_end, rig_plan_t **plan, rig_stream_t stream) {
    ABI_BEGIN
    if (!plan) throw Error(RIG_ERR_INVALID, "plan is NULL");
    *plan = make_plan(A, scale_rows, drop_tol, flags, row_begin, row_end, (cudaStream_t)stream);
    return RIG_OK;
    ABI_END
}

int rig_plan_query(const rig_plan_t *plan, int64_t *nnz_upper, int64_t *products, size_t *workspace_bytes) {
    ABI_BEGIN
    if (!plan) throw Error(RIG_ERR_INVALID, "plan is NULL");
    if (nnz_upper) *nnz_upper = plan->nnz_upper;
    if (products) *products = plan->h.products;
    if (workspace_bytes) *workspace_bytes = 0;  // temporaries are stream-ordered pool allocations
    return RIG_OK;
    ABI_END
}

int rig_plan_execute(rig_plan_t *plan, void *workspace, rig_graph_t *out, rig_stream_t stream) {
    ABI_BEGIN
    (void)workspace;
    if (!plan || !out) throw Error(RIG_ERR_INVALID, "plan/out is NULL");
    if (!out->row_ptr || ((!out->col_idx || !out->w) && plan->nnz_upper > 0))
        throw Error(RIG_ERR_INVALID, "output arrays are NULL");
    if ((plan->flags & RIG_FLAG_DIAG) && !out->diag && plan->nloc > 0)
        throw Error(RIG_ERR_INVALID, "RIG_FLAG_DIAG needs out->diag");
    plan->s = (cudaStream_t)stream;
    Arena tmp(plan->s);
    const int64_t g = plan_numeric(plan, out->col_idx, out->w, out->diag, out->row_ptr, tmp, nullptr, plan->nnz_upper);
    out->n = plan->nloc;
    out->nnz = g;
    return RIG_OK;
    ABI_END
}

int rig_plan_destroy(rig_plan_t *plan) {
    ABI_BEGIN
    delete plan;
    return RIG_OK;
    ABI_END
}

int rig_row_split(const rig_csr_t *A, int32_t parts, int64_t *split, rig_stream_t stream) {
    ABI_BEGIN
    check_csr(A);
    if (parts < 1 || !split) throw Error(RIG_ERR_INVALID, "parts < 1 or split NULL");
    ensure_pool();
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar(s);
    const int64_t n = A->nrows, m = A->ncols;
    Csr A0{n, m, A->nnz, A->row_ptr, A->col_idx, A->val};
    Layout L;
    const size_t o_ctr = L.add(sizeof(DevCounters));
    const size_t o_cnt = L.add(sizeof(unsigned) * (size_t)m);
    const size_t o_st1 = L.add(scan_tmp_bytes(m));
    const size_t o_st2 = L.add(scan_tmp_bytes(n));
    const size_t zero_bytes = L.bytes;
    const size_t o_cp = L.add(sizeof(int64_t) * (size_t)(m + 1));
    const size_t o_f = L.add(sizeof(int64_t) * (size_t)n);
    const size_t o_fp = L.add(sizeof(int64_t) * (size_t)(n + 1));
    const size_t o_sp = L.add(sizeof(int64_t) * (size_t)(parts + 1));
    unsigned char *ws = ar.raw(L.bytes);
    CK(cudaMemsetAsync(ws, 0, zero_bytes, s));
    DevCounters *ctr = reinterpret_cast<DevCounters *>(ws + o_ctr);
    unsigned *cnt = reinterpret_cast<unsigned *>(ws + o_cnt);
    int64_t *cp = reinterpret_cast<int64_t *>(ws + o_cp);
    int64_t *f = reinterpret_cast<int64_t *>(ws + o_f);
    int64_t *fp = reinterpret_cast<int64_t *>(ws + o_fp);
    int64_t *sp = reinterpret_cast<int64_t *>(ws + o_sp);
    Prof pf(P_SPLIT, s);
    if (A->nnz > 0) launch_col_hist(A0, cnt, nullptr, s);
    scan_u32(cnt, m, cp, ws + o_st1, 0, s);
    if (n > 0) launch_analyze(A0, cp, 0, n, f, ctr, s);
    scan_i64(f, n, fp, ScanOp::Identity, ws + o_st2, 0, s);
    launch_split(fp, n, parts, sp, s);
    check_launch("split");
    CK(cudaMemcpyAsync(split, sp, sizeof(int64_t) * (size_t)(parts + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return RIG_OK;
    ABI_END
}

int rig_sparsify(const rig_csr_t *A, int scale_rows, uint32_t flags, rig_csr_t *out, rig_stream_t stream) {
    ABI_BEGIN
    if (!out) throw Error(RIG_ERR_INVALID, "out is NULL");
    std::memset(out, 0, sizeof(*out));
    cudaStream_t s = (cudaStream_t)stream;
    rig_plan *p = new_plan(A, scale_rows, 0.0, (flags & RIG_FLAG_VALIDATE) | RIG_FLAG_SPARSIFY, 0, 0, s);
    p->cached = true;
    unsigned char *block = nullptr;
    try {
        plan_build(p, A);
        const Csr &At = p->A;
        Layout L;
        const size_t o_rp = L.add(sizeof(int64_t) * (size_t)(At.nrows + 1));
        const size_t o_ci = L.add(sizeof(int32_t) * (size_t)At.nnz);
        const size_t o_v = L.add(sizeof(double) * (size_t)At.nnz);
        CK(cudaMallocAsync((void **)&block, L.bytes, s));
        CK(cudaMemcpyAsync(block + o_rp, At.rp, sizeof(int64_t) * (size_t)(At.nrows + 1), cudaMemcpyDeviceToDevice, s));
        if (At.nnz > 0) {
            CK(cudaMemcpyAsync(block + o_ci, At.ci, sizeof(int32_t) * (size_t)At.nnz, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(block + o_v, At.v, sizeof(double) * (size_t)At.nnz, cudaMemcpyDeviceToDevice, s));
        }
        out->nrows = At.nrows;
        out->ncols = At.ncols;
        out->nnz = At.nnz;
        out->row_ptr = reinterpret_cast<const int64_t *>(block + o_rp);
        out->col_idx = reinterpret_cast<const int32_t *>(block + o_ci);
        out->val = reinterpret_cast<const double *>(block + o_v);
        std::lock_guard<std::mutex> lk(g_own_mu);
        g_owned[block] = nullptr;
    } catch (...) {
        if (block) cudaFreeAsync(block, s);
        delete p;
        throw;
    }
    delete p;
    return RIG_OK;
    ABI_END
}

int rig_csr_free(rig_csr_t *A, rig_stream_t stream) {
    ABI_BEGIN
    if (!A) throw Error(RIG_ERR_INVALID, "NULL argument");
    if (!A->row_ptr) return RIG_OK;
    void *key = const_cast<int64_t *>(A->row_ptr);
    {
        std::lock_guard<std::mutex> lk(g_own_mu);
        auto it = g_owned.find(key);
        if (it == g_owned.end() || it->second != nullptr) throw Error(RIG_ERR_INVALID, "matrix was not allocated by rig_sparsify");
        g_owned.erase(it);
    }
    CK(cudaFreeAsync(key, (cudaStream_t)stream));
    std::memset(A, 0, sizeof(*A));
    return RIG_OK;
    ABI_END
}

int rig_hem_match(const int64_t *row_ptr, const int32_t *col, const int64_t *wgt, int64_t n, int32_t rounds,
                  int32_t *match, rig_stream_t stream) {
    ABI_BEGIN
    if (n < 0 || rounds < 0 || (n > 0 && (!row_ptr || !col || !wgt || !match)))
        throw Error(RIG_ERR_INVALID, "NULL argument, n < 0 or rounds < 0");
    if (n == 0) return RIG_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar(s);
    int32_t *cand = ar.get<int32_t>(n);
    CK(cudaMemsetAsync(match, 0xff, sizeof(int32_t) * (size_t)n, s));  // -1: unmatched
    for (int r = 0; r < rounds; ++r) launch_hem_round(row_ptr, col, wgt, n, match, cand, s);
    check_launch("hem_match");
    return RIG_OK;
    ABI_END
}

int rig_coarsen(const int64_t *row_ptr, const int32_t *col, const int64_t *wgt, const int64_t *vwgt, int64_t n,
                const int32_t *match, rig_coarse_t *out, rig_stream_t stream) {
    ABI_BEGIN
    if (!out || n < 0 || (n > 0 && (!row_ptr || !col || !wgt || !match))) throw Error(RIG_ERR_INVALID, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    if (n == 0) return RIG_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar(s);
    int64_t *flag = ar.get<int64_t>(n);
    int64_t *cid = ar.get<int64_t>(n + 1);
    void *st = ar.raw(scan_tmp_bytes(n));
    int32_t *lead = ar.get<int32_t>(n);
    int64_t *cvw_tmp = ar.get<int64_t>(n);
    int64_t *citems = ar.get<int64_t>(n);
    unsigned long long *maxit = ar.get<unsigned long long>(1);
    CK(cudaMemsetAsync(maxit, 0, sizeof(unsigned long long), s));
    unsigned char *block = nullptr;
    try {
        // cmap lives in the output block; allocate it with the vertex arrays once nc is known
        int32_t *cmap_tmp = ar.get<int32_t>(n);
        launch_leader_flags(match, n, flag, s);
        scan_i64(flag, n, cid, ScanOp::Identity, st, 0, s);
        launch_coarse_map(row_ptr, match, vwgt, n, cid, cmap_tmp, lead, cvw_tmp, citems, maxit, s);
        check_launch("coarse map");
        HostStage *hs = host_stage();
        CK(cudaMemcpyAsync(&hs->v[0], cid + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&hs->v[1], maxit, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int64_t nc = hs->v[0], maxitems = hs->v[1];
        int64_t *ccnt = ar.get<int64_t>(nc);
        int64_t *crp_tmp = ar.get<int64_t>(nc + 1);
        int64_t *toff = ar.get<int64_t>(nc + 1);
        void *st2 = ar.raw(scan_tmp_bytes(nc));
        // coarse rows beyond 1024 items: per-warp global scratch (keys + weights)
        int64_t gcap = 1;
        while (gcap < maxitems) gcap <<= 1;
        const int big_warps = maxitems > 1024 ? 4 * num_sms() : 0;
        uint64_t *gs = big_warps ? ar.get<uint64_t>((size_t)big_warps * 2 * (size_t)gcap) : nullptr;
        // one sorting pass: rows into a temporary at their item bounds, with counts
        scan_i64(citems, nc, toff, ScanOp::Identity, st2, 0, s);
        CK(cudaMemcpyAsync(&hs->v[2], toff + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int64_t tslots = std::max<int64_t>(hs->v[2], 1);
        int32_t *tcol = ar.get<int32_t>(tslots);
        int64_t *tw = ar.get<int64_t>(tslots);
        launch_coarse_rows(2, row_ptr, col, wgt, match, cmap_tmp, lead, nc, ccnt, toff, tcol, tw, gs, gcap, big_warps,
                           s);
        scan_i64(ccnt, nc, crp_tmp, ScanOp::Identity, st2, 0, s);
        check_launch("coarse rows");
        CK(cudaMemcpyAsync(&hs->v[0], crp_tmp + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int64_t cnnz = hs->v[0];
        Layout L;
        const size_t o_rp = L.add(sizeof(int64_t) * (size_t)(nc + 1));
        const size_t o_col = L.add(sizeof(int32_t) * (size_t)std::max<int64_t>(cnnz, 1));
        const size_t o_w = L.add(sizeof(int64_t) * (size_t)std::max<int64_t>(cnnz, 1));
        const size_t o_vw = L.add(sizeof(int64_t) * (size_t)nc);
        const size_t o_cm = L.add(sizeof(int32_t) * (size_t)n);
        CK(cudaMallocAsync((void **)&block, L.bytes, s));
        out->row_ptr = reinterpret_cast<int64_t *>(block + o_rp);
        out->col_idx = reinterpret_cast<int32_t *>(block + o_col);
        out->wgt = reinterpret_cast<int64_t *>(block + o_w);
        out->vwgt = reinterpret_cast<int64_t *>(block + o_vw);
        out->cmap = reinterpret_cast<int32_t *>(block + o_cm);
        CK(cudaMemcpyAsync(out->row_ptr, crp_tmp, sizeof(int64_t) * (size_t)(nc + 1), cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(out->vwgt, cvw_tmp, sizeof(int64_t) * (size_t)nc, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(out->cmap, cmap_tmp, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        launch_coarse_copy(toff, out->row_ptr, nc, tcol, tw, out->col_idx, out->wgt, s);
        check_launch("coarse rows");
        out->n = nc;
        out->nnz = cnnz;
        std::lock_guard<std::mutex> lk(g_own_mu);
        g_owned[block] = reinterpret_cast<void *>(1);  // tag: a coarse graph
    } catch (...) {
        if (block) cudaFreeAsync(block, s);
        std::memset(out, 0, sizeof(*out));
        throw;
    }
    return RIG_OK;
    ABI_END
}

int rig_coarse_free(rig_coarse_t *c, rig_stream_t stream) {
    ABI_BEGIN
    if (!c) throw Error(RIG_ERR_INVALID, "NULL argument");
    if (!c->row_ptr) return RIG_OK;
    void *key = c->row_ptr;
    {
        std::lock_guard<std::mutex> lk(g_own_mu);
        auto it = g_owned.find(key);
        if (it == g_owned.end() || it->second != reinterpret_cast<void *>(1))
            throw Error(RIG_ERR_INVALID, "graph was not allocated by rig_coarsen");
        g_owned.erase(it);
    }
    CK(cudaFreeAsync(key, (cudaStream_t)stream));
    std::memset(c, 0, sizeof(*c));
    return RIG_OK;
    ABI_END
}

int rig_int_weights(const double *w, int64_t n, int64_t alpha, int64_t *wgt, rig_stream_t stream) {
    ABI_BEGIN
    if (n < 0 || (n > 0 && (!w || !wgt))) throw Error(RIG_ERR_INVALID, "NULL argument or n < 0");
    if (alpha < 1 || alpha > ((int64_t)1 << 53)) throw Error(RIG_ERR_INVALID, "alpha outside [1, 2^53]");
    launch_int_weights(w, n, alpha, wgt, (cudaStream_t)stream);
    check_launch("int_weights");
    return RIG_OK;
    ABI_END
}

int rig_cutsize(const rig_graph_t *g, int64_t row_begin, int64_t n_global, const int32_t *part, int32_t K,
                double *cut_dev, rig_stream_t stream) {
    ABI_BEGIN
    if (!g || !part || !cut_dev) throw Error(RIG_ERR_INVALID, "NULL argument");
    if (K < 1 || n_global < 0 || row_begin < 0 || row_begin + g->n > n_global)
        throw Error(RIG_ERR_INVALID, "bad K / row range");
    if (!g->row_ptr || (g->nnz > 0 && (!g->col_idx || !g->w))) throw Error(RIG_ERR_INVALID, "graph arrays NULL");
    ensure_pool();
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar(s);
    const int nb = cutsize_blocks();
    double *partials = ar.get<double>(nb + 1);
    Prof pf(P_CUTSIZE, s);
    launch_cutsize(g->row_ptr, g->col_idx, g->w, g->n, row_begin, n_global, part, K, partials, nb, cut_dev, s);
    check_launch("cutsize");
    return RIG_OK;
    ABI_END
}

int rig_partition_ip(const rig_graph_t *g, int64_t row_begin, int64_t n_global, const int32_t *part, int32_t K,
                     const int64_t *a_row_ptr, int64_t *acc, int64_t *W, rig_stream_t stream) {
    ABI_BEGIN
    if (!g || !part || !acc || !W) throw Error(RIG_ERR_INVALID, "NULL argument");
    if (K < 1 || K > 65536 || n_global < 0 || row_begin < 0 || row_begin + g->n > n_global)
        throw Error(RIG_ERR_INVALID, "bad K / row range");
    if (!g->row_ptr || (g->nnz > 0 && (!g->col_idx || !g->w))) throw Error(RIG_ERR_INVALID, "graph arrays NULL");
    cudaStream_t s = (cudaStream_t)stream;
    Prof pf(P_CUTSIZE, s);
    unsigned long long *a = reinterpret_cast<unsigned long long *>(acc);
    launch_partition_ip(g->row_ptr, g->col_idx, g->w, g->n, row_begin, n_global, part, K, a_row_ptr, a,
                        reinterpret_cast<unsigned long long *>(W), reinterpret_cast<int *>(a + 4 * (int64_t)K * K), s);
    check_launch("partition_ip");
    return RIG_OK;
    ABI_END
}

int rig_partition_ip_finalize(const int64_t *acc_host, int32_t K, double *ip_host) {
    ABI_BEGIN
    if (!acc_host || !ip_host || K < 1) throw Error(RIG_ERR_INVALID, "NULL argument or K < 1");
    const int64_t cells = (int64_t)K * K;
    if (acc_host[4 * cells]) throw Error(RIG_ERR_INVALID, "part id outside [0, K) or weight outside [0, 2^63)");
    for (int64_t c = 0; c < cells; ++c) {
        const uint64_t *l = reinterpret_cast<const uint64_t *>(acc_host + 4 * c);
        // value * 2^64 = l3 2^96 + l2 2^64 + l1 2^32 + l0 (each limb sum < 2^63)
        const unsigned __int128 lo = ((unsigned __int128)l[1] << 32) + l[0];
        const unsigned __int128 hi = ((unsigned __int128)l[3] << 32) + l[2];  // integer part - carry
        const unsigned __int128 ip = hi + (lo >> 64);
        const uint64_t fr = (uint64_t)lo;
        if ((ip >> 63) == 0) {  // fits 127 bits: one correctly rounded conversion
            const unsigned __int128 v = (ip << 64) | fr;
            ip_host[c] = std::ldexp((double)v, -64);
        } else {
            ip_host[c] = (double)ip + std::ldexp((double)fr, -64);
        }
    }
    return RIG_OK;
    ABI_END
}

int rig_build_host(const rig_csr_t *Ah, int scale_rows, double drop_tol, uint32_t flags, const int32_t *part_host,
                   int32_t K, rig_graph_t *out_host, int64_t capacity, double *cut_host, rig_stream_t stream) {
    ABI_BEGIN
    check_csr(Ah);
    if (!out_host || !out_host->row_ptr) throw Error(RIG_ERR_INVALID, "out_host arrays are NULL");
    if (part_host && K < 1) throw Error(RIG_ERR_INVALID, "K < 1");
    ensure_pool();
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar(s);
    const int64_t n = Ah->nrows, nnz = Ah->nnz;
    Layout L;
    const size_t o_rp = L.add(sizeof(int64_t) * (size_t)(n + 1));
    const size_t o_ci = L.add(sizeof(int32_t) * (size_t)nnz);
    const size_t o_v = L.add(sizeof(double) * (size_t)nnz);
    const size_t o_part = L.add(sizeof(int32_t) * (size_t)n);
    const size_t o_cut = L.add(sizeof(double));
    unsigned char *ws = ar.raw(L.bytes);
    int64_t *rp = reinterpret_cast<int64_t *>(ws + o_rp);
    int32_t *ci = reinterpret_cast<int32_t *>(ws + o_ci);
    double *v = reinterpret_cast<double *>(ws + o_v);
    int32_t *part = part_host ? reinterpret_cast<int32_t *>(ws + o_part) : nullptr;
    double *cut_dev = reinterpret_cast<double *>(ws + o_cut);
    CK(cudaMemcpyAsync(rp, Ah->row_ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
        CK(cudaMemcpyAsync(ci, Ah->col_idx, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(v, Ah->val, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice, s));
    }
    if (part) CK(cudaMemcpyAsync(part, part_host, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, s));
    rig_csr_t Ad{n, Ah->ncols, nnz, rp, ci, v};
    rig_graph_t g{};
    CutReq cr;
    cr.part = part;
    cr.K = K;
    cr.cut_dev = cut_dev;
    build_owned(&Ad, scale_rows, drop_tol, flags, 0, n, &g, s, part ? &cr : nullptr);
    struct Guard {
        rig_graph_t *g;
        cudaStream_t s;
        ~Guard() {
            try {
                free_owned(g, s);
            } catch (...) {
            }
        }
    } guard{&g, s};
    if (g.nnz > capacity) {
        out_host->nnz = g.nnz;
        throw Error(RIG_ERR_INVALID, "capacity too small for the graph");
    }
    CK(cudaMemcpyAsync(out_host->row_ptr, g.row_ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyDeviceToHost, s));
    if (g.nnz > 0) {
        if (!out_host->col_idx || !out_host->w) throw Error(RIG_ERR_INVALID, "out_host col/w NULL");
        CK(cudaMemcpyAsync(out_host->col_idx, g.col_idx, sizeof(int32_t) * (size_t)g.nnz, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(out_host->w, g.w, sizeof(double) * (size_t)g.nnz, cudaMemcpyDeviceToHost, s));
    }
    if ((flags & RIG_FLAG_DIAG) && out_host->diag && n > 0)
        CK(cudaMemcpyAsync(out_host->diag, g.diag, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, s));
    HostStage *hs = host_stage();
    if (part) CK(cudaMemcpyAsync(&hs->v[2], cut_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double cut = std::nan("");
    if (part) std::memcpy(&cut, &hs->v[2], sizeof(double));
    if (cut_host) *cut_host = cut;
    out_host->n = n;
    out_host->nnz = g.nnz;
    return RIG_OK;
    ABI_END
}

}  // extern "C"

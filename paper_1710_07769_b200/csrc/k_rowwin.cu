// k_rowwin.cu -- steps a5 + a6 (+ the fused a7 partial) for shards whose rows
// are all off the merge path (banded / FEM-like rows of many entries, e.g.
// BASELINE configs[4]): one warp per row of C = A_hat A_hat^T (Gustavson,
// PAPER.md:560-562), every row placed straight into the graph.  There is no
// symbolic pass and no graph-sized temporary: a row's kept count is
// published as soon as it is known, and its graph offset comes from a
// decoupled look-back over the counts of the rows before it.  Rows are handed
// out in order by a ticket counter.  So that a warp never idles waiting for
// slower rows in flight, a finished row goes to a small per-warp staging
// slot (L2-resident) and is copied to its offset after the warp has computed
// its NEXT row -- by then the rows before it have published their counts.
//
// Per row i (ordering contract, DESIGN.md §3 R4: every c_ij is the fma chain
// over the shared columns k in ascending k, from +0.0):
//  * units: the row's entries k ascending, each column cut into 32-row chunks
//    (keys inside one column are distinct, so a unit has no conflicts); a
//    per-row table in shared memory holds each unit's CSC offset, lane count
//    and a_ik.  The (j, a_jk) gathers run kRwDepth units ahead.
//  * near keys -kRwWH <= j - i < kRwWH accumulate in a direct-mapped shared window
//    wv[j - i + kRwWH] (+0.0 initially; a slot never touched stays +0.0 and is
//    never kept, since kept means |c| > drop_tol >= 0).  Invalid lanes of a
//    unit carry j = -1, b = 0: never far, and near only on the slot of key
//    -1, which no real key uses and which stays +0.0.
//  * far keys are appended (key << 6 | unit, a_jk) to a far list in arrival
//    (= ascending k) order; the packed words are unique and ordered by (key,
//    arrival), so sorting them is the stable key sort: value buckets filled
//    in arrival order; each lane then insertion-sorts its own short buckets,
//    and the warp ranks the rare long bucket found out of order.  Equal keys
//    are folded in arrival order.
//  * one pass folds, counts (kept: j != i and |c| > tol, PAPER.md:295-315,
//    352) and writes the row in ascending j (far-below, window, far-above)
//    to the warp's staging slot; the count is published, and the row is
//    copied to its offset after the warp's next row; the row's cut edges (j
//    > i, part[i] != part[j]) go to per-lane sums there,
//    reduced in fixed trees (deterministic).
//  * rows of more than 32 entries or more than kRwTcap units, and rows whose
//    far list outgrows the shared one, run with their far list in a per-warp
//    slice of global scratch (capacity >= the largest f_i, host-checked).
#include "common.cuh"

namespace rig {

constexpr int kRwThreads = 128;
constexpr int kRwWarps = kRwThreads / 32;
#ifndef RIG_RW_WH
#define RIG_RW_WH 112
#endif
constexpr int kRwWH = RIG_RW_WH;     // window: -kRwWH <= j - i < kRwWH
constexpr int kRwW = 2 * kRwWH;      // window slots
#ifndef RIG_RW_FCAP
#define RIG_RW_FCAP 192
#endif
constexpr int kRwFcap = RIG_RW_FCAP; // far items in shared memory
#ifndef RIG_RW_NB
#define RIG_RW_NB 128
#endif
constexpr int kRwNB = RIG_RW_NB;     // sort buckets (shared mode)
constexpr int kRwGNB = 512;          // sort buckets (global mode)
#ifndef RIG_RW_TCAP
#define RIG_RW_TCAP 40
#endif
constexpr int kRwTcap = RIG_RW_TCAP; // units per table fill
#ifndef RIG_RW_SMALLB
#define RIG_RW_SMALLB 8
#endif
constexpr int kRwSmallBucket = RIG_RW_SMALLB;  // buckets up to this size: per-lane insertion sort
constexpr int kRwStageCap = 512;     // entries per staging slot (>= kRwFcap + kRwW); slots are 128-byte aligned
#ifndef RIG_RW_DISCARD
#define RIG_RW_DISCARD 1
#endif
#ifndef RIG_RW_DEPTH
#define RIG_RW_DEPTH 3  // fits the 56-register budget of 9 CTAs per SM
#endif
constexpr int kRwDepth = RIG_RW_DEPTH;  // units in flight
// shared far items: the unit (< 2^kFarPack table slots) packed under the key
constexpr int kFarPack = 6;
static_assert(kRwTcap + 2 * kRwDepth <= (1 << kFarPack), "unit ids must fit kFarPack bits");
constexpr int64_t kRowWinMaxRows = int64_t{1} << (31 - kFarPack);  // packed keys fit int32

struct RwSmem {
    double wv[kRwW];      // window (every access is guarded by t < kRwW)
    double fb[kRwFcap];   // far: a_jk; after the count pass, at a group's head item: |c| (or -1: not kept)
    // units: padded up to a multiple of kRwDepth, plus kRwDepth look-ahead slots
    double ta[kRwTcap + 2 * kRwDepth];  // unit: a_ik
    int2 tcs[kRwTcap + 2 * kRwDepth];   // unit: (CSC offset of its first lane, lane count); tmp of the bucket rank
    int fk[kRwFcap];      // far: key j << kFarPack | unit (a_ik = ta[unit]); rows < 2^25 on this path
    int bc[kRwNB];        // bucket cursors / ends
    unsigned bad[kRwNB / 32];
    int nbad;
    int badlist[32];
    uint16_t perm[kRwFcap];
};

// far list storage: shared memory (FarS, one batch of <= 32 entries and
// <= kRwTcap units: a_ik comes from the unit table) or a per-warp slice of
// global scratch (FarG, a_ik stored per item); same accessors.
struct FarS {
    RwSmem *S;
    static constexpr int nb = kRwNB;
    static constexpr int pack = kFarPack;  // raw = key << pack | unit: ordered by (key, unit) = (key, arrival)
    __device__ __forceinline__ int cap() const { return kRwFcap; }
    __device__ __forceinline__ double a(int x) const { return S->ta[S->fk[x] & ((1 << kFarPack) - 1)]; }
    __device__ __forceinline__ int key(int x) const { return S->fk[x] >> kFarPack; }
    __device__ __forceinline__ void put(int pos, int j, double b, double, int u) const {
        S->fk[pos] = (j << kFarPack) | u;
        S->fb[pos] = b;
    }
    __device__ __forceinline__ double *fb() const { return S->fb; }
    __device__ __forceinline__ int *fk() const { return S->fk; }
    __device__ __forceinline__ int *bc() const { return S->bc; }
    __device__ __forceinline__ unsigned *bad() const { return S->bad; }
    __device__ __forceinline__ uint16_t *perm() const { return S->perm; }
    __device__ __forceinline__ uint16_t *tmp() const { return reinterpret_cast<uint16_t *>(S->tcs); }
    __device__ __forceinline__ int tmp_cap() const { return (kRwTcap + 2 * kRwDepth) * 4; }
    __device__ __forceinline__ int *nbad_ptr() const { return &S->nbad; }
    __device__ __forceinline__ void nbad_set(int v) const { S->nbad = v; }
    __device__ __forceinline__ int nbad_get() const { return *reinterpret_cast<volatile int *>(&S->nbad); }
    __device__ __forceinline__ int *badlist() const { return S->badlist; }
};

__host__ __device__ __forceinline__ size_t rw_slice_bytes(int gcap) {
    const size_t b = (size_t)gcap * (8 + 8 + 4 + 2 + 2) + (size_t)kRwGNB * 4 + (kRwGNB / 32) * 4 + 33 * 4;
    return (b + 255) & ~(size_t)255;
}

struct FarG {
    unsigned char *base;
    int gcap;
    static constexpr int nb = kRwGNB;
    static constexpr int pack = 0;  // raw = key
    __device__ __forceinline__ int cap() const { return gcap; }
    __device__ __forceinline__ double *fa() const { return reinterpret_cast<double *>(base); }
    __device__ __forceinline__ double *fb() const { return fa() + gcap; }
    __device__ __forceinline__ int *fk() const { return reinterpret_cast<int *>(fb() + gcap); }
    __device__ __forceinline__ int *bc() const { return fk() + gcap; }
    __device__ __forceinline__ unsigned *bad() const { return reinterpret_cast<unsigned *>(bc() + kRwGNB); }
    __device__ __forceinline__ uint16_t *perm() const { return reinterpret_cast<uint16_t *>(bad() + kRwGNB / 32); }
    __device__ __forceinline__ uint16_t *tmp() const { return perm() + gcap; }
    __device__ __forceinline__ int tmp_cap() const { return gcap; }
    __device__ __forceinline__ int *nbad_ptr() const { return reinterpret_cast<int *>(tmp() + gcap); }
    __device__ __forceinline__ void nbad_set(int v) const { *nbad_ptr() = v; }
    __device__ __forceinline__ int nbad_get() const { return *reinterpret_cast<volatile int *>(nbad_ptr()); }
    __device__ __forceinline__ int *badlist() const { return nbad_ptr() + 1; }
    __device__ __forceinline__ double a(int x) const { return fa()[x]; }
    __device__ __forceinline__ int key(int x) const { return fk()[x]; }
    __device__ __forceinline__ void put(int pos, int j, double b, double at, int) const {
        fk()[pos] = j;
        fb()[pos] = b;
        fa()[pos] = at;
    }
};

// Cut sums: CutSum (common.cuh), plain per-lane sums of positive weights;
// RIG_RW_CUT_COMP=1: Neumaier per lane instead.
#if RIG_RW_CUT_COMP
#define CutSum Comp
#endif

// look-back status words and lookback(): common.cuh

// Stable sort of the n far items by key: F.perm()[sorted position] = item
// (items are numbered in arrival order).  Sorts the raw values fk[] (key <<
// F_::pack | unit in the shared list: unique, ordered by (key, arrival)).  Value buckets (monotone fp32 map of
// key - min) filled in arrival order; each lane insertion-sorts its own
// buckets of <= kRwSmallBucket items; a longer bucket found out of order is
// ranked by (key, arrival) by the whole warp.
template <class F_>
__device__ __forceinline__ bool far_sort(const F_ &F, int n, int key_bits) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    constexpr int NB = F_::nb, PER = NB / 32;
    constexpr int NBB = NB == 128 ? 7 : (NB == 256 ? 8 : (NB == 512 ? 9 : (NB == 64 ? 6 : 10)));
    static_assert((1 << NBB) == NB, "NB must be a power of two in [64, 1024]");
    int *fk = F.fk(), *bc = F.bc();
    uint16_t *perm = F.perm();
    // fixed-width value buckets over [0, 2^raw_bits) (keys are row ids):
    // monotone in the key, no min / max pass
    const int raw_bits = key_bits + F_::pack;
    const int sh = raw_bits > NBB ? raw_bits - NBB : 0;
    auto bucket = [&](int k) { return k >> sh; };
#pragma unroll
    for (int u = 0; u < PER; ++u) bc[l * PER + u] = 0;
    if (l < PER) F.bad()[l] = 0u;
    __syncwarp();
    for (int p = l; p < n; p += 32) atomicAdd(&bc[bucket(fk[p])], 1);
    __syncwarp();
    int c[PER], tot = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        c[u] = bc[l * PER + u];
        tot += c[u];
    }
    const int start = warp_incl_scan(tot) - tot;
    int base = start;
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        bc[l * PER + u] = base;  // running cursor; ends as the bucket end
        base += c[u];
    }
    __syncwarp();
    for (int p0 = 0; p0 < n; p0 += 32) {  // arrival order: stable
        const int p = p0 + l;
        const int b = p < n ? bucket(fk[p]) : NB + l;
        const unsigned g = __match_any_sync(kFull, b);
        if (p < n) {
            RIG_CHECK(b >= 0 && b < NB && bc[b] + __popc(g & lt) < n);
            perm[bc[b] + __popc(g & lt)] = (uint16_t)p;
        }
        __syncwarp();
        if (p < n && (g & lt) == 0) bc[b] += __popc(g);
        __syncwarp();
    }
    // buckets holding keys of several columns may be out of order: find
    // descents (adjacent sorted positions, same bucket since buckets are
    // ordered by value), list each such bucket once
    if (l == 0) F.nbad_set(0);
    __syncwarp();
    for (int p = l + 1; p < n; p += 32) {
        const int k2 = fk[perm[p]];
        if (fk[perm[p - 1]] > k2) {
            const int b = bucket(k2);
            const unsigned bit = 1u << (b & 31);
            if (!(atomicOr(&F.bad()[b >> 5], bit) & bit)) {
                const int t = atomicAdd(F.nbad_ptr(), 1);
                if (t < 32) F.badlist()[t] = b;
            }
        }
    }
    __syncwarp();
    const int nbad = F.nbad_get();
    if (nbad == 0) return true;
    // one lane per short bad bucket: insertion sort (key ties keep arrival
    // order = item index); long ones (or > 32 bad buckets): the warp ranks
    bool big = nbad > 32;
    if (l < nbad && l < 32) {
        const int b = F.badlist()[l];
        const int e1 = bc[b], e0 = b > 0 ? bc[b - 1] : 0;
        if (e1 - e0 <= kRwSmallBucket) {
            for (int q = e0 + 1; q < e1; ++q) {
                const int x = perm[q], kx = fk[x];
                int p = q - 1;
                int y = perm[p];
                while (fk[y] > kx) {
                    perm[p + 1] = (uint16_t)y;
                    if (--p < e0) break;
                    y = perm[p];
                }
                perm[p + 1] = (uint16_t)x;
            }
            const unsigned bit = 1u << (b & 31);
            atomicAnd(&F.bad()[b >> 5], ~bit);  // done
        } else {
            big = true;
        }
    }
    if (!__any_sync(kFull, big)) return true;
    __syncwarp();
    uint16_t *tmp = F.tmp();
    for (int wd = 0; wd < PER; ++wd) {
        unsigned m = F.bad()[wd];
        while (m) {
            const int b = wd * 32 + __ffs(m) - 1;
            m &= m - 1;
            const int e1 = bc[b], e0 = b > 0 ? bc[b - 1] : 0, sz = e1 - e0;
            if (sz > F.tmp_cap()) return false;  // the caller redoes the row with a global far list
            RIG_CHECK(e0 >= 0 && e1 <= n && sz >= 0);
            if (sz <= 32) {
                // the bucket in arrival order is a few ascending runs (one per
                // column it holds keys of): an item's rank = its index in its
                // run + for every other run, the items before it (keys < its
                // key; <= for earlier runs: equal keys keep arrival order),
                // found by a binary search over that run's lanes
                const int x = l < sz ? (int)perm[e0 + l] : 0;
                const int kx = l < sz ? fk[x] : INT_MAX;
                const int kp = __shfl_up_sync(kFull, kx, 1);
                const unsigned starts = __ballot_sync(kFull, l < sz && (l == 0 || kx < kp));
                const int rs = 31 - __clz(starts & (0xffffffffu >> (31 - l)));  // my run's start
                int rank = l - rs;
                unsigned m = starts;
                while (m) {
                    const int s0 = __ffs(m) - 1;
                    m &= m - 1;
                    const int s1 = m ? __ffs(m) - 1 : sz;  // run [s0, s1)
                    const bool earlier = s0 < rs;
                    int lo = s0, hi = s1;
#pragma unroll
                    for (int it = 0; it < 5; ++it) {  // runs are <= 32 long
                        const int mid = (lo + hi) >> 1;
                        const int km = __shfl_sync(kFull, kx, mid & 31);
                        if (lo < hi) {
                            if (earlier ? km <= kx : km < kx)
                                lo = mid + 1;
                            else
                                hi = mid;
                        }
                    }
                    if (s0 != rs) rank += lo - s0;
                }
                __syncwarp();
                if (l < sz) perm[e0 + rank] = (uint16_t)x;
                __syncwarp();
                continue;
            }
            for (int q = l; q < sz; q += 32) tmp[q] = perm[e0 + q];
            __syncwarp();
            for (int r0 = 0; r0 < sz; r0 += 32) {
                const int x = r0 + l < sz ? (int)tmp[r0 + l] : INT_MAX;
                const int kx = x != INT_MAX ? fk[x] : INT_MAX;
                int rank = 0;
                for (int s0 = 0; s0 < sz; s0 += 32) {
                    const int y = s0 + l < sz ? (int)tmp[s0 + l] : INT_MAX;
                    const int ky = y != INT_MAX ? fk[y] : INT_MAX;
                    const int cnt = min(32, sz - s0);
                    for (int t = 0; t < cnt; ++t) {
                        const int yt = __shfl_sync(kFull, y, t);
                        const int kt = __shfl_sync(kFull, ky, t);
                        rank += (kt < kx) || (kt == kx && yt < x);
                    }
                }
                if (x != INT_MAX) perm[e0 + rank] = (uint16_t)x;
            }
            __syncwarp();
        }
    }
    return true;
}

// 32-bit row ids and entry offsets: on this path nnz + ncols < 2^31 (CSC
// offsets fit int32), so rows and A's entry offsets fit too -- fewer live
// registers in the row loop (the kernel runs at 56 registers)
struct RowMeta {
    int i = 0;           // global row id
    int s = 0, e = 0;
    int k = 0;           // lane t: column of entry t
    int cs = 0, cl = 0;  // lane t: CSC offset (sentinel layout) and length of column k
    double av = 0.0;     // lane t: a_hat_ik
    int32_t pi = 0;      // part[i]
};

// Row metadata in three dependent stages (row pointers; entries; column
// bounds), issued at points of the previous row where their latency hides.
template <bool TEMP>
__device__ __forceinline__ void meta_rows(const RowArgs &a, int idx, int nrows, RowMeta &M) {
    M.s = M.e = 0;
    if (idx >= nrows) return;
    const int i = TEMP ? a.list[idx] : (int)a.rb + idx;  // TEMP: the mixed path's row list
    if (TEMP) M.i = i;
    M.s = (int)a.A.rp[i];
    M.e = (int)a.A.rp[i + 1];
    if (a.part) M.pi = __ldg(&a.part[i]);
}
__device__ __forceinline__ void meta_entries(const RowArgs &a, RowMeta &M) {
    const int l = lane_id();
    M.k = -1;
    if (l < M.e - M.s) {
        M.k = a.A.ci[M.s + l];
        M.av = a.A.v[M.s + l];
    }
}
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// stage 3; with `pf`, each lane also prefetches its column (rows, values)
// into L2, so that the row's gathers hit L2 when the row starts
__device__ __forceinline__ void meta_cols(const RowArgs &a, RowMeta &M, bool pf) {
    M.cl = 0;
    if (M.k >= 0) {
        const int64_t c0 = a.T.cp[M.k];
        M.cl = (int)(a.T.cp[M.k + 1] - c0);
        M.cs = (int)(c0 + M.k);
        if (pf) {
            const char *r0 = reinterpret_cast<const char *>(a.T.ri + M.cs);
            const char *v0 = reinterpret_cast<const char *>(a.T.vt + M.cs);
            for (int off = 0; off < M.cl * 4; off += 128) prefetch_l2(r0 + off);
            for (int off = 0; off < M.cl * 8; off += 128) prefetch_l2(v0 + off);
        }
    }
}

// Accumulate row i (window + far list).  Returns the number of far products
// (> F.cap(): the list overflowed and is incomplete).
template <class F_>
__device__ __forceinline__ int accumulate(const RowArgs &a, RwSmem &S, const F_ &F, int i,
                                          const RowMeta &M) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    const int wbase = i - kRwWH;
    int nfar = 0;
    for (int bb = M.s; bb < M.e; bb += 32) {
        const int nent = min(32, M.e - bb);
        int cs = 0, cl = 0;
        double av = 0.0;
        if (bb == M.s) {
            cs = M.cs;
            cl = M.cl;
            av = M.av;
        } else if (l < nent) {
            const int k = a.A.ci[bb + l];
            const int64_t c0 = a.T.cp[k];
            cl = (int)(a.T.cp[k + 1] - c0);
            cs = (int)(c0 + k);
            av = a.A.v[bb + l];
        }
        const int nch = l < nent ? (cl + 31) >> 5 : 0;
        const int incl = warp_incl_scan(nch);
        const int U = __shfl_sync(kFull, incl, 31);
        auto apply = [&](int j, double b, double at, int u) {
            const int d = j - wbase;
            const bool near = (unsigned)d < (unsigned)kRwW;
            RIG_CHECK(j >= -1 && j < a.A.nrows);
            if (near) S.wv[d] = __fma_rn(at, b, S.wv[d]);
            const bool far = !near && j >= 0;
            const unsigned fm = __ballot_sync(kFull, far);
            if (fm) {
                const int pos = nfar + __popc(fm & lt);
                if (far && pos < F.cap()) F.put(pos, j, b, at, u);
                nfar += __popc(fm);
            }
        };
        if (U <= kRwTcap) {
            // the table is padded with empty units up to a multiple of
            // kRwDepth (+ kRwDepth for the look-ahead): no bounds checks in
            // the pipeline
            const int Up = (U + kRwDepth - 1) / kRwDepth * kRwDepth;
            for (int c = 0, ex = incl - nch; c < nch; ++c) {
                RIG_CHECK(ex + c < kRwTcap + 2 * kRwDepth);
                RIG_CHECK(cs >= 0 && (int64_t)cs + cl <= a.A.nnz + a.A.ncols);
                S.tcs[ex + c] = make_int2(cs + 32 * c, min(32, cl - 32 * c));
                S.ta[ex + c] = av;
            }
            RIG_CHECK(Up + kRwDepth <= kRwTcap + 2 * kRwDepth);
            if (l < Up + kRwDepth - U) {
                S.tcs[U + l] = make_int2(0, 0);
                S.ta[U + l] = 0.0;
            }
            __syncwarp();
            int pj[kRwDepth];
            double pb[kRwDepth];
            auto issue = [&](int u, int &j, double &b) {
                const int2 t = S.tcs[u];
                j = -1;
                b = 0.0;
                if (l < t.y) {
                    j = __ldg(&a.T.ri[t.x + l]);
                    b = __ldg(&a.T.vt[t.x + l]);
                }
            };
#pragma unroll
            for (int d = 0; d < kRwDepth; ++d) issue(d, pj[d], pb[d]);
            for (int u0 = 0; u0 < Up; u0 += kRwDepth) {
#pragma unroll
                for (int d = 0; d < kRwDepth; ++d) {
                    apply(pj[d], pb[d], S.ta[u0 + d], u0 + d);
                    issue(u0 + d + kRwDepth, pj[d], pb[d]);
                }
            }
        } else {  // very long columns: unit by unit (global far list: a_ik per item)
            for (int t = 0; t < nent; ++t) {
                const int tcs = __shfl_sync(kFull, cs, t), tcl = __shfl_sync(kFull, cl, t);
                const double at = __shfl_sync(kFull, av, t);
                for (int off = 0; off < tcl; off += 32) {
                    int j = -1;
                    double b = 0.0;
                    if (off + l < tcl) {
                        j = a.T.ri[tcs + off + l];
                        b = a.T.vt[tcs + off + l];
                    }
                    apply(j, b, at, 0);
                }
            }
        }
        __syncwarp();
    }
    return nfar;
}

// Number of sorted far items with key < wbase (the far keys are either
// below the window or above it): two rounds of 32 probes narrow the
// boundary instead of a pass over every item.
template <class F_>
__device__ __forceinline__ int far_below(const F_ &F, int n, int wbase) {
    const int l = lane_id();
    int lo = 0, hi = n;  // boundary in [lo, hi]
    while (hi - lo > 32) {
        const int step = (hi - lo + 31) / 32;
        const int p = lo + l * step;  // probe positions lo, lo + step, ...
        const bool below = p < hi && F.key(F.perm()[p]) < wbase;
        const int c = __popc(__ballot_sync(kFull, below));  // probes below: a prefix
        const int nlo = lo + (c > 0 ? (c - 1) * step + 1 : 0);
        hi = min(hi, lo + c * step);
        lo = nlo;
    }
    const int p = lo + l;
    return lo + __popc(__ballot_sync(kFull, p < hi && F.key(F.perm()[p]) < wbase));
}

// Count pass over a sorted far list: the head of each equal-key group folds
// the group in arrival order (the R4 chain of that key) and stores |c| (or
// -1: not kept) in fb of the head item.  Returns kept far entries; nbelow =
// far items with key < wbase.
template <class F_>
__device__ __forceinline__ int far_count(const F_ &F, int n, int wbase, double tol, int &nbelow) {
    const int l = lane_id();
    int kept = 0;
    nbelow = 0;
    const uint16_t *perm = F.perm();
    double *fb = F.fb();
    for (int p0 = 0; p0 < n; p0 += 32) {
        const int p = p0 + l;
        bool keep = false, below = false;
        if (p < n) {
            const int x = perm[p];
            const int key = F.key(x);
            below = key < wbase;
            if (p == 0 || F.key(perm[p - 1]) != key) {
                double acc = __fma_rn(F.a(x), fb[x], +0.0);
                for (int q = p + 1; q < n; ++q) {
                    const int y = perm[q];
                    if (F.key(y) != key) break;
                    acc = __fma_rn(F.a(y), fb[y], acc);
                }
                const double w = fabs(acc);
                keep = w > tol;
                fb[x] = keep ? w : -1.0;
            }
        }
        __syncwarp();
        nbelow += __popc(__ballot_sync(kFull, below));
        kept += __popc(__ballot_sync(kFull, keep));
    }
    return kept;
}

// Emit a row in ascending j to dst (col, w) from position 0: far below the
// window, the window (re-zeroed), far above; returns the kept count.  FOLD:
// group heads fold their far groups here (else far_count stored |c| / -1 in
// fb).  Cut edges (j > i, part differs) go to acc; diag[idx] = c_ii.
template <bool FOLD, bool CUT, class F_>
__device__ __forceinline__ int emit_row(const RowArgs &a, RwSmem &S, const F_ &F, int i, int r, int n,
                                        int nbelow,
                                        int32_t *dcol, double *dw, bool write, int32_t pi, CutSum &acc) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    const int wbase = (int)i - kRwWH;
    const bool cut = CUT && a.part != nullptr;
    int o = 0;
    auto put = [&](bool keep, int key, double w) {
        const unsigned bal = __ballot_sync(kFull, keep);
        if (keep && write) {
            const int pos = o + __popc(bal & lt);
            dcol[pos] = key;
            dw[pos] = w;
        }
        o += __popc(bal);
    };
    auto far_range = [&](int f0, int f1) {
        for (int b0 = f0; b0 < f1; b0 += 32) {
            const int p = b0 + l;
            bool keep = false;
            int key = 0;
            double w = 0.0;
            if (p < f1) {
                const int x = F.perm()[p];
                key = F.key(x);
                if (p == 0 || F.key(F.perm()[p - 1]) != key) {
                    if (FOLD) {
                        double c = __fma_rn(F.a(x), F.fb()[x], +0.0);
                        for (int q = p + 1; q < n; ++q) {  // the group, in arrival order
                            const int y = F.perm()[q];
                            if (F.key(y) != key) break;
                            c = __fma_rn(F.a(y), F.fb()[y], c);
                        }
                        w = fabs(c);
                        keep = w > a.tol;
                    } else {
                        w = F.fb()[x];
                        keep = w >= 0.0;
                    }
                }
            }
            if (cut && keep && key > i) {
                const int32_t pj = __ldg(&a.part[key]);
                if (pj != pi) acc.add(w);
            }
            put(keep, key, w);
        }
    };
    far_range(0, nbelow);
#pragma unroll
    for (int t0 = 0; t0 < kRwW; t0 += 32) {
        const int t = t0 + l;
        const int key = wbase + t;
        double c = 0.0;
        if (t < kRwW) {
            c = S.wv[t];
            S.wv[t] = +0.0;
        }
        if (t == kRwWH && a.diag) a.diag[r] = c;
        const double w = fabs(c);
        const bool keep = t < kRwW && t != kRwWH && w > a.tol;
        if (cut && keep && t > kRwWH) {
            const int32_t pj = __ldg(&a.part[key]);
            if (pj != pi) acc.add(w);
        }
        put(keep, key, w);
    }
    far_range(nbelow, n);
    return o;
}

// Copy a staged row (n entries) to the graph at g0 (coalesced, streaming;
// kCopyU rounds of loads in flight), and take the row's cut edges there (j >
// i, part[j] != part[i]: PAPER.md:393-405) -- the part[] gathers are batched
// with the copy instead of stalling the emission.
#ifndef RIG_RW_COPYU
#define RIG_RW_COPYU 3
#endif
constexpr int kCopyU = RIG_RW_COPYU;  // 3 rounds of 32 per iteration: a config-5 row (~283 entries) is 3 iterations
__device__ __forceinline__ void copy_staged(const RowArgs &a, const int32_t *scol, const double *sw, int n, int64_t g0,
                                            bool write, int i, int32_t pi, CutSum &acc) {
    const int l = lane_id();
    const bool cut = a.part != nullptr;
#pragma unroll 1
    for (int t0 = 0; t0 < n; t0 += 32 * kCopyU) {
        int32_t c[kCopyU], pj[kCopyU];
        double w[kCopyU];
#pragma unroll
        for (int u = 0; u < kCopyU; ++u) {
            const int t = t0 + 32 * u + l;
            c[u] = -1;
            w[u] = 0.0;
            if (t < n) {
                c[u] = __ldcs(scol + t);
                w[u] = __ldcs(sw + t);
            }
        }
#pragma unroll
        for (int u = 0; u < kCopyU; ++u) {
            const int t = t0 + 32 * u + l;
            if (t < n && write) {
                __stcs(a.gcol + g0 + t, c[u]);
                __stcs(a.gw + g0 + t, w[u]);
            }
            pj[u] = pi;
            if (cut && c[u] > i) pj[u] = __ldg(&a.part[c[u]]);
        }
        if (cut) {
#pragma unroll
            for (int u = 0; u < kCopyU; ++u) {
                if (pj[u] != pi) acc.add(w[u]);
            }
        }
    }
#if RIG_RW_DISCARD
    // the staged lines are dead now: drop them from L2 without a write-back
    // (a dirty staged line would otherwise reach DRAM when evicted)
    __syncwarp();
    const int lc = (n * 4 + 127) / 128, lw = (n * 8 + 127) / 128;
    for (int t = l; t < lc + lw; t += 32) {
        const char *pl = t < lc ? reinterpret_cast<const char *>(scol) + 128 * t
                                : reinterpret_cast<const char *>(sw) + 128 * (t - lc);
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(pl) : "memory");
    }
#endif
}

// part[] ids were range-checked up front (k_part_check): no check here
__device__ __forceinline__ void finish_cut(const RowArgs &a, int idx, CutSum &acc) {
    const int l = lane_id();
    double v = acc.value();  // fixed lane tree: deterministic per row
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    if (l == 0) a.cutrow[idx] = v;
}

#ifndef RIG_RW_MINB
#define RIG_RW_MINB 9  // CTAs per SM the register budget (56) is fitted to; shared memory allows 9
#endif
// TEMP = false: every row of the shard, placed by look-back (row-window
// path).  TEMP = true: the rows of a.list (mixed path's mid rows), each
// written with its exact kept count to the temporary at toff[r] (cnt[r] =
// kept + 1, as the mid kernels); k_copy_rows places them and takes their cut.
template <bool TEMP>
__global__ void __launch_bounds__(kRwThreads, RIG_RW_MINB) k_row_win(RowArgs a) {
    extern __shared__ __align__(16) unsigned char rw_smem[];
    const int wid = threadIdx.x >> 5;
    RwSmem &S = reinterpret_cast<RwSmem *>(rw_smem)[wid];
    const int l = lane_id();
    for (int t = l; t < kRwW; t += 32) S.wv[t] = +0.0;
    __syncwarp();
    const FarS FS{&S};
    const int64_t gw = (int64_t)blockIdx.x * kRwWarps + wid;
    const FarG FG{a.gscratch ? static_cast<unsigned char *>(a.gscratch) + (size_t)gw * rw_slice_bytes(a.gcap)
                             : nullptr,
                  a.gcap};
    // staging: two slots per warp
    int32_t *stc = a.stage_col + gw * 2 * kRwStageCap;
    double *stw = a.stage_w + gw * 2 * kRwStageCap;
    const bool staging = !(a.dbg & 2);
    int pidx = -1;  // staged row waiting for its offset
    int pkept = 0, pslot = 0;
    const int nrows = (int)(TEMP ? *a.count_dev : a.nloc);
    const int key_bits = a.A.nrows > 1 ? 64 - __clzll((unsigned long long)(a.A.nrows - 1)) : 1;  // keys < 2^key_bits
    int idx = 0;
    if (l == 0) idx = (int)atomicAdd(a.ticket, 1ull);
    idx = __shfl_sync(kFull, idx, 0);
    RowMeta cur, nxt;
    meta_rows<TEMP>(a, idx, nrows, cur);
    meta_entries(a, cur);
    meta_cols(a, cur, false);
    // the staged row: look back for its offset, copy it into place
    int32_t ppi = 0;  // part of the staged row
    auto flush = [&]() {
        if (TEMP || pidx < 0) return;
        const int64_t g0 = lookback(a.chain, pidx, pkept);
        const bool fits = g0 + pkept <= a.cap;
        CutSum acc;
        copy_staged(a, stc + pslot * kRwStageCap, stw + pslot * kRwStageCap, pkept, g0, fits, (int)a.rb + pidx, ppi, acc);
        if (a.part) finish_cut(a, pidx, acc);
        if (l == 0) {
            a.row_ptr[pidx + 1] = g0 + pkept;
            if (pidx == 0) a.row_ptr[0] = 0;
            if (!fits) atomicOr(a.overflow, 1);
        }
        pidx = -1;
    };
    auto finish = [&](const auto &F, int nfar, bool shared_list) {
        const int i = TEMP ? cur.i : (int)a.rb + idx;
        const int wbase = (int)i - kRwWH;
        CutSum acc;
        int nidx = 0;
        if constexpr (TEMP) {
            // exact row into the temporary (room f_i - len_i >= kept), one pass
            if (l == 0) nidx = (int)atomicAdd(a.ticket, 1ull);
            const int nbelow = far_below(F, nfar, wbase);
            const int r = i - (int)a.rb;
            const int64_t t0 = a.toff[r];
            const int kept = emit_row<true, false>(a, S, F, i, r, nfar, nbelow, a.tcol + t0, a.tw + t0, true, cur.pi,
                                                   acc);
            RIG_CHECK(kept <= a.toff[r + 1] - a.toff[r]);
            if (l == 0) a.cnt[r] = kept + 1;  // the graph scan subtracts the diagonal slot
            nidx = __shfl_sync(kFull, nidx, 0);
            meta_rows<TEMP>(a, nidx, nrows, nxt);
        } else if (staging && shared_list) {
            // one pass: fold, count and write the row into the free staging
            // slot (kept <= far items + window slots <= kRwStageCap)
            const int nbelow = far_below(F, nfar, wbase);
            const int slot = pslot ^ 1;
            const int kept = emit_row<true, false>(a, S, F, i, idx, nfar, nbelow, stc + slot * kRwStageCap,
                                                   stw + slot * kRwStageCap, true, cur.pi, acc);
            RIG_CHECK(kept <= kRwStageCap);
            // publish the count; take the next ticket now (a ticket taken
            // earlier would be held while this warp waits, and rows behind it
            // would wait on it); then place the previously staged row
            if (l == 0) st_relaxed(&a.chain[idx], (idx == 0 ? kPre : kAgg) | (unsigned long long)kept);
            if (l == 0) nidx = (int)atomicAdd(a.ticket, 1ull);
            flush();
            pidx = idx;
            pkept = kept;
            pslot = slot;
            ppi = cur.pi;
            nidx = __shfl_sync(kFull, nidx, 0);
            meta_rows<TEMP>(a, nidx, nrows, nxt);
        } else {  // count, publish, wait for the offset, write in place
            int nbelow = 0;
            int kept = far_count(F, nfar, wbase, a.tol, nbelow);
#pragma unroll
            for (int t0 = 0; t0 < kRwW; t0 += 32) {
                const int t = t0 + l;
                kept += __popc(__ballot_sync(kFull, t < kRwW && t != kRwWH && fabs(S.wv[t]) > a.tol));
            }
            if (l == 0) st_relaxed(&a.chain[idx], (idx == 0 ? kPre : kAgg) | (unsigned long long)kept);
            if (l == 0) nidx = (int)atomicAdd(a.ticket, 1ull);
            flush();
            nidx = __shfl_sync(kFull, nidx, 0);
            meta_rows<TEMP>(a, nidx, nrows, nxt);
            const int64_t g0 = (a.dbg & 1) ? min((int64_t)idx * 280, a.cap - 1024) : lookback(a.chain, idx, kept);
            const bool fits = g0 + kept <= a.cap;
            emit_row<false, true>(a, S, F, i, idx, nfar, nbelow, a.gcol + g0, a.gw + g0, fits, cur.pi, acc);
            if (l == 0) {
                a.row_ptr[idx + 1] = g0 + kept;
                if (idx == 0) a.row_ptr[0] = 0;
                if (!fits) atomicOr(a.overflow, 1);
            }
            if (a.part) finish_cut(a, idx, acc);
        }
        meta_entries(a, nxt);
        meta_cols(a, nxt, !(a.dbg & 4));
        __syncwarp();
        return nidx;
    };
    while (idx < nrows) {
        const int i = TEMP ? cur.i : (int)a.rb + idx;
        if (TEMP && a.fskip_list && a.fnm[i - a.rb] + (cur.e - cur.s) > a.fskip) {
            // long row: left to the CTA-per-row kernel
            int nidx = 0;
            if (l == 0) {
                a.fskip_list[atomicAdd((unsigned long long *)a.fskip_count, 1ull)] = (int32_t)i;
                nidx = (int)atomicAdd(a.ticket, 1ull);
            }
            nidx = __shfl_sync(kFull, nidx, 0);
            meta_rows<TEMP>(a, nidx, nrows, nxt);
            meta_entries(a, nxt);
            meta_cols(a, nxt, false);
            idx = nidx;
            cur = nxt;
            continue;
        }
        const bool one_batch = cur.e - cur.s <= 32;
        int nfar = 0;
        bool global = !one_batch;
        if (one_batch) {
            // more than kRwTcap units leave no a_ik table: global
            const int nch = l < (int)(cur.e - cur.s) ? (cur.cl + 31) >> 5 : 0;
            global = __reduce_add_sync(kFull, (unsigned)nch) > (unsigned)kRwTcap;
        }
        if (!global) {
            nfar = accumulate(a, S, FS, i, cur);
            // far list overflow, or a long out-of-order sort bucket beyond the
            // shared scratch: redo the row with the global far list
            bool redo = nfar > FS.cap();
            if (!redo) {
                if (nfar > 1)
                    redo = !far_sort(FS, nfar, key_bits);
                else if (nfar == 1 && l == 0)
                    FS.perm()[0] = 0;
                __syncwarp();
            }
            if (redo) {
                for (int t = l; t < kRwW; t += 32) S.wv[t] = +0.0;
                __syncwarp();
                global = true;
            }
        }
        int nidx;
        if (!global) {
            nidx = finish(FS, nfar, true);
        } else {
            nfar = accumulate(a, S, FG, i, cur);
            if (nfar > FG.cap()) {  // cannot happen when gcap >= max f_i (host check)
                if (l == 0) atomicOr(a.overflow, 2);
                nfar = FG.cap();
            }
            if (nfar > 1)
                far_sort(FG, nfar, key_bits);  // tmp_cap = gcap: always sorts
            else if (nfar == 1 && l == 0)
                FG.perm()[0] = 0;
            __syncwarp();
            nidx = finish(FG, nfar, false);
        }
        idx = nidx;
        cur = nxt;
    }
    flush();
}

// Per-row cut partials -> kRowCutBlocks partials (fixed segments, fixed trees).
constexpr int kRowCutThreads = 256, kRowCutBlocks = 256;
__global__ void __launch_bounds__(kRowCutThreads) k_rowcut_partials(const double *__restrict__ cutrow, int64_t n,
                                                                    double *partials, int *used) {
    const int64_t seg = (n + kRowCutBlocks - 1) / kRowCutBlocks;
    const int64_t r0 = (int64_t)blockIdx.x * seg, r1 = min(n, r0 + seg);
    Comp c;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += kRowCutThreads) c.add(cutrow[r]);
    const double v = block_tree_sum<kRowCutThreads>(c.value());
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = v;
        if (blockIdx.x == 0) *used = kRowCutBlocks;
    }
}

static int rowwin_ctas_per_sm() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        const size_t smem = (size_t)kRwWarps * sizeof(RwSmem);
        cudaFuncSetAttribute(k_row_win<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_row_win<false>, kRwThreads, smem);
        cache[dev] = per_sm > 0 ? per_sm : 1;
    }
    return cache[dev];
}

int rowwin_grid() { return num_sms() * rowwin_ctas_per_sm(); }
size_t rowwin_scratch_bytes(int gcap) { return (size_t)rowwin_grid() * kRwWarps * rw_slice_bytes(gcap); }
size_t rowwin_stage_entries() { return (size_t)rowwin_grid() * kRwWarps * 2 * kRwStageCap; }
int rowwin_max_gcap() { return 65535; }  // perm entries are 16-bit
int64_t rowwin_max_rows() { return kRowWinMaxRows; }  // packed far keys (key << kFarPack | unit) fit int32

void launch_row_win(const RowArgs &a, cudaStream_t s) {
    const size_t smem = (size_t)kRwWarps * sizeof(RwSmem);
    if (a.list) {
        cudaFuncSetAttribute(k_row_win<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_row_win<true><<<rowwin_grid(), kRwThreads, smem, s>>>(a);
    } else {
        cudaFuncSetAttribute(k_row_win<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_row_win<false><<<rowwin_grid(), kRwThreads, smem, s>>>(a);
    }
    note_launch();
}

void launch_rowcut_partials(const double *cutrow, int64_t n, double *partials, int *used, cudaStream_t s) {
    k_rowcut_partials<<<kRowCutBlocks, kRowCutThreads, 0, s>>>(cutrow, n, partials, used);
    note_launch();
}

}  // namespace rig

// k_midrow.cu -- steps a5 + a6 for rows off the merge path (A-row longer
// than kMergeMaxLen, or many products): one warp per row of
// C = A_hat A_hat^T (Gustavson), written with its exact
// kept count to a temporary; k_copy_rows moves it to its final graph slots
// once all counts are scanned, and takes these rows' share of the cut (a7).
// No symbolic pass is needed.
//
// Per row i (ordering contract, DESIGN.md §3 R4: every c_ij is the fma chain
// over the shared columns k in ascending k from +0.0):
//  * the row's entries k are taken in ascending order; column k of the CSC
//    (rows j ascending) is one 32-lane step when it has <= 32 rows (a longer
//    one, several).  Keys inside a column are distinct: no conflicts.  The
//    gathers run 8 columns ahead of the column being applied.
//  * near keys, |j - i| < kMidWinHalf, accumulate in a direct-mapped window
//    wv[j - i + kMidWinHalf]: columns are applied in ascending k, so each slot
//    sees its chain in order, and the window is already sorted by j.
//  * far keys are appended with both factors (a_ik, a_jk) to a far list in
//    arrival (= ascending k) order, as unique items (key << 32 | position);
//    sorting the items by value orders them by key and, for equal keys, by
//    arrival -- ascending k.  The sort distributes them into 32 value buckets
//    (each column's far keys arrive as an ascending run, so buckets are nearly
//    sorted) and insertion-sorts each bucket; equal keys are then folded in
//    order.
//  * output in ascending j: far keys below the window, the window, far keys
//    above it; kept iff j != i and |c| > tol.
// A row whose far list exceeds the capacity, or whose far keys crowd one
// bucket, is deferred to the CTA-per-row huge path.
#include "common.cuh"

namespace rig {

constexpr int kMidThreads = 64;  // 2 warps per CTA: fine-grained shared-memory occupancy
constexpr int kMidWarps = kMidThreads / 32;
constexpr int kMidWinHalf = 128;
constexpr int kMidWin = 2 * kMidWinHalf;
constexpr int kWideWinHalf = 2048, kWideCap = 64;  // a later pass over the deferred rows
#ifndef RIG_MID_BIG_CAP
#define RIG_MID_BIG_CAP 768  // measured: 512 / 768 / 1024 on configs 4 and 6
#endif
constexpr int kMidBigFarCap = RIG_MID_BIG_CAP;      // the pass between: long far lists (random columns)
constexpr int kMidGlobalFarCap = 4096;              // far lists in global scratch: rows up to f_i ~ 4096
constexpr int kMaxBucket = 96;

// far-sort buckets: 32 for the small far lists, FCAP/8 for bigger ones
template <int FCAP>
__host__ __device__ constexpr int far_buckets() { return FCAP <= 256 ? 32 : FCAP / 8; }

// GFAR: the far list lives in a per-warp slice of global scratch (MidArgs::
// fscratch) instead of shared memory -- long lists, few rows.
template <int FCAP, int WIN = kMidWin, bool GFAR = false>
struct MidSmem {
    static constexpr int FS = GFAR ? 1 : FCAP;
    double wv[WIN];
    double fa[FS], fb[FS];        // factors of the far products (arrival order)
    uint64_t m0[FS], m1[FS];      // far items (key << 32 | arrival position); sorted copy
    int64_t ecs[32];              // batch of row entries: CSC start, length, a_hat_ik
    int elen[32];
    double ea[32];
    int bcnt[far_buckets<FCAP>()];  // bucket counts / cursors of the far sort
    int bst[far_buckets<FCAP>()];   // bucket starts
};

__device__ __forceinline__ int it_key(uint64_t v) { return (int)(uint32_t)(v >> 32); }
__device__ __forceinline__ int it_pos(uint64_t v) { return (int)(uint32_t)v; }

// Sort n unique far items in place (a, via tmp): NB value buckets (NB/32 per
// lane) filled stably in arrival order (tmp), then every item is placed at its
// bucket's start plus its rank in the bucket (the count of smaller items there;
// items are unique), back into a.  NB ~ n/4 keeps buckets short for uniform
// keys.  Returns false (nothing usable) if a bucket would exceed kMaxBucket.
template <int NB>
__device__ __forceinline__ bool bucket_sort_far(uint64_t *__restrict__ a, uint64_t *__restrict__ tmp, int *cnt,
                                                int *bst, int n) {
    constexpr int PER = NB / 32;
    const int l = lane_id();
    int mn = INT_MAX, mx = INT_MIN;
    for (int p = l; p < n; p += 32) {
        const int k = it_key(a[p]);
        mn = min(mn, k);
        mx = max(mx, k);
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    // bucket(k) = floor((k - mn) * mul / 2^32) in [0, NB), monotone in k
    const uint64_t mul = (((uint64_t)NB << 32) - 1) / (uint64_t)((int64_t)mx - mn + 1);
    auto bucket = [&](uint64_t v) { return (int)(((uint64_t)(uint32_t)(it_key(v) - mn) * mul) >> 32); };
#pragma unroll
    for (int u = 0; u < PER; ++u) cnt[l * PER + u] = 0;
    __syncwarp();
    for (int p = l; p < n; p += 32) atomicAdd(&cnt[bucket(a[p])], 1);
    __syncwarp();
    int c[PER], tot = 0, big = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        c[u] = cnt[l * PER + u];
        tot += c[u];
        big |= c[u] > kMaxBucket;
    }
    if (__any_sync(kFull, big)) return false;
    int base = warp_incl_scan(tot) - tot;
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PER; ++u) {  // running cursors, bucket starts
        cnt[l * PER + u] = base;
        bst[l * PER + u] = base;
        base += c[u];
    }
    __syncwarp();
    const unsigned lt = lanemask_lt();
    for (int p0 = 0; p0 < n; p0 += 32) {  // arrival order (stable)
        const int p = p0 + l;
        const uint64_t v = p < n ? a[p] : 0ull;
        const int b = p < n ? bucket(v) : NB + l;
        const unsigned g = __match_any_sync(kFull, b);
        if (p < n) tmp[cnt[b] + __popc(g & lt)] = v;
        __syncwarp();
        if (p < n && (g & lt) == 0) cnt[b] += __popc(g);
        __syncwarp();
    }
    // rank in the bucket: [bst[b], cnt[b]) holds bucket b
    for (int p = l; p < n; p += 32) {
        const uint64_t v = tmp[p];
        const int b = bucket(v);
        const int b0 = bst[b], b1 = cnt[b];
        int rank = 0;
        for (int q = b0; q < b1; ++q) rank += tmp[q] < v;
        a[b0 + rank] = v;
    }
    __syncwarp();
    return true;
}

// WH: window half-width.  kMidWinHalf for the mid bins; kWideWinHalf for the
// rows the first pass deferred (their far list overflowed): rows of banded or
// FEM-like matrices with long rows keep every key within a few thousand of
// the diagonal, and a wide window takes them all without sorting.
template <int FCAP, int WH, bool GFAR>
__global__ void __launch_bounds__(kMidThreads, 8) k_num_mid(MidArgs a) {
    constexpr int kMidWinHalf = WH, kMidWin = 2 * WH;
    extern __shared__ __align__(16) unsigned char mid_smem[];
    MidSmem<FCAP, kMidWin, GFAR> &S = reinterpret_cast<MidSmem<FCAP, kMidWin, GFAR> *>(mid_smem)[threadIdx.x >> 5];
    double *far_a = S.fa, *far_b = S.fb;
    uint64_t *far_m0 = S.m0, *far_m1 = S.m1;
    if constexpr (GFAR) {  // this warp's slice: m0, m1, fa, fb (FCAP each)
        const int64_t gw = (int64_t)blockIdx.x * kMidWarps + (threadIdx.x >> 5);
        uint64_t *base = reinterpret_cast<uint64_t *>(a.fscratch) + gw * 4 * (int64_t)FCAP;
        far_m0 = base;
        far_m1 = base + FCAP;
        far_a = reinterpret_cast<double *>(base + 2 * FCAP);
        far_b = reinterpret_cast<double *>(base + 3 * FCAP);
    }
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    for (int t = l; t < kMidWin; t += 32) S.wv[t] = +0.0;
    __syncwarp();
    const int64_t n = *a.count;
    const int64_t nw = (int64_t)gridDim.x * kMidWarps;
    // row metadata (first batch of entries: lane t holds entry t), loaded one
    // row ahead so its dependent gathers (row_ptr -> col -> col_ptr) overlap
    // the current row
    struct Meta {
        int64_t i = 0, s = 0, e = 0, cs = 0;
        int len = 0;
        double av = 0.0;
    };
    auto load_meta = [&](int64_t id, Meta &M) {
        M.len = 0;
        if (id >= n) return;
        M.i = a.list[id];
        M.s = a.A.rp[M.i];
        M.e = a.A.rp[M.i + 1];
        if (l < M.e - M.s) {
            const int k = a.A.ci[M.s + l];
            const int64_t c0 = a.T.cp[k];
            M.len = (int)(a.T.cp[k + 1] - c0);
            M.cs = c0 + k;  // sentinel layout (csc_begin)
            M.av = a.A.v[M.s + l];
        }
    };
    Meta cur, nxt;
    int64_t idx = blockIdx.x * (int64_t)kMidWarps + (threadIdx.x >> 5);
    load_meta(idx, cur);
    for (; idx < n; idx += nw) {
        const int64_t i = cur.i;
        const int64_t r = i - a.rb;
        const int64_t s = cur.s, e = cur.e;
        const int wbase = (int)i - kMidWinHalf;
        int nfar = 0;
        bool prefetched = false;
        if (GFAR && a.fnm && a.fnm[r] > 2 * (int64_t)FCAP) {  // far beyond this pass: on to the huge kernel
            if (l == 0) a.defer_list[atomicAdd((unsigned long long *)a.defer_count, 1ull)] = (int32_t)i;
            load_meta(idx + nw, nxt);
            cur = nxt;
            __syncwarp();
            continue;
        }
        // one column step: lanes hold rows j of a column of a_ik = at
        auto apply = [&](int j, double b, double at, bool v) {
            const int d = j - wbase;
            const bool near = v && (unsigned)d < (unsigned)kMidWin;
            if (near) S.wv[d] = __fma_rn(at, b, S.wv[d]);
            const bool far = v && !near;
            const unsigned fm = __ballot_sync(kFull, far);
            const int pos = nfar + __popc(fm & lt);
            if (far && pos < FCAP && !(a.dbg & 2)) {
                far_m0[pos] = ((uint64_t)(uint32_t)j << 32) | (uint32_t)pos;
                far_a[pos] = at;
                far_b[pos] = b;
            }
            nfar += __popc(fm);
        };
        for (int64_t bb = s; bb < e; bb += 32) {
            const int nent = (int)min((int64_t)32, e - bb);
            int clen = 0;
            if (bb == s) {
                clen = cur.len;
                if (l < nent) {
                    S.ecs[l] = cur.cs;
                    S.elen[l] = clen;
                    S.ea[l] = cur.av;
                }
            } else if (l < nent) {
                const int k = a.A.ci[bb + l];
                const int64_t c0 = a.T.cp[k];
                clen = (int)(a.T.cp[k + 1] - c0);
                S.ecs[l] = c0 + k;
                S.elen[l] = clen;
                S.ea[l] = a.A.v[bb + l];
            }
            const bool short_cols = __all_sync(kFull, clen <= 32);
            __syncwarp();
            if (!prefetched) {  // next row's metadata, overlapping this row
                load_meta(idx + nw, nxt);
                prefetched = true;
            }
            if (short_cols) {
#ifndef RIG_MID_DEPTH
#define RIG_MID_DEPTH 12  // measured 4, 8, 12, 16 on config 5
#endif
                constexpr int kDepth = RIG_MID_DEPTH;  // columns in flight
                int pj[kDepth];
                double pb[kDepth];
#pragma unroll
                for (int u = 0; u < kDepth; ++u) {
                    pj[u] = 0;
                    pb[u] = 0.0;
                    if (u < nent && l < S.elen[u]) {
                        const int64_t q = S.ecs[u] + l;
                        pj[u] = a.T.ri[q];
                        pb[u] = a.T.vt[q];
                    }
                }
                for (int t0 = 0; t0 < nent; t0 += kDepth) {
#pragma unroll
                    for (int u = 0; u < kDepth; ++u) {
                        const int t = t0 + u;
                        if (t < nent) {
                            apply(pj[u], pb[u], S.ea[t], l < S.elen[t]);
                            const int tn = t + kDepth;
                            if (tn < nent && l < S.elen[tn]) {
                                const int64_t q = S.ecs[tn] + l;
                                pj[u] = a.T.ri[q];
                                pb[u] = a.T.vt[q];
                            }
                        }
                    }
                }
            } else {
                for (int t = 0; t < nent; ++t) {
                    const int64_t q0 = S.ecs[t];
                    const int len = S.elen[t];
                    const double at = S.ea[t];
                    for (int off = 0; off < len; off += 32) {
                        const bool v = off + l < len;
                        int j = 0;
                        double b = 0.0;
                        if (v) {
                            j = a.T.ri[q0 + off + l];
                            b = a.T.vt[q0 + off + l];
                        }
                        apply(j, b, at, v);
                    }
                }
            }
            __syncwarp();
            if (FCAP != kMidSmallCap && nfar > FCAP) break;  // later passes: the row goes on
        }
        if (!prefetched) load_meta(idx + nw, nxt);
        cur = nxt;
        __syncwarp();
        // ---- sort the far items (or defer the row to the huge path)
        const uint64_t *srt = far_m0;
        bool ok = nfar <= FCAP;
        if (a.dbg & 2) nfar = 0;
        if (ok && nfar > 1 && !(a.dbg & 1)) {
            ok = bucket_sort_far<far_buckets<FCAP>()>(far_m0, far_m1, S.bcnt, S.bst, nfar);  // sorted in place (m0)
        }
        if (!ok) {
            for (int t = l; t < kMidWin; t += 32) S.wv[t] = +0.0;
            if (l == 0) a.defer_list[atomicAdd((unsigned long long *)a.defer_count, 1ull)] = (int32_t)i;
            __syncwarp();
            continue;
        }
        // ---- emit in ascending j: far below, window, far above
        const int64_t g0 = a.toff[r];
        int64_t o = 0;
        auto emit = [&](bool keep, int key, double w) {
            const unsigned bal = __ballot_sync(kFull, keep);
            if (keep && !(a.dbg & 4)) {
                const int64_t pos = g0 + o + __popc(bal & lt);
                __stcs(a.tcol + pos, key);  // streamed: keeps the CSC gathers in L2
                __stcs(a.tw + pos, w);
            }
            o += __popc(bal);
        };
        // far items: the first of each equal-key group folds the group in order
        auto emit_far = [&](int f0, int f1) {
            for (int b0 = f0; b0 < f1; b0 += 32) {
                const int p = b0 + l;
                bool keep = false;
                int key = 0;
                double w = 0.0;
                if (p < f1) {
                    key = it_key(srt[p]);
                    if (p == 0 || it_key(srt[p - 1]) != key) {
                        double acc = +0.0;
                        int q = p;
                        do {
                            const int x = it_pos(srt[q]);
                            acc = __fma_rn(far_a[x], far_b[x], acc);
                            ++q;
                        } while (q < nfar && it_key(srt[q]) == key);
                        w = fabs(acc);
                        keep = w > a.tol;
                    }
                }
                emit(keep, key, w);
            }
        };
        int nbelow = 0;
        for (int b0 = 0; b0 < nfar; b0 += 32) {
            const int p = b0 + l;
            nbelow += __popc(__ballot_sync(kFull, p < nfar && it_key(srt[p]) < wbase));
        }
        emit_far(0, nbelow);
        for (int t = l; t < kMidWin; t += 32) {
            const int key = wbase + t;
            const double c = S.wv[t];
            S.wv[t] = +0.0;
            if ((int64_t)key == i && a.diag) a.diag[r] = c;
            const double w = fabs(c);
            emit((int64_t)key != i && w > a.tol, key, w);  // untouched slots hold +0.0: never kept
        }
        emit_far(nbelow, nfar);
        if (l == 0) a.cnt[r] = o + 1;  // the scan subtracts the diagonal slot
        __syncwarp();
    }
}

template <int FCAP, int WH, bool GFAR = false>
static void launch_mid_t(const MidArgs &a, cudaStream_t s) {
    const size_t smem = (size_t)kMidWarps * sizeof(MidSmem<FCAP, 2 * WH, GFAR>);
    cudaFuncSetAttribute(k_num_mid<FCAP, WH, GFAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_num_mid<FCAP, WH, GFAR>, kMidThreads, smem);
    if (per_sm < 1) per_sm = 1;
    int g = num_sms() * per_sm;
    if (g > kCutSlotsPerLaunch) g = kCutSlotsPerLaunch;
    if (GFAR) {  // the global far lists: a slice per warp
        const int64_t cap = a.fscratch_bytes / ((int64_t)kMidWarps * 4 * 8 * FCAP);
        if (g > cap) g = (int)cap;
        if (g < 1) return;
    }
    k_num_mid<FCAP, WH, GFAR><<<g, kMidThreads, smem, s>>>(a);
    note_launch();
}

void launch_num_mid(const MidArgs &a, int fcap, cudaStream_t s) {
    (void)fcap;
    launch_mid_t<kMidSmallCap, kMidWinHalf>(a, s);
}

void launch_num_mid_wide(const MidArgs &a, cudaStream_t s) { launch_mid_t<kWideCap, kWideWinHalf>(a, s); }

void launch_num_mid_big(const MidArgs &a, cudaStream_t s) { launch_mid_t<kMidBigFarCap, kMidWinHalf>(a, s); }

void launch_num_mid_gfar(const MidArgs &a, cudaStream_t s) { launch_mid_t<kMidGlobalFarCap, kMidWinHalf, true>(a, s); }

size_t mid_gfar_scratch_bytes() { return (size_t)num_sms() * 16 * kMidWarps * 4 * 8 * kMidGlobalFarCap; }

// Rows off the merge path: temporary (toff[r], exact count) -> final graph
// slots [gptr[r], gptr[r+1]).  One warp per row, coalesced.  The fused cut
// (a7) of these rows is taken here, on the streamed entries: every kept edge
// (i, j), j > i, with part[j] != part[i].
constexpr int kCopyThreads = 256;
__global__ void __launch_bounds__(kCopyThreads) k_copy_rows(const int32_t *__restrict__ list, const int64_t *count,
                                                            int64_t rb, const int64_t *__restrict__ toff,
                                                            const int64_t *__restrict__ gptr,
                                                            const int32_t *__restrict__ tcol,
                                                            const double *__restrict__ tw, int32_t *gcol, double *gw,
                                                            CutOut cut) {
    const int l = lane_id();
    const int64_t n = *count;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    Comp acc;
    int badp = 0;
    for (int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < n; idx += nw) {
        const int64_t i = list[idx];
        const int64_t r = i - rb;
        const int64_t src = toff[r], d = gptr[r], len = gptr[r + 1] - d;
        int32_t pi = 0;
        if (cut.part) {
            pi = __ldg(&cut.part[i]);
            badp |= (pi < 0) | (pi >= cut.K);
        }
        constexpr int U = 4;  // 4 chunks of loads (and part gathers) in flight per lane
        for (int64_t t0 = 0; t0 < len; t0 += 32 * U) {
            int32_t j[U], pj[U];
            double w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t t = t0 + 32 * u + l;
                j[u] = -1;
                w[u] = 0.0;
                if (t < len) {  // streamed: the temporary is read once
                    j[u] = __ldcs(tcol + src + t);
                    w[u] = __ldcs(tw + src + t);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t t = t0 + 32 * u + l;
                if (t < len) {
                    __stcs(gcol + d + t, j[u]);
                    __stcs(gw + d + t, w[u]);
                }
                pj[u] = pi;
                if (cut.part && (int64_t)j[u] > i) pj[u] = __ldg(&cut.part[j[u]]);
            }
            if (cut.part) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    badp |= (pj[u] < 0) | (pj[u] >= cut.K);
                    if (pj[u] != pi) acc.add(w[u]);
                }
            }
        }
    }
    if (cut.part) {
        const double v = block_tree_sum<kCopyThreads>(acc.value());
        if (threadIdx.x == 0) {
            cut.cutp[blockIdx.x] = v;
            if (blockIdx.x == 0) *cut.used = (int)gridDim.x;
        }
        if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(cut.bad, 1);
    }
}

void launch_copy_rows(const int32_t *list, const int64_t *count, int64_t rb, const int64_t *toff, const int64_t *gptr,
                      const int32_t *tcol, const double *tw, int32_t *gcol, double *gw, const CutOut &cut,
                      cudaStream_t s) {
    k_copy_rows<<<num_sms() * 8, kCopyThreads, 0, s>>>(list, count, rb, toff, gptr, tcol, tw, gcol, gw, cut);
    note_launch();
}

}  // namespace rig

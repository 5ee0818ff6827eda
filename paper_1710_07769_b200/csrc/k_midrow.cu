// k_midrow.cu -- steps a5 + a6 (+ a7 partials) for rows off the merge path
// (A-row longer than kMergeMaxLen, or many products): one warp per row of
// C = A_hat A_hat^T (Gustavson), written with its exact
// kept count to a temporary; k_copy_rows moves it to its final graph slots
// once all counts are scanned.  No symbolic pass is needed.
//
// Per row i (ordering contract, DESIGN.md §3 R4: every c_ij is the fma chain
// over the shared columns k in ascending k from +0.0):
//  * the row's entries k are taken in ascending order; column k of the CSC
//    (rows j ascending) is walked in pieces of 32 lanes.  Keys inside a
//    column are distinct, so a piece has no conflicts.
//  * near keys, |j - i| < kWinHalf, accumulate in a direct-mapped window
//    wv[j - i + kWinHalf]: pieces are applied in ascending k, so each window
//    slot sees its chain in order.  The window is also already sorted by j.
//  * far keys are appended, with both factors (a_ik, a_jk), to a far list in
//    arrival (= ascending k) order, as unique items (key, run, index).  They
//    are sorted by a stable 32-bucket distribution plus per-bucket insertion
//    sorts (each column's far keys arrive as an ascending run, so buckets are
//    nearly sorted); skewed rows fall back to pairwise merges of the runs by a
//    warp merge path.  Equal keys end adjacent in ascending k and their
//    products are folded in that order.
//  * output in ascending j: far keys below the window, the window, far keys
//    above it; kept iff j != i and |c| > tol.
// A row whose far list would exceed the kernel's capacity is deferred to the
// next (larger) capacity, and finally to the CTA-per-row huge path.
#include "common.cuh"

namespace rig {

constexpr int kMidThreads = 64;  // 2 warps per CTA: fine-grained shared-memory occupancy
constexpr int kMidWarps = kMidThreads / 32;
constexpr int kMidWinHalf = 128;
constexpr int kMidWin = 2 * kMidWinHalf;
template <int FCAP>
struct MidSmem {
    double wv[kMidWin];
    double ra[FCAP];              // a_hat_ik of each far run (a run = one column's far keys)
    double fb[FCAP];              // a_hat_jk of each far product (arrival order)
    uint64_t m0[FCAP], m1[FCAP];  // far items: (key << 32) | (run << 16) | arrival index; sort output
    int64_t ecs[32];              // batch of row entries: CSC start, length, a_hat_ik
    int elen[32];
    double ea[32];
    uint16_t rs[FCAP + 1];        // run starts in the far list
    int bcnt[32];                 // bucket counts / cursors of the far sort
};

__device__ __forceinline__ uint64_t mk_item(int key, int run, int idx) {
    return ((uint64_t)(uint32_t)key << 32) | ((uint64_t)(uint32_t)run << 16) | (uint64_t)(uint32_t)idx;
}
__device__ __forceinline__ int it_key(uint64_t v) { return (int)(uint32_t)(v >> 32); }
__device__ __forceinline__ int it_run(uint64_t v) { return (int)((v >> 16) & 0xffffu); }
__device__ __forceinline__ int it_idx(uint64_t v) { return (int)(v & 0xffffu); }

// One level of the far-run merge: segments of 2^lv runs (boundaries
// rs[min(s << lv, nruns)]) are merged pairwise from src into dst.  Items are
// unique 64-bit values (key, run, index), so merging by plain < is stable in
// run order -- equal keys stay in ascending k.  Merge path: lane l produces the
// output positions [l*E, l*E + E); per merged segment it co-ranks its first
// position with one binary search and then merges sequentially.
__device__ __forceinline__ void merge_level(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst,
                                            const uint16_t *__restrict__ rs, int nruns, int lv, int n) {
    const int l = lane_id();
    const int E = (n + 31) >> 5;
    int p = l * E;
    const int pend = min(p + E, n);
    while (p < pend) {
        // merged segment m (runs [2m << lv, (2m+2) << lv)) containing p
        int m = 0, hi = ((nruns - 1) >> (lv + 1)) + 1;  // number of merged segments
        while (hi - m > 1) {
            const int mid = (m + hi) >> 1;
            if (rs[min((2 * mid) << lv, nruns)] <= p)
                m = mid;
            else
                hi = mid;
        }
        const int a0 = rs[min((2 * m) << lv, nruns)], a1 = rs[min((2 * m + 1) << lv, nruns)];
        const int b1 = rs[min((2 * m + 2) << lv, nruns)];
        const int la = a1 - a0, lb = b1 - a1;
        const int q = p - a0;
        int lo = max(0, q - lb), h2 = min(q, la);  // co-rank: items taken from A
        while (lo < h2) {
            const int mid = (lo + h2) >> 1;
            if (src[a0 + mid] < src[a1 + q - 1 - mid])
                lo = mid + 1;
            else
                h2 = mid;
        }
        int ia = a0 + lo, ib = a1 + (q - lo);
        const int stop = min(pend, b1);
        uint64_t va = ia < a1 ? src[ia] : ~0ull, vb = ib < b1 ? src[ib] : ~0ull;
        for (; p < stop; ++p) {
            if (va < vb) {
                dst[p] = va;
                ++ia;
                va = ia < a1 ? src[ia] : ~0ull;
            } else {
                dst[p] = vb;
                ++ib;
                vb = ib < b1 ? src[ib] : ~0ull;
            }
        }
    }
}

// Stable distribution of the far items into 32 value buckets (one per lane)
// in arrival order, then a per-lane insertion sort of each bucket.  Items are
// unique, buckets are nearly sorted (a far column's keys arrive as one
// ascending run), so the insertion sorts are close to linear.  Returns false
// (nothing written) if a bucket would exceed kMaxBucket: the caller then
// uses the merge path.
constexpr int kMaxBucket = 96;
__device__ __forceinline__ bool bucket_sort_far(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst,
                                                int *cnt, int n) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    int mn = INT_MAX, mx = INT_MIN;
    for (int p = l; p < n; p += 32) {
        const int k = it_key(src[p]);
        mn = min(mn, k);
        mx = max(mx, k);
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    // bucket(k) = floor((k - mn) * mul / 2^32) in [0, 32), monotone in k
    const uint64_t mul = ((1ull << 37) - 1) / (uint64_t)((int64_t)mx - mn + 1);
    cnt[l] = 0;
    __syncwarp();
    for (int p = l; p < n; p += 32) {
        const int b = (int)(((uint64_t)(uint32_t)(it_key(src[p]) - mn) * mul) >> 32);
        atomicAdd(&cnt[b], 1);
    }
    __syncwarp();
    const int c = cnt[l];
    if (__any_sync(kFull, c > kMaxBucket)) return false;
    const int base = warp_incl_scan(c) - c;
    __syncwarp();
    cnt[l] = base;  // running cursor of bucket l
    __syncwarp();
    for (int p0 = 0; p0 < n; p0 += 32) {  // arrival order: stable
        const int p = p0 + l;
        const uint64_t v = p < n ? src[p] : 0ull;
        const int b = p < n ? (int)(((uint64_t)(uint32_t)(it_key(v) - mn) * mul) >> 32) : 32 + l;
        const unsigned g = __match_any_sync(kFull, b);
        if (p < n) dst[cnt[b] + __popc(g & lt)] = v;
        __syncwarp();
        if (p < n && (g & lt) == 0) cnt[b] += __popc(g);
        __syncwarp();
    }
    // insertion sort of bucket l
    for (int q = base + 1; q < base + c; ++q) {
        const uint64_t v = dst[q];
        int t = q - 1;
        while (t >= base && dst[t] > v) {
            dst[t + 1] = dst[t];
            --t;
        }
        dst[t + 1] = v;
    }
    __syncwarp();
    return true;
}

template <int FCAP>
__global__ void __launch_bounds__(kMidThreads, 8) k_num_mid(MidArgs a) {
    extern __shared__ __align__(16) unsigned char mid_smem[];
    MidSmem<FCAP> &S = reinterpret_cast<MidSmem<FCAP> *>(mid_smem)[threadIdx.x >> 5];
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
        const int64_t wbase = i - kMidWinHalf;
        bool prefetched = false;
        int nfar = 0, nruns = 0;
        // ---- accumulate: entries in ascending k.  A column of <= 32 rows is
        // one stage; stages are software-pipelined 4 deep so later columns'
        // gathers are in flight while one is applied.  Batches with a longer
        // column go through 32-lane pieces without the pipeline.
        auto apply = [&](int j, double b, double at, bool valid) {  // one piece of one column
            const int d = (int)((int64_t)j - wbase);
            const bool near = valid && (unsigned)d < (unsigned)kMidWin;
            if (near && !(a.dbg & 16)) S.wv[d] = __fma_rn(at, b, S.wv[d]);
            const bool far = valid && !near && !(a.dbg & 32);
            const unsigned fm = __ballot_sync(kFull, far);
            const int pos = nfar + __popc(fm & lt);
            if (far && pos < FCAP) {
                S.m0[pos] = mk_item(j, nruns < FCAP ? nruns : 0, pos);
                S.fb[pos] = b;
            }
            return fm;
        };
        auto close_run = [&](int cnt, double at) {  // a column's far keys form one run
            if (cnt) {
                if (l == 0 && nruns < FCAP && nfar < FCAP) {
                    S.rs[nruns] = (uint16_t)nfar;
                    S.ra[nruns] = at;
                }
                nfar += cnt;
                ++nruns;
            }
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
                S.ecs[l] = c0 + k;  // sentinel layout (csc_begin)
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
                // columns of <= 32 rows: lane l holds row l of column t.  The
                // gathers run kDepth columns ahead of the column being applied.
                constexpr int kDepth = 8;
                int pj[kDepth];
                double pb[kDepth];
#pragma unroll
                for (int u = 0; u < kDepth; ++u) {
                    pj[u] = 0;
                    pb[u] = 0.0;
                    const int len = __shfl_sync(kFull, clen, u < nent ? u : 0);
                    if (u < nent && l < len) {
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
                            const int len = __shfl_sync(kFull, clen, t);
                            const double at = S.ea[t];
                            close_run(__popc(apply(pj[u], pb[u], at, l < len)), at);
                            const int tn = t + kDepth;
                            const int lenn = __shfl_sync(kFull, clen, tn < nent ? tn : 0);
                            if (tn < nent && l < lenn) {
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
                    int cnt = 0;
                    for (int off = 0; off < len; off += 32) {
                        const bool valid = off + l < len;
                        int j = 0;
                        double b = 0.0;
                        if (valid) {
                            j = a.T.ri[q0 + off + l];
                            b = a.T.vt[q0 + off + l];
                        }
                        nfar += cnt;  // the pieces of one column extend one run
                        const unsigned fm = apply(j, b, at, valid);
                        nfar -= cnt;
                        cnt += __popc(fm);
                    }
                    close_run(cnt, at);
                }
            }
            __syncwarp();
        }
        if (!prefetched) load_meta(idx + nw, nxt);
        cur = nxt;
        __syncwarp();
        if (nfar > FCAP) {  // far list overflow: reset, defer the row to the next capacity
            for (int t = l; t < kMidWin; t += 32) S.wv[t] = +0.0;
            if (l == 0) a.defer_list[atomicAdd((unsigned long long *)a.defer_count, 1ull)] = (int32_t)i;
            __syncwarp();
            continue;
        }
        // ---- sort the far items: buckets (usual) or stable pairwise run merges
        const uint64_t *srt = S.m0;
        if (nruns > 1 && !(a.dbg & 1)) {
            uint64_t *dst = S.m1;
            if (bucket_sort_far(S.m0, dst, S.bcnt, nfar)) {
                srt = dst;
            } else {
                uint64_t *src = S.m0;
                if (l == 0) S.rs[nruns] = (uint16_t)nfar;
                __syncwarp();
                for (int lv = 0; (1 << lv) < nruns; ++lv) {
                    merge_level(src, dst, S.rs, nruns, lv, nfar);
                    __syncwarp();
                    uint64_t *tmp = src;
                    src = dst;
                    dst = tmp;
                }
                srt = src;
            }
        }
        // ---- emit in ascending j: far below, window, far above
        const int64_t g0 = a.toff[r];
        int64_t o = 0;
        auto emit = [&](bool keep, int key, double w) {
            const unsigned bal = __ballot_sync(kFull, keep);
            if (keep && !(a.dbg & 4)) {
                const int64_t pos = g0 + o + __popc(bal & lt);
                a.tcol[pos] = key;
                a.tw[pos] = w;
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
                    const uint64_t v = srt[p];
                    key = it_key(v);
                    if (p == 0 || it_key(srt[p - 1]) != key) {
                        double acc = +0.0;
                        int q = p;
                        do {
                            const uint64_t x = srt[q];
                            acc = __fma_rn(S.ra[it_run(x)], S.fb[it_idx(x)], acc);
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
            nbelow += __popc(__ballot_sync(kFull, p < nfar && (int64_t)it_key(srt[p]) < wbase));
        }
        if (a.dbg & 2) nbelow = nfar = 0;
        emit_far(0, nbelow);
        for (int t = l; t < kMidWin; t += 32) {
            const int64_t key = wbase + t;
            const double c = S.wv[t];
            S.wv[t] = +0.0;
            if (key == i && a.diag) a.diag[r] = c;
            const double w = fabs(c);
            emit(key != i && w > a.tol, (int)key, w);  // untouched slots hold +0.0: never kept
        }
        emit_far(nbelow, nfar);
        if (l == 0) a.cnt[r] = o + 1;  // the scan subtracts the diagonal slot
        __syncwarp();
    }
}

template <int FCAP>
static void launch_mid_t(const MidArgs &a, cudaStream_t s) {
    const size_t smem = (size_t)kMidWarps * sizeof(MidSmem<FCAP>);
    cudaFuncSetAttribute(k_num_mid<FCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_num_mid<FCAP>, kMidThreads, smem);
    if (per_sm < 1) per_sm = 1;
    int g = num_sms() * per_sm;
    if (g > kCutSlotsPerLaunch) g = kCutSlotsPerLaunch;
    k_num_mid<FCAP><<<g, kMidThreads, smem, s>>>(a);
    note_launch();
}

void launch_num_mid(const MidArgs &a, int fcap, cudaStream_t s) {
    if (fcap <= 256)
        launch_mid_t<256>(a, s);
    else
        launch_mid_t<2048>(a, s);
}

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
        for (int64_t t = l; t < len; t += 32) {
            const int32_t j = tcol[src + t];
            const double w = tw[src + t];
            gcol[d + t] = j;
            gw[d + t] = w;
            if (cut.part && (int64_t)j > i) {
                const int32_t pj = __ldg(&cut.part[j]);
                badp |= (pj < 0) | (pj >= cut.K);
                if (pj != pi) acc.add(w);
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

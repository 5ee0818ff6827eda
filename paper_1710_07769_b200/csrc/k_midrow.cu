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
//    arrival (= ascending k) order.  Each piece's far keys ascend (the column
//    is sorted), so the list is a concatenation of sorted runs; runs are
//    merged pairwise by a warp merge path (stable: on equal keys the earlier
//    run first) in ceil(log2 runs) rounds.  Equal keys are then adjacent in
//    ascending k and their products are folded in that order.
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
    uint64_t m0[FCAP], m1[FCAP];  // merge buffers: (key << 32) | (run << 16) | arrival index
    int64_t ecs[32];              // batch of row entries: CSC start, length, a_hat_ik
    int elen[32];
    double ea[32];
    uint16_t rs[FCAP + 1];        // run starts in the far list
};

// One column (<= 64 rows) of a row's batch: lane l holds rows l and l + 32.
struct Stage {
    int j0, j1;
    double b0, b1;  // a_hat_jk
    double a;       // a_hat_ik (uniform)
    bool v0, v1;
};

__device__ __forceinline__ bool is_near(int j, int64_t wbase) {
    const int64_t d = (int64_t)j - wbase;
    return d >= 0 && d < kMidWin;
}

__device__ __forceinline__ void fetch_stage(const Csc &T, const int64_t *ecs, const int *elen, const double *ea, int t,
                                            int nent, Stage &P) {
    const int l = lane_id();
    P.v0 = P.v1 = false;
    P.j0 = P.j1 = 0;
    P.b0 = P.b1 = 0.0;
    P.a = 0.0;
    if (t >= nent) return;
    const int64_t q0 = ecs[t];
    const int len = elen[t];
    P.a = ea[t];
    P.v0 = l < len;
    P.v1 = l + 32 < len;
    if (P.v0) {
        P.j0 = T.ri[q0 + l];
        P.b0 = T.vt[q0 + l];
    }
    if (P.v1) {
        P.j1 = T.ri[q0 + 32 + l];
        P.b1 = T.vt[q0 + 32 + l];
    }
}

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

template <int FCAP>
__global__ void __launch_bounds__(kMidThreads, 8) k_num_mid(MidArgs a) {
    extern __shared__ __align__(16) unsigned char mid_smem[];
    MidSmem<FCAP> &S = reinterpret_cast<MidSmem<FCAP> *>(mid_smem)[threadIdx.x >> 5];
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    Comp cut;
    int badp = 0;
    for (int t = l; t < kMidWin; t += 32) S.wv[t] = +0.0;
    __syncwarp();
    const int64_t n = *a.count;
    const int64_t nw = (int64_t)gridDim.x * kMidWarps;
    for (int64_t idx = blockIdx.x * (int64_t)kMidWarps + (threadIdx.x >> 5); idx < n; idx += nw) {
        const int64_t i = a.list[idx];
        const int64_t r = i - a.rb;
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        const int64_t wbase = i - kMidWinHalf;
        int nfar = 0, nruns = 0;
        // ---- accumulate: entries in ascending k.  A column of <= 64 rows is
        // one stage (two elements per lane); stages are software-pipelined 4
        // deep so later columns' gathers are in flight while one is applied.
        // Longer columns go through 32-lane pieces without the pipeline.
        auto apply = [&](int j, double b, double at, bool valid) {
            const int64_t d = (int64_t)j - wbase;
            const bool near = valid && d >= 0 && d < kMidWin;
            if (near) S.wv[d] = __fma_rn(at, b, S.wv[d]);
            const bool far = valid && !near;
            const unsigned fm = __ballot_sync(kFull, far);
            if (fm) {
                const int pos = nfar + __popc(fm & lt);
                if (far && pos < FCAP) {
                    S.m0[pos] = mk_item(j, nruns < FCAP ? nruns : 0, pos);
                    S.fb[pos] = b;
                }
                return true;
            }
            return false;
        };
        auto close_run = [&](unsigned any, int cnt, double at) {  // one far run per column
            if (any) {
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
            if (l < nent) {
                const int k = a.A.ci[bb + l];
                const int64_t c0 = a.T.cp[k];
                clen = (int)(a.T.cp[k + 1] - c0);
                S.ecs[l] = c0 + k;  // sentinel layout (csc_begin)
                S.elen[l] = clen;
                S.ea[l] = a.A.v[bb + l];
            }
            const bool short_cols = __all_sync(kFull, clen <= 64);
            __syncwarp();
            if (short_cols) {
                Stage P[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) fetch_stage(a.T, S.ecs, S.elen, S.ea, u, nent, P[u]);
                for (int t0 = 0; t0 < nent; t0 += 4) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (t0 + u < nent) {
                            Stage &Q = P[u];
                            // lower half then upper half: the column's keys ascend
                            const unsigned f0 = __ballot_sync(kFull, Q.v0 && !is_near(Q.j0, wbase));
                            apply(Q.j0, Q.b0, Q.a, Q.v0);
                            const int c0n = __popc(f0);
                            // the upper half appends after the lower half of the same run
                            nfar += c0n;
                            const unsigned f1 = __ballot_sync(kFull, Q.v1 && !is_near(Q.j1, wbase));
                            apply(Q.j1, Q.b1, Q.a, Q.v1);
                            nfar -= c0n;
                            close_run(f0 | f1, c0n + __popc(f1), Q.a);
                            fetch_stage(a.T, S.ecs, S.elen, S.ea, t0 + u + 4, nent, Q);
                        }
                    }
                }
            } else {
                for (int t = 0; t < nent; ++t) {
                    const int64_t q0 = S.ecs[t];
                    const int len = S.elen[t];
                    const double at = S.ea[t];
                    int cnt = 0;
                    unsigned any = 0;
                    for (int off = 0; off < len; off += 32) {
                        const bool valid = off + l < len;
                        int j = 0;
                        double b = 0.0;
                        if (valid) {
                            j = a.T.ri[q0 + off + l];
                            b = a.T.vt[q0 + off + l];
                        }
                        const unsigned fm = __ballot_sync(kFull, valid && !is_near(j, wbase));
                        nfar += cnt;
                        apply(j, b, at, valid);
                        nfar -= cnt;
                        cnt += __popc(fm);
                        any |= fm;
                    }
                    close_run(any, cnt, at);
                }
            }
            __syncwarp();
        }
        __syncwarp();
        if (nfar > FCAP) {  // far list overflow: reset, defer the row to the next capacity
            for (int t = l; t < kMidWin; t += 32) S.wv[t] = +0.0;
            if (l == 0) a.defer_list[atomicAdd((unsigned long long *)a.defer_count, 1ull)] = (int32_t)i;
            __syncwarp();
            continue;
        }
        // ---- stable pairwise merges of the far runs
        uint64_t *src = S.m0, *dst = S.m1;
        if (l == 0) S.rs[nruns] = (uint16_t)nfar;
        __syncwarp();
        for (int lv = 0; (1 << lv) < nruns; ++lv) {
            merge_level(src, dst, S.rs, nruns, lv, nfar);
            __syncwarp();
            uint64_t *tmp = src;
            src = dst;
            dst = tmp;
        }
        // ---- emit in ascending j: far below, window, far above
        const int64_t g0 = a.toff[r];
        int32_t pi = 0;
        if (a.part) {
            pi = a.part[i];
            badp |= (pi < 0) | (pi >= a.K);
        }
        int64_t o = 0;
        auto emit = [&](bool keep, int key, double w) {
            const unsigned bal = __ballot_sync(kFull, keep);
            if (keep) {
                const int64_t pos = g0 + o + __popc(bal & lt);
                a.tcol[pos] = key;
                a.tw[pos] = w;
                if (a.part && (int64_t)key > i) {
                    const int32_t pj = a.part[key];
                    badp |= (pj < 0) | (pj >= a.K);
                    if (pj != pi) cut.add(w);
                }
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
                    const uint64_t v = src[p];
                    key = it_key(v);
                    if (p == 0 || it_key(src[p - 1]) != key) {
                        double acc = +0.0;
                        int q = p;
                        do {
                            const int x = it_idx(src[q]);
                            acc = __fma_rn(S.ra[it_run(src[q])], S.fb[x], acc);
                            ++q;
                        } while (q < nfar && it_key(src[q]) == key);
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
            nbelow += __popc(__ballot_sync(kFull, p < nfar && (int64_t)it_key(src[p]) < wbase));
        }
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
    if (a.part) {
        const double v = block_tree_sum<kMidThreads>(cut.value());
        if (threadIdx.x == 0) {
            a.cutp[blockIdx.x] = v;
            if (blockIdx.x == 0) *a.cut_used = (int)gridDim.x;
        }
        if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(a.bad_part, 1);
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
// slots [gptr[r], gptr[r+1]).  One warp per row, coalesced.
__global__ void __launch_bounds__(256) k_copy_rows(const int32_t *__restrict__ list, const int64_t *count,
                                                   int64_t rb, const int64_t *__restrict__ toff,
                                                   const int64_t *__restrict__ gptr, const int32_t *__restrict__ tcol,
                                                   const double *__restrict__ tw, int32_t *gcol, double *gw) {
    const int l = lane_id();
    const int64_t n = *count;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < n; idx += nw) {
        const int64_t r = list[idx] - rb;
        const int64_t src = toff[r], d = gptr[r], len = gptr[r + 1] - d;
        for (int64_t t = l; t < len; t += 32) {
            gcol[d + t] = tcol[src + t];
            gw[d + t] = tw[src + t];
        }
    }
}

void launch_copy_rows(const int32_t *list, const int64_t *count, int64_t rb, const int64_t *toff, const int64_t *gptr,
                      const int32_t *tcol, const double *tw, int32_t *gcol, double *gw, cudaStream_t s) {
    k_copy_rows<<<num_sms() * 8, 256, 0, s>>>(list, count, rb, toff, gptr, tcol, tw, gcol, gw);
    note_launch();
}

}  // namespace rig

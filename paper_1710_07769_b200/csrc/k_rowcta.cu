// k_rowcta.cu -- steps a5 + a6 for long rows of scattered columns (the mixed
// path's tail: power-law rows, SURVEY §8(d) D2 config 4, and f3's config 6):
// one CTA per row of C = A_hat A_hat^T (Gustavson) in
// shared memory, expand -> stable sort -> fold (ESC).  These rows have no
// window locality (their keys are spread over all of [0, n)), so the
// row-window kernel's window is useless to them and its far list spills to
// global scratch; here the whole row lives in shared memory.
//
// Per row i (ordering contract, DESIGN.md §3 R4):
//  * expand: the row's entries k ascending, 256 at a time; each thread writes
//    its column's products (key j, a_ik, a_jk) at its exclusive-scan offset,
//    so the items are numbered in arrival (= ascending k) order;
//  * sort: stable LSD radix sort of (key, item) by key, 8-bit digits, as many
//    passes as n needs; each warp ranks its own contiguous slice of items in
//    order (match_any inside a round, rounds in order) and the offsets are
//    scanned digit-major, warp-minor -- stable, so equal keys stay in arrival
//    order;
//  * fold: the first item of each equal-key group folds the group in that
//    order (the R4 chain), kept iff j != i and |c| > tol (PAPER.md:295-315,
//    352); the kept entries are written with the row's exact count to the
//    temporary at toff[r] (cnt[r] = kept + 1, as the other mid-row kernels),
//    and k_copy_rows places them and takes their cut.
// Rows with more products than the shared arrays hold go to `rest` (the
// wide-window / global-far-list / CTA-accumulator chain), or, in the RANGE
// instantiation (a second launch with larger arrays), through key ranges:
//  * expand the row's f items in arrival order into this CTA's slice of
//    global scratch (key, a_ik, a_jk);
//  * one stable counting pass by the key's top 8 bits (256 buckets, the same
//    per-warp ordered ranking) into the slice's second half: each bucket's
//    items stay in arrival order;
//  * consecutive buckets are grouped into ranges of at most fmax items; each
//    range is loaded into shared memory (relative keys), sorted by the stable
//    LSD passes its width needs and folded as above -- ranges ascend, so the
//    row comes out in ascending j.  A bucket of more than fmax items, or a row
//    beyond the slice, goes to `rest`.
#include "common.cuh"

namespace rig {

constexpr int kRcThreads = 256;
constexpr int kRcWarps = kRcThreads / 32;
constexpr int kRcBins = 256;

__host__ __device__ constexpr size_t rc_item_bytes() { return 4 + 4 + 2 + 2 + 8 + 8; }
size_t rowcta_smem_bytes(int fmax, bool range) {
    return (size_t)fmax * rc_item_bytes() + (size_t)kRcWarps * kRcBins * 4 + 32 * 4 + 8 * 8 +
           (range ? (size_t)(kRcWarps + 1) * (kRcBins + 4) * 4 + (size_t)kRcBins * 16 : 0);
}
size_t rowcta_scratch_bytes(int64_t scap, int grid) { return (size_t)grid * (size_t)scap * (2 * 4 + 4 * 8); }

// Block-wide exclusive scan of one int per thread (256 threads); *total gets
// the sum.  Uses `ws` (kRcWarps + 1 ints of shared memory).
__device__ __forceinline__ int rc_block_scan(int v, int *ws, int *total) {
    const int l = lane_id(), w = threadIdx.x >> 5;
    const int inc = warp_incl_scan(v);
    if (l == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int x = l < kRcWarps ? ws[l] : 0;
        const int xi = warp_incl_scan(x);
        if (l < kRcWarps) ws[l] = xi - x;
        if (l == kRcWarps - 1) ws[kRcWarps] = xi;
    }
    __syncthreads();
    const int r = ws[w] + inc - v;
    *total = ws[kRcWarps];
    __syncthreads();
    return r;
}

// Shared arrays of one CTA (fmax items).
struct RcSmem {
    double *ia, *ib;         // a_ik, a_jk of item
    unsigned *key0, *key1;   // (relative) keys, ping-pong
    unsigned *hist;          // [warp][bin], then offsets
    int *ws;                 // block-scan scratch
    int64_t *misc;           // broadcast slots
    int *bst;                // RANGE: bucket starts [kRcBins + 1]
    int *sub;                // RANGE: per-warp sub-bucket starts [kRcWarps][kRcBins + 4]
    int2 *dsc;               // RANGE: ranges (first, end bucket) [kRcBins]
    int *kept, *koff;        // RANGE: kept count, output offset per range [kRcBins]
    uint16_t *idx0, *idx1;   // item numbers, ping-pong
};

__device__ __forceinline__ RcSmem rc_carve(unsigned char *smem, int F, bool range) {
    RcSmem S;
    S.ia = reinterpret_cast<double *>(smem);
    S.ib = S.ia + F;
    S.key0 = reinterpret_cast<unsigned *>(S.ib + F);
    S.key1 = S.key0 + F;
    S.hist = S.key1 + F;
    S.ws = reinterpret_cast<int *>(S.hist + kRcWarps * kRcBins);
    S.misc = reinterpret_cast<int64_t *>(S.ws + 32);
    S.bst = reinterpret_cast<int *>(S.misc + 8);
    S.sub = S.bst + kRcBins + 4;
    S.dsc = reinterpret_cast<int2 *>(S.sub + kRcWarps * (kRcBins + 4));
    S.kept = reinterpret_cast<int *>(S.dsc + kRcBins);
    S.koff = S.kept + kRcBins;
    S.idx0 = reinterpret_cast<uint16_t *>(range ? S.koff + kRcBins : S.bst);
    S.idx1 = S.idx0 + F;
    return S;
}

// Digit-major, warp-minor exclusive offsets of the per-warp digit counts in
// hist (thread b owns digit b); returns digit tid's total, and its start in
// *start.
__device__ __forceinline__ int rc_offsets(unsigned *hist, int *ws, int *start) {
    const int tid = threadIdx.x;
    int c[kRcWarps], sum = 0;
#pragma unroll
    for (int u = 0; u < kRcWarps; ++u) {
        c[u] = hist[u * kRcBins + tid];
        sum += c[u];
    }
    int tot;
    int run = rc_block_scan(sum, ws, &tot);
    *start = run;
#pragma unroll
    for (int u = 0; u < kRcWarps; ++u) {
        hist[u * kRcBins + tid] = run;
        run += c[u];
    }
    __syncthreads();
    return sum;
}

// Stable LSD radix sort of the nit items in shared memory by their relative
// key (key0, `passes` 8-bit digits), then the first item of each equal-key
// group folds the group in arrival order (the R4 chain); kept entries (key
// klo + k, j != i, |c| > tol) go to tcol/tw from t0.  Returns the kept count.
__device__ __forceinline__ int rc_sort_fold(const RcArgs &a, const RcSmem &S, int nit, int64_t klo, int passes,
                                            int64_t i, int64_t r, int64_t t0) {
    const int tid = threadIdx.x, l = lane_id(), w = tid >> 5;
    const unsigned lt = lanemask_lt();
    unsigned *kin = S.key0, *kout = S.key1;
    uint16_t *xin = S.idx0, *xout = S.idx1;
    const int chunk = ((nit + kRcWarps - 1) / kRcWarps + 31) / 32 * 32;
    const int w0 = min(nit, w * chunk), w1 = min(nit, w0 + chunk);
    for (int d = 0; d < passes; ++d) {
        const int sh = 8 * d;
        for (int b = tid; b < kRcWarps * kRcBins; b += kRcThreads) S.hist[b] = 0;
        __syncthreads();
        unsigned *hw = S.hist + w * kRcBins;
        for (int p0 = w0; p0 < w1; p0 += 32) {  // this warp's slice, in order
            const int p = p0 + l;
            const int dg = p < w1 ? (int)((kin[p] >> sh) & 255u) : kRcBins + l;
            const unsigned g = __match_any_sync(kFull, dg);
            if (p < w1 && (g & lt) == 0) hw[dg] += __popc(g);
            __syncwarp();
        }
        __syncthreads();
        int start;
        rc_offsets(S.hist, S.ws, &start);
        for (int p0 = w0; p0 < w1; p0 += 32) {
            const int p = p0 + l;
            unsigned k = 0;
            int dg = kRcBins + l;
            if (p < w1) {
                k = kin[p];
                dg = (int)((k >> sh) & 255u);
            }
            const unsigned g = __match_any_sync(kFull, dg);
            if (p < w1) {
                const int pos = (int)hw[dg] + __popc(g & lt);
                kout[pos] = k;
                xout[pos] = xin[p];
            }
            __syncwarp();
            if (p < w1 && (g & lt) == 0) hw[dg] += __popc(g);
            __syncwarp();
        }
        __syncthreads();
        unsigned *tk = kin;
        kin = kout;
        kout = tk;
        uint16_t *tx = xin;
        xin = xout;
        xout = tx;
    }
    // ---- fold equal keys in arrival order, write the kept entries
    int obase = 0;
    for (int p0 = 0; p0 < nit; p0 += kRcThreads) {
        const int p = p0 + tid;
        bool keep = false;
        unsigned key = 0;
        double wv = 0.0;
        if (p < nit) {
            key = kin[p];
            if (p == 0 || kin[p - 1] != key) {
                double acc = +0.0;
                for (int q = p; q < nit && kin[q] == key; ++q) {
                    const int x = xin[q];
                    acc = __fma_rn(S.ia[x], S.ib[x], acc);
                }
                if (klo + (int64_t)key == i) {
                    if (a.diag) a.diag[r] = acc;
                } else {
                    wv = fabs(acc);
                    keep = wv > a.tol;
                }
            }
        }
        int tot;
        const int pos = obase + rc_block_scan(keep ? 1 : 0, S.ws, &tot);
        if (keep) {
            a.tcol[t0 + pos] = (int32_t)(klo + key);
            a.tw[t0 + pos] = wv;
        }
        obase += tot;
    }
    return obase;
}

// Number of 8-bit LSD passes for keys in [0, width).
__device__ __forceinline__ int rc_passes(int64_t width) {
    int passes = 0;
    for (int64_t m = width - 1; m > 0; m >>= 8) ++passes;
    return passes;
}

// ---- RANGE mode (see the header): warp-level pieces.  A warp works on up
// to kRcFw items in its slice of the shared arrays (fmax = kRcWarps * kRcFw).
#ifndef RIG_RC_FW
#define RIG_RC_FW 384
#endif
constexpr int kRcFw = RIG_RC_FW;

struct RcWarp {
    double *ia, *ib;
    unsigned *k0, *k1;
    uint16_t *x0, *x1;
    unsigned *hist;  // 256 counters
    int *sub;        // 257 sub-bucket starts (crowded buckets)
};
__device__ __forceinline__ RcWarp rc_warp_view(const RcSmem &S, int w) {
    RcWarp W;
    W.ia = S.ia + w * kRcFw;
    W.ib = S.ib + w * kRcFw;
    W.k0 = S.key0 + w * kRcFw;
    W.k1 = S.key1 + w * kRcFw;
    W.x0 = S.idx0 + w * kRcFw;
    W.x1 = S.idx1 + w * kRcFw;
    W.hist = S.hist + w * kRcBins;
    W.sub = S.sub + w * (kRcBins + 4);
    return W;
}

// Warp-level stable counting pass of m items by digit dig(k): counts into
// hist, exclusive offsets (+ base) left in hist and, if `starts`, copied to
// starts[0..256] (starts[256] = base + m).  Items are read through `key(p)`
// and placed through `put(pos, p, k)`.
template <class Key, class Dig, class Put>
__device__ __forceinline__ void rc_warp_count_pass(unsigned *hist, int m, int base, int *starts, Key key, Dig dig,
                                                   Put put) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int q = 0; q < kRcBins / 32; ++q) hist[q * 32 + l] = 0;
    __syncwarp();
    for (int p0 = 0; p0 < m; p0 += 32) {
        const int p = p0 + l;
        const int dg = p < m ? dig(key(p)) : kRcBins + l;
        const unsigned g = __match_any_sync(kFull, dg);
        if (p < m && (g & lt) == 0) hist[dg] += __popc(g);
        __syncwarp();
    }
    // lane l owns bins [8l, 8l + 8)
    int c[kRcBins / 32], sum = 0;
#pragma unroll
    for (int q = 0; q < kRcBins / 32; ++q) {
        c[q] = (int)hist[l * (kRcBins / 32) + q];
        sum += c[q];
    }
    int run = base + warp_incl_scan(sum) - sum;
#pragma unroll
    for (int q = 0; q < kRcBins / 32; ++q) {
        hist[l * (kRcBins / 32) + q] = run;
        if (starts) starts[l * (kRcBins / 32) + q] = run;
        run += c[q];
    }
    if (starts && l == 31) starts[kRcBins] = run;
    __syncwarp();
    for (int p0 = 0; p0 < m; p0 += 32) {
        const int p = p0 + l;
        unsigned k = 0;
        int dg = kRcBins + l;
        if (p < m) {
            k = key(p);
            dg = dig(k);
        }
        const unsigned g = __match_any_sync(kFull, dg);
        if (p < m) put((int)hist[dg] + __popc(g & lt), p, k);
        __syncwarp();
        if (p < m && (g & lt) == 0) hist[dg] += __popc(g);
        __syncwarp();
    }
}

// One warp: m <= kRcFw items of keys in [klo, klo + 2^(8 passes)) from
// (gk, ga, gb)[0, m) -> stable sort in shared memory -> fold (R4 chain) ->
// kept (klo + key, |c|) to (ok, ow) from 0.  Returns the kept count.
__device__ int rc_warp_range(const RcArgs &a, const RcWarp &W, const int32_t *gk, const double *ga,
                             const double *gb, int m, int64_t klo, int passes, int64_t i, int64_t r, int32_t *ok,
                             double *ow) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    constexpr int U = 4;  // rounds per step: their global loads in flight together
    for (int p0 = l; p0 < m; p0 += 32 * U) {
        int kk[U];
        double xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = p0 + 32 * u;
            kk[u] = 0;
            xa[u] = xb[u] = 0.0;
            if (p < m) {
                kk[u] = gk[p];
                xa[u] = ga[p];
                xb[u] = gb[p];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = p0 + 32 * u;
            if (p < m) {
                W.k0[p] = (unsigned)(kk[u] - klo);
                W.x0[p] = (uint16_t)p;
                W.ia[p] = xa[u];
                W.ib[p] = xb[u];
            }
        }
    }
    __syncwarp();
    unsigned *kin = W.k0, *kout = W.k1;
    uint16_t *xin = W.x0, *xout = W.x1;
    for (int d = 0; d < passes; ++d) {
        const int sh = 8 * d;
        rc_warp_count_pass(
            W.hist, m, 0, nullptr, [&](int p) { return kin[p]; }, [&](unsigned k) { return (int)((k >> sh) & 255u); },
            [&](int pos, int p, unsigned k) {
                kout[pos] = k;
                xout[pos] = xin[p];
            });
        unsigned *tk = kin;
        kin = kout;
        kout = tk;
        uint16_t *tx = xin;
        xin = xout;
        xout = tx;
    }
    int o = 0;
    for (int p0 = 0; p0 < m; p0 += 32) {
        const int p = p0 + l;
        bool keep = false;
        unsigned key = 0;
        double wv = 0.0;
        if (p < m) {
            key = kin[p];
            if (p == 0 || kin[p - 1] != key) {
                double acc = +0.0;
                for (int q = p; q < m && kin[q] == key; ++q) {
                    const int x = xin[q];
                    acc = __fma_rn(W.ia[x], W.ib[x], acc);
                }
                if (klo + (int64_t)key == i) {
                    if (a.diag) a.diag[r] = acc;
                } else {
                    wv = fabs(acc);
                    keep = wv > a.tol;
                }
            }
        }
        const unsigned bal = __ballot_sync(kFull, keep);
        if (keep) {
            const int pos = o + __popc(bal & lt);
            ok[pos] = (int32_t)(klo + key);
            ow[pos] = wv;
        }
        o += __popc(bal);
    }
    __syncwarp();
    return o;
}

__device__ __forceinline__ int rc_bits(int64_t width) {
    int b = 0;
    while ((int64_t{1} << b) < width) ++b;
    return b;
}

// Expand row entries [s, e) in arrival order (entries k ascending, each
// column's rows ascending): per chunk of 256 entries a block scan of the
// column lengths, then the chunk's items are dealt to the threads round-robin
// (consecutive items to consecutive threads: coalesced stores, independent
// gathers); item q finds its entry by binary search over the chunk's
// offsets.  emit(o, j, a_ik, a_jk) for item o.  Uses the hist region for the
// chunk's entry metadata.  Returns the item count.
template <class Emit>
__device__ __forceinline__ int rc_expand(const RcArgs &a, int64_t s, int64_t e, const RcSmem &S, Emit emit) {
    const int tid = threadIdx.x;
    int *mofs = reinterpret_cast<int *>(S.hist);
    int *mcs = mofs + kRcThreads;
    double *mav = reinterpret_cast<double *>(mcs + kRcThreads);
    int base = 0;
    for (int64_t e0 = s; e0 < e; e0 += kRcThreads) {
        const int64_t p = e0 + tid;
        int cl = 0, cs = 0;
        double av = 0.0;
        if (p < e) {
            const int k = a.A.ci[p];
            const int64_t c0 = a.T.cp[k];
            cl = (int)(a.T.cp[k + 1] - c0);
            cs = (int)(c0 + k);  // CSC offsets fit int32 on this path (csc_fits_i32)
            av = a.A.v[p];
        }
        int tot;
        const int off = rc_block_scan(cl, S.ws, &tot);
        mofs[tid] = off;
        mcs[tid] = cs;
        mav[tid] = av;
        __syncthreads();
        const int ne = (int)min((int64_t)kRcThreads, e - e0);
#pragma unroll 4
        for (int q = tid; q < tot; q += kRcThreads) {
            int lo = 0, hi = ne - 1;  // the last entry whose offset is <= q
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (mofs[mid] <= q) lo = mid;
                else hi = mid - 1;
            }
            const int x = mcs[lo] + (q - mofs[lo]);
            emit(base + q, a.T.ri[x], mav[lo], a.T.vt[x]);
        }
        base += tot;
        __syncthreads();
    }
    return base;
}

// RANGE mode for one row of f > fmax items; returns false (nothing counted)
// if a key sub-bucket holds more than kRcFw items.
//  1. expand in arrival order into slice half 0 (key, a_ik, a_jk);
//  2. CTA-wide stable counting pass by bucket = key >> bsh (256 buckets)
//     into half 1; bucket starts in bst;
//  3. thread 0 groups consecutive buckets into ranges of <= kRcFw items (a
//     bucket beyond that is a range of its own: "crowded");
//  4. warps take ranges: sort + fold one range in shared memory (a crowded
//     bucket: first a warp-level counting pass by the next 8 key bits back
//     into half 0, then its sub-ranges in order; a sub-bucket still beyond
//     kRcFw fails the row); each range's kept entries are staged at its own
//     item offset (outputs never overtake inputs);
//  5. block scan of the ranges' kept counts, copy to the temporary in order.
__device__ __noinline__ bool rc_range_row(const RcArgs &a, const RcSmem &S, int64_t i, int64_t r, int64_t s,
                                          int64_t e, int f) {  // f: the row's products (key i included)
    const int tid = threadIdx.x, l = lane_id(), w = tid >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t sc = a.scap;
    int32_t *gk0 = a.skey + (int64_t)blockIdx.x * 2 * sc, *gk1 = gk0 + sc;
    double *ga0 = a.sval + (int64_t)blockIdx.x * 4 * sc, *gb0 = ga0 + sc, *ga1 = gb0 + sc, *gb1 = ga1 + sc;
    const int nb = rc_bits(a.A.nrows);
    const int bsh = nb > 8 ? nb - 8 : 0;
    const int bsh2 = bsh > 8 ? bsh - 8 : 0;
    // ---- 1. expand in arrival order into half 0.  Key i is dropped by the
    // bucket pass: every column k of row i holds i once, so c_ii is the chain
    // over the row's entries of a_ik * a_ik (thread 0; only for diag), and no
    // other key has more products than two rows share columns.
    if (tid == 0 && a.diag) {
        double acc = +0.0;
        for (int64_t p = s; p < e; ++p) {
            const double v = a.A.v[p];
            acc = __fma_rn(v, v, acc);
        }
        a.diag[r] = acc;
    }
    f = rc_expand(a, s, e, S, [&](int o, int j, double av, double b) {
        gk0[o] = j;
        ga0[o] = av;
        gb0[o] = b;
    });
    // ---- 2. stable counting pass by bucket into half 1 (warp slices in
    // order), without key i
    const int chunk = ((f + kRcWarps - 1) / kRcWarps + 31) / 32 * 32;
    const int w0 = min(f, w * chunk), w1 = min(f, w0 + chunk);
    for (int b = tid; b < kRcWarps * kRcBins; b += kRcThreads) S.hist[b] = 0;
    __syncthreads();
    unsigned *hw = S.hist + w * kRcBins;
    constexpr int U = 4;  // rounds per step: their global loads in flight together
    for (int p00 = w0; p00 < w1; p00 += 32 * U) {
        int kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = p00 + 32 * u + l;
            kk[u] = p < w1 ? gk0[p] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int dg = (kk[u] >= 0 && kk[u] != (int)i) ? kk[u] >> bsh : kRcBins + l;
            const unsigned g = __match_any_sync(kFull, dg);
            if (dg < kRcBins && (g & lt) == 0) hw[dg] += __popc(g);
            __syncwarp();
        }
    }
    __syncthreads();
    int start;
    const int bcnt = rc_offsets(S.hist, S.ws, &start);
    S.bst[tid] = start;
    if (tid == kRcThreads - 1) S.bst[kRcBins] = start + bcnt;
    for (int p00 = w0; p00 < w1; p00 += 32 * U) {
        int kk[U];
        double xx[U], yy[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = p00 + 32 * u + l;
            kk[u] = -1;
            xx[u] = yy[u] = 0.0;
            if (p < w1) {
                kk[u] = gk0[p];
                xx[u] = ga0[p];
                yy[u] = gb0[p];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int dg = (kk[u] >= 0 && kk[u] != (int)i) ? kk[u] >> bsh : kRcBins + l;
            const unsigned g = __match_any_sync(kFull, dg);
            if (dg < kRcBins) {
                const int pos = (int)hw[dg] + __popc(g & lt);
                gk1[pos] = kk[u];
                ga1[pos] = xx[u];
                gb1[pos] = yy[u];
            }
            __syncwarp();
            if (dg < kRcBins && (g & lt) == 0) hw[dg] += __popc(g);
            __syncwarp();
        }
    }
    __syncthreads();
    // ---- 3. ranges of consecutive buckets (in parallel, bucket per thread):
    // a bucket of more than T = kRcFw / 2 items is a range of its own; the
    // others group by start / T, so a group holds < T + T items
    constexpr int T = kRcFw / 2;
    const int st = S.bst[tid];
    const bool big = bcnt > T;
    const bool bigp = tid > 0 && S.bst[tid] - S.bst[tid - 1] > T;
    const bool flag = tid == 0 || big || bigp || st / T != S.bst[tid - 1] / T;
    int nr;
    const int rid = rc_block_scan(flag ? 1 : 0, S.ws, &nr);  // exclusive: ranges before this bucket's
    const int myr = rid + (flag ? 1 : 0) - 1;
    if (flag) S.dsc[myr].x = tid;
    if (tid == 0) {
        S.misc[2] = 0;  // failure flag
        S.misc[3] = 0;  // range queue
    }
    // a range ends where the next one starts
    if (flag && tid > 0) S.dsc[myr - 1].y = tid;
    if (tid == kRcThreads - 1) S.dsc[myr].y = kRcBins;
    __syncthreads();
    // ---- 4. warps take ranges from a queue
    const RcWarp W = rc_warp_view(S, w);
    for (;;) {
        int d = 0;
        if (l == 0) d = atomicAdd(reinterpret_cast<int *>(&S.misc[3]), 1);
        d = __shfl_sync(kFull, d, 0);
        if (d >= nr) break;
        const int lo = S.dsc[d].x, hi = S.dsc[d].y;
        const int b0 = S.bst[lo], m = S.bst[hi] - b0;
        const int64_t klo = (int64_t)lo << bsh;
        int kept = 0;
        if (m <= kRcFw) {
            const int64_t width = min((int64_t)(hi - lo) << bsh, a.A.nrows - klo);
            kept = rc_warp_range(a, W, gk1 + b0, ga1 + b0, gb1 + b0, m, klo, (rc_bits(width) + 7) / 8, i, r,
                                 gk0 + b0, ga0 + b0);
        } else {  // crowded bucket: sub-buckets by the next 8 key bits, into half 0
            rc_warp_count_pass(
                W.hist, m, 0, W.sub, [&](int p) { return (unsigned)gk1[b0 + p]; },
                [&](unsigned k) { return (int)((k >> bsh2) & 255u); },
                [&](int pos, int p, unsigned k) {
                    gk0[b0 + pos] = (int32_t)k;
                    ga0[b0 + pos] = ga1[b0 + p];
                    gb0[b0 + pos] = gb1[b0 + p];
                });
            __syncwarp();
            for (int sl = 0; sl < kRcBins;) {
                int sh_ = sl + 1;
                while (sh_ < kRcBins && W.sub[sh_ + 1] - W.sub[sl] <= kRcFw) ++sh_;
                const int sb0 = W.sub[sl], sm = W.sub[sh_] - sb0;
                if (sm > kRcFw) {  // one sub-bucket too crowded: the row goes to the fallback chain
                    if (l == 0) S.misc[2] = 1;
                    break;
                }
                if (sm > 0) {
                    const int64_t sklo = klo + ((int64_t)sl << bsh2);
                    const int64_t width = min((int64_t)(sh_ - sl) << bsh2, a.A.nrows - sklo);
                    // outputs go to half 1 of this bucket (consumed by the sub pass)
                    kept += rc_warp_range(a, W, gk0 + b0 + sb0, ga0 + b0 + sb0, gb0 + b0 + sb0, sm, sklo,
                                          (rc_bits(width) + 7) / 8, i, r, gk1 + b0 + kept, ga1 + b0 + kept);
                }
                sl = sh_;
            }
        }
        if (l == 0) S.kept[d] = kept;
    }
    __syncthreads();
    if (S.misc[2]) return false;
    // ---- 5. offsets of the ranges' outputs, copy to the temporary in order
    int tot;
    const int myk = tid < nr ? S.kept[tid] : 0;
    const int off = rc_block_scan(myk, S.ws, &tot);
    if (tid < nr) S.koff[tid] = off;
    __syncthreads();
    const int64_t t0 = a.toff[r];
    for (int d = w; d < nr; d += kRcWarps) {
        const int lo = S.dsc[d].x, hi = S.dsc[d].y;
        const int b0 = S.bst[lo], m = S.bst[hi] - b0;
        const int32_t *sk = m <= kRcFw ? gk0 + b0 : gk1 + b0;
        const double *sw = m <= kRcFw ? ga0 + b0 : ga1 + b0;
        const int kd = S.kept[d], od = S.koff[d];
        for (int p = l; p < kd; p += 32) {
            a.tcol[t0 + od + p] = sk[p];
            a.tw[t0 + od + p] = sw[p];
        }
    }
    if (tid == 0) a.cnt[r] = tot + 1;
    return true;
}

#ifndef RIG_RC_MINB
#define RIG_RC_MINB 2
#endif
template <bool RANGE>
__global__ void __launch_bounds__(kRcThreads, RANGE ? RIG_RC_MINB : 1) k_row_cta(RcArgs a) {
    extern __shared__ __align__(16) unsigned char rc_smem[];
    const int F = a.fmax;
    const RcSmem S = rc_carve(rc_smem, F, RANGE);
    const int tid = threadIdx.x;
    const int64_t n0 = *a.count0, n1 = a.list1 ? *a.count1 : 0;
    const int passes = rc_passes(a.A.nrows);
    // with ticket2: two rounds over the list, the rows beyond bigf products
    // first (longest work first: a long row started last would hold the
    // launch's tail), a ticket each
    for (int round = 0; round < (a.ticket2 ? 2 : 1); ++round)
    for (;;) {
        if (tid == 0) S.misc[0] = (int64_t)atomicAdd(round ? a.ticket2 : a.ticket, 1ull);
        __syncthreads();
        const int64_t t = S.misc[0];
        __syncthreads();
        if (t >= n0 + n1) break;
        const int64_t i = t < n0 ? a.list0[t] : a.list1[t - n0];
        const int64_t r = i - a.rb;
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        const int64_t f = a.fnm[r] + (e - s);
        if (a.ticket2 && ((f > a.bigf) != (round == 0))) continue;
        if (f > F) {
            const bool done = RANGE && f <= a.scap && rc_range_row(a, S, i, r, s, e, (int)f);
            if (!done && tid == 0) a.rest[atomicAdd((unsigned long long *)a.rest_count, 1ull)] = (int32_t)i;
            __syncthreads();
            continue;
        }
        // ---- expand in arrival order
        const int base = rc_expand(a, s, e, S, [&](int o, int j, double av, double b) {
            S.key0[o] = (unsigned)j;
            S.idx0[o] = (uint16_t)o;
            S.ia[o] = av;
            S.ib[o] = b;
        });
        const int nit = base;  // == f
        const int obase = rc_sort_fold(a, S, nit, 0, passes, i, r, a.toff[r]);
        if (tid == 0) a.cnt[r] = obase + 1;  // the graph scan subtracts the diagonal slot
        if (e == s && tid == 0 && a.diag) a.diag[r] = 0.0;
        __syncthreads();
    }
}

int rowcta_range_fmax() { return kRcWarps * kRcFw; }

// Grid of a launch for fmax (the RANGE launch's scratch is per CTA).
int rowcta_grid(int fmax, bool range) {
    const size_t smem = rowcta_smem_bytes(fmax, range);
    auto kern = range ? k_row_cta<true> : k_row_cta<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRcThreads, smem);
    if (per_sm < 1) per_sm = 1;
    return num_sms() * per_sm;
}

void launch_row_cta(const RcArgs &a, cudaStream_t s) {
    const bool range = a.skey != nullptr;
    const size_t smem = rowcta_smem_bytes(a.fmax, range);
    const int grid = rowcta_grid(a.fmax, range);
    if (range)
        k_row_cta<true><<<grid, kRcThreads, smem, s>>>(a);
    else
        k_row_cta<false><<<grid, kRcThreads, smem, s>>>(a);
    note_launch();
}

}  // namespace rig

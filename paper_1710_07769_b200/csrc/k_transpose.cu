// k_transpose.cu -- steps a1 (row scaling) + a2 (column access: CSC of A_hat)
// as a bucketed, deterministic transpose:
//
//   1. k_col_hist (k_prep.cu): per-column counts -> scan -> col_ptr cp.
//   2. k_bucket_scatter: a warp owns 32 consecutive rows; lane l computes the
//      norm of its row (ordered fma chain), then the warp
//      walks the rows' entries 32 at a time (coalesced), writes a_hat (coalesced)
//      and appends a 16-byte record (col, row, a_hat) to the entry's column
//      bucket (kBucketCols columns per bucket).  Lanes hitting the same bucket
//      share one atomic (__match_any_sync) and write contiguous records.
//   3. k_bucket_sort: one CTA per bucket loads its records into shared memory,
//      places them by column (counting sort), orders each column by row, and
//      writes the bucket's CSC slice with fully coalesced stores.
//
// CSC layout: column k occupies [cp[k] + k, cp[k+1] + k) followed by one
// sentinel (row = INT_MAX, value 0) at cp[k+1] + k, so consumers walking a
// column need no end bound (csc_begin()).  Rows ascend within each column.
#include <algorithm>

#include "common.cuh"

namespace rig {

// Bucket width 2^shift columns, chosen per matrix so an average bucket holds
// about kBucketTarget records; a warp sorts a bucket whose records plus one
// sentinel per column fit kBucketSlots, larger buckets go to a CTA-wide pass.
constexpr int kMinShift = 3, kMaxShift = 9;
constexpr int kMaxBucketCols = 1 << kMaxShift;
#ifndef RIG_BUCKET_TARGET
#define RIG_BUCKET_TARGET 256
#endif
constexpr int kBucketTarget = RIG_BUCKET_TARGET;
#ifndef RIG_BUCKET_SLOTS
#define RIG_BUCKET_SLOTS 640
#endif
constexpr int kBucketSlots = RIG_BUCKET_SLOTS;
#ifndef RIG_SMALL_BUCKET_SLOTS
#define RIG_SMALL_BUCKET_SLOTS 256
#endif
constexpr int kSmallBucketSlots = RIG_SMALL_BUCKET_SLOTS, kSmallBucketCols = 64;

struct __align__(16) Rec {
    int32_t col, row;
    double x;
};

// a /_rn b for b > 0 normal, given y = RN(1/b) (one reciprocal per row).
// Markstein: q0 = a*y, r = a - q0*b (exact by fma), q1 = q0 + r*y.  q1 is
// returned only if it is PROVEN to be RN(a/b): q1 normal and not a power of
// two (symmetric rounding interval) and the exact remainder a - q1*b, which
// the fma gives rounded monotonically, strictly inside b*ulp(q1)/2 (h is a
// power-of-two multiple of b, exact while normal).  Anything else falls back
// to __ddiv_rn, so the result is bit-identical to the IEEE division
// (R5) -- the fast path only skips work.
__device__ __forceinline__ double div_rn_fast(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-q0, b, a);
    const double q1 = __fma_rn(r, y, q0);
    const double r1 = __fma_rn(-q1, b, a);
    const long long bits = __double_as_longlong(q1);
    const int e = (int)((bits >> 52) & 0x7ff);
    if (e > 54 && e < 2046 && (bits & 0xfffffffffffffll) != 0) {
        const double h = __dmul_rn(b, __longlong_as_double((long long)(e - 53) << 52));  // b * ulp(q1) / 2
        if (h >= 0x1p-1000 && fabs(r1) < h) return q1;
    }
    return __ddiv_rn(a, b);
}

constexpr int kScatterThreads = 256;

// One warp per tile of 32 consecutive rows.  Lane l computes the norm of row
// r0 + l (ordered fma chain) and its reciprocal; the
// warp then walks the tile's entries 32 at a time (coalesced), finds each
// entry's row from the bitmask of row starts inside the chunk (no search),
// scales it, writes a_hat and appends a 16-byte record (col, row, a_hat) to
// the column's bucket; lanes hitting the same bucket share one atomic.
#ifdef RIG_SCATTER_MINB
#define RIG_SCATTER_BOUNDS __launch_bounds__(kScatterThreads, RIG_SCATTER_MINB)
#else
#define RIG_SCATTER_BOUNDS __launch_bounds__(kScatterThreads)
#endif
__global__ void RIG_SCATTER_BOUNDS k_bucket_scatter(Csr A, int scale, double *__restrict__ ahat,
                                                                    const int64_t *__restrict__ cp,
                                                                    unsigned long long *bcur, Rec *__restrict__ rec,
                                                                    int *err, int shift, const int *guard) {
    if (guard_skip(guard)) return;
    __shared__ int s_nz[kScatterThreads / 32][32];  // lane of the k-th nonempty row of the tile
    const int l = lane_id(), w = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t ntiles = (A.nrows + 31) / 32;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntiles; tile += nw) {
        const int64_t r0 = tile * 32;
        const int rows = (int)min((int64_t)32, A.nrows - r0);
        const int64_t hi = A.rp[r0 + rows];
        const int64_t my_s = l < rows ? A.rp[r0 + l] : hi;
        const int64_t my_e = l < rows ? A.rp[r0 + l + 1] : hi;
        double nrm = 1.0, y = 1.0;
        int bad = 0;
        if (scale && l < rows) {
            double ss = +0.0;
            for (int64_t p0 = my_s; p0 < my_e; p0 += 8) {  // 8 loads in flight, chain in order
                double av[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) av[u] = p0 + u < my_e ? A.v[p0 + u] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (p0 + u < my_e) ss = __fma_rn(av[u], av[u], ss);
            }
            if (!isfinite(ss)) {
                bad = kErrNonFinite;
            } else if (ss == 0.0) {
                bad = kErrZeroRow;
            } else {
                nrm = __dsqrt_rn(ss);
                y = __drcp_rn(nrm);
            }
        }
        if (bad) atomicOr(err, bad);
        const bool ne = my_e > my_s;
        const unsigned NE = __ballot_sync(kFull, ne);
        if (ne) s_nz[w][__popc(NE & lt)] = l;
        __syncwarp();
        const int64_t lo = __shfl_sync(kFull, my_s, 0);
        int cnt = NE ? 1 : 0;  // nonempty rows starting at or before c0
#ifndef RIG_SCATTER_U
#define RIG_SCATTER_U 2
#endif
        constexpr int U = RIG_SCATTER_U;  // chunks per group: their bucket atomics are in flight together
        for (int64_t g0 = lo; g0 < hi; g0 += 32 * U) {
            int kk[U], row[U], bb[U];
            double xx[U], av[U];
            unsigned gg[U];
            unsigned long long off[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {  // every chunk's loads first: in flight together
                const int64_t p = g0 + 32 * u + l;
                kk[u] = 0;
                av[u] = 0.0;
                if (p < hi) {
                    kk[u] = A.ci[p];
                    av[u] = A.v[p];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t c0 = g0 + 32 * u;
                // bit (rel - 1) for nonempty rows starting at c0 + rel, 1 <= rel <= 32
                const int64_t rel = my_s - c0;
                const unsigned S = __reduce_or_sync(kFull, (ne && rel >= 1 && rel <= 32) ? (1u << (rel - 1)) : 0u);
                const int k_row = cnt + __popc(S & ((1u << l) - 1u));  // nonempty starts <= c0 + l
                cnt += __popc(S);
                row[u] = s_nz[w][(k_row > 0 ? k_row : 1) - 1];
                const double rn = shfl_d(nrm, row[u]), ry = shfl_d(y, row[u]);
                const int64_t p = c0 + l;
                const bool valid = p < hi;
                xx[u] = 0.0;
                if (valid) {
                    xx[u] = scale ? div_rn_fast(av[u], rn, ry) : av[u];
                    if (scale) ahat[p] = xx[u];
                }
                bb[u] = valid ? (kk[u] >> shift) : -1 - l;
                gg[u] = __match_any_sync(kFull, bb[u]);
                off[u] = 0;
                if (valid && l == __ffs(gg[u]) - 1) off[u] = atomicAdd(&bcur[bb[u]], (unsigned long long)__popc(gg[u]));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned long long o = __shfl_sync(kFull, off[u], __ffs(gg[u]) - 1);
                if (bb[u] >= 0) {
                    const int64_t pos = (int64_t)o + __popc(gg[u] & lt);  // bcur holds absolute positions
                    Rec r;
                    r.col = kk[u];
                    r.row = (int32_t)(r0 + row[u]);
                    r.x = xx[u];
                    rec[pos] = r;
                }
            }
        }
        __syncwarp();
    }
}

// Ascending-only bitonic network over a virtual power-of-two length with
// +inf padding past `len` (pairs whose upper index is >= len never swap).
template <typename KeyAt, typename Swap>
__device__ void bitonic_sort_block(int64_t len, KeyAt key, Swap swap) {
    int64_t P = 1;
    while (P < len) P <<= 1;
    for (int64_t size = 2; size <= P; size <<= 1) {
        const int64_t half = size >> 1;
        for (int64_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
            const int64_t blk = t / half, off = t % half;
            const int64_t i = blk * size + off, j = blk * size + size - 1 - off;
            if (j < len && key(i) > key(j)) swap(i, j);
        }
        __syncthreads();
        for (int64_t str = size >> 2; str > 0; str >>= 1) {
            for (int64_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
                const int64_t i = (t / str) * 2 * str + (t % str), j = i + str;
                if (j < len && key(i) > key(j)) swap(i, j);
            }
            __syncthreads();
        }
    }
}

// Bucket cursors start at the bucket's first record slot (cp of its first
// column), so the scatter's atomics return absolute positions.
__global__ void k_bucket_init(const int64_t *__restrict__ cp, int64_t nb, int shift, unsigned long long *bcur,
                              const int *guard) {
    if (guard_skip(guard)) return;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        bcur[b] = (unsigned long long)cp[b << shift];
}

#ifndef RIG_RANK_U4
#define RIG_RANK_U4 1
#endif
// r += (a < b), as a compare and a predicated add
__device__ __forceinline__ void count_lt(int &r, int a, int b) {
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p add.s32 %0, %0, 1; }" : "+r"(r) : "r"(a), "r"(b));
}

#ifndef RIG_RANK_PAD
#define RIG_RANK_PAD 1  // small buckets: padded key copies, four compares per shared load (config 5 sort 1.07 -> 0.99 ms)
#endif
#ifndef RIG_SMALL_RANK
#define RIG_SMALL_RANK 1  // small buckets: rank (1) or per-lane insertion sorts (0; measured)
#endif
constexpr int kSortThreads = 64;  // 2 warps: one bucket per warp
constexpr int kSortWarps = kSortThreads / 32;

// One warp per bucket: records are placed by column into their CSC slots
// (column c of the bucket occupies [loff[c], loff[c+1] - 1), then its
// sentinel), each entry is ranked by row within its column, and the slice --
// entries and sentinels, in rank order -- is written with fully coalesced
// stores.  Buckets that do not fit are listed for
// k_bucket_sort_big.
// SLOTS / MAXC: shared capacity of a bucket (records + sentinels) and of its
// column count; a small instantiation (more warps per SM) serves matrices
// whose buckets are small, larger buckets go to the big list as usual.
template <bool RANK, int SLOTS = kBucketSlots, int MAXC = kMaxBucketCols>
__global__ void __launch_bounds__(kSortThreads) k_bucket_sort(const Rec *__restrict__ rec,
                                                              const int64_t *__restrict__ cp, int64_t ncols,
                                                              int32_t *ri, double *vt, int shift, int *big_list,
                                                              int *big_count, const int *guard) {
    if (guard_skip(guard)) return;
    __shared__ int32_t s_ri[kSortWarps][SLOTS];
    __shared__ double s_vt[kSortWarps][SLOTS];
    constexpr int RS = RANK ? SLOTS : 1;
    __shared__ uint16_t s_col[kSortWarps][RS];  // local column of a slot (0xffff: sentinel)
    __shared__ uint16_t s_inv[kSortWarps][RS];  // sorted position -> slot
    __shared__ uint16_t s_off[kSortWarps][MAXC + 1];
    __shared__ unsigned s_cur[kSortWarps][MAXC];
    // PAD (small instantiation): the rows once more, each column's keys from
    // a 16-byte aligned start and padded with INT_MAX to a multiple of four,
    // so the rank loop compares four keys per shared load and has no tail
    constexpr bool PAD = RANK && RIG_RANK_PAD != 0 && MAXC <= 64;
    constexpr int RKS = PAD ? SLOTS + 3 * MAXC + 8 : 4;
    __shared__ __align__(16) int32_t s_rk[kSortWarps][RKS];
    __shared__ uint16_t s_pdel[kSortWarps][PAD ? MAXC + 1 : 1];  // key slot - record slot of a column
    const int w = threadIdx.x >> 5, l = lane_id();
    int32_t *sr = s_ri[w];
    double *sv = s_vt[w];
    uint16_t *scol = s_col[w], *inv = s_inv[w];
    (void)scol;
    (void)inv;
    uint16_t *loff = s_off[w];
    unsigned *cur = s_cur[w];
    int32_t *srk = s_rk[w];
    uint16_t *pdel = s_pdel[w];
    (void)srk;
    (void)pdel;
    const int bcols = 1 << shift;
    const int64_t nb = (ncols + bcols - 1) / bcols;
    for (int64_t b = (int64_t)blockIdx.x * kSortWarps + w; b < nb; b += (int64_t)gridDim.x * kSortWarps) {
        const int64_t c0 = b << shift;
        const int ncb = (int)min((int64_t)bcols, ncols - c0);
        const int64_t e0 = cp[c0];
        const int64_t E = cp[c0 + ncb] - e0;
        if (E + ncb > SLOTS || ncb > MAXC) {
            if (l == 0) big_list[atomicAdd(big_count, 1)] = (int)b;
            continue;
        }
        // slot offsets include one sentinel per earlier column
        for (int c = l; c <= ncb; c += 32) {
            const int o = (int)(cp[c0 + c] - e0) + c;
            loff[c] = (uint16_t)o;
            if (c < ncb) cur[c] = (unsigned)o;
            if (RANK && c > 0) scol[o - 1] = 0xffff;  // sentinel slot of column c - 1
            // key slots: align4(entries before c + 3 c) (>= the previous
            // column's start + its length rounded up to four)
            if (PAD) pdel[c] = (uint16_t)((((o - c) + 3 * c + 3) & ~3) - o);
        }
        if (PAD) {
            const int tot4 = ((int)E + 3 * ncb + 6) / 4 + 1;
            for (int t = l; t < tot4; t += 32)
                reinterpret_cast<int4 *>(srk)[t] = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);
        }
        __syncwarp();
        for (int t0 = 0; t0 < (int)E; t0 += 128) {  // 4 record loads in flight per lane
            Rec rr[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + 32 * u + l;
                if (t < (int)E) {  // streamed: each record is read once
                    const int4 q = __ldcs(reinterpret_cast<const int4 *>(rec + e0 + t));
                    rr[u].col = q.x;
                    rr[u].row = q.y;
                    rr[u].x = __hiloint2double(q.w, q.z);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (t0 + 32 * u + l < (int)E) {
                    const int lc = rr[u].col - (int)c0;
                    const int pos = (int)atomicAdd(&cur[lc], 1u);
                    sr[pos] = rr[u].row;
                    sv[pos] = rr[u].x;
                    if (RANK) scol[pos] = (uint16_t)lc;
                    if (PAD) srk[pos + pdel[lc]] = rr[u].row;
                }
            }
        }
        __syncwarp();
        const int n = (int)E + ncb;
        if (RANK) {
            // order each column by row: an entry's rank in its column is the
            // number of entries of that column with a smaller row (rows are
            // distinct), so every slot is ranked independently -- no serial
            // insertion chains on long columns
            for (int q = l; q < n; q += 32) {
                const int c = scol[q];
                if (c == 0xffff) {
                    inv[q] = 0xffff;  // a sentinel stays at the end of its column
                    continue;
                }
                const int s0 = loff[c], e1 = loff[c + 1] - 1;
                const int rq = sr[q];
                if (PAD) {
                    const int4 *kp = reinterpret_cast<const int4 *>(srk + s0 + pdel[c]);
                    const int nv = (e1 - s0 + 3) >> 2;
                    int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
                    for (int v = 0; v < nv; ++v) {
                        const int4 k = kp[v];
                        // compare + predicated increment (two instructions per key;
                        // the compiler's own form is three)
                        count_lt(r0, k.x, rq);
                        count_lt(r1, k.y, rq);
                        count_lt(r2, k.z, rq);
                        count_lt(r3, k.w, rq);
                    }
                    inv[s0 + (r0 + r1) + (r2 + r3)] = (uint16_t)q;
                    continue;
                }
#if RIG_RANK_U4
                // four independent counts: the compares issue back to back
                // instead of one per loop trip (the loop was 2/3 of the kernel)
                int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
                int t = s0;
                for (; t + 4 <= e1; t += 4) {
                    count_lt(r0, sr[t], rq);
                    count_lt(r1, sr[t + 1], rq);
                    count_lt(r2, sr[t + 2], rq);
                    count_lt(r3, sr[t + 3], rq);
                }
                for (; t < e1; ++t) count_lt(r0, sr[t], rq);
                const int rank = (r0 + r1) + (r2 + r3);
#else
                int rank = 0;
                for (int t = s0; t < e1; ++t) rank += sr[t] < rq;
#endif
                inv[s0 + rank] = (uint16_t)q;
            }
        } else {
            // short columns: insertion sort by one lane per column
            for (int c = l; c < ncb; c += 32) {
                const int s0 = loff[c], e1 = loff[c + 1] - 1;  // [s0, e1) entries, e1 = sentinel slot
                for (int q = s0 + 1; q < e1; ++q) {
                    const int kr = sr[q];
                    const double kv = sv[q];
                    int t = q - 1;
                    while (t >= s0 && sr[t] > kr) {
                        sr[t + 1] = sr[t];
                        sv[t + 1] = sv[t];
                        --t;
                    }
                    sr[t + 1] = kr;
                    sv[t + 1] = kv;
                }
                sr[e1] = INT_MAX;
                sv[e1] = 0.0;
            }
        }
        __syncwarp();
        const int64_t out0 = e0 + c0;
        for (int t = l; t < n; t += 32) {
            const int q = RANK ? (int)inv[t] : t;
            ri[out0 + t] = q == 0xffff ? INT_MAX : sr[q];
            vt[out0 + t] = q == 0xffff ? 0.0 : sv[q];
        }
        __syncwarp();
    }
}

// Buckets too large for one warp: place with global per-column cursors, then
// sort each column in global memory (correct for any skew, slower).
__global__ void __launch_bounds__(128) k_bucket_sort_big(const Rec *__restrict__ rec, const int64_t *__restrict__ cp,
                                                         int64_t ncols, unsigned *gcur, int32_t *ri, double *vt,
                                                         int shift, const int *big_list, const int *big_count,
                                                         const int *guard) {
    if (guard_skip(guard)) return;
    const int bcols = 1 << shift;
    const int nbig = *big_count;
    for (int q = blockIdx.x; q < nbig; q += gridDim.x) {
        const int64_t b = big_list[q];
        const int64_t c0 = b << shift;
        const int ncb = (int)min((int64_t)bcols, ncols - c0);
        const int64_t e0 = cp[c0], E = cp[c0 + ncb] - e0;
        for (int64_t t = threadIdx.x; t < E; t += blockDim.x) {
            const Rec r = rec[e0 + t];
            const int64_t o = cp[r.col] + r.col + atomicAdd(&gcur[r.col], 1u);
            ri[o] = r.row;
            vt[o] = r.x;
        }
        for (int c = threadIdx.x; c < ncb; c += blockDim.x) {
            const int64_t o = cp[c0 + c + 1] + c0 + c;
            ri[o] = INT_MAX;
            vt[o] = 0.0;
        }
        __threadfence_block();
        __syncthreads();
        for (int c = 0; c < ncb; ++c) {
            const int64_t s = cp[c0 + c] + c0 + c, len = cp[c0 + c + 1] - cp[c0 + c];
            int32_t *gk = ri + s;
            double *gv = vt + s;
            bitonic_sort_block(
                len, [&](int64_t i) { return gk[i]; },
                [&](int64_t i, int64_t j) {
                    const int32_t tk = gk[i];
                    gk[i] = gk[j];
                    gk[j] = tk;
                    const double tv = gv[i];
                    gv[i] = gv[j];
                    gv[j] = tv;
                });
        }
        __syncthreads();
    }
}

int transpose_shift(int64_t nnz, int64_t ncols) {
    const double avg = ncols > 0 ? (double)nnz / (double)ncols : 1.0;
    int sh = kMinShift;
    while (sh < kMaxShift && (double)(1 << (sh + 1)) * (avg + 1.0) <= kBucketTarget) ++sh;
    return sh;
}

int64_t transpose_buckets(int64_t nnz, int64_t ncols) {
    const int sh = transpose_shift(nnz, ncols);
    return (ncols + (1 << sh) - 1) >> sh;
}

void launch_transpose(const Csr &A, int scale, const int64_t *cp, double *ahat, unsigned long long *bcur,
                      void *rec, unsigned *gcur, int *big, int32_t *ri, double *vt, int *err, cudaStream_t s,
                      const int *guard) {
    const int shift = transpose_shift(A.nnz, A.ncols);
    if (A.ncols > 0) {
        const int64_t nb = (A.ncols + (1 << shift) - 1) >> shift;
        int64_t g = (nb + 255) / 256;
        g = g > (int64_t)num_sms() * 4 ? (int64_t)num_sms() * 4 : g;
        k_bucket_init<<<(unsigned)g, 256, 0, s>>>(cp, nb, shift, bcur, guard);
        note_launch();
    }
    if (A.nrows > 0) {
        int64_t g = (A.nrows + kScatterThreads - 1) / kScatterThreads;
        const int64_t cap = (int64_t)num_sms() * 8;
        g = g < 1 ? 1 : (g > cap ? cap : g);
        k_bucket_scatter<<<(unsigned)g, kScatterThreads, 0, s>>>(A, scale, ahat, cp, bcur, static_cast<Rec *>(rec),
                                                                 err, shift, guard);
        note_launch();
    }
    if (A.ncols > 0) {
        const int64_t nb = (A.ncols + (1 << shift) - 1) >> shift;
        const int64_t cap = (int64_t)num_sms() * 16;
        int64_t g = (nb + kSortWarps - 1) / kSortWarps;
        g = g < cap ? g : cap;
        // big[0] = count of big buckets, big[1..] = their ids
        // long columns: parallel ranking; short ones: per-lane insertion sorts
        // buckets of <= ~200 records on average (2^shift <= 64 columns): the
        // small-capacity instantiation (a third of the shared memory per warp)
        const int64_t mean_bucket = A.nnz / (nb > 0 ? nb : 1) + (1 << shift);
        const bool small = (1 << shift) <= kSmallBucketCols && mean_bucket <= kSmallBucketSlots * 3 / 4;
        if (A.nnz > (int64_t)12 * A.ncols && small)
            k_bucket_sort<RIG_SMALL_RANK != 0, kSmallBucketSlots, kSmallBucketCols><<<(unsigned)std::min<int64_t>(
                                                                          (nb + kSortWarps - 1) / kSortWarps,
                                                                          (int64_t)num_sms() * 24),
                                                                      kSortThreads, 0, s>>>(
                static_cast<const Rec *>(rec), cp, A.ncols, ri, vt, shift, big + 1, big, guard);
        else if (A.nnz > (int64_t)12 * A.ncols)
            k_bucket_sort<true><<<(unsigned)g, kSortThreads, 0, s>>>(static_cast<const Rec *>(rec), cp, A.ncols, ri,
                                                                     vt, shift, big + 1, big, guard);
        else
            k_bucket_sort<false><<<(unsigned)g, kSortThreads, 0, s>>>(static_cast<const Rec *>(rec), cp, A.ncols, ri,
                                                                      vt, shift, big + 1, big, guard);
        k_bucket_sort_big<<<(unsigned)num_sms(), 128, 0, s>>>(static_cast<const Rec *>(rec), cp, A.ncols, gcur, ri,
                                                              vt, shift, big + 1, big, guard);
        note_launch(2);
    }
}

// ------------------------------------------------------------------ pattern-symmetric fast path
static int sym_grid(int64_t work, int block, int per_sm) {
    int64_t g = (work + block - 1) / block;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// Row norms for the gather: nrm_i = sqrt_rn(ordered fma chain of a_ik^2), y_i =
// RN(1/nrm_i) (the same arithmetic as k_bucket_scatter, R5).
__global__ void k_row_norms(Csr A, double *nrm, double *y, int *err, const int *fail) {
    if (*reinterpret_cast<const volatile int *>(fail)) return;  // the probe found a missing mirror
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.nrows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = A.rp[i], e = A.rp[i + 1];
        double ss = +0.0;
        for (int64_t p0 = s; p0 < e; p0 += 8) {  // 8 loads in flight, chain in order
            double av[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) av[u] = p0 + u < e ? A.v[p0 + u] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (p0 + u < e) ss = __fma_rn(av[u], av[u], ss);
        }
        double nm = 1.0, yy = 1.0;
        if (!isfinite(ss)) {
            atomicOr(err, kErrNonFinite);
        } else if (ss == 0.0) {
            atomicOr(err, kErrZeroRow);
        } else {
            nm = __dsqrt_rn(ss);
            yy = __drcp_rn(nm);
        }
        nrm[i] = nm;
        y[i] = yy;
    }
}

// Probe before the gather: 4096 entries spread over A; one without its mirror
// (or in a row longer than 64) sets *fail, so a non-symmetric matrix costs a
// few skipped launches instead of a failed gather.
__global__ void k_sym_probe(Csr A, int *fail) {
    const int64_t nprobe = 4096;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nprobe && t < A.nrows;
         t += (int64_t)gridDim.x * blockDim.x) {
        // row k spread over the matrix, an entry of it chosen by t
        const int64_t k = A.nrows <= nprobe ? t : t * (A.nrows / nprobe);
        const int64_t s = A.rp[k], e = A.rp[k + 1];
        if (e == s) continue;
        const int j = A.ci[s + (t % (e - s))];
        const int64_t sj = A.rp[j], ej = A.rp[j + 1];
        bool found = false;
        if (ej - sj <= 64)
            for (int64_t q = sj; q < ej && !found; ++q) found = A.ci[q] == (int)k;
        if (!found) atomicOr(fail, 1);
    }
}

// Column k of the CSC is row k's column list (mirror pattern), so
// col_ptr[k+1] = row_ptr[k+1] and CSR entry p of row k goes to CSC slot p + k
// (one sentinel per earlier column).  A warp takes 32 consecutive rows and
// walks their entries 32 at a time (coalesced loads and stores); lane p finds
// its row k by a shuffle binary search over the tile's row pointers, and the
// value a_hat_jk of the mirror entry (j, k) in row j: first at the mirrored
// position (stencil rows share their offset pattern: entry t of row k and
// entry len_j - 1 - t of row j are each other's mirror), else by a search of
// row j.  A missing mirror sets *fail; every warp then stops at its next chunk.
constexpr int kSymThreads = 128;
#ifndef RIG_SYM_MINB  // CTAs per SM the register budget is fitted to (measured 1, 6, 8)
#define RIG_SYM_MINB 8
#endif
__global__ void __launch_bounds__(kSymThreads, RIG_SYM_MINB) k_sym_transpose(Csr A, int scale, const double *__restrict__ nrm,
                                                               const double *__restrict__ y, double *ahat, int64_t *cp,
                                                               int32_t *ri, double *vt, int *fail) {
    const int l = lane_id();
    const int64_t ntiles = (A.nrows + 31) / 32;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntiles; tile += nw) {
        if (*reinterpret_cast<volatile int *>(fail)) return;
        const int64_t r0 = tile * 32;
        const int rows = (int)min((int64_t)32, A.nrows - r0);
        const int64_t my_s = l < rows ? A.rp[r0 + l] : A.rp[r0 + rows];
        const int64_t hi = A.rp[r0 + rows];
        if (l < rows) {
            cp[r0 + l + 1] = A.rp[r0 + l + 1];
            ri[A.rp[r0 + l + 1] + r0 + l] = INT_MAX;  // sentinel of column r0 + l
            vt[A.rp[r0 + l + 1] + r0 + l] = 0.0;
        }
        if (r0 == 0 && l == 0) cp[0] = 0;
        const double my_n = scale && l < rows ? nrm[r0 + l] : 1.0, my_y = scale && l < rows ? y[r0 + l] : 1.0;
#ifndef RIG_SYM_U
#define RIG_SYM_U 2  // measured 1, 2, 4 on config 3 (with 8 CTAs per SM: 2)
#endif
        constexpr int U = RIG_SYM_U;  // chunks of 32 entries in flight per warp
        for (int64_t c0 = __shfl_sync(kFull, my_s, 0); c0 < hi; c0 += 32 * U) {
            if (*reinterpret_cast<volatile int *>(fail)) return;
            int64_t p[U], k[U], q[U];
            int j[U], cq[U];
            double akj[U], nk[U], yk[U], nj[U], yj[U], vq[U];
#pragma unroll
            for (int t = 0; t < U; ++t) {  // round 1: the entry, its row (shuffle search)
                p[t] = c0 + 32 * t + l;
                int u = 0;
#pragma unroll
                for (int b = 16; b > 0; b >>= 1) {
                    const int64_t sv = __shfl_sync(kFull, my_s, u + b < rows ? u + b : rows - 1);
                    if (u + b < rows && sv <= p[t]) u += b;
                }
                k[t] = r0 + u;
                q[t] = __shfl_sync(kFull, my_s, u);  // row start, for the mirror guess
                nk[t] = shfl_d(my_n, u);
                yk[t] = shfl_d(my_y, u);
                j[t] = p[t] < hi ? A.ci[p[t]] : -1;
                akj[t] = p[t] < hi ? A.v[p[t]] : 0.0;
            }
            int64_t sj[U], ej[U];
#pragma unroll
            for (int t = 0; t < U; ++t) {  // round 2: row j's bounds and scale
                sj[t] = 0;
                ej[t] = 0;
                nj[t] = 1.0;
                yj[t] = 1.0;
                if (j[t] >= 0) {
                    sj[t] = A.rp[j[t]];
                    ej[t] = A.rp[j[t] + 1];
                    if (scale) {
                        nj[t] = nrm[j[t]];
                        yj[t] = y[j[t]];
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < U; ++t) {  // round 3: the mirrored position, column and value together
                q[t] = ej[t] - 1 - (p[t] - q[t]);
                cq[t] = -1;
                vq[t] = 0.0;
                if (j[t] >= 0 && q[t] >= sj[t] && q[t] < ej[t]) {
                    cq[t] = A.ci[q[t]];
                    vq[t] = A.v[q[t]];
                }
            }
#pragma unroll
            for (int t = 0; t < U; ++t) {
                if (j[t] < 0) continue;
                if (cq[t] != (int)k[t]) {  // search row j (short rows only: a longer one ends the attempt)
                    q[t] = -1;
                    if (ej[t] - sj[t] <= 64) {
                        for (int64_t b0 = sj[t]; b0 < ej[t] && q[t] < 0; b0 += 8) {
                            int cc[8];
#pragma unroll
                            for (int z = 0; z < 8; ++z) cc[z] = b0 + z < ej[t] ? A.ci[b0 + z] : -1;
#pragma unroll
                            for (int z = 0; z < 8; ++z)
                                if (cc[z] == (int)k[t]) q[t] = b0 + z;
                        }
                    }
                    if (q[t] < 0) {  // no mirror entry (j, k): not pattern-symmetric
                        atomicOr(fail, 1);
                        continue;
                    }
                    vq[t] = A.v[q[t]];
                }
                ri[p[t] + k[t]] = j[t];
                vt[p[t] + k[t]] = scale ? div_rn_fast(vq[t], nj[t], yj[t]) : vq[t];
                if (scale) ahat[p[t]] = div_rn_fast(akj[t], nk[t], yk[t]);
            }
        }
    }
}

// Shape statistics (DevCounters, see scan_u32_shape) from the row pointers:
// with a mirror pattern column k has as many entries as row k.  Runs only if
// the gather succeeded (guard = fail, inverted).
__global__ void k_sym_shape(const int64_t *__restrict__ rp, int64_t n, int64_t rb, int64_t re, DevCounters *ctr,
                            const int *fail) {
    if (*reinterpret_cast<const volatile int *>(fail)) return;
    unsigned long long ps = 0, mc = 0, mr = 0, mn = 0;  // mn: max of kMinRowBias - len
#pragma unroll 4
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long len = (unsigned long long)(rp[k + 1] - rp[k]);
        ps += len * len;
        mc = max(mc, len);
        if (k >= rb && k < re) {
            mr = max(mr, len);
            mn = max(mn, (unsigned long long)kMinRowBias - len);
        }
    }
    ps = warp_sum(ps);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mc = max(mc, __shfl_xor_sync(kFull, mc, o));
        mr = max(mr, __shfl_xor_sync(kFull, mr, o));
        mn = max(mn, __shfl_xor_sync(kFull, mn, o));
    }
    __shared__ unsigned long long red[4][8];  // one atomic per counter per CTA (<= 256 threads)
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        red[0][w] = ps;
        red[1][w] = mc;
        red[2][w] = mr;
        red[3][w] = mn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            ps += red[0][k];
            mc = max(mc, red[1][k]);
            mr = max(mr, red[2][k]);
            mn = max(mn, red[3][k]);
        }
        if (ps) atomicAdd((unsigned long long *)&ctr->p_full, ps);
        if (mc) atomicMax((unsigned long long *)&ctr->max_col, mc);
        if (mr) atomicMax((unsigned long long *)&ctr->max_row, mr);
        if (mn) atomicMax((unsigned long long *)&ctr->min_row_c, mn);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->shard_nnz = rp[re] - rp[rb];
}

void launch_sym_transpose(const Csr &A, int scale, double *nrm, double *y, double *ahat, int64_t *cp, int32_t *ri,
                          double *vt, int *fail, int *err, DevCounters *shape, int64_t rb, int64_t re, cudaStream_t s) {
    if (A.nrows <= 0) return;
    k_sym_probe<<<16, 256, 0, s>>>(A, fail);
    note_launch();
    if (scale) {
        k_row_norms<<<sym_grid(A.nrows, 256, 8), 256, 0, s>>>(A, nrm, y, err, fail);
        note_launch();
    }
    k_sym_transpose<<<sym_grid((A.nrows + 31) / 32 * 32, kSymThreads, 16), kSymThreads, 0, s>>>(A, scale, nrm, y, ahat, cp, ri, vt, fail);
    note_launch();
    if (shape) {
        k_sym_shape<<<sym_grid(A.nrows, 256, 8), 256, 0, s>>>(A.rp, A.nrows, rb, re, shape, fail);
        note_launch();
    }
}

}  // namespace rig

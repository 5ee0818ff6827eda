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
#include "common.cuh"

namespace rig {

// Bucket width 2^shift columns, chosen per matrix so an average bucket holds
// about kBucketTarget records (transpose_shift).
constexpr int kMinShift = 3, kMaxShift = 9;
constexpr int kMaxBucketCols = 1 << kMaxShift;
constexpr int kBucketTarget = 512;
constexpr int kBucketCap = 1024;  // records per bucket sorted in shared memory (16 KB)

struct __align__(16) Rec {
    int32_t col, row;
    double x;
};

__global__ void __launch_bounds__(256) k_bucket_scatter(Csr A, int scale, double *__restrict__ ahat,
                                                        const int64_t *__restrict__ cp, unsigned long long *bcur,
                                                        Rec *__restrict__ rec, int *err, int shift) {
    const int l = lane_id();
    const unsigned lt = lanemask_lt();
    const int64_t ntiles = (A.nrows + 31) / 32;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntiles; tile += nw) {
        const int64_t r0 = tile * 32;
        const int rows = (int)min((int64_t)32, A.nrows - r0);
        const int64_t hi = A.rp[r0 + rows];
        const int64_t my_s = l < rows ? A.rp[r0 + l] : hi;
        const int64_t my_e = l < rows ? A.rp[r0 + l + 1] : hi;
        double nrm = 1.0;
        int bad = 0;
        if (scale && l < rows) {
            double ss = +0.0;
            for (int64_t p0 = my_s; p0 < my_e; p0 += 8) {  // 8 loads in flight, chain in order
                double a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = p0 + u < my_e ? A.v[p0 + u] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (p0 + u < my_e) ss = __fma_rn(a[u], a[u], ss);
            }
            if (!isfinite(ss))
                bad = kErrNonFinite;
            else if (ss == 0.0)
                bad = kErrZeroRow;
            else
                nrm = __dsqrt_rn(ss);
        }
        if (bad) atomicOr(err, bad);
        const int64_t lo = __shfl_sync(kFull, my_s, 0);
        const int64_t last = __shfl_sync(kFull, my_s, 31);
        for (int64_t base = lo; base < hi; base += 32) {
            const int64_t p = base + l;
            int t = 0;  // row of entry p: (number of lanes with start <= p) - 1
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const int64_t v = __shfl_sync(kFull, my_s, t + step - 1);
                if (v <= p) t += step;
            }
            if (t == 31 && last <= p) t = 32;
            const int row = t > 0 ? t - 1 : 0;
            const double rn = __shfl_sync(kFull, nrm, row);
            const bool valid = p < hi;
            int k = 0;
            double x = 0.0;
            if (valid) {
                k = A.ci[p];
                x = scale ? __ddiv_rn(A.v[p], rn) : A.v[p];
                if (scale) ahat[p] = x;
            }
            const int b = valid ? (k >> shift) : -1 - l;
            const unsigned g = __match_any_sync(kFull, b);
            const int leader = __ffs(g) - 1;
            unsigned long long off = 0;
            if (valid && l == leader) off = atomicAdd(&bcur[b], (unsigned long long)__popc(g));
            off = __shfl_sync(kFull, off, leader);
            if (valid) {
                const int64_t pos = cp[(int64_t)b << shift] + (int64_t)off + __popc(g & lt);
                Rec r;
                r.col = k;
                r.row = (int32_t)(r0 + row);
                r.x = x;
                rec[pos] = r;
            }
        }
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

constexpr int kSortThreads = 128;

__global__ void __launch_bounds__(kSortThreads) k_bucket_sort(const Rec *__restrict__ rec,
                                                              const int64_t *__restrict__ cp, int64_t ncols,
                                                              unsigned *gcur, int32_t *ri, double *vt, int shift) {
    __shared__ Rec srec[kBucketCap];
    __shared__ int loff[kMaxBucketCols + 1];
    __shared__ int cur[kMaxBucketCols];
    const int bcols = 1 << shift;
    const int64_t nb = (ncols + bcols - 1) / bcols;
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t c0 = b << shift;
        const int ncb = (int)min((int64_t)bcols, ncols - c0);
        const int64_t e0 = cp[c0], e1 = cp[c0 + ncb];
        const int64_t E = e1 - e0;
        const int64_t out0 = e0 + c0;  // CSC slot of the bucket's first entry
        if (E <= kBucketCap) {
            for (int c = threadIdx.x; c <= ncb; c += kSortThreads) loff[c] = (int)(cp[c0 + c] - e0);
            for (int c = threadIdx.x; c < ncb; c += kSortThreads) cur[c] = 0;
            __syncthreads();
            // counting placement by column (order within a column fixed below)
            for (int64_t t = threadIdx.x; t < E; t += kSortThreads) {
                const Rec r = rec[e0 + t];
                const int lc = r.col - (int)c0;
                srec[loff[lc] + atomicAdd(&cur[lc], 1)] = r;
            }
            __syncthreads();
            // each column ascending by row (columns are short: insertion sort)
            for (int c = threadIdx.x; c < ncb; c += kSortThreads) {
                const int s = loff[c], e = loff[c + 1];
                for (int a2 = s + 1; a2 < e; ++a2) {
                    const Rec key = srec[a2];
                    int q = a2 - 1;
                    while (q >= s && srec[q].row > key.row) {
                        srec[q + 1] = srec[q];
                        --q;
                    }
                    srec[q + 1] = key;
                }
            }
            __syncthreads();
            // coalesced write-out: entry j of column lc goes to out0 + j + lc
            for (int64_t j = threadIdx.x; j < E; j += kSortThreads) {
                const Rec r = srec[j];
                const int64_t o = out0 + j + (r.col - c0);
                ri[o] = r.row;
                vt[o] = r.x;
            }
            for (int c = threadIdx.x; c < ncb; c += kSortThreads) {
                const int64_t o = out0 + loff[c + 1] + c;
                ri[o] = INT_MAX;
                vt[o] = 0.0;
            }
            __syncthreads();
        } else {
            // large bucket: place with global per-column cursors, then sort each
            // column in global memory (correct for any skew, slower)
            for (int64_t t = threadIdx.x; t < E; t += kSortThreads) {
                const Rec r = rec[e0 + t];
                const int64_t o = cp[r.col] + r.col + atomicAdd(&gcur[r.col], 1u);
                ri[o] = r.row;
                vt[o] = r.x;
            }
            for (int c = threadIdx.x; c < ncb; c += kSortThreads) {
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
}

int transpose_shift(int64_t nnz, int64_t ncols) {
    const double avg = ncols > 0 ? (double)nnz / (double)ncols : 1.0;
    int sh = kMinShift;
    while (sh < kMaxShift && (double)(1 << (sh + 1)) * avg <= kBucketTarget) ++sh;
    return sh;
}

int64_t transpose_buckets(int64_t nnz, int64_t ncols) {
    const int sh = transpose_shift(nnz, ncols);
    return (ncols + (1 << sh) - 1) >> sh;
}

void launch_transpose(const Csr &A, int scale, const int64_t *cp, double *ahat, unsigned long long *bcur,
                      void *rec, unsigned *gcur, int32_t *ri, double *vt, int *err, cudaStream_t s) {
    const int shift = transpose_shift(A.nnz, A.ncols);
    if (A.nrows > 0) {
        int64_t g = (A.nrows + 255) / 256;
        const int64_t cap = (int64_t)num_sms() * 8;
        g = g < 1 ? 1 : (g > cap ? cap : g);
        k_bucket_scatter<<<(unsigned)g, 256, 0, s>>>(A, scale, ahat, cp, bcur, static_cast<Rec *>(rec), err, shift);
        note_launch();
    }
    if (A.ncols > 0) {
        const int64_t nb = (A.ncols + (1 << shift) - 1) >> shift;
        const int64_t cap = (int64_t)num_sms() * 16;
        k_bucket_sort<<<(unsigned)(nb < cap ? nb : cap), kSortThreads, 0, s>>>(static_cast<const Rec *>(rec), cp,
                                                                                A.ncols, gcur, ri, vt, shift);
        note_launch();
    }
}

}  // namespace rig

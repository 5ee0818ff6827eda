// k_prep.cu -- steps a0-a3 of the hot path:
//   a0 validate (flag-gated), a1 row scaling fused into the a2 transpose
//   scatter, a2 column access (CSC of A_hat), a3 flop count + binning.
#include "common.cuh"

namespace rig {

static int grid_for(int64_t work, int block, int per_sm = 8) {
    int64_t g = (work + block - 1) / block;
    int64_t cap = (int64_t)num_sms() * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ------------------------------------------------------------------ a0
// Canonical CSR: row_ptr[0]=0, non-decreasing,
// row_ptr[n]=nnz, columns strictly increasing in [0,ncols), values finite.
__global__ void k_validate(Csr A, int *err) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0 && (A.rp[0] != 0 || A.rp[A.nrows] != A.nnz)) atomicOr(err, kErrNonCanonical);
    for (int64_t i = tid; i < A.nrows; i += stride) {
        const int64_t s = A.rp[i], e = A.rp[i + 1];
        if (s < 0 || e < s || e > A.nnz) {
            atomicOr(err, kErrNonCanonical);
            continue;
        }
        int prev = -1;
        bool bad = false, nonfinite = false;
        for (int64_t p = s; p < e; ++p) {
            const int c = A.ci[p];
            bad |= (c <= prev) | ((int64_t)c >= A.ncols);
            prev = c;
            nonfinite |= !isfinite(A.v[p]);
        }
        if (bad) atomicOr(err, kErrNonCanonical);
        if (nonfinite) atomicOr(err, kErrNonFinite);
    }
}

void launch_validate(const Csr &A, int *err, cudaStream_t s) {
    k_validate<<<grid_for(A.nrows, 256), 256, 0, s>>>(A, err);
    note_launch();
}

// ------------------------------------------------------------------ a2 (histogram)
// Column counts; with `rank`, also each entry's arrival slot in its column
// (the returned old count), so the scatter needs no atomics.
__global__ void k_col_hist(const int32_t *__restrict__ ci, int64_t nnz, unsigned *cnt, unsigned *rank) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (rank) {
        for (; p + 3 * stride < nnz; p += 4 * stride) {  // 4 returning atomics in flight
            unsigned r[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) r[u] = atomicAdd(&cnt[ci[p + u * stride]], 1u);
#pragma unroll
            for (int u = 0; u < 4; ++u) rank[p + u * stride] = r[u];
        }
        for (; p < nnz; p += stride) rank[p] = atomicAdd(&cnt[ci[p]], 1u);
    } else {
        for (; p < nnz; p += stride) atomicAdd(&cnt[ci[p]], 1u);
    }
}

void launch_col_hist(const Csr &A, unsigned *cnt, unsigned *rank, cudaStream_t s) {
    k_col_hist<<<grid_for(A.nnz, 256, 16), 256, 0, s>>>(A.ci, A.nnz, cnt, rank);
    note_launch();
}

// ------------------------------------------------------------------ a1 + a2 (scatter)
// a1: ss_i = fma-chain of a_ik^2 in ascending k from
// +0.0; nrm_i = sqrt_rn(ss_i); a_hat = a /_rn nrm_i (DESIGN.md §3 R5).
// Fused with the CSC scatter so the scaled value written to the CSR copy and
// to the CSC slot is the same double.  Slot of entry p in the CSC:
// cp[ci[p]] + rank[p] (rank from k_col_hist).
// Warp-tile variant: a warp owns 32 consecutive rows.  Lane l computes the
// norm of row r0+l (the ordered fma chain is per row and sequential), then the
// warp walks the tile's entries [rp[r0], rp[r0+32]) 32 at a time: coalesced
// loads of col / value / rank, coalesced a_hat stores, scattered CSC stores.
__global__ void __launch_bounds__(256) k_scale_scatter_tile(Csr A, int scale, double *__restrict__ ahat,
                                                            const int64_t *__restrict__ cp,
                                                            const unsigned *__restrict__ rank, int32_t *ri,
                                                            double *vt, int *err) {
    const int l = lane_id();
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
            for (int64_t p = my_s; p < my_e; ++p) {
                const double a = A.v[p];
                ss = __fma_rn(a, a, ss);
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
            // row of entry p: (number of lanes with start <= p) - 1
            int t = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const int64_t v = __shfl_sync(kFull, my_s, t + step - 1);
                if (v <= p) t += step;
            }
            if (t == 31 && last <= p) t = 32;
            const int row = t > 0 ? t - 1 : 0;
            const double rn = __shfl_sync(kFull, nrm, row);
            if (p < hi) {
                const double x = scale ? __ddiv_rn(A.v[p], rn) : A.v[p];
                if (scale) ahat[p] = x;
                const int64_t q = cp[A.ci[p]] + rank[p];
                ri[q] = (int32_t)(r0 + row);
                vt[q] = x;
            }
        }
    }
}

void launch_scale_scatter(const Csr &A, int scale, double *ahat, const int64_t *cp, const unsigned *rank,
                          int32_t *ri, double *vt, int *err, cudaStream_t s) {
    int64_t g = (A.nrows + 255) / 256;  // 8 tiles of 32 rows per CTA
    const int64_t cap = (int64_t)num_sms() * 8;
    g = g < 1 ? 1 : (g > cap ? cap : g);
    k_scale_scatter_tile<<<(unsigned)g, 256, 0, s>>>(A, scale, ahat, cp, rank, ri, vt, err);
    note_launch();
}

// ------------------------------------------------------------------ a2 (column sort)
// The scatter order inside a column is arbitrary (atomics); the merge path
// needs each column's rows ascending.  Short columns: insertion sort by one
// thread; long ones go to a list sorted by a CTA.
constexpr int kShortCol = 32;
constexpr int kRegCol = 8;

// Odd-even transposition network on registers (static indices only).
template <int N>
__device__ __forceinline__ void sort_regs(int32_t (&k)[N], double (&v)[N]) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
        for (int i = r & 1; i + 1 < N; i += 2) {
            const bool sw = k[i] > k[i + 1];
            const int32_t ka = sw ? k[i + 1] : k[i], kb = sw ? k[i] : k[i + 1];
            const double va = sw ? v[i + 1] : v[i], vb = sw ? v[i] : v[i + 1];
            k[i] = ka; k[i + 1] = kb; v[i] = va; v[i + 1] = vb;
        }
    }
}

__global__ void k_col_sort_short(int64_t ncols, const int64_t *__restrict__ cp, int32_t *ri, double *vt,
                                 int32_t *long_list, unsigned *long_count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ncols; k += stride) {
        const int64_t s = cp[k], len = cp[k + 1] - s;
        if (len > kShortCol) {
            long_list[atomicAdd(long_count, 1u)] = (int32_t)k;
            continue;
        }
        if (len <= kRegCol) {
            int32_t kk[kRegCol];
            double vv[kRegCol];
            bool sorted = true;
#pragma unroll
            for (int t = 0; t < kRegCol; ++t) {
                kk[t] = t < len ? ri[s + t] : INT_MAX;
                if (t > 0) sorted &= kk[t - 1] <= kk[t];
            }
            if (sorted) continue;  // values are only read when the keys need sorting
#pragma unroll
            for (int t = 0; t < kRegCol; ++t) vv[t] = t < len ? vt[s + t] : 0.0;
            sort_regs<kRegCol>(kk, vv);
#pragma unroll
            for (int t = 0; t < kRegCol; ++t) {
                if (t < len) {
                    ri[s + t] = kk[t];
                    vt[s + t] = vv[t];
                }
            }
            continue;
        }
        for (int64_t a = 1; a < len; ++a) {
            const int32_t key = ri[s + a];
            const double v = vt[s + a];
            int64_t b = a - 1;
            while (b >= 0 && ri[s + b] > key) {
                ri[s + b + 1] = ri[s + b];
                vt[s + b + 1] = vt[s + b];
                --b;
            }
            ri[s + b + 1] = key;
            vt[s + b + 1] = v;
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

constexpr int kSmemSortCap = 4096;

__global__ void k_col_sort_long(const int64_t *__restrict__ cp, int32_t *ri, double *vt,
                                const int32_t *__restrict__ list, const unsigned *count) {
    extern __shared__ unsigned char smem_raw[];
    int32_t *sk = reinterpret_cast<int32_t *>(smem_raw + kSmemSortCap * sizeof(double));
    double *sv = reinterpret_cast<double *>(smem_raw);
    const unsigned n = *count;
    for (unsigned c = blockIdx.x; c < n; c += gridDim.x) {
        const int k = list[c];
        const int64_t s = cp[k], len = cp[k + 1] - s;
        if (len <= kSmemSortCap) {
            for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
                sk[t] = ri[s + t];
                sv[t] = vt[s + t];
            }
            __syncthreads();
            bitonic_sort_block(
                len, [&](int64_t i) { return sk[i]; },
                [&](int64_t i, int64_t j) {
                    int32_t tk = sk[i];
                    sk[i] = sk[j];
                    sk[j] = tk;
                    double tv = sv[i];
                    sv[i] = sv[j];
                    sv[j] = tv;
                });
            for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
                ri[s + t] = sk[t];
                vt[s + t] = sv[t];
            }
        } else {  // in place in global memory (correct, slow; pathological inputs only)
            int32_t *gk = ri + s;
            double *gv = vt + s;
            bitonic_sort_block(
                len, [&](int64_t i) { return gk[i]; },
                [&](int64_t i, int64_t j) {
                    int32_t tk = gk[i];
                    gk[i] = gk[j];
                    gk[j] = tk;
                    double tv = gv[i];
                    gv[i] = gv[j];
                    gv[j] = tv;
                });
        }
        __syncthreads();
    }
}

void launch_col_sort(int64_t ncols, const int64_t *cp, int32_t *ri, double *vt, int32_t *long_list,
                     unsigned *long_count, cudaStream_t s) {
    k_col_sort_short<<<grid_for(ncols, 256), 256, 0, s>>>(ncols, cp, ri, vt, long_list, long_count);
    const size_t smem = kSmemSortCap * (sizeof(double) + sizeof(int32_t));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_col_sort_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_col_sort_long<<<num_sms(), 512, smem, s>>>(cp, ri, vt, long_list, long_count);
    note_launch(2);
}

// ------------------------------------------------------------------ a3
// f_i = sum over k in row i of nnz(column k) (Gustavson products).  Rows off
// the merge path go to symbolic bin ceil(log2(2 f_i)) in [6, 12], or to the
// huge bin (index 7) above that.
__device__ __forceinline__ int ceil_log2_2x(int64_t m) {
    const int64_t m2 = 2 * (m > 1 ? m : 1);
    return 64 - __clzll(m2 - 1);
}

__global__ void k_analyze(Csr A, const int64_t *__restrict__ cp, int64_t rb, int64_t re, int64_t *f,
                          int32_t *sym_lists, int64_t cap, DevCounters *ctr) {
    const int64_t nloc = re - rb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t local = 0;
    int maxlen = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc; r += stride) {
        const int64_t i = rb + r;
        const int64_t s = A.rp[i], e = A.rp[i + 1];
        int64_t fi = 0;
        for (int64_t p = s; p < e; ++p) {
            const int k = A.ci[p];
            fi += cp[k + 1] - cp[k];
        }
        if (f) f[r] = fi;
        local += fi;
        const bool merge = e - s <= kMergeMaxLen && fi <= kMergeMaxF;
        if (merge) maxlen = max(maxlen, (int)(e - s));
        if (sym_lists && !merge) {
            int lg = ceil_log2_2x(fi);
            if (lg < kSymBinMinLog) lg = kSymBinMinLog;
            const int b = lg > kSymBinMaxLog ? kNumSymBins : lg - kSymBinMinLog;
            const unsigned long long pos = atomicAdd((unsigned long long *)&ctr->sym_count[b], 1ull);
            sym_lists[b * cap + (int64_t)pos] = (int32_t)i;
            atomicAdd((unsigned long long *)&ctr->n_mid, 1ull);
        }
    }
    maxlen = __reduce_max_sync(kFull, maxlen);
    if (lane_id() == 0 && maxlen) atomicMax(&ctr->max_len, maxlen);
    local = warp_sum(local);
    __shared__ int64_t part[32];
    if (lane_id() == 0) part[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0;
        v = warp_sum(v);
        if (threadIdx.x == 0 && v) atomicAdd((unsigned long long *)&ctr->products, (unsigned long long)v);
    }
}

void launch_analyze(const Csr &A, const int64_t *cp, int64_t rb, int64_t re, int64_t *f, int32_t *sym_lists,
                    int64_t cap, DevCounters *ctr, cudaStream_t s) {
    k_analyze<<<grid_for(re - rb, 256), 256, 0, s>>>(A, cp, rb, re, f, sym_lists, cap, ctr);
    note_launch();
}

// Numeric bins by nnzC_i: table T = 2^ceil(log2(2 nnzC_i)) in [64, 2048];
// larger -> huge bin (index 6).
__global__ void k_bin_num(const int32_t *__restrict__ sym_lists, int64_t sym_cap, const DevCounters *ctr,
                          const int64_t *__restrict__ nnzc, int64_t rb, int32_t *num_lists, int64_t num_cap,
                          int64_t *num_count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int b = 0; b < kSymBins; ++b) {
        const int64_t n = ctr->sym_count[b];
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride) {
            const int32_t i = sym_lists[b * sym_cap + t];
            int lg = ceil_log2_2x(nnzc[i - rb]);
            if (lg < kNumBinMinLog) lg = kNumBinMinLog;
            const int nb = lg > kNumBinMaxLog ? kNumNumBins : lg - kNumBinMinLog;
            const unsigned long long pos = atomicAdd((unsigned long long *)&num_count[nb], 1ull);
            num_lists[nb * num_cap + (int64_t)pos] = i;
        }
    }
}

void launch_bin_num(const int32_t *sym_lists, int64_t sym_cap, const DevCounters *ctr, const int64_t *nnzc,
                    int64_t rb, int32_t *num_lists, int64_t num_cap, int64_t *num_count, cudaStream_t s) {
    k_bin_num<<<grid_for(num_cap, 256), 256, 0, s>>>(sym_lists, sym_cap, ctr, nnzc, rb, num_lists, num_cap,
                                                      num_count);
    note_launch();
}

}  // namespace rig

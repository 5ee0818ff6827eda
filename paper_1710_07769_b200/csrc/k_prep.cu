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

// a1 + a2 (scaling, CSC): k_transpose.cu

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
                          const int32_t *__restrict__ farc, int64_t rb, int32_t *num_lists, int64_t num_cap,
                          int64_t *num_count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int b = 0; b < kSymBins; ++b) {
        const int64_t n = ctr->sym_count[b];
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride) {
            const int32_t i = sym_lists[b * sym_cap + t];
            int lg = ceil_log2_2x(farc[i - rb]);
            if (lg < kNumBinMinLog) lg = kNumBinMinLog;
            const int nb = lg > kNumBinMaxLog ? kNumNumBins : lg - kNumBinMinLog;
            const unsigned long long pos = atomicAdd((unsigned long long *)&num_count[nb], 1ull);
            num_lists[nb * num_cap + (int64_t)pos] = i;
        }
    }
}

void launch_bin_num(const int32_t *sym_lists, int64_t sym_cap, const DevCounters *ctr, const int32_t *farc,
                    int64_t rb, int32_t *num_lists, int64_t num_cap, int64_t *num_count, cudaStream_t s) {
    k_bin_num<<<grid_for(num_cap, 256), 256, 0, s>>>(sym_lists, sym_cap, ctr, farc, rb, num_lists, num_cap,
                                                      num_count);
    note_launch();
}

}  // namespace rig

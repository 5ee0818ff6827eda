// k_prep.cu -- steps a0-a3 of the hot path:
//   a0 validate (flag-gated), a1 row scaling fused into the a2 transpose
//   scatter, a2 column access (CSC of A_hat), a3 flop count + binning.
#include <algorithm>

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

// Partition ids (a7): every part[v], v < n, in [0, K) -- the oracle's check
// (orc_cutsize) -- else *bad = 1 and the fused cut becomes NaN.  One read of
// part[] up front, so the fused numeric kernels gather part[j] unchecked.
__global__ void k_part_check(const int32_t *__restrict__ part, int64_t n, int32_t K, int *bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int b = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
        const int32_t x = part[v];
        b |= (x < 0) | (x >= K);
    }
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

void launch_part_check(const int32_t *part, int64_t n, int32_t K, int *bad, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t g = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_part_check<<<(unsigned)g, 256, 0, s>>>(part, n, K, bad);
    note_launch();
}

// ------------------------------------------------------------------ a2 (histogram)
// Column counts; with `rank`, also each entry's arrival slot in its column
// (the returned old count), so the scatter needs no atomics.
__global__ void k_col_hist(const int32_t *__restrict__ ci, int64_t nnz, unsigned *cnt, unsigned *rank,
                           const int *guard) {
    if (guard_skip(guard)) return;
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

// Column counts without ranks, privatised: each CTA counts a chunk of
// kHistChunk consecutive entries into a shared window of kHistWin columns
// starting just below the chunk's first column (banded / stencil rows keep
// most columns near the row index, so most entries stay on chip), entries
// outside the window go straight to global atomics, and the window's
// non-zero bins are added to the global counts once.  Counts are sums:
// the result does not depend on the order.
constexpr int kHistThreads = 256, kHistWin = 2048, kHistChunk = 4096, kHistSlack = 64;
__global__ void __launch_bounds__(kHistThreads) k_col_hist_win(const int32_t *__restrict__ ci, int64_t nnz,
                                                                int64_t ncols, unsigned *cnt, const int *guard) {
    if (guard_skip(guard)) return;
    __shared__ unsigned h[kHistWin];
    const int64_t nch = (nnz + kHistChunk - 1) / kHistChunk;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        const int64_t e0 = c * kHistChunk, e1 = min(nnz, e0 + kHistChunk);
        for (int t = threadIdx.x; t < kHistWin; t += kHistThreads) h[t] = 0u;
        const int64_t base = max((int64_t)0, (int64_t)__ldg(&ci[e0]) - kHistSlack);
        __syncthreads();
        for (int64_t p0 = e0 + threadIdx.x; p0 < e1; p0 += 4 * kHistThreads) {  // 4 loads in flight
            int k[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t p = p0 + (int64_t)u * kHistThreads;
                k[u] = p < e1 ? __ldcs(&ci[p]) : -1;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k[u] < 0) continue;
                const int64_t d = (int64_t)k[u] - base;
                if (d >= 0 && d < kHistWin)
                    atomicAdd(&h[d], 1u);
                else
                    atomicAdd(&cnt[k[u]], 1u);
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < kHistWin; t += kHistThreads) {
            const unsigned v = h[t];
            if (v && base + t < ncols) atomicAdd(&cnt[base + t], v);
        }
        __syncthreads();
    }
}

void launch_col_hist(const Csr &A, unsigned *cnt, unsigned *rank, cudaStream_t s, const int *guard) {
    if (rank) {
        k_col_hist<<<grid_for(A.nnz, 256, 16), 256, 0, s>>>(A.ci, A.nnz, cnt, rank, guard);
    } else {
        const int64_t nch = (A.nnz + kHistChunk - 1) / kHistChunk;
        const int64_t g = std::min<int64_t>(nch, (int64_t)num_sms() * 16);
        k_col_hist_win<<<(unsigned)std::max<int64_t>(g, 1), kHistThreads, 0, s>>>(A.ci, A.nnz, A.ncols, cnt, guard);
    }
    note_launch();
}

// a1 + a2 (scaling, CSC): k_transpose.cu

// ------------------------------------------------------------------ a3
// f_i = sum over k in row i of nnz(column k) (Gustavson products), for the
// flop-balanced row split.  (The build path computes f_i in k_analyze_sym.)

__global__ void k_analyze(Csr A, const int64_t *__restrict__ cp, int64_t rb, int64_t re, int64_t *f,
                          DevCounters *ctr) {
    const int64_t nloc = re - rb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t local = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc; r += stride) {
        const int64_t i = rb + r;
        const int64_t s = A.rp[i], e = A.rp[i + 1];
        int64_t fi = 0;
        for (int64_t p = s; p < e; ++p) {
            const int k = A.ci[p];
            fi += cp[k + 1] - cp[k];
        }
        f[r] = fi;
        local += fi;
    }
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

void launch_analyze(const Csr &A, const int64_t *cp, int64_t rb, int64_t re, int64_t *f, DevCounters *ctr,
                    cudaStream_t s) {
    k_analyze<<<grid_for(re - rb, 256), 256, 0, s>>>(A, cp, rb, re, f, ctr);
    note_launch();
}

// ------------------------------------------------------------------ row lists
// Rows off the merge path are listed in ASCENDING row order (list 0: mid
// rows, list 1: huge rows), so the warps that run at the same time work on
// neighbouring rows and share their CSC columns in L2 (banded / stencil
// inputs).  Deterministic three-step partition: per-tile counts -> exclusive
// scan -> ordered scatter.  Merge-path rows (bin8 = kBinNone) are in no list.
constexpr int kBinThreads = 256;
constexpr int kBinRounds = 4;
constexpr int64_t kBinTile = (int64_t)kBinThreads * kBinRounds;
constexpr int kBinWarps = kBinThreads / 32;
constexpr int kLists = 2;

__device__ __forceinline__ int row_list(const uint8_t *__restrict__ bin8, int64_t r) {
    const int b = bin8[r];
    if (b == kBinNone) return -1;
    return b == kNumSymBins ? 1 : 0;
}

__global__ void __launch_bounds__(kBinThreads) k_bin_count(const uint8_t *__restrict__ bin8, int64_t nloc,
                                                           unsigned *cnt, int64_t nt) {
    __shared__ unsigned sc[kLists];
    for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x) {
        if (threadIdx.x < kLists) sc[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kBinRounds; ++j) {
            const int64_t r = tile * kBinTile + j * kBinThreads + threadIdx.x;
            const int b = r < nloc ? row_list(bin8, r) : -1;
#pragma unroll
            for (int q = 0; q < kLists; ++q) {
                const unsigned m = __ballot_sync(kFull, b == q);
                if (lane_id() == 0 && m) atomicAdd(&sc[q], (unsigned)__popc(m));
            }
        }
        __syncthreads();
        if (threadIdx.x < kLists) cnt[(int64_t)threadIdx.x * nt + tile] = sc[threadIdx.x];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBinThreads) k_bin_scatter(const uint8_t *__restrict__ bin8, int64_t rb,
                                                             int64_t nloc, const int64_t *__restrict__ off, int64_t nt,
                                                             int32_t *lists, int64_t cap, int64_t *counts) {
    __shared__ unsigned wc[kBinWarps][kLists];
    __shared__ int64_t run[kLists];
    const int w = threadIdx.x >> 5, l = lane_id();
    if (counts && blockIdx.x == 0 && threadIdx.x < kLists)
        counts[threadIdx.x] = off[(int64_t)(threadIdx.x + 1) * nt] - off[(int64_t)threadIdx.x * nt];
    for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x) {
        if (threadIdx.x < kLists)
            run[threadIdx.x] = off[(int64_t)threadIdx.x * nt + tile] - off[(int64_t)threadIdx.x * nt];
        __syncthreads();
        for (int j = 0; j < kBinRounds; ++j) {
            const int64_t r = tile * kBinTile + j * kBinThreads + threadIdx.x;
            const int b = r < nloc ? row_list(bin8, r) : -1;
            unsigned m[kLists];
#pragma unroll
            for (int q = 0; q < kLists; ++q) {
                m[q] = __ballot_sync(kFull, b == q);
                if (l == 0) wc[w][q] = (unsigned)__popc(m[q]);
            }
            __syncthreads();
            if (b >= 0) {
                int64_t pos = run[b] + __popc(m[b] & lanemask_lt());
                for (int v = 0; v < w; ++v) pos += wc[v][b];
                lists[(int64_t)b * cap + pos] = (int32_t)(rb + r);
            }
            __syncthreads();
            if (threadIdx.x < kLists) {
                unsigned t = 0;
                for (int v = 0; v < kBinWarps; ++v) t += wc[v][threadIdx.x];
                run[threadIdx.x] += t;
            }
            __syncthreads();
        }
    }
}

size_t bins_count_elems(int64_t nloc) { return (size_t)kLists * (size_t)((nloc + kBinTile - 1) / kBinTile); }

void launch_bins(const uint8_t *bin8, int64_t rb, int64_t nloc, unsigned *cnt, int64_t *off, void *scan_tmp,
                 int32_t *lists, int64_t cap, int64_t *counts, cudaStream_t s) {
    const int64_t nt = (nloc + kBinTile - 1) / kBinTile;
    if (nt == 0) return;
    const unsigned g = (unsigned)std::min<int64_t>(nt, (int64_t)num_sms() * 8);
    k_bin_count<<<g, kBinThreads, 0, s>>>(bin8, nloc, cnt, nt);
    note_launch();
    scan_u32(cnt, (int64_t)kLists * nt, off, scan_tmp, 0, s);
    k_bin_scatter<<<g, kBinThreads, 0, s>>>(bin8, rb, nloc, off, nt, lists, cap, counts);
    note_launch();
}

}  // namespace rig

// k_sparsify.cu -- SURVEY.md §8(f) f1, the steps next to the hot path:
//
//   * dense-column sparsification A~ (§2.3): a column with
//     more than T = ceil(sqrt(n)) nonzeros keeps the T entries of largest
//     |a_hat| (ties: the lower row; readings R20-R21);
//   * integer edge weights wgt = ceil(alpha * w) for the partitioner
//     (PAPER.md:611-613), exact.
//
// Sparsification runs on the CSC of A_hat that the transpose already built
// (rows ascending per column, values bit-identical to the CSR ones):
//   k_dense_cols    list of columns with cnt > T
//   k_col_cutoff    CTA per dense column: radix select of the T-th largest
//                   |value| key (8 passes of 8 bits over the column), then
//                   the row of the last tie that survives (in row order)
//   k_filter_rows   warp per CSR row: keep (i,k) iff column k is not dense,
//                   or key > cutoff_k, or key == cutoff_k and i <= row_k;
//                   pass 0 counts per row, pass 1 writes A~ at the scanned
//                   offsets (ballot compaction keeps the column order)
// |value| keys: the IEEE bit pattern of fabs(v) orders non-negative doubles.
#include <algorithm>

#include "common.cuh"

namespace rig {

namespace {

__device__ __forceinline__ unsigned long long mag_key(double v) {
    return (unsigned long long)__double_as_longlong(fabs(v));
}

__global__ void k_dense_cols(const unsigned *__restrict__ cnt, int64_t m, int64_t T, int32_t *list, int *count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x; k0 < m; k0 += stride) {
        const int64_t k = k0 + threadIdx.x;
        const bool dense = k < m && (int64_t)cnt[k] > T;
        const unsigned b = __ballot_sync(0xffffffffu, dense);
        if (!b) continue;
        const int lane = threadIdx.x & 31;
        int base = 0;
        if (lane == 0) base = atomicAdd(count, __popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (dense) list[base + __popc(b & ((1u << lane) - 1u))] = (int32_t)k;
    }
}

constexpr int kCutThreads = 256;

__global__ void __launch_bounds__(kCutThreads) k_col_cutoff(Csc Tc, const int32_t *__restrict__ list,
                                                            const int *__restrict__ count, int64_t T,
                                                            unsigned long long *__restrict__ ckey,
                                                            int32_t *__restrict__ crow) {
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_rem;
    __shared__ int s_wsum[kCutThreads / 32];
    __shared__ int s_found;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nd = *count;
    for (int d = blockIdx.x; d < nd; d += gridDim.x) {
        const int k = list[d];
        const int64_t b = csc_begin(Tc, k), e = Tc.cp[k + 1] + k;
        unsigned long long prefix = 0, mask = 0;
        if (tid == 0) s_rem = T;
        for (int shift = 56; shift >= 0; shift -= 8) {
            hist[tid] = 0;
            __syncthreads();
            for (int64_t p = b + tid; p < e; p += kCutThreads) {
                const unsigned long long key = mag_key(Tc.vt[p]);
                if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (tid == 0) {
                long long rem = s_rem, acc = 0;
                int sel = 0;
                for (int dg = 255; dg >= 0; --dg) {
                    if (acc + hist[dg] >= rem) {
                        sel = dg;
                        break;
                    }
                    acc += hist[dg];
                }
                s_rem = rem - acc;  // ties of the selected key still to keep (>= 1 at the end)
                s_prefix = prefix | ((unsigned long long)sel << shift);
            }
            __syncthreads();
            prefix = s_prefix;
            mask |= 255ull << shift;
        }
        // the s_rem-th entry (in row order) whose key equals the cutoff
        const long long need = s_rem;
        if (tid == 0) s_found = 0;
        long long seen = 0;
        __syncthreads();
        for (int64_t base = b; base < e; base += kCutThreads) {
            const int64_t p = base + tid;
            const bool eq = p < e && mag_key(Tc.vt[p]) == prefix;
            const unsigned bal = __ballot_sync(0xffffffffu, eq);
            if (lane == 0) s_wsum[wid] = __popc(bal);
            __syncthreads();
            long long before = seen;
            int total = 0;
            for (int w = 0; w < kCutThreads / 32; ++w) {
                if (w < wid) before += s_wsum[w];
                total += s_wsum[w];
            }
            before += __popc(bal & ((1u << lane) - 1u));
            if (eq && before + 1 == need) {
                ckey[k] = prefix;
                crow[k] = Tc.ri[p];
                s_found = 1;
            }
            seen += total;
            __syncthreads();
            if (s_found) break;
        }
        __syncthreads();
    }
}

// pass 0: nk[i] = kept entries of row i; pass 1: write them at rp2[i]
template <int PASS>
__global__ void k_filter_rows(Csr A, const unsigned *__restrict__ cnt, int64_t T,
                              const unsigned long long *__restrict__ ckey, const int32_t *__restrict__ crow,
                              int64_t *__restrict__ nk, const int64_t *__restrict__ rp2, int32_t *__restrict__ ci2,
                              double *__restrict__ v2) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < A.nrows; i += nwarps) {
        const int64_t s = A.rp[i], e = A.rp[i + 1];
        int64_t o = PASS ? rp2[i] : 0;
        for (int64_t base = s; base < e; base += 32) {
            const int64_t p = base + lane;
            bool keep = false;
            int c = 0;
            double v = 0.0;
            if (p < e) {
                c = A.ci[p];
                v = A.v[p];
                keep = (int64_t)cnt[c] <= T;
                if (!keep) {
                    const unsigned long long key = mag_key(v), ck = ckey[c];
                    keep = key > ck || (key == ck && (int32_t)i <= crow[c]);
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (PASS && keep) {
                const int64_t q = o + __popc(bal & ((1u << lane) - 1u));
                ci2[q] = c;
                v2[q] = v;
            }
            o += __popc(bal);
        }
        if (!PASS && lane == 0) nk[i] = o;
    }
}

// wgt = ceil(alpha * w), exact.  With p = RN(alpha * w) and
// the exact remainder r = fma(alpha, w, -p): if p is not an integer, the
// exact product lies within ulp(p)/2 of p, strictly between the integers
// around p, so the ceiling is ceil(p); if p is an integer (p >= 1, no
// underflow in r), the ceiling is p + ceil(r).  Invalid elements (w < 0,
// non-finite, result beyond 2^62) give -1.
__global__ void k_int_weights(const double *__restrict__ w, int64_t n, double alpha, int64_t *__restrict__ wgt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
        const double x = w[e];
        int64_t out;
        if (!(x >= 0.0) || !isfinite(x)) {
            out = -1;
        } else {
            const double p = __dmul_rn(alpha, x);
            const double c = ceil(p);
            if (!(p <= 4611686018427387904.0)) {  // 2^62
                out = -1;
            } else if (c != p) {
                out = (int64_t)c;
            } else {
                const double r = __fma_rn(alpha, x, -p);
                out = (int64_t)p + (int64_t)ceil(r);
                if (out > (int64_t)1 << 62) out = -1;
            }
        }
        wgt[e] = out;
    }
}

int sm_grid(int per_sm) { return num_sms() * per_sm; }

}  // namespace

void launch_sparsify_cutoffs(const unsigned *cnt, int64_t m, int64_t T, const Csc &Tc, int32_t *list, int *count,
                             unsigned long long *ckey, int32_t *crow, cudaStream_t s) {
    if (m <= 0) return;
    const int64_t g = std::min<int64_t>((m + 255) / 256, (int64_t)sm_grid(8));
    k_dense_cols<<<(int)g, 256, 0, s>>>(cnt, m, T, list, count);
    k_col_cutoff<<<sm_grid(2), kCutThreads, 0, s>>>(Tc, list, count, T, ckey, crow);
    note_launch(2);
}

void launch_sparsify_filter(int pass, const Csr &A, const unsigned *cnt, int64_t T, const unsigned long long *ckey,
                            const int32_t *crow, int64_t *nk, const int64_t *rp2, int32_t *ci2, double *v2,
                            cudaStream_t s) {
    if (A.nrows <= 0) return;
    const int64_t g = std::min<int64_t>((A.nrows * 32 + 255) / 256, (int64_t)sm_grid(8));
    if (pass == 0)
        k_filter_rows<0><<<(int)g, 256, 0, s>>>(A, cnt, T, ckey, crow, nk, rp2, ci2, v2);
    else
        k_filter_rows<1><<<(int)g, 256, 0, s>>>(A, cnt, T, ckey, crow, nk, rp2, ci2, v2);
    note_launch();
}

void launch_int_weights(const double *w, int64_t n, int64_t alpha, int64_t *wgt, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t g = std::min<int64_t>((n + 255) / 256, (int64_t)sm_grid(8));
    k_int_weights<<<(int)g, 256, 0, s>>>(w, n, (double)alpha, wgt);
    note_launch();
}

}  // namespace rig

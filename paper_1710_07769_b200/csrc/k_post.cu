// k_post.cu -- a6 compaction (only when the numeric pass dropped entries),
// a7 cutsize (§2.2; eq. partcut) and the
// flop-balanced row split for multi-GPU sharding.
#include <algorithm>

#include "common.cuh"

namespace rig {

// ------------------------------------------------------------------ a6 (holes path)
// The numeric pass writes each row's kept entries at the front of its
// structural slot range [gptr_ub[r], gptr_ub[r+1]) and marks the rest -1.
__global__ void k_count_kept(const int64_t *__restrict__ gptr_ub, int64_t nloc, const int32_t *__restrict__ gcol,
                             int64_t *kept) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int l = lane_id();
    for (int64_t r = w; r < nloc; r += nw) {
        const int64_t s = gptr_ub[r], e = gptr_ub[r + 1];
        int64_t c = 0;
        for (int64_t t = s + l; t < e; t += 32) c += gcol[t] >= 0;
        c = warp_sum(c);
        if (l == 0) kept[r] = c;
    }
}

void launch_count_kept(const int64_t *gptr_ub, int64_t nloc, const int32_t *gcol, int64_t *kept, cudaStream_t s) {
    int64_t g = (nloc * 32 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    g = g < 1 ? 1 : (g > cap ? cap : g);
    k_count_kept<<<(unsigned)g, 256, 0, s>>>(gptr_ub, nloc, gcol, kept);
    note_launch();
}

__global__ void k_compact_move(const int64_t *__restrict__ gptr_ub, const int64_t *__restrict__ gptr, int64_t nloc,
                               const int32_t *__restrict__ gcol_in, const double *__restrict__ gw_in, int32_t *gcol,
                               double *gw) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int l = lane_id();
    for (int64_t r = w; r < nloc; r += nw) {
        const int64_t s = gptr_ub[r], d = gptr[r], len = gptr[r + 1] - d;
        for (int64_t t = l; t < len; t += 32) {
            gcol[d + t] = gcol_in[s + t];
            gw[d + t] = gw_in[s + t];
        }
    }
}

void launch_compact_move(const int64_t *gptr_ub, const int64_t *gptr, int64_t nloc, const int32_t *gcol_in,
                         const double *gw_in, int32_t *gcol, double *gw, cudaStream_t s) {
    int64_t g = (nloc * 32 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    g = g < 1 ? 1 : (g > cap ? cap : g);
    k_compact_move<<<(unsigned)g, 256, 0, s>>>(gptr_ub, gptr, nloc, gcol_in, gw_in, gcol, gw);
    note_launch();
}

// ------------------------------------------------------------------ a7 cutsize
// Each undirected edge counted once (stored j > i), DESIGN.md §3 R8.
// Per-thread Neumaier sums, fixed-shape tree per CTA, then a fixed-order
// final reduction: deterministic for a given graph.
constexpr int kCutThreads = 256;

__device__ __forceinline__ void neumaier_add(double &s, double &c, double x) {
    const double t = s + x;
    if (fabs(s) >= fabs(x))
        c += (s - t) + x;
    else
        c += (x - t) + s;
    s = t;
}

__global__ void __launch_bounds__(kCutThreads) k_cutsize(const int64_t *__restrict__ grp,
                                                         const int32_t *__restrict__ gcol,
                                                         const double *__restrict__ gw, int64_t nloc, int64_t rb,
                                                         int64_t n_global, const int32_t *__restrict__ part,
                                                         int32_t K, double *partials, int *bad) {
    const int l = lane_id();
    const int64_t wg = ((int64_t)blockIdx.x * kCutThreads + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * kCutThreads) >> 5;
    double s = 0.0, c = 0.0;
    int badp = 0;
    // part ids must lie in [0, K)
    for (int64_t v = (int64_t)blockIdx.x * kCutThreads + threadIdx.x; v < n_global;
         v += (int64_t)gridDim.x * kCutThreads) {
        const int32_t p = part[v];
        badp |= (p < 0) | (p >= K);
    }
    const int64_t ntiles = (nloc + 31) / 32;
    for (int64_t tile = wg; tile < ntiles; tile += nwg) {
        const int64_t r0 = tile * 32;
        const int rows = (int)min((int64_t)32, nloc - r0);
        const int64_t hi = grp[r0 + rows];
        const int64_t my_start = l < rows ? grp[r0 + l] : hi;
        const int32_t pi = l < rows ? part[rb + r0 + l] : 0;
        const int64_t lo = __shfl_sync(kFull, my_start, 0);
        const int64_t last = __shfl_sync(kFull, my_start, 31);
        constexpr int U = 4;  // chunks of 32 edges in flight per iteration
        for (int64_t base = lo; base < hi; base += 32 * U) {
            int32_t j[U], pj[U];
            double wv[U];
            int64_t e[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                e[u] = base + 32 * u + l;
                const bool v = e[u] < hi;
                j[u] = v ? gcol[e[u]] : 0;
                wv[u] = v ? gw[e[u]] : 0.0;
            }
#pragma unroll
            // j < 0 marks an unfilled slot of the upper-bound layout: skipped
            for (int u = 0; u < U; ++u) pj[u] = (e[u] < hi && j[u] >= 0) ? part[j[u]] : 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                // row of edge e: (number of lanes with start <= e) - 1
                int t = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const int64_t v = __shfl_sync(kFull, my_start, t + step - 1);
                    if (v <= e[u]) t += step;
                }
                if (t == 31 && last <= e[u]) t = 32;
                const int row = t - 1;
                const int32_t prow = __shfl_sync(kFull, pi, row < 0 ? 0 : row);
                if (e[u] < hi && (int64_t)j[u] > rb + r0 + row && pj[u] != prow) neumaier_add(s, c, wv[u]);
            }
        }
    }
    __shared__ double red[kCutThreads];
    red[threadIdx.x] = s + c;
    __syncthreads();
    for (int h = kCutThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
    if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(bad, 1);
}

// One CTA: strided Neumaier sums, then a fixed-shape tree (deterministic).
__global__ void __launch_bounds__(kCutThreads) k_cutsize_final(const double *partials, int n, const int *bad,
                                                               double *cut) {
    double s = 0.0, c = 0.0;
    for (int k = threadIdx.x; k < n; k += kCutThreads) neumaier_add(s, c, partials[k]);
    __shared__ double red[kCutThreads];
    red[threadIdx.x] = s + c;
    __syncthreads();
    for (int h = kCutThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) *cut = *bad ? __longlong_as_double(0x7ff8000000000000ll) : red[0];
}

int cutsize_blocks() { return num_sms() * 8; }

// Fused-cut partials: nseg segments of `stride` slots, segment g holding
// used[g] partials.  Fixed order: deterministic.
__global__ void __launch_bounds__(kCutThreads) k_cut_final_seg(const double *partials, const int *used, int nseg,
                                                               int stride, const int *bad, double *cut) {
    double s = 0.0, c = 0.0;
    for (int g = 0; g < nseg; ++g) {
        const int n = used[g];
        for (int k = threadIdx.x; k < n; k += kCutThreads) neumaier_add(s, c, partials[(int64_t)g * stride + k]);
    }
    __shared__ double red[kCutThreads];
    red[threadIdx.x] = s + c;
    __syncthreads();
    for (int h = kCutThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) *cut = *bad ? __longlong_as_double(0x7ff8000000000000ll) : red[0];
}

void launch_cut_final(const double *partials, const int *used, int nseg, int stride, const int *bad, double *cut,
                      cudaStream_t s) {
    k_cut_final_seg<<<1, kCutThreads, 0, s>>>(partials, used, nseg, stride, bad, cut);
    note_launch();
}

void launch_cutsize(const int64_t *grp, const int32_t *gcol, const double *gw, int64_t nloc, int64_t rb,
                    int64_t n_global, const int32_t *part, int32_t K, double *partials, int nblocks, double *cut,
                    cudaStream_t s) {
    int *bad = reinterpret_cast<int *>(partials + nblocks);
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    k_cutsize<<<nblocks, kCutThreads, 0, s>>>(grp, gcol, gw, nloc, rb, n_global, part, K, partials, bad);
    k_cutsize_final<<<1, kCutThreads, 0, s>>>(partials, nblocks, bad, cut);
    note_launch(2);
}

// ------------------------------------------------------------------ f2: IP matrix, part weights
// ip_km = sum of the stored weights w_ij with part[i] = k != m = part[j]
// (eq. ip_km), W_k = sum of w(v_i) over part k, w = 1 or
// nnz(r_i) (eq16, 1141-1146 eq. Wk).  Every weight is added
// as the fixed-point value trunc(w * 2^64) split into four 32-bit limbs, each
// summed in its own 64-bit counter: integer sums, so the result is exact and
// independent of the summation order (deterministic under any schedule and
// across GPUs: ranks allreduce the counters as integers).  For K <= 32 a CTA
// accumulates in shared memory first.
constexpr int kIpThreads = 256;
constexpr int kIpSmemK = 32;

__device__ __forceinline__ bool add_fixed(unsigned long long *acc4, double w) {
    if (!(w >= 0.0) || w >= 9.2233720368547758e18) return false;  // 2^63: outside the fixed-point range
    const unsigned long long hi = (unsigned long long)w;            // floor (w >= 0)
    const unsigned long long lo = __double2ull_rz((w - (double)hi) * 18446744073709551616.0);  // frac * 2^64
    const unsigned long long l[4] = {lo & 0xffffffffull, lo >> 32, hi & 0xffffffffull, hi >> 32};
#pragma unroll
    for (int t = 0; t < 4; ++t)
        if (l[t]) atomicAdd(&acc4[t], l[t]);
    return true;
}

__global__ void __launch_bounds__(kIpThreads) k_partition_ip(const int64_t *__restrict__ grp,
                                                             const int32_t *__restrict__ gcol,
                                                             const double *__restrict__ gw, int64_t nloc, int64_t rb,
                                                             int64_t n_global, const int32_t *__restrict__ part,
                                                             int32_t K, const int64_t *__restrict__ arp,
                                                             unsigned long long *acc, unsigned long long *wsum,
                                                             int *bad) {
    __shared__ unsigned long long s_acc[4 * kIpSmemK * kIpSmemK];
    __shared__ unsigned long long s_w[kIpSmemK];
    const bool priv = K <= kIpSmemK;
    if (priv) {
        for (int t = threadIdx.x; t < 4 * K * K; t += kIpThreads) s_acc[t] = 0ull;
        for (int t = threadIdx.x; t < K; t += kIpThreads) s_w[t] = 0ull;
        __syncthreads();
    }
    const int l = lane_id();
    int badp = 0;
    for (int64_t v = (int64_t)blockIdx.x * kIpThreads + threadIdx.x; v < n_global; v += (int64_t)gridDim.x * kIpThreads) {
        const int32_t p = part[v];
        badp |= (p < 0) | (p >= K);
    }
    if (__syncthreads_or(badp)) {  // ids are checked before any use as an index
        if (threadIdx.x == 0) atomicOr(bad, 1);
        return;
    }
    const int64_t nwarps = ((int64_t)gridDim.x * kIpThreads) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * kIpThreads + threadIdx.x) >> 5; r < nloc; r += nwarps) {
        const int64_t i = rb + r;
        const int32_t k = part[i];
        if (l == 0) {
            const unsigned long long wv = arp ? (unsigned long long)(arp[i + 1] - arp[i]) : 1ull;
            atomicAdd(priv ? &s_w[k] : &wsum[k], wv);
        }
        for (int64_t e = grp[r] + l; e < grp[r + 1]; e += 32) {
            const int32_t m = part[gcol[e]];
            if (m == k) continue;
            const int64_t cell = (int64_t)k * K + m;
            if (!add_fixed(priv ? &s_acc[4 * cell] : &acc[4 * cell], gw[e])) badp = 1;
        }
    }
    if (priv) {
        __syncthreads();
        for (int t = threadIdx.x; t < 4 * K * K; t += kIpThreads)
            if (s_acc[t]) atomicAdd(&acc[t], s_acc[t]);
        for (int t = threadIdx.x; t < K; t += kIpThreads)
            if (s_w[t]) atomicAdd(&wsum[t], s_w[t]);
    }
    if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(bad, 1);
}

void launch_partition_ip(const int64_t *grp, const int32_t *gcol, const double *gw, int64_t nloc, int64_t rb,
                         int64_t n_global, const int32_t *part, int32_t K, const int64_t *arp, unsigned long long *acc,
                         unsigned long long *wsum, int *bad, cudaStream_t s) {
    int64_t g = (std::max<int64_t>(nloc, 1) * 32 + kIpThreads - 1) / kIpThreads;
    const int64_t cap = (int64_t)num_sms() * 8;
    g = g < 1 ? 1 : (g > cap ? cap : g);
    k_partition_ip<<<(unsigned)g, kIpThreads, 0, s>>>(grp, gcol, gw, nloc, rb, n_global, part, K, arp, acc, wsum,
                                                      bad);
    note_launch();
}

// ------------------------------------------------------------------ row split
// split[g] = smallest r with fprefix[r] >= ceil(g * P / parts); split[parts] = n.
__global__ void k_split(const int64_t *__restrict__ fprefix, int64_t n, int32_t parts, int64_t *split) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g > parts) return;
    const int64_t P = fprefix[n];
    if (g == parts) {
        split[g] = n;
        return;
    }
    const int64_t target = (int64_t)(((__int128)g * P + parts - 1) / parts);
    int64_t lo = 0, hi = n;  // first r in [0, n] with fprefix[r] >= target
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (fprefix[mid] >= target)
            hi = mid;
        else
            lo = mid + 1;
    }
    split[g] = lo;
}

void launch_split(const int64_t *fprefix, int64_t n, int32_t parts, int64_t *split, cudaStream_t s) {
    k_split<<<(parts + 1 + 127) / 128, 128, 0, s>>>(fprefix, n, parts, split);
    note_launch();
}

}  // namespace rig

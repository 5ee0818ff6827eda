// k_scan.cu -- device-wide exclusive prefix sum with int64 output (CSC column
// pointers, graph row pointers, flop prefix).  Two variants:
//  * single pass (k_scan_1p, the default when no shape statistics are
//    wanted): tiles of kTile items taken in order from a ticket; each tile
//    publishes its total, then finds its prefix by a decoupled look-back over
//    the earlier tiles' 64-bit status words (2 flag bits + a 62-bit value).
//    Assumptions: every prefix is < 2^62; forward progress holds because a
//    tile only waits on tiles with lower tickets, which were taken by CTAs
//    already running (tickets are handed out by resident CTAs only).
//  * two launches (k_tile_sum + k_tile_scan, used with the shape statistics
//    or an event between the passes): per-tile totals, then each CTA adds the
//    totals of all earlier tiles (tiles are few: <= n / 4096), so there is no
//    serial chain between CTAs.
#include "common.cuh"

namespace rig {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int64_t kTile = (int64_t)kScanThreads * kScanItems;

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

template <typename T>
__device__ __forceinline__ int64_t scan_load(const T *in, int64_t i, ScanOp op) {
    int64_t x = (int64_t)in[i];
    if (op == ScanOp::UbOffDiag) x = x > 0 ? x - 1 : 0;  // structural off-diagonal nnz
    return x;
}

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *total) {
    __shared__ int64_t wsum[kScanThreads / 32];
    const int w = threadIdx.x >> 5, l = lane_id();
    const int64_t inc = warp_incl_scan(v);
    if (l == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int64_t x = l < kScanThreads / 32 ? wsum[l] : 0;
        const int64_t xi = warp_incl_scan(x);
        if (l < kScanThreads / 32) wsum[l] = xi - x;
        if (l == kScanThreads / 32 - 1) *total = xi;
    }
    __syncthreads();
    const int64_t r = wsum[w] + inc - v;
    __syncthreads();
    return r;
}

// Optional shape statistics, taken on the column counts while they are summed
// (and on the row pointers of the shard): max column, sum of len^2, max row,
// shard nnz -- see DevCounters.
struct ShapeOut {
    DevCounters *ctr;  // null: no statistics
    const int64_t *rp;
    int64_t rb, re;
};

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sum(const T *__restrict__ in, int64_t n, ScanOp op,
                                                           int64_t *tile_sums, ShapeOut so, const int *guard) {
    if (guard_skip(guard)) return;
    const int64_t base = blockIdx.x * kTile;
    int64_t s = 0;
    unsigned long long ps = 0, mc = 0, mr = 0, mn = 0;  // mn: max of kMinRowBias - len
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) {
            const int64_t x = scan_load(in, i, op);
            s += x;
            ps += (unsigned long long)x * (unsigned long long)x;
            mc = max(mc, (unsigned long long)x);
        }
    }
    s = warp_sum(s);
    __shared__ int64_t ws[kScanThreads / 32];
    if (lane_id() == 0) ws[threadIdx.x >> 5] = s;
    if (so.ctr) {
        const int64_t stride = (int64_t)gridDim.x * kScanThreads;
#pragma unroll 8
        for (int64_t i = so.rb + blockIdx.x * (int64_t)kScanThreads + threadIdx.x; i < so.re; i += stride)
        {
            const unsigned long long len = (unsigned long long)(so.rp[i + 1] - so.rp[i]);
            mr = max(mr, len);
            mn = max(mn, (unsigned long long)kMinRowBias - len);
        }
        ps = warp_sum(ps);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mc = max(mc, __shfl_xor_sync(kFull, mc, o));
            mr = max(mr, __shfl_xor_sync(kFull, mr, o));
            mn = max(mn, __shfl_xor_sync(kFull, mn, o));
        }
        __shared__ unsigned long long red[4][kScanThreads / 32];
        if (lane_id() == 0) {
            red[0][threadIdx.x >> 5] = ps;
            red[1][threadIdx.x >> 5] = mc;
            red[2][threadIdx.x >> 5] = mr;
            red[3][threadIdx.x >> 5] = mn;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < kScanThreads / 32; ++k) {
                ps += red[0][k];
                mc = max(mc, red[1][k]);
                mr = max(mr, red[2][k]);
                mn = max(mn, red[3][k]);
            }
            if (ps) atomicAdd((unsigned long long *)&so.ctr->p_full, ps);
            if (mc) atomicMax((unsigned long long *)&so.ctr->max_col, mc);
            if (mr) atomicMax((unsigned long long *)&so.ctr->max_row, mr);
            if (mn) atomicMax((unsigned long long *)&so.ctr->min_row_c, mn);
            if (blockIdx.x == 0) so.ctr->shard_nnz = so.rp[so.re] - so.rp[so.rb];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int k = 0; k < kScanThreads / 32; ++k) t += ws[k];
        tile_sums[blockIdx.x] = t;
    }
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T *__restrict__ in, int64_t n, ScanOp op,
                                                            const int64_t *__restrict__ tile_sums, int64_t ntiles,
                                                            int64_t *out, const int *guard) {
    if (guard_skip(guard)) return;
    __shared__ int64_t sv[kTile + kTile / 16];  // padded: conflict-free blocked <-> striped transpose
    __shared__ int64_t tot_s, pre_s;
    // prefix of the earlier tiles' totals
    int64_t pre = 0;
    for (int64_t t = threadIdx.x; t < blockIdx.x; t += kScanThreads) pre += tile_sums[t];
    pre = warp_sum(pre);
    __shared__ int64_t ws[kScanThreads / 32];
    if (lane_id() == 0) ws[threadIdx.x >> 5] = pre;
    const int64_t base = blockIdx.x * kTile;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {  // coalesced blocked load
        const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        sv[pad(j * kScanThreads + threadIdx.x)] = i < n ? scan_load(in, i, op) : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int k = 0; k < kScanThreads / 32; ++k) t += ws[k];
        pre_s = t;
    }
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = sv[pad(threadIdx.x * kScanItems + j)];
        s += v[j];
    }
    const int64_t ex = block_excl_scan(s, &tot_s);  // (contains __syncthreads: pre_s visible after)
    int64_t run = pre_s + ex;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        sv[pad(threadIdx.x * kScanItems + j)] = run;
        run += v[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) out[i] = sv[pad(j * kScanThreads + threadIdx.x)];
    }
    if (blockIdx.x == ntiles - 1 && threadIdx.x == 0) out[n] = pre_s + tot_s;
}

// Single-pass variant (no shape statistics): tiles are taken in order from a
// ticket, each publishes its total and then its inclusive prefix, found by a
// decoupled look-back over the previous tiles' status words (a tile only waits
// on tiles that started before it, so the chain always completes).  tmp holds
// the status words [ntiles] and the ticket, zeroed before the launch.
constexpr unsigned long long kScanAgg = 1ull << 62, kScanPre = 2ull << 62, kScanVal = (1ull << 62) - 1;

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_1p(const T *__restrict__ in, int64_t n, ScanOp op,
                                                          unsigned long long *status, unsigned *ticket, int64_t *out,
                                                          const int *guard) {
    if (guard_skip(guard)) return;
    __shared__ int64_t sv[kTile + kTile / 16];
    __shared__ int64_t tot_s, pre_s;
    __shared__ unsigned tile_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t base = tile * kTile;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {  // coalesced blocked load
        const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        sv[pad(j * kScanThreads + threadIdx.x)] = i < n ? scan_load(in, i, op) : 0;
    }
    __syncthreads();
    int64_t v[kScanItems];
    int64_t sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = sv[pad(threadIdx.x * kScanItems + j)];
        sum += v[j];
    }
    const int64_t ex = block_excl_scan(sum, &tot_s);
    if (threadIdx.x < 32) {  // warp 0: publish the total, look back, publish the prefix
        const int l = lane_id();
        const unsigned long long tot = (unsigned long long)tot_s;
        int64_t excl = 0;
        if (tile == 0) {
            if (l == 0) {
                __threadfence();
                atomicExch(&status[0], kScanPre | tot);
            }
        } else {
            if (l == 0) {
                __threadfence();
                atomicExch(&status[tile], kScanAgg | tot);
            }
            int64_t b = tile - 1;
            while (true) {
                const int64_t j = b - l;
                unsigned long long st = 2ull << 62;  // before tile 0: an inclusive prefix of 0
                if (j >= 0) st = *reinterpret_cast<volatile unsigned long long *>(&status[j]);
                const unsigned pm = __ballot_sync(kFull, (st & kScanPre) != 0);
                const unsigned zm = __ballot_sync(kFull, (st & (kScanPre | kScanAgg)) == 0);
                const int fp = pm ? __ffs(pm) - 1 : 31;
                const unsigned need = fp == 31 ? kFull : ((2u << fp) - 1u);
                if (zm & need) continue;  // a needed earlier tile has not published yet
                __threadfence();
                excl += warp_sum(((need >> l) & 1u) ? (int64_t)(st & kScanVal) : (int64_t)0);
                if (pm) break;
                b -= 32;
            }
            if (l == 0) {
                __threadfence();
                atomicExch(&status[tile], kScanPre | (unsigned long long)(excl + (int64_t)tot));
            }
        }
        if (l == 0) pre_s = excl;
    }
    __syncthreads();
    int64_t run = pre_s + ex;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        sv[pad(threadIdx.x * kScanItems + j)] = run;
        run += v[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) out[i] = sv[pad(j * kScanThreads + threadIdx.x)];
    }
    if (base + kTile >= n && threadIdx.x == 0) out[n] = pre_s + tot_s;
}

size_t scan_tmp_bytes(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    return (size_t)(ntiles + 1) * sizeof(int64_t);
}

template <typename T>
static void scan_impl(const T *in, int64_t n, int64_t *out, ScanOp op, void *tmp, cudaStream_t s,
                      ShapeOut so = ShapeOut{nullptr, nullptr, 0, 0}, cudaEvent_t after_sum = nullptr,
                      const int *guard = nullptr) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    if (ntiles == 0) {
        cudaMemsetAsync(out, 0, sizeof(int64_t), s);
        return;
    }
    if (!so.ctr && !after_sum) {  // single pass
        auto *st = static_cast<unsigned long long *>(tmp);
        cudaMemsetAsync(st, 0, sizeof(unsigned long long) * (size_t)(ntiles + 1), s);
        k_scan_1p<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, op, st, reinterpret_cast<unsigned *>(st + ntiles),
                                                                out, guard);
        note_launch();
        return;
    }
    int64_t *ts = static_cast<int64_t *>(tmp);
    k_tile_sum<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, op, ts, so, guard);
    if (after_sum) cudaEventRecord(after_sum, s);
    k_tile_scan<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, op, ts, ntiles, out, guard);
    note_launch(2);
}

void scan_i64(const int64_t *in, int64_t n, int64_t *out, ScanOp op, void *tmp, size_t, cudaStream_t s) {
    scan_impl<int64_t>(in, n, out, op, tmp, s);
}

void scan_u32(const unsigned *in, int64_t n, int64_t *out, void *tmp, size_t, cudaStream_t s, const int *guard) {
    scan_impl<unsigned>(in, n, out, ScanOp::Identity, tmp, s, ShapeOut{nullptr, nullptr, 0, 0}, nullptr, guard);
}

void scan_u32_shape(const unsigned *in, int64_t n, int64_t *out, void *tmp, DevCounters *ctr, const int64_t *rp,
                    int64_t rb, int64_t re, void *host_copy, cudaEvent_t ready, cudaStream_t s,
                    const int *guard) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    if (ntiles == 0) {  // no columns: the statistics are zeros except the shard
        cudaMemsetAsync(out, 0, sizeof(int64_t), s);
        cudaMemcpyAsync(host_copy, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ready, s);
        return;
    }
    int64_t *ts = static_cast<int64_t *>(tmp);
    k_tile_sum<unsigned><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, ScanOp::Identity, ts,
                                                                    ShapeOut{ctr, rp, rb, re}, guard);
    // the statistics go to the host from a side stream (per thread and
    // device), so the build's stream never waits on the PCIe round trip; the
    // host reads only the shape fields, which nothing on `s` writes again
    // before the host has waited on `ready`
    struct Side {
        int dev = -1;
        cudaStream_t st = nullptr;
        cudaEvent_t done = nullptr;
    };
    static thread_local Side side[8];
    int dev = 0;
    cudaGetDevice(&dev);
    Side *sd = dev >= 0 && dev < 8 ? &side[dev] : nullptr;
    if (sd && !sd->st) {
        if (cudaStreamCreateWithFlags(&sd->st, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd->done, cudaEventDisableTiming) != cudaSuccess)
            sd->st = nullptr;
    }
    if (sd && sd->st) {
        cudaEventRecord(sd->done, s);
        cudaStreamWaitEvent(sd->st, sd->done, 0);
        cudaMemcpyAsync(host_copy, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, sd->st);
        cudaEventRecord(ready, sd->st);
    } else {
        cudaMemcpyAsync(host_copy, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ready, s);
    }
    k_tile_scan<unsigned><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, ScanOp::Identity, ts, ntiles, out, guard);
    note_launch(2);
}

}  // namespace rig

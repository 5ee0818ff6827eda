// k_scan.cu -- device-wide exclusive prefix sum, int64 output (used for the
// CSC column pointers, the graph row pointers and the flop prefix).
// Three launches: per-tile reduce, one-CTA scan of tile sums, per-tile scan.
#include "common.cuh"

namespace rig {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int64_t kTile = (int64_t)kScanThreads * kScanItems;

template <typename T>
struct Load {
    __device__ __forceinline__ int64_t operator()(const T *in, int64_t i, ScanOp op) const {
        int64_t x = (int64_t)in[i];
        if (op == ScanOp::UbOffDiag) x = x > 0 ? x - 1 : 0;  // structural off-diagonal nnz
        return x;
    }
};

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *total) {
    __shared__ int64_t wsum[kScanThreads / 32];
    const int w = threadIdx.x >> 5, l = lane_id();
    int64_t inc = warp_incl_scan(v);
    if (l == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        int64_t x = l < kScanThreads / 32 ? wsum[l] : 0;
        int64_t xi = warp_incl_scan(x);
        if (l < kScanThreads / 32) wsum[l] = xi - x;
        if (l == kScanThreads / 32 - 1) *total = xi;
    }
    __syncthreads();
    const int64_t r = wsum[w] + inc - v;
    __syncthreads();
    return r;
}

template <typename T>
__global__ void k_tile_reduce(const T *__restrict__ in, int64_t n, ScanOp op, int64_t *tile_sums) {
    const int64_t base = blockIdx.x * kTile;
    int64_t s = 0;
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) s += Load<T>()(in, i, op);
    }
    __shared__ int64_t tot;
    int64_t dummy = block_excl_scan(s, &tot);
    (void)dummy;
    __syncthreads();
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void k_scan_tiles(int64_t *tile_sums, int64_t ntiles, int64_t *out_total) {
    __shared__ int64_t carry_s;
    __shared__ int64_t tot;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int64_t base = 0; base < ntiles; base += kScanThreads) {
        const int64_t i = base + threadIdx.x;
        const int64_t v = i < ntiles ? tile_sums[i] : 0;
        const int64_t ex = block_excl_scan(v, &tot);
        const int64_t c = carry_s;
        if (i < ntiles) tile_sums[i] = c + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = c + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *out_total = carry_s;
}

template <typename T>
__global__ void k_tile_scan(const T *__restrict__ in, int64_t n, ScanOp op, const int64_t *tile_offs,
                            int64_t *out) {
    const int64_t base = blockIdx.x * kTile + (int64_t)threadIdx.x * kScanItems;
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + j;
        v[j] = i < n ? Load<T>()(in, i, op) : 0;
        s += v[j];
    }
    __shared__ int64_t tot;
    int64_t run = block_excl_scan(s, &tot) + tile_offs[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
}

size_t scan_tmp_bytes(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    return (size_t)(ntiles + 1) * sizeof(int64_t);
}

template <typename T>
static void scan_impl(const T *in, int64_t n, int64_t *out, ScanOp op, void *tmp, cudaStream_t s) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    int64_t *tile = static_cast<int64_t *>(tmp);
    if (ntiles == 0) {
        cudaMemsetAsync(out, 0, sizeof(int64_t), s);
        return;
    }
    k_tile_reduce<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, op, tile);
    k_scan_tiles<<<1, kScanThreads, 0, s>>>(tile, ntiles, out + n);
    k_tile_scan<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, n, op, tile, out);
    note_launch(3);
}

void scan_i64(const int64_t *in, int64_t n, int64_t *out, ScanOp op, void *tmp, size_t, cudaStream_t s) {
    scan_impl<int64_t>(in, n, out, op, tmp, s);
}

void scan_u32(const unsigned *in, int64_t n, int64_t *out, void *tmp, size_t, cudaStream_t s) {
    scan_impl<unsigned>(in, n, out, ScanOp::Identity, tmp, s);
}

}  // namespace rig

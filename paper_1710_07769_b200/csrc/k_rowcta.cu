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
// wide-window / global-far-list / CTA-accumulator chain).
#include "common.cuh"

namespace rig {

constexpr int kRcThreads = 256;
constexpr int kRcWarps = kRcThreads / 32;
constexpr int kRcBins = 256;

__host__ __device__ constexpr size_t rc_item_bytes() { return 4 + 4 + 2 + 2 + 8 + 8; }
size_t rowcta_smem_bytes(int fmax) {
    return (size_t)fmax * rc_item_bytes() + (size_t)kRcWarps * kRcBins * 4 + 64 * 8;
}

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

__global__ void __launch_bounds__(kRcThreads) k_row_cta(RcArgs a) {
    extern __shared__ __align__(16) unsigned char rc_smem[];
    const int F = a.fmax;
    double *ia = reinterpret_cast<double *>(rc_smem);  // a_ik of item
    double *ib = ia + F;                                // a_jk of item
    unsigned *key0 = reinterpret_cast<unsigned *>(ib + F);
    unsigned *key1 = key0 + F;
    unsigned *hist = key1 + F;                          // [warp][bin], then offsets
    int *ws = reinterpret_cast<int *>(hist + kRcWarps * kRcBins);
    int64_t *misc = reinterpret_cast<int64_t *>(ws + 32);
    uint16_t *idx0 = reinterpret_cast<uint16_t *>(misc + 8);
    uint16_t *idx1 = idx0 + F;
    const int tid = threadIdx.x, l = lane_id(), w = tid >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t n0 = *a.count0, n1 = a.list1 ? *a.count1 : 0;
    int passes = 0;
    for (int64_t m = a.A.nrows - 1; m > 0; m >>= 8) ++passes;
    for (;;) {
        if (tid == 0) misc[0] = (int64_t)atomicAdd(a.ticket, 1ull);
        __syncthreads();
        const int64_t t = misc[0];
        __syncthreads();
        if (t >= n0 + n1) break;
        const int64_t i = t < n0 ? a.list0[t] : a.list1[t - n0];
        const int64_t r = i - a.rb;
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        const int64_t f = a.fnm[r] + (e - s);
        if (f > F) {
            if (tid == 0) a.rest[atomicAdd((unsigned long long *)a.rest_count, 1ull)] = (int32_t)i;
            continue;
        }
        // ---- expand in arrival order
        int base = 0;
        for (int64_t e0 = s; e0 < e; e0 += kRcThreads) {
            const int64_t p = e0 + tid;
            int cl = 0;
            int64_t cs = 0;
            double av = 0.0;
            if (p < e) {
                const int k = a.A.ci[p];
                const int64_t c0 = a.T.cp[k];
                cl = (int)(a.T.cp[k + 1] - c0);
                cs = c0 + k;
                av = a.A.v[p];
            }
            int tot;
            const int off = base + rc_block_scan(cl, ws, &tot);
            for (int q = 0; q < cl; ++q) {
                const int it = off + q;
                key0[it] = (unsigned)a.T.ri[cs + q];
                idx0[it] = (uint16_t)it;
                ia[it] = av;
                ib[it] = a.T.vt[cs + q];
            }
            base += tot;
        }
        const int nit = base;  // == f
        __syncthreads();
        // ---- stable LSD radix sort of (key, item) by key
        unsigned *kin = key0, *kout = key1;
        uint16_t *xin = idx0, *xout = idx1;
        const int chunk = ((nit + kRcWarps - 1) / kRcWarps + 31) / 32 * 32;
        const int w0 = min(nit, w * chunk), w1 = min(nit, w0 + chunk);
        for (int d = 0; d < passes; ++d) {
            const int sh = 8 * d;
            for (int b = tid; b < kRcWarps * kRcBins; b += kRcThreads) hist[b] = 0;
            __syncthreads();
            unsigned *hw = hist + w * kRcBins;
            for (int p0 = w0; p0 < w1; p0 += 32) {  // this warp's slice, in order
                const int p = p0 + l;
                const int dg = p < w1 ? (int)((kin[p] >> sh) & 255u) : kRcBins + l;
                const unsigned g = __match_any_sync(kFull, dg);
                if (p < w1 && (g & lt) == 0) hw[dg] += __popc(g);
                __syncwarp();
            }
            __syncthreads();
            // offsets, digit-major then warp: thread b owns digit b's 8 counters
            int c[kRcWarps], sum = 0;
#pragma unroll
            for (int u = 0; u < kRcWarps; ++u) {
                c[u] = hist[u * kRcBins + tid];
                sum += c[u];
            }
            int tot;
            int run = rc_block_scan(sum, ws, &tot);
#pragma unroll
            for (int u = 0; u < kRcWarps; ++u) {
                hist[u * kRcBins + tid] = run;
                run += c[u];
            }
            __syncthreads();
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
        const int64_t t0 = a.toff[r];
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
                        acc = __fma_rn(ia[x], ib[x], acc);
                    }
                    if ((int64_t)key == i) {
                        if (a.diag) a.diag[r] = acc;
                    } else {
                        wv = fabs(acc);
                        keep = wv > a.tol;
                    }
                }
            }
            int tot;
            const int pos = obase + rc_block_scan(keep ? 1 : 0, ws, &tot);
            if (keep) {
                a.tcol[t0 + pos] = (int32_t)key;
                a.tw[t0 + pos] = wv;
            }
            obase += tot;
        }
        if (tid == 0) a.cnt[r] = obase + 1;  // the graph scan subtracts the diagonal slot
        if (e == s && tid == 0 && a.diag) a.diag[r] = 0.0;
        __syncthreads();
    }
}

void launch_row_cta(const RcArgs &a, cudaStream_t s) {
    const size_t smem = rowcta_smem_bytes(a.fmax);
    cudaFuncSetAttribute(k_row_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_row_cta, kRcThreads, smem);
    if (per_sm < 1) per_sm = 1;
    k_row_cta<<<num_sms() * per_sm, kRcThreads, smem, s>>>(a);
    note_launch();
}

}  // namespace rig

// k_coarsen.cu -- SURVEY.md §8(f) f4: the first stage of a multilevel
// partitioner on G_RIP (the paper hands G_RIP with integer edge weights to
// METIS, and proposes a parallel partitioner, PAPER.md:
// 1119-1122): heavy-edge matching and one coarsening step, on a symmetric
// CSR graph with int64 edge weights (rig_int_weights of G_RIP).  Readings:
// DESIGN.md R23 (matching), R24 (coarse vertices), R25 (coarse edges).
//
//  * k_hem_pick: one warp per unmatched vertex v picks its heaviest unmatched
//    neighbour (ties to the smaller index) -- a warp reduction of (w, -u).
//  * k_hem_match: v matches u iff v picked u and u picked v (each side writes
//    its own entry: no races).  Rounds repeat on the vertices left over.
//  * k_coarse_map: leaders (v unmatched, or v < match(v)) are counted by a
//    scan: coarse id = rank of the leader; cmap, lead, coarse vertex weights.
//  * k_coarse_rows<PASS, BIG>: one warp per coarse vertex gathers the mapped
//    neighbour lists of its members as items (cmap(j) << 32 | position),
//    bitonic-sorts them (shared memory up to 1024 items; a per-warp slice of
//    global scratch beyond, in a separate launch), sums the weights of equal
//    keys (integers: order-free, exact) and drops its own id, writing the row
//    with its exact count into a temporary at offsets from the rows' item
//    bounds (pass 2); after the scan of the counts, k_coarse_copy places the
//    rows (pass 0/1: count, then write at the scanned offsets, sort twice).
#include "common.cuh"

namespace rig {

constexpr int kCoarseThreads = 64;  // 2 warps: 32 KB of static shared memory
constexpr int kCoarseWarps = kCoarseThreads / 32;
constexpr int kSmemItems = 1024;

__global__ void k_hem_pick(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                           const int64_t *__restrict__ wgt, int64_t n, const int32_t *__restrict__ match,
                           int32_t *cand) {
    const int l = lane_id();
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
        if (match[v] >= 0) {
            if (l == 0) cand[v] = -1;
            continue;
        }
        bool have = false;
        int64_t bw = 0;
        int bu = INT_MAX;
        for (int64_t p = rp[v] + l; p < rp[v + 1]; p += 32) {
            const int u = col[p];
            if ((int64_t)u == v || match[u] >= 0) continue;
            const int64_t w = wgt[p];
            if (!have || w > bw || (w == bw && u < bu)) {
                have = true;
                bw = w;
                bu = u;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const bool oh = __shfl_xor_sync(kFull, (int)have, o);
            const int64_t ow = __shfl_xor_sync(kFull, bw, o);
            const int ou = __shfl_xor_sync(kFull, bu, o);
            if (oh && (!have || ow > bw || (ow == bw && ou < bu))) {
                have = true;
                bw = ow;
                bu = ou;
            }
        }
        if (l == 0) cand[v] = have ? bu : -1;
    }
}

__global__ void k_hem_match(const int32_t *__restrict__ cand, int64_t n, int32_t *match) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int u = cand[v];
        if (match[v] < 0 && u >= 0 && (int64_t)cand[u] == v) match[v] = u;
    }
}

__global__ void k_leader_flags(const int32_t *__restrict__ match, int64_t n, int64_t *flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int m = match[v];
        flag[v] = (m < 0 || v < (int64_t)m) ? 1 : 0;
    }
}

// cid: exclusive scan of the leader flags ([n + 1], cid[n] = nc).  maxit:
// the largest item count of a coarse row (the members' degrees).
__global__ void k_coarse_map(const int64_t *__restrict__ rp, const int32_t *__restrict__ match,
                             const int64_t *__restrict__ vwgt, int64_t n, const int64_t *__restrict__ cid,
                             int32_t *cmap, int32_t *lead, int64_t *cvwgt, int64_t *citems,
                             unsigned long long *maxit) {
    unsigned long long mx = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int m = match[v];
        const int64_t ld = (m < 0 || v < (int64_t)m) ? v : (int64_t)m;
        const int64_t c = cid[ld];
        cmap[v] = (int32_t)c;
        if (ld == v) {
            lead[c] = (int32_t)v;
            int64_t w = vwgt ? vwgt[v] : 1;
            int64_t it = rp[v + 1] - rp[v];
            if (m >= 0) {
                w += vwgt ? vwgt[m] : 1;
                it += rp[m + 1] - rp[m];
            }
            cvwgt[c] = w;
            citems[c] = it;  // >= the coarse row's entries: its slots in the temporary
            mx = max(mx, (unsigned long long)it);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane_id() == 0 && mx) atomicMax(maxit, mx);
}

// Ascending bitonic sort of N (a power of two) 64-bit keys by one warp.
__device__ __forceinline__ void warp_bitonic(uint64_t *key, int N) {
    const int l = lane_id();
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = l; i < N; i += 32) {
                const int p = i ^ j;
                if (p > i) {
                    const uint64_t a = key[i], b = key[p];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        key[i] = b;
                        key[p] = a;
                    }
                }
            }
            __syncwarp();
        }
    }
}

struct CoarseArgs {
    const int64_t *rp;
    const int32_t *col;
    const int64_t *wgt;
    const int32_t *match;
    const int32_t *cmap;
    const int32_t *lead;
    int64_t nc;
    int64_t *ccnt;        // pass 0: kept entries per coarse row
    const int64_t *crp;   // pass 1: coarse row pointers
    int32_t *ccol;
    int64_t *cw;
    uint64_t *gscratch;   // BIG: per warp [2 * gcap] (keys, then weights)
    int64_t gcap;
};

template <int PASS, bool BIG>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_rows(CoarseArgs a) {
    __shared__ uint64_t s_key[BIG ? 1 : kCoarseWarps][BIG ? 1 : kSmemItems];
    __shared__ int64_t s_w[BIG ? 1 : kCoarseWarps][BIG ? 1 : kSmemItems];
    const int w = threadIdx.x >> 5, l = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t *key = BIG ? a.gscratch + gw * 2 * a.gcap : &s_key[0][0] + (BIG ? 0 : w * kSmemItems);
    int64_t *wt = BIG ? reinterpret_cast<int64_t *>(a.gscratch + gw * 2 * a.gcap + a.gcap)
                      : &s_w[0][0] + (BIG ? 0 : w * kSmemItems);
    const unsigned lt = lanemask_lt();
    for (int64_t c = gw; c < a.nc; c += nw) {
        const int v = a.lead[c];
        const int u = a.match[v];
        const int64_t sv = a.rp[v], ev = a.rp[v + 1];
        const int64_t su = u >= 0 ? a.rp[u] : 0, eu = u >= 0 ? a.rp[u + 1] : 0;
        const int64_t nv = ev - sv, nit = nv + (eu - su);
        if ((nit > kSmemItems) != BIG) continue;  // the other launch takes it
        int N = 1;
        while (N < nit) N <<= 1;
        for (int64_t t = l; t < N; t += 32) {
            if (t < nit) {
                const int64_t p = t < nv ? sv + t : su + (t - nv);
                key[t] = ((uint64_t)(uint32_t)a.cmap[a.col[p]] << 32) | (uint64_t)t;
                wt[t] = a.wgt[p];
            } else {
                key[t] = ~0ull;
            }
        }
        __syncwarp();
        warp_bitonic(key, N);
        // runs of equal coarse id: the first item of a run sums it
        int64_t base = PASS ? a.crp[c] : 0;  // PASS 2: crp holds the temporary offsets
        int64_t kept = 0;
        for (int64_t t0 = 0; t0 < nit; t0 += 32) {
            const int64_t t = t0 + l;
            bool head = false;
            int64_t sum = 0;
            uint32_t kc = 0;
            if (t < nit) {
                kc = (uint32_t)(key[t] >> 32);
                head = (t == 0 || (uint32_t)(key[t - 1] >> 32) != kc) && (int64_t)kc != c;
                if (head) {
                    int64_t q = t;
                    do {
                        sum += wt[(uint32_t)key[q]];
                        ++q;
                    } while (q < nit && (uint32_t)(key[q] >> 32) == kc);
                }
            }
            const unsigned bal = __ballot_sync(kFull, head);
            if (PASS && head) {
                const int64_t pos = base + kept + __popc(bal & lt);
                a.ccol[pos] = (int32_t)kc;
                a.cw[pos] = sum;
            }
            kept += __popc(bal);
        }
        if (PASS != 1 && l == 0) a.ccnt[c] = kept;
        __syncwarp();
    }
}

// Coarse rows from the temporary (toff, exact counts) to their final slots.
__global__ void k_coarse_copy(const int64_t *__restrict__ toff, const int64_t *__restrict__ crp, int64_t nc,
                              const int32_t *__restrict__ tcol, const int64_t *__restrict__ tw, int32_t *ccol,
                              int64_t *cw) {
    const int l = lane_id();
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nc; c += nw) {
        const int64_t src = toff[c], dst = crp[c], len = crp[c + 1] - dst;
        for (int64_t t = l; t < len; t += 32) {
            ccol[dst + t] = tcol[src + t];
            cw[dst + t] = tw[src + t];
        }
    }
}

void launch_coarse_copy(const int64_t *toff, const int64_t *crp, int64_t nc, const int32_t *tcol, const int64_t *tw,
                        int32_t *ccol, int64_t *cw, cudaStream_t s) {
    if (nc <= 0) return;
    int64_t g = (nc * 32 + 255) / 256;
    if (g > (int64_t)num_sms() * 16) g = (int64_t)num_sms() * 16;
    k_coarse_copy<<<(unsigned)g, 256, 0, s>>>(toff, crp, nc, tcol, tw, ccol, cw);
    note_launch();
}

void launch_hem_round(const int64_t *rp, const int32_t *col, const int64_t *wgt, int64_t n, int32_t *match,
                      int32_t *cand, cudaStream_t s) {
    if (n <= 0) return;
    int64_t g = (n * 32 + 255) / 256;
    if (g > (int64_t)num_sms() * 32) g = (int64_t)num_sms() * 32;
    k_hem_pick<<<(unsigned)g, 256, 0, s>>>(rp, col, wgt, n, match, cand);
    int64_t g2 = (n + 255) / 256;
    if (g2 > (int64_t)num_sms() * 16) g2 = (int64_t)num_sms() * 16;
    k_hem_match<<<(unsigned)g2, 256, 0, s>>>(cand, n, match);
    note_launch(2);
}

void launch_leader_flags(const int32_t *match, int64_t n, int64_t *flag, cudaStream_t s) {
    int64_t g = (n + 255) / 256;
    g = g < 1 ? 1 : (g > (int64_t)num_sms() * 16 ? (int64_t)num_sms() * 16 : g);
    k_leader_flags<<<(unsigned)g, 256, 0, s>>>(match, n, flag);
    note_launch();
}

void launch_coarse_map(const int64_t *rp, const int32_t *match, const int64_t *vwgt, int64_t n, const int64_t *cid,
                       int32_t *cmap, int32_t *lead, int64_t *cvwgt, int64_t *citems, unsigned long long *maxit,
                       cudaStream_t s) {
    int64_t g = (n + 255) / 256;
    g = g < 1 ? 1 : (g > (int64_t)num_sms() * 16 ? (int64_t)num_sms() * 16 : g);
    k_coarse_map<<<(unsigned)g, 256, 0, s>>>(rp, match, vwgt, n, cid, cmap, lead, cvwgt, citems, maxit);
    note_launch();
}

// Rows of up to 1024 items in shared memory; beyond, `big_warps` warps with
// a global scratch slice each (caller-provided, 2 * gcap uint64 per warp).
void launch_coarse_rows(int pass, const int64_t *rp, const int32_t *col, const int64_t *wgt, const int32_t *match,
                        const int32_t *cmap, const int32_t *lead, int64_t nc, int64_t *ccnt, const int64_t *crp,
                        int32_t *ccol, int64_t *cw, uint64_t *gscratch, int64_t gcap, int big_warps,
                        cudaStream_t s) {
    if (nc <= 0) return;
    CoarseArgs a{rp, col, wgt, match, cmap, lead, nc, ccnt, crp, ccol, cw, gscratch, gcap};
    int64_t g = (nc + kCoarseWarps - 1) / kCoarseWarps;
    if (g > (int64_t)num_sms() * 16) g = (int64_t)num_sms() * 16;
    if (pass == 2)
        k_coarse_rows<2, false><<<(unsigned)g, kCoarseThreads, 0, s>>>(a);
    else if (pass == 0)
        k_coarse_rows<0, false><<<(unsigned)g, kCoarseThreads, 0, s>>>(a);
    else
        k_coarse_rows<1, false><<<(unsigned)g, kCoarseThreads, 0, s>>>(a);
    note_launch();
    if (gscratch && big_warps > 0) {
        const unsigned gb = (unsigned)((big_warps + kCoarseWarps - 1) / kCoarseWarps);
        if (pass == 2)
            k_coarse_rows<2, true><<<gb, kCoarseThreads, 0, s>>>(a);
        else if (pass == 0)
            k_coarse_rows<0, true><<<gb, kCoarseThreads, 0, s>>>(a);
        else
            k_coarse_rows<1, true><<<gb, kCoarseThreads, 0, s>>>(a);
        note_launch();
    }
}

}  // namespace rig

// k_spgemm.cu -- steps a4 (symbolic) and a5+a6 (numeric, fused with abs /
// drop / diagonal strip) of the hot path: row i of C = A_hat A_hat^T by
// Gustavson's row-by-row SpGEMM (§2.3), kept as G_RIP edges
// (PAPER.md:293-315, 321-325, 352).
//
// Ordering contract (DESIGN.md §3 R4): every c_ij is the fma-chain over the
// shared columns k in ASCENDING k from +0.0.  Each path below preserves it:
//  * merge path (row length <= 8): one thread per row performs a k-way merge
//    of the row's column runs (sorted by j); for the current minimum j it
//    folds the runs in ascending k -- exactly the chain.
//  * warp-hash path: products are enumerated in (k ascending, column order)
//    and processed in chunks of 32 lanes in that order; lanes with the same j
//    (__match_any_sync) pass the accumulator down the group in lane order, so
//    each key's chain is applied in ascending k.  Then an LSD radix sort
//    orders the row by j.
//  * huge path (one CTA per row): warp w owns the keys with (j/32) % W == w
//    and walks the whole product stream in order, so again every chain runs in
//    ascending k; the dense accumulator's bitmap yields j-sorted output.
#include "common.cuh"

namespace rig {

static int g_sms_cache = 0;

// ======================================================== merge path
// One thread per row i.  The row's R column runs (column k of A_hat^T, rows j
// ascending) are merged; for the current minimum j the runs holding it are
// folded in ascending k: c_ij = fma(a_ik, a_jk, c_ij) -- the ordered chain.
// IdxT: int32 CSC offsets when nnz < 2^31 (fewer registers), else int64.
// Columns end in an INT_MAX sentinel (csc_begin), so a run needs no end bound.
template <int R, typename IdxT>
__device__ __forceinline__ int64_t sym_merge_row(const Csr &A, const Csc &T, int64_t s) {
    int32_t h[R];
    IdxT q[R];
    int64_t f = 0;
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int k = A.ci[s + t];
        const int64_t c0 = T.cp[k], c1 = T.cp[k + 1];
        q[t] = (IdxT)(c0 + k);
        f += c1 - c0;
    }
    if (f > kMergeMaxF) return -1;
#pragma unroll
    for (int t = 0; t < R; ++t) h[t] = T.ri[q[t]];
    int64_t cnt = 0;
    while (true) {
        int m = h[0];
#pragma unroll
        for (int t = 1; t < R; ++t) m = min(m, h[t]);
        if (m == INT_MAX) break;
        ++cnt;
#pragma unroll
        for (int t = 0; t < R; ++t) {
            if (h[t] == m) h[t] = T.ri[++q[t]];
        }
    }
    return cnt;
}

// Writes the kept entries of row i to (oc, ow)[0..), pads the structural
// slots it did not fill ([kept, ub)) with col = -1 and raises *holes.
// With a.part set, kept edges (i,j), j > i, part[j] != pi also go to `cut`.
template <int R, typename IdxT>
__device__ __forceinline__ void num_merge_row(const NumArgs &a, int64_t i, int64_t r, int64_t s, int32_t *oc,
                                              double *ow, int64_t ub, Comp &cut, int32_t pi, int &badp) {
    int32_t h[R];
    IdxT q[R];
    double av[R], hv[R];
    int64_t f = 0;
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int k = a.A.ci[s + t];
        av[t] = a.A.v[s + t];
        const int64_t c0 = a.T.cp[k], c1 = a.T.cp[k + 1];
        q[t] = (IdxT)(c0 + k);
        f += c1 - c0;
    }
    if (f > kMergeMaxF) return;
#pragma unroll
    for (int t = 0; t < R; ++t) {
        h[t] = a.T.ri[q[t]];
        hv[t] = a.T.vt[q[t]];
    }
    int64_t o = 0;
    while (true) {
        int m = h[0];
#pragma unroll
        for (int t = 1; t < R; ++t) m = min(m, h[t]);
        if (m == INT_MAX) break;
        double acc = +0.0;
#pragma unroll
        for (int t = 0; t < R; ++t) {
            if (h[t] == m) {  // runs visited in ascending k: the ordered chain
                acc = __fma_rn(av[t], hv[t], acc);
                ++q[t];
                h[t] = a.T.ri[q[t]];  // the column's sentinel stops the run
                hv[t] = a.T.vt[q[t]];
            }
        }
        if ((int64_t)m == i) {
            if (a.diag) a.diag[r] = acc;
        } else {
            const double w = fabs(acc);
            if (w > a.tol) {
                oc[o] = m;
                ow[o] = w;
                ++o;
                if (a.part && (int64_t)m > i) {
                    const int32_t pj = a.part[m];
                    badp |= (pj < 0) | (pj >= a.K);
                    if (pj != pi) cut.add(w);
                }
            }
        }
    }
    if (o < ub) {
        for (int64_t t = o; t < ub; ++t) oc[t] = -1;
        atomicOr(a.holes, 1);
    }
}

constexpr int kMergeThreads = 256;
constexpr int kMergeWarps = kMergeThreads / 32;
// staged graph entries per warp: NumArgs::stage_cap (dynamic shared memory)

template <int RMAX, typename IdxT>
__global__ void __launch_bounds__(kMergeThreads) k_sym_merge(SymArgs a) {
    const int64_t nloc = a.re - a.rb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc; r += stride) {
        const int64_t i = a.rb + r;
        const int64_t s = a.A.rp[i];
        const int len = (int)min(a.A.rp[i + 1] - s, (int64_t)kMergeMaxLen + 1);
        int64_t c = -1;
        switch (len) {
            case 0: c = 0; break;
            case 1: c = sym_merge_row<1, IdxT>(a.A, a.T, s); break;
            case 2: c = sym_merge_row<2, IdxT>(a.A, a.T, s); break;
            case 3: c = sym_merge_row<3, IdxT>(a.A, a.T, s); break;
            case 4: c = sym_merge_row<4, IdxT>(a.A, a.T, s); break;
            case 5: if constexpr (RMAX >= 5) c = sym_merge_row<5, IdxT>(a.A, a.T, s); break;
            case 6: if constexpr (RMAX >= 6) c = sym_merge_row<6, IdxT>(a.A, a.T, s); break;
            case 7: if constexpr (RMAX >= 7) c = sym_merge_row<7, IdxT>(a.A, a.T, s); break;
            case 8: if constexpr (RMAX >= 8) c = sym_merge_row<8, IdxT>(a.A, a.T, s); break;
            default: break;
        }
        if (c >= 0) a.nnzc[r] = c;
    }
}

// Each warp takes 32 consecutive rows (one per lane).  Their graph slots are
// contiguous, so when they fit the stage capacity the lanes write into shared memory
// and the warp streams the range out with coalesced stores.
template <int RMAX, typename IdxT>
__global__ void __launch_bounds__(kMergeThreads) k_num_merge(NumArgs a) {
    extern __shared__ __align__(16) unsigned char merge_smem[];
    const int cap = a.stage_cap;
    const int w = threadIdx.x >> 5, l = lane_id();
    double *st_wp = reinterpret_cast<double *>(merge_smem) + (size_t)w * cap;
    int32_t *st_cp = reinterpret_cast<int32_t *>(merge_smem + (size_t)kMergeWarps * cap * sizeof(double)) + (size_t)w * cap;
    const int64_t nloc = a.re - a.rb;
    const int64_t ntiles = (nloc + 31) / 32;
    Comp cut;
    int badp = 0;
    for (int64_t tile = (int64_t)blockIdx.x * kMergeWarps + w; tile < ntiles;
         tile += (int64_t)gridDim.x * kMergeWarps) {
        const int64_t r0 = tile * 32;
        const int rows = (int)min((int64_t)32, nloc - r0);
        const int64_t r = r0 + l;
        const int64_t g0 = a.gptr[r0];
        const int64_t span = a.gptr[r0 + rows] - g0;
        const bool staged = span <= cap;
        if (l < rows) {
            const int64_t i = a.rb + r;
            const int64_t s = a.A.rp[i];
            const int len = (int)min(a.A.rp[i + 1] - s, (int64_t)kMergeMaxLen + 1);
            const int64_t gr = a.gptr[r], ub = a.gptr[r + 1] - gr;
            int32_t *oc = staged ? st_cp + (gr - g0) : a.gcol + gr;
            double *ow = staged ? st_wp + (gr - g0) : a.gw + gr;
            int32_t pi = 0;
            if (a.part) {
                pi = a.part[i];
                badp |= (pi < 0) | (pi >= a.K);
            }
            switch (len) {
                case 0:
                    if (a.diag) a.diag[r] = 0.0;
                    break;
                case 1: num_merge_row<1, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 2: num_merge_row<2, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 3: num_merge_row<3, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 4: num_merge_row<4, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 5: if constexpr (RMAX >= 5) num_merge_row<5, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 6: if constexpr (RMAX >= 6) num_merge_row<6, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 7: if constexpr (RMAX >= 7) num_merge_row<7, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                case 8: if constexpr (RMAX >= 8) num_merge_row<8, IdxT>(a, i, r, s, oc, ow, ub, cut, pi, badp); break;
                default: break;
            }
        }
        if (staged) {
            __syncwarp();
            for (int64_t t = l; t < span; t += 32) {
                a.gcol[g0 + t] = st_cp[t];
                a.gw[g0 + t] = st_wp[t];
            }
            __syncwarp();
        }
    }
    if (a.part) {  // fused a7: per-CTA partial of the cut
        const double v = block_tree_sum<kMergeThreads>(cut.value());
        if (threadIdx.x == 0) {
            a.cutp[blockIdx.x] = v;
            if (blockIdx.x == 0) *a.cut_used = (int)gridDim.x;
        }
        if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(a.bad_part, 1);
    }
}

static int sms() {
    if (!g_sms_cache) g_sms_cache = num_sms();
    return g_sms_cache;
}

// a3 + a4 fused for the merge path: per row, f_i = sum of column lengths;
// merge-path rows get their structural nnz(C_i) right away, the others are
// binned for the warp-hash / huge symbolic kernels by ceil(log2(2 f_i)).
template <typename IdxT>
__global__ void __launch_bounds__(kMergeThreads) k_analyze_sym(SymArgs a, uint8_t *bin8, DevCounters *ctr) {
    const int64_t nloc = a.re - a.rb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t local = 0;
    int maxlen = 0;
    // per-thread bin counts, two 32-bit counters per register (bins 0..7;
    // a thread sees at most nloc / stride rows, far below 2^32)
    unsigned long long pc0 = 0, pc1 = 0, pc2 = 0, pc3 = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nloc; r += stride) {
        const int64_t i = a.rb + r;
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        int64_t fi = 0;
        for (int64_t p0 = s; p0 < e; p0 += 8) {  // 8 independent gathers in flight
            int k[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) k[u] = p0 + u < e ? a.A.ci[p0 + u] : -1;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k[u] >= 0) fi += a.T.cp[k[u] + 1] - a.T.cp[k[u]];
        }
        local += fi;
        const int len = (int)min(e - s, (int64_t)kMergeMaxLen + 1);
        if (len <= kMergeMaxLen && fi <= kMergeMaxF) {
            maxlen = max(maxlen, len);
            int64_t c = 0;
            switch (len) {
                case 1: c = sym_merge_row<1, IdxT>(a.A, a.T, s); break;
                case 2: c = sym_merge_row<2, IdxT>(a.A, a.T, s); break;
                case 3: c = sym_merge_row<3, IdxT>(a.A, a.T, s); break;
                case 4: c = sym_merge_row<4, IdxT>(a.A, a.T, s); break;
                case 5: c = sym_merge_row<5, IdxT>(a.A, a.T, s); break;
                case 6: c = sym_merge_row<6, IdxT>(a.A, a.T, s); break;
                case 7: c = sym_merge_row<7, IdxT>(a.A, a.T, s); break;
                case 8: c = sym_merge_row<8, IdxT>(a.A, a.T, s); break;
                default: break;
            }
            a.nnzc[r] = c;
            bin8[r] = kBinNone;
        } else {
            const int64_t m2 = 2 * (fi > 1 ? fi : 1);
            int lg = 64 - __clzll(m2 - 1);
            if (lg < kSymBinMinLog) lg = kSymBinMinLog;
            const int b = lg > kSymBinMaxLog ? kNumSymBins : lg - kSymBinMinLog;
            bin8[r] = (uint8_t)b;
            const unsigned long long inc = 1ull << (32 * (b & 1));
            pc0 += (b >> 1) == 0 ? inc : 0ull;
            pc1 += (b >> 1) == 1 ? inc : 0ull;
            pc2 += (b >> 1) == 2 ? inc : 0ull;
            pc3 += (b >> 1) == 3 ? inc : 0ull;
        }
    }
    pc0 = warp_sum(pc0);
    pc1 = warp_sum(pc1);
    pc2 = warp_sum(pc2);
    pc3 = warp_sum(pc3);
    if (lane_id() == 0 && (pc0 | pc1 | pc2 | pc3)) {
        const unsigned long long pcs[4] = {pc0, pc1, pc2, pc3};
        unsigned long long mid = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const unsigned long long lo = pcs[q] & 0xffffffffull, hi = pcs[q] >> 32;
            if (lo) atomicAdd((unsigned long long *)&ctr->sym_count[2 * q], lo);
            if (hi) atomicAdd((unsigned long long *)&ctr->sym_count[2 * q + 1], hi);
            mid += lo + hi;
        }
        atomicAdd((unsigned long long *)&ctr->n_mid, mid);
    }
    maxlen = __reduce_max_sync(kFull, maxlen);
    if (lane_id() == 0 && maxlen) atomicMax(&ctr->max_len, maxlen);
    local = warp_sum(local);
    if (lane_id() == 0 && local) atomicAdd((unsigned long long *)&ctr->products, (unsigned long long)local);
}

void launch_analyze_sym(const SymArgs &a, uint8_t *bin8, DevCounters *ctr, cudaStream_t s) {
    const int64_t nloc = a.re - a.rb;
    int64_t g = (nloc + kMergeThreads - 1) / kMergeThreads;
    g = g < 1 ? 1 : (g > (int64_t)sms() * 16 ? (int64_t)sms() * 16 : g);
    if (a.A.nnz <= INT32_MAX)
        k_analyze_sym<int32_t><<<(unsigned)g, kMergeThreads, 0, s>>>(a, bin8, ctr);
    else
        k_analyze_sym<int64_t><<<(unsigned)g, kMergeThreads, 0, s>>>(a, bin8, ctr);
    note_launch();
}

template <int RMAX, typename IdxT>
static void launch_merge_t(const SymArgs *sa, const NumArgs *na, cudaStream_t s) {
    if (sa) {
        const int64_t nloc = sa->re - sa->rb;
        int64_t g = (nloc + kMergeThreads - 1) / kMergeThreads;
        g = g < 1 ? 1 : (g > (int64_t)sms() * 16 ? (int64_t)sms() * 16 : g);
        k_sym_merge<RMAX, IdxT><<<(unsigned)g, kMergeThreads, 0, s>>>(*sa);
    } else {
        const int64_t nloc = na->re - na->rb;
        int64_t g = (nloc + kMergeThreads - 1) / kMergeThreads;
        g = g < 1 ? 1 : (g > (int64_t)sms() * 16 ? (int64_t)sms() * 16 : g);
        const size_t smem = (size_t)kMergeWarps * (size_t)na->stage_cap * (sizeof(double) + sizeof(int32_t));
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_num_merge<RMAX, IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kMergeWarps * kMaxStageCap * (sizeof(double) + sizeof(int32_t))));
            attr = true;
        }
        k_num_merge<RMAX, IdxT><<<(unsigned)g, kMergeThreads, smem, s>>>(*na);
    }
    note_launch();
}

template <typename IdxT>
static void launch_merge_r(int maxlen, const SymArgs *sa, const NumArgs *na, cudaStream_t s) {
    if (maxlen <= 4)
        launch_merge_t<4, IdxT>(sa, na, s);
    else if (maxlen == 5)
        launch_merge_t<5, IdxT>(sa, na, s);
    else if (maxlen == 6)
        launch_merge_t<6, IdxT>(sa, na, s);
    else if (maxlen == 7)
        launch_merge_t<7, IdxT>(sa, na, s);
    else
        launch_merge_t<8, IdxT>(sa, na, s);
}

void launch_sym_merge(const SymArgs &a, int maxlen, cudaStream_t s) {
    if (a.A.nnz <= INT32_MAX)
        launch_merge_r<int32_t>(maxlen, &a, nullptr, s);
    else
        launch_merge_r<int64_t>(maxlen, &a, nullptr, s);
}

void launch_num_merge(const NumArgs &a, int maxlen, cudaStream_t s) {
    if (a.A.nnz <= INT32_MAX)
        launch_merge_r<int32_t>(maxlen, nullptr, &a, s);
    else
        launch_merge_r<int64_t>(maxlen, nullptr, &a, s);
}

// ======================================================== product enumeration
// Row entries of row i are taken 32 at a time; for each, the column segment
// [cp[k], cp[k+1]) of the CSC.  Products of the batch are numbered 0..total-1
// in (k ascending, column order); lane L of a chunk handles product c0+L.
struct Batch {
    int64_t incl;  // inclusive prefix of column lengths (this lane's entry)
    int64_t excl;
    int64_t cs;    // column start
    double a;      // a_hat_ik of this lane's entry
    int64_t total;
};

__device__ __forceinline__ Batch load_batch(const Csr &A, const Csc &T, int64_t base, int64_t e, bool need_a) {
    Batch b;
    const int64_t p = base + lane_id();
    int64_t cl = 0;
    b.cs = 0;
    b.a = 0.0;
    if (p < e) {
        const int k = A.ci[p];
        const int64_t c0 = T.cp[k];
        cl = T.cp[k + 1] - c0;
        b.cs = c0 + k;  // sentinel layout (csc_begin)
        if (need_a) b.a = A.v[p];
    }
    b.incl = warp_incl_scan(cl);
    b.excl = b.incl - cl;
    b.total = __shfl_sync(kFull, b.incl, 31);
    return b;
}

// Segment (lane index) holding product pp: number of lanes with incl <= pp.
__device__ __forceinline__ int find_seg(const Batch &b, int64_t pp) {
    int t = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        const int64_t v = __shfl_sync(kFull, b.incl, t + step - 1);
        if (v <= pp) t += step;
    }
    return t;
}

// One product per lane for the chunk [c0, c0+32) of a batch.  The lane's
// segment (row entry) comes from an OR-reduced bitmask of the segment starts
// that fall inside the chunk -- no shuffle search.  Lanes past the batch get
// j = -2 - lane (negative and pairwise distinct).
struct Chunk {
    int j;
    double b;  // a_hat_jk
    double a;  // a_hat_ik
};

template <bool NEED_VAL>
__device__ __forceinline__ Chunk fetch_chunk(const Csc &T, const Batch &b, int64_t c0) {
    const int l = lane_id();
    const int64_t rel = b.excl - c0;
    const unsigned starts = __reduce_or_sync(kFull, (rel > 0 && rel < 32) ? (1u << (int)rel) : 0u);
    const int seg0 = __popc(__ballot_sync(kFull, b.incl <= c0));
    const int seg = (seg0 + __popc(starts & ((2u << l) - 1u))) & 31;
    const int64_t pp = c0 + l;
    Chunk c;
    const bool valid = pp < b.total;
    const int64_t q = __shfl_sync(kFull, b.cs - b.excl, seg) + pp;
    c.a = NEED_VAL ? shfl_d(b.a, seg) : 0.0;
    c.j = valid ? T.ri[q] : -2 - l;
    c.b = (NEED_VAL && valid) ? T.vt[q] : 0.0;
    return c;
}

// One column segment (or a 32-entry piece of a longer one) of row entry t of
// a batch: lane l takes entry off + l of column k_t.  Keys inside a piece are
// distinct (rows of one column), so a piece updates its accumulators with no
// conflicts and no chains -- the segment mode of the numeric warp kernel.
struct Piece {
    int j;      // -1: lane idle
    double b;   // a_hat_jk
    double a;   // a_hat_ik (uniform)
    int64_t len;  // column length (uniform)
};

__device__ __forceinline__ Piece fetch_piece(const Csc &T, const Batch &b, int t, int64_t off) {
    const int l = lane_id();
    Piece p;
    const int64_t cs = __shfl_sync(kFull, b.cs, t);
    p.len = __shfl_sync(kFull, b.incl - b.excl, t);
    p.a = shfl_d(b.a, t);
    const bool valid = off + l < p.len;
    const int64_t q = cs + off + l;
    p.j = valid ? T.ri[q] : -1;
    p.b = valid ? T.vt[q] : 0.0;
    return p;
}

__device__ __forceinline__ unsigned hash_key(int j, int logt) {
    return ((unsigned)j * 0x9E3779B1u) >> (32 - logt);
}

// ======================================================== warp paths
// Rows off the merge path.  Keys j inside the row's window
// [i - kWinHalf, i + kWinHalf) go to a direct-mapped window (occupancy bitmap
// + values): no hashing, and already in order for the output.  Other ("far")
// keys use an open-addressing table in shared memory.  Banded rows (config 5)
// keep most keys in the window; random rows (config 4) keep most in the table.
// Chunks are software-pipelined: the next chunk's gathers are issued before
// the current chunk is accumulated.
constexpr int kWarpHashThreads = 128;  // 4 warps per CTA, many CTAs per SM
constexpr int kWinHalf = 128;
constexpr int kWin = 2 * kWinHalf;
constexpr int kWinSeenWords = kWin / 4;  // symbolic: one byte per window slot
constexpr int kFarHuge = 1 << 30;  // farc marker: route the numeric pass to the huge path

template <int LOGT>
__global__ void __launch_bounds__(kWarpHashThreads) k_sym_warp(SymArgs a, const int32_t *__restrict__ list,
                                                               const int64_t *count) {
    constexpr int T = 1 << LOGT;
    extern __shared__ int32_t sym_tab[];
    const int w = threadIdx.x >> 5, l = lane_id();
    int32_t *keys = sym_tab + w * (T + kWinSeenWords);
    unsigned *seenw = reinterpret_cast<unsigned *>(keys + T);  // one byte per window slot
    unsigned char *seen = reinterpret_cast<unsigned char *>(seenw);
    const int64_t n = *count;
    for (int s = l; s < T; s += 32) keys[s] = -1;
    for (int s = l; s < kWinSeenWords; s += 32) seenw[s] = 0u;
    __syncwarp();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t idx = blockIdx.x * (int64_t)(blockDim.x >> 5) + w; idx < n; idx += nw) {
        const int64_t i = list[idx];
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        const int64_t wbase = i - kWinHalf;
        int nfar = 0;
        for (int64_t base = s; base < e; base += 32) {
            const Batch b = load_batch(a.A, a.T, base, e, false);
            Chunk cur = fetch_chunk<false>(a.T, b, 0);
            for (int64_t c0 = 0; c0 < b.total; c0 += 32) {
                Chunk nxt = cur;
                if (c0 + 32 < b.total) nxt = fetch_chunk<false>(a.T, b, c0 + 32);
                const int64_t d = (int64_t)cur.j - wbase;
                if (cur.j >= 0) {
                    if (d >= 0 && d < kWin) {
                        seen[d] = 1;  // idempotent: no atomics, duplicates harmless
                    } else {
                        unsigned sl = hash_key(cur.j, LOGT);
                        while (true) {
                            const int prev = atomicCAS(&keys[sl], -1, cur.j);
                            if (prev == -1) {
                                ++nfar;
                                break;
                            }
                            if (prev == cur.j) break;
                            sl = (sl + 1) & (T - 1);
                        }
                    }
                }
                cur = nxt;
            }
        }
        __syncwarp();
        int nnear = 0;
        for (int s2 = l; s2 < kWinSeenWords; s2 += 32) nnear += __popc(seenw[s2]);  // bytes are 0 / 1
        nnear = warp_sum(nnear);
        nfar = warp_sum(nfar);
        if (l == 0) {
            a.nnzc[i - a.rb] = nnear + nfar;
            a.farc[i - a.rb] = nfar;
        }
        __syncwarp();
        for (int s2 = l; s2 < T; s2 += 32) keys[s2] = -1;
        for (int s2 = l; s2 < kWinSeenWords; s2 += 32) seenw[s2] = 0u;
        __syncwarp();
    }
}

template <int LOGT>
static void launch_sym_warp_t(const SymArgs &a, const int32_t *list, const int64_t *count, cudaStream_t s) {
    constexpr int T = 1 << LOGT;
    const size_t smem = (size_t)(kWarpHashThreads / 32) * (T + kWinSeenWords) * sizeof(int32_t);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sym_warp<LOGT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int per_sm = (int)((200 * 1024) / smem);
    per_sm = per_sm < 1 ? 1 : (per_sm > 16 ? 16 : per_sm);
    k_sym_warp<LOGT><<<sms() * per_sm, kWarpHashThreads, smem, s>>>(a, list, count);
    note_launch();
}

void launch_sym_warp(const SymArgs &a, const int32_t *lists, int64_t cap, const int64_t *counts,
                     const int64_t *hcounts, cudaStream_t s) {
    if (hcounts[0]) launch_sym_warp_t<6>(a, lists + 0 * cap, counts + 0, s);
    if (hcounts[1]) launch_sym_warp_t<7>(a, lists + 1 * cap, counts + 1, s);
    if (hcounts[2]) launch_sym_warp_t<8>(a, lists + 2 * cap, counts + 2, s);
    if (hcounts[3]) launch_sym_warp_t<9>(a, lists + 3 * cap, counts + 3, s);
    if (hcounts[4]) launch_sym_warp_t<10>(a, lists + 4 * cap, counts + 4, s);
    if (hcounts[5]) launch_sym_warp_t<11>(a, lists + 5 * cap, counts + 5, s);
    if (hcounts[6]) launch_sym_warp_t<12>(a, lists + 6 * cap, counts + 6, s);
}

// Numeric, per warp (T = 2^LOGT far-table slots >= 2 * far keys):
//   wv[kWin] window values, vals[T] / keys[T] far table (+0.0 / -1 when
//   empty; reused as the second radix buffer), radix buffer of T/2
//   (key, value), hist[256].  Every accumulator starts at +0.0, so the first
//   fma of a chain sees +0.0 exactly as in the ordering contract; an
//   untouched window slot reads +0.0 and is never emitted (|c| > tol >= 0).
template <int LOGT>
struct NumWarpSmem {
    static constexpr int T = 1 << LOGT;
    static constexpr size_t bytes = (size_t)kWin * 8 + (size_t)T * 8 + (size_t)T * 4 + (size_t)(T / 2) * 12 + 256 * 4;
};

// Segment mode when the batch's mean column length is at least this.
constexpr int kSegMinMean = 12;

template <int LOGT>
__device__ __forceinline__ double *far_slot(int32_t *keys, double *vals, int j) {
    constexpr int T = 1 << LOGT;
    unsigned sl = hash_key(j, LOGT);
    while (true) {
        const int prev = atomicCAS(&keys[sl], -1, j);
        if (prev == -1 || prev == j) break;
        sl = (sl + 1) & (T - 1);
    }
    return vals + sl;
}

template <int LOGT>
__global__ void __launch_bounds__(kWarpHashThreads, 1) k_num_warp(NumArgs a, const int32_t *__restrict__ list,
                                                               const int64_t *count) {
    constexpr int T = 1 << LOGT;
    constexpr int H = T / 2;
    constexpr int WPB = kWarpHashThreads / 32;
    extern __shared__ __align__(16) unsigned char num_smem[];
    const int w = threadIdx.x >> 5, l = lane_id();
    unsigned char *base = num_smem + (size_t)w * NumWarpSmem<LOGT>::bytes;
    double *wv = reinterpret_cast<double *>(base);
    double *vals = wv + kWin;
    double *av = vals + T;
    int32_t *keys = reinterpret_cast<int32_t *>(av + H);
    int32_t *ak = keys + T;
    int32_t *hist = ak + H;
    const unsigned lt = lanemask_lt();
    Comp cut;
    int badp = 0;

    for (int s = l; s < T; s += 32) {
        keys[s] = -1;
        vals[s] = +0.0;
    }
    for (int s = l; s < kWin; s += 32) wv[s] = +0.0;
    __syncwarp();
    const int64_t n = *count;
    const int64_t nw = (int64_t)gridDim.x * WPB;
    for (int64_t idx = blockIdx.x * (int64_t)WPB + w; idx < n; idx += nw) {
        const int64_t i = list[idx];
        const int64_t r = i - a.rb;
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        const int64_t wbase = i - kWinHalf;
        // ---- accumulate (ordered chains: products applied in ascending k)
        for (int64_t bb = s; bb < e; bb += 32) {
            const Batch b = load_batch(a.A, a.T, bb, e, true);
            const int nent = (int)min((int64_t)32, e - bb);
            if (b.total >= (int64_t)kSegMinMean * nent) {
                // segment mode: one column (piece) per round, keys distinct
                int t = 0;
                int64_t off = 0;
                Piece cur = fetch_piece(a.T, b, 0, 0);
                while (true) {
                    int tn = t;
                    int64_t offn = off + 32;
                    if (offn >= cur.len) {
                        tn = t + 1;
                        offn = 0;
                    }
                    const bool more = tn < nent;
                    Piece nxt = cur;
                    if (more) nxt = fetch_piece(a.T, b, tn, offn);
                    if (cur.j >= 0) {
                        const int64_t d = (int64_t)cur.j - wbase;
                        double *acc = (d >= 0 && d < kWin) ? wv + d : far_slot<LOGT>(keys, vals, cur.j);
                        *acc = __fma_rn(cur.a, cur.b, *acc);
                    }
                    __syncwarp();
                    if (!more) break;
                    cur = nxt;
                    t = tn;
                    off = offn;
                }
                continue;
            }
            // chunk mode: 32 products per round; a key repeated inside the
            // chunk (several columns) is chained through its lanes in order
            Chunk cur = fetch_chunk<true>(a.T, b, 0);
            for (int64_t c0 = 0; c0 < b.total; c0 += 32) {
                Chunk nxt = cur;
                if (c0 + 32 < b.total) nxt = fetch_chunk<true>(a.T, b, c0 + 32);
                const int j = cur.j;
                const bool valid = j >= 0;
                const int64_t d = (int64_t)j - wbase;
                const bool near = valid && d >= 0 && d < kWin;
                const unsigned g = __match_any_sync(kFull, j);
                const int leader = __ffs(g) - 1;
                const int rank = __popc(g & lt);
                const int cnt = __popc(g);
                double *accp = wv;
                double acc = 0.0;
                if (valid && l == leader) {
                    accp = near ? wv + d : far_slot<LOGT>(keys, vals, j);
                    acc = *accp;
                }
                const int pred = rank ? 31 - __clz(g & lt) : l;
                const int maxc = __reduce_max_sync(kFull, valid ? cnt : 0);
                for (int it = 0; it < maxc; ++it) {
                    const double x = shfl_d(acc, pred);
                    if (valid && rank == it) acc = __fma_rn(cur.a, cur.b, rank == 0 ? acc : x);
                }
                // the last lane of each key's group stores the chain's value
                const int last = 31 - __clz(g);
                const unsigned long long pa = __shfl_sync(kFull, (unsigned long long)accp, leader);
                if (valid && l == last) *reinterpret_cast<double *>(pa) = acc;
                __syncwarp();
                cur = nxt;
            }
        }
        // ---- far keys: compact the table into (ak, av)
        int L = 0;
        int jmin = INT_MAX, jmax = -1;
        for (int b0 = 0; b0 < T; b0 += 32) {
            const int sidx = b0 + l;
            const int k = keys[sidx];
            const bool occ = k >= 0;
            const unsigned bal = __ballot_sync(kFull, occ);
            if (occ) {
                const int pos = L + __popc(bal & lt);
                ak[pos] = k;
                av[pos] = vals[sidx];
                jmin = min(jmin, k);
                jmax = max(jmax, k);
            }
            L += __popc(bal);
        }
        jmin = __reduce_min_sync(kFull, jmin);
        jmax = __reduce_max_sync(kFull, jmax);
        __syncwarp();
        // ---- LSD radix sort of the far keys on (key - jmin), 8-bit digits,
        // stable; the (now copied-out) table region is the second buffer
        const unsigned span = L > 1 ? (unsigned)(jmax - jmin) : 0u;
        const int bits = span ? 32 - __clz(span) : 0;
        int32_t *ck = ak, *nk = keys;
        double *cv = av, *nv = vals;
        for (int sh = 0; sh < bits; sh += 8) {
            for (int h = l; h < 256; h += 32) hist[h] = 0;
            __syncwarp();
            for (int rd = 0; rd < L; rd += 32) {
                const int e2 = rd + l;
                const bool v = e2 < L;
                const int dig = v ? (int)(((unsigned)(ck[e2] - jmin) >> sh) & 255u) : 256 + l;
                const unsigned g = __match_any_sync(kFull, dig);
                if (v && l == __ffs(g) - 1) hist[dig] += __popc(g);
                __syncwarp();
            }
            {
                int loc[8], sum = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    loc[u] = hist[l * 8 + u];
                    sum += loc[u];
                }
                const int inc = warp_incl_scan(sum);
                int run = inc - sum;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    hist[l * 8 + u] = run;
                    run += loc[u];
                }
            }
            __syncwarp();
            for (int rd = 0; rd < L; rd += 32) {
                const int e2 = rd + l;
                const bool v = e2 < L;
                const int key = v ? ck[e2] : 0;
                const int dig = v ? (int)(((unsigned)(key - jmin) >> sh) & 255u) : 256 + l;
                const unsigned g = __match_any_sync(kFull, dig);
                if (v) {
                    const int pos = hist[dig] + __popc(g & lt);
                    nk[pos] = key;
                    nv[pos] = cv[e2];
                }
                __syncwarp();
                if (v && l == 31 - __clz(g)) hist[dig] += __popc(g);
                __syncwarp();
            }
            int32_t *tk = ck;
            ck = nk;
            nk = tk;
            double *tv = cv;
            cv = nv;
            nv = tv;
        }
        // far keys below the window sort first
        int nbelow = 0;
        for (int rd = 0; rd < L; rd += 32) {
            const int e2 = rd + l;
            nbelow += __popc(__ballot_sync(kFull, e2 < L && (int64_t)ck[e2] < wbase));
        }
        // ---- write the row in ascending j: far-below, window, far-above
        const int64_t g0 = a.gptr[r], ub = a.gptr[r + 1] - g0;
        int32_t pi = 0;
        if (a.part) {
            pi = a.part[i];
            badp |= (pi < 0) | (pi >= a.K);
        }
        int64_t o = 0;
        auto emit = [&](bool v, int key, double c) {
            const bool isdiag = v && (int64_t)key == i;
            if (isdiag && a.diag) a.diag[r] = c;
            const bool keep = v && !isdiag && fabs(c) > a.tol;
            const unsigned bal = __ballot_sync(kFull, keep);
            if (keep) {
                const int64_t pos = g0 + o + __popc(bal & lt);
                a.gcol[pos] = key;
                a.gw[pos] = fabs(c);
                if (a.part && (int64_t)key > i) {
                    const int32_t pj = a.part[key];
                    badp |= (pj < 0) | (pj >= a.K);
                    if (pj != pi) cut.add(fabs(c));
                }
            }
            o += __popc(bal);
        };
        for (int rd = 0; rd < nbelow; rd += 32) {
            const int e2 = rd + l;
            const bool v = e2 < nbelow;
            emit(v, v ? ck[e2] : -1, v ? cv[e2] : 0.0);
        }
        for (int slot = l; slot < kWin; slot += 32) {  // untouched slots hold +0.0: never kept
            const int64_t key = wbase + slot;
            emit(key >= 0, (int)key, wv[slot]);
            wv[slot] = +0.0;
        }
        for (int rd = nbelow; rd < L; rd += 32) {
            const int e2 = rd + l;
            const bool v = e2 < L;
            emit(v, v ? ck[e2] : -1, v ? cv[e2] : 0.0);
        }
        __syncwarp();
        // reset the far table (it also served as a radix buffer) and the bitmap
        for (int s2 = l; s2 < T; s2 += 32) {
            keys[s2] = -1;
            vals[s2] = +0.0;
        }
        if (o < ub) {
            for (int64_t t = o + l; t < ub; t += 32) a.gcol[g0 + t] = -1;
            if (l == 0) atomicOr(a.holes, 1);
        }
        __syncwarp();
    }
    if (a.part) {
        const double v = block_tree_sum<kWarpHashThreads>(cut.value());
        if (threadIdx.x == 0) {
            a.cutp[blockIdx.x] = v;
            if (blockIdx.x == 0) *a.cut_used = (int)gridDim.x;
        }
        if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(a.bad_part, 1);
    }
}

template <int LOGT>
static void launch_num_warp_t(const NumArgs &a, const int32_t *list, const int64_t *count, cudaStream_t s) {
    const size_t smem = (size_t)(kWarpHashThreads / 32) * NumWarpSmem<LOGT>::bytes;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_num_warp<LOGT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int per_sm = (int)((220 * 1024) / smem);
    per_sm = per_sm < 1 ? 1 : (per_sm > 16 ? 16 : per_sm);
    int g = sms() * per_sm;
    if (g > kCutSlotsPerLaunch) g = kCutSlotsPerLaunch;
    k_num_warp<LOGT><<<g, kWarpHashThreads, smem, s>>>(a, list, count);
    note_launch();
}

void launch_num_warp(const NumArgs &a, const int32_t *lists, int64_t cap, const int64_t *counts,
                     const int64_t *hcounts, cudaStream_t s) {
    // fused-cut partial slots: launch slot 0 = merge, 1..6 = these bins, 7 = huge
    NumArgs b[6];
    for (int k = 0; k < 6; ++k) {
        b[k] = a;
        if (a.cutp) {
            b[k].cutp = a.cutp + (int64_t)(1 + k) * kCutSlotsPerLaunch;
            b[k].cut_used = a.cut_used + 1 + k;
        }
    }
    if (hcounts[0]) launch_num_warp_t<6>(b[0], lists + 0 * cap, counts + 0, s);
    if (hcounts[1]) launch_num_warp_t<7>(b[1], lists + 1 * cap, counts + 1, s);
    if (hcounts[2]) launch_num_warp_t<8>(b[2], lists + 2 * cap, counts + 2, s);
    if (hcounts[3]) launch_num_warp_t<9>(b[3], lists + 3 * cap, counts + 3, s);
    if (hcounts[4]) launch_num_warp_t<10>(b[4], lists + 4 * cap, counts + 4, s);
    if (hcounts[5]) launch_num_warp_t<11>(b[5], lists + 5 * cap, counts + 5, s);
}

// ======================================================== huge rows
// One CTA per row; per-CTA scratch slot = bitmap over j (nrows bits) and, for
// the numeric pass, a dense accumulator acc[nrows].  The bitmap is all-zero
// between rows (each row clears what it set).
constexpr int kHugeThreads = 512;
constexpr int kHugeWarps = kHugeThreads / 32;

static int64_t bitmap_words(int64_t nrows) { return (nrows + 31) / 32; }

// Scratch layout: [slots bitmaps][slots dense accumulators]; only the bitmap
// prefix (huge_bitmap_bytes) needs zeroing -- each row clears what it set.
static size_t bitmap_stride(int64_t nrows) { return ((size_t)bitmap_words(nrows) * 4 + 255) & ~(size_t)255; }

size_t huge_bitmap_bytes(int64_t nrows, int slots) { return bitmap_stride(nrows) * (size_t)slots; }

size_t huge_scratch_bytes(int64_t nrows, int slots, bool numeric) {
    return huge_bitmap_bytes(nrows, slots) + (numeric ? (size_t)nrows * 8 * (size_t)slots : 0);
}

int huge_slots(int64_t nrows, int64_t n_huge) {
    const size_t per = huge_scratch_bytes(nrows, 1, true);
    int64_t budget = (int64_t)(4ull << 30) / (int64_t)(per ? per : 1);
    int64_t s = 2 * (int64_t)sms();
    if (s > budget) s = budget;
    if (s > n_huge) s = n_huge;
    if (s < 1) s = 1;
    return (int)s;
}

struct BlockBatch {
    int64_t total;
};

// CTA-level batch of up to kHugeThreads row entries: prefix of column
// lengths in shared memory.
__device__ __forceinline__ int64_t block_batch(const Csr &A, const Csc &T, int64_t base, int64_t e,
                                               int64_t *s_incl, int64_t *s_cs, double *s_a) {
    __shared__ int64_t wsum[kHugeWarps];
    const int tid = threadIdx.x, w = tid >> 5, l = lane_id();
    const int64_t p = base + tid;
    int64_t cl = 0, cs = 0;
    double av = 0.0;
    if (p < e) {
        const int k = A.ci[p];
        const int64_t c0 = T.cp[k];
        cl = T.cp[k + 1] - c0;
        cs = c0 + k;  // sentinel layout (csc_begin)
        if (s_a) av = A.v[p];
    }
    const int64_t inc = warp_incl_scan(cl);
    if (l == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int64_t x = l < kHugeWarps ? wsum[l] : 0;
        const int64_t xi = warp_incl_scan(x);
        if (l < kHugeWarps) wsum[l] = xi - x;
    }
    __syncthreads();
    s_incl[tid] = inc + wsum[w];
    s_cs[tid] = cs;
    if (s_a) s_a[tid] = av;
    __syncthreads();
    const int64_t total = s_incl[kHugeThreads - 1];
    return total;
}

// index of the entry holding product pp: number of entries with incl <= pp
__device__ __forceinline__ int block_find(const int64_t *s_incl, int64_t pp) {
    int lo = 0, hi = kHugeThreads;  // first index with incl > pp
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_incl[mid] <= pp)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t block_sum(int64_t v) {
    __shared__ int64_t red[kHugeWarps];
    v = warp_sum(v);
    if (lane_id() == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
    for (int k = 0; k < kHugeWarps; ++k) t += red[k];
    __syncthreads();
    return t;
}

// Second-level bitmap in shared memory: bit (w & 31) of word w >> 5 is set iff
// the row's L1 bitmap word w (global) is non-zero, so output and clearing
// touch only non-empty L1 words instead of all nrows/32.
__host__ __device__ __forceinline__ int64_t l2_words(int64_t nwords) { return (nwords + 31) / 32; }

__global__ void __launch_bounds__(kHugeThreads) k_sym_huge(SymArgs a, const int32_t *__restrict__ list,
                                                           const int64_t *count, unsigned char *scratch,
                                                           size_t slot_bytes, int64_t nwords) {
    extern __shared__ unsigned l2[];
    __shared__ int64_t s_incl[kHugeThreads], s_cs[kHugeThreads];
    const int64_t nw2 = l2_words(nwords);
    unsigned *bm = reinterpret_cast<unsigned *>(scratch + slot_bytes * blockIdx.x);
    for (int64_t t = threadIdx.x; t < nw2; t += kHugeThreads) l2[t] = 0u;
    __syncthreads();
    const int64_t n = *count;
    for (int64_t idx = blockIdx.x; idx < n; idx += gridDim.x) {
        const int64_t i = list[idx];
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        int64_t cnt = 0;
        for (int64_t base = s; base < e; base += kHugeThreads) {
            const int64_t total = block_batch(a.A, a.T, base, e, s_incl, s_cs, nullptr);
            for (int64_t pp = threadIdx.x; pp < total; pp += kHugeThreads) {
                const int t = block_find(s_incl, pp);
                const int64_t ex = t ? s_incl[t - 1] : 0;
                const int j = a.T.ri[s_cs[t] + pp - ex];
                const unsigned bit = 1u << (j & 31);
                const unsigned old = atomicOr(&bm[j >> 5], bit);
                if (!(old & bit)) {
                    ++cnt;
                    if (old == 0u) atomicOr(&l2[j >> 10], 1u << ((j >> 5) & 31));
                }
            }
            __syncthreads();
        }
        cnt = block_sum(cnt);
        if (threadIdx.x == 0) {
            a.nnzc[i - a.rb] = cnt;
            a.farc[i - a.rb] = kFarHuge;
        }
        // clear the touched L1 words and the L2 bitmap
        for (int64_t t = threadIdx.x; t < nw2; t += kHugeThreads) {
            for (unsigned m = l2[t]; m; m &= m - 1) bm[t * 32 + __ffs(m) - 1] = 0u;
            l2[t] = 0u;
        }
        __syncthreads();
    }
}

// Numeric: the row's products are enumerated 512 at a time (one 32-product
// sub-chunk per warp) and routed, in product order, into shared-memory queues
// of their owner warp ((j >> 5) % 16).  Each owner then applies its queue in
// order (ordered __match_any_sync chains) to the dense accumulator, so every
// chain runs in ascending k and each product is handled once.
__global__ void __launch_bounds__(kHugeThreads) k_num_huge(NumArgs a, const int32_t *__restrict__ list,
                                                           const int64_t *count, unsigned char *scratch,
                                                           size_t slot_bytes, int64_t nwords) {
    extern __shared__ unsigned l2[];
    __shared__ int64_t s_incl[kHugeThreads], s_cs[kHugeThreads];
    __shared__ double s_a[kHugeThreads];
    __shared__ int32_t q_j[kHugeThreads];
    __shared__ double q_a[kHugeThreads], q_b[kHugeThreads];
    __shared__ int cnt[kHugeWarps][kHugeWarps + 1];
    __shared__ int otot[kHugeWarps], obase[kHugeWarps + 1];
    __shared__ int64_t s_scan[kHugeWarps];
    const int64_t nw2 = l2_words(nwords);
    unsigned *bm = reinterpret_cast<unsigned *>(scratch + slot_bytes * blockIdx.x);
    double *acc_g = reinterpret_cast<double *>(scratch + slot_bytes * gridDim.x) + (size_t)blockIdx.x * a.A.nrows;
    const int tid = threadIdx.x, w = tid >> 5, l = lane_id();
    const unsigned lt = lanemask_lt();
    for (int64_t t = tid; t < nw2; t += kHugeThreads) l2[t] = 0u;
    __syncthreads();
    Comp cut;
    int badp = 0;
    const int64_t n = *count;
    for (int64_t idx = blockIdx.x; idx < n; idx += gridDim.x) {
        const int64_t i = list[idx];
        const int64_t r = i - a.rb;
        const int64_t s = a.A.rp[i], e = a.A.rp[i + 1];
        for (int64_t base = s; base < e; base += kHugeThreads) {
            const int64_t total = block_batch(a.A, a.T, base, e, s_incl, s_cs, s_a);
            for (int64_t c0 = 0; c0 < total; c0 += kHugeThreads) {
                // ---- enumerate: warp w takes products c0 + 32 w + l
                const int64_t pp = c0 + tid;
                const bool valid = pp < total;
                int j = 0, o = 32 + l;
                double aik = 0.0, bjk = 0.0;
                if (valid) {
                    const int t = block_find(s_incl, pp);
                    const int64_t ex = t ? s_incl[t - 1] : 0;
                    const int64_t q = s_cs[t] + pp - ex;
                    j = a.T.ri[q];
                    bjk = a.T.vt[q];
                    aik = s_a[t];
                    o = (j >> 5) & (kHugeWarps - 1);
                }
                const unsigned g = __match_any_sync(kFull, o);
                const int rank = __popc(g & lt);
                if (l < kHugeWarps) cnt[w][l] = 0;
                __syncwarp();
                if (valid && l == __ffs(g) - 1) cnt[w][o] = __popc(g);
                __syncthreads();
                if (tid < kHugeWarps) {  // owner tid: offsets of each sub-chunk in its queue
                    int run = 0;
                    for (int ww = 0; ww < kHugeWarps; ++ww) {
                        const int c = cnt[ww][tid];
                        cnt[ww][tid] = run;
                        run += c;
                    }
                    otot[tid] = run;
                }
                __syncthreads();
                if (tid == 0) {
                    int sum = 0;
                    for (int oo = 0; oo < kHugeWarps; ++oo) {
                        obase[oo] = sum;
                        sum += otot[oo];
                    }
                    obase[kHugeWarps] = sum;
                }
                __syncthreads();
                if (valid) {
                    const int pos = obase[o] + cnt[w][o] + rank;
                    q_j[pos] = j;
                    q_a[pos] = aik;
                    q_b[pos] = bjk;
                }
                __syncthreads();
                // ---- owner warp w applies its queue segment in order
                const int qe = obase[w + 1];
                for (int qs = obase[w]; qs < qe; qs += 32) {
                    const int ee = qs + l;
                    const bool v = ee < qe;
                    const int jj = v ? q_j[ee] : -2 - l;
                    const unsigned gg = __match_any_sync(kFull, jj);
                    const int rk = __popc(gg & lt);
                    const int cn = __popc(gg);
                    double acc = 0.0;
                    if (v && rk == 0) {
                        const unsigned bit = 1u << (jj & 31);
                        const unsigned old = atomicOr(&bm[jj >> 5], bit);
                        if (old == 0u) atomicOr(&l2[jj >> 10], 1u << ((jj >> 5) & 31));
                        acc = (old & bit) ? acc_g[jj] : +0.0;
                    }
                    const int pred = rk ? 31 - __clz(gg & lt) : l;
                    const int maxc = __reduce_max_sync(kFull, v ? cn : 0);
                    const double qa = v ? q_a[ee] : 0.0, qb = v ? q_b[ee] : 0.0;
                    for (int it = 0; it < maxc; ++it) {
                        const double x = shfl_d(acc, pred);
                        if (v && rk == it) acc = __fma_rn(qa, qb, rk == 0 ? acc : x);
                    }
                    if (v && rk == cn - 1) acc_g[jj] = acc;
                    __syncwarp();
                }
                __syncthreads();
            }
        }
        __threadfence_block();
        __syncthreads();
        // ---- emit in ascending j: walk the non-empty L1 words via the L2 bitmap
        const int64_t g0 = a.gptr[r], ub = a.gptr[r + 1] - g0;
        int32_t pi = 0;
        if (a.part) {
            pi = a.part[i];
            badp |= (pi < 0) | (pi >= a.K);
        }
        int64_t o = 0;
        for (int64_t rb2 = 0; rb2 < nw2; rb2 += kHugeThreads) {
            const int64_t t2 = rb2 + tid;
            const unsigned m2 = t2 < nw2 ? l2[t2] : 0u;
            int keep = 0;
            for (unsigned mm = m2; mm; mm &= mm - 1) {
                const int64_t w1 = t2 * 32 + __ffs(mm) - 1;
                for (unsigned m = bm[w1]; m; m &= m - 1) {
                    const int64_t j = w1 * 32 + __ffs(m) - 1;
                    const double c = acc_g[j];
                    if (j == i) {
                        if (a.diag) a.diag[r] = c;
                    } else if (fabs(c) > a.tol) {
                        ++keep;
                    }
                }
            }
            const int64_t inc = warp_incl_scan((int64_t)keep);
            if (l == 31) s_scan[w] = inc;
            __syncthreads();
            int64_t wofs = 0, tot = 0;
            for (int k = 0; k < kHugeWarps; ++k) {
                if (k < w) wofs += s_scan[k];
                tot += s_scan[k];
            }
            int64_t pos = g0 + o + wofs + inc - keep;
            for (unsigned mm = m2; mm; mm &= mm - 1) {
                const int64_t w1 = t2 * 32 + __ffs(mm) - 1;
                for (unsigned m = bm[w1]; m; m &= m - 1) {
                    const int64_t j = w1 * 32 + __ffs(m) - 1;
                    const double c = acc_g[j];
                    if (j != i && fabs(c) > a.tol) {
                        a.gcol[pos] = (int32_t)j;
                        a.gw[pos] = fabs(c);
                        ++pos;
                        if (a.part && j > i) {
                            const int32_t pj = a.part[j];
                            badp |= (pj < 0) | (pj >= a.K);
                            if (pj != pi) cut.add(fabs(c));
                        }
                    }
                }
                bm[w1] = 0u;
            }
            if (t2 < nw2) l2[t2] = 0u;
            o += tot;
            __syncthreads();
        }
        if (o < ub) {
            for (int64_t t = o + tid; t < ub; t += kHugeThreads) a.gcol[g0 + t] = -1;
            if (tid == 0) atomicOr(a.holes, 1);
        }
        __syncthreads();
    }
    if (a.part) {
        const double v = block_tree_sum<kHugeThreads>(cut.value());
        if (threadIdx.x == 0) {
            a.cutp[blockIdx.x] = v;
            if (blockIdx.x == 0) *a.cut_used = (int)gridDim.x;
        }
        if (__syncthreads_or(badp) && threadIdx.x == 0) atomicOr(a.bad_part, 1);
    }
}

void launch_sym_huge(const SymArgs &a, const int32_t *list, const int64_t *count, int slots, void *scratch,
                     cudaStream_t s) {
    const size_t slot_bytes = bitmap_stride(a.A.nrows);
    const int64_t nw = bitmap_words(a.A.nrows);
    const size_t smem = (size_t)l2_words(nw) * sizeof(unsigned);
    cudaFuncSetAttribute(k_sym_huge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sym_huge<<<slots, kHugeThreads, smem, s>>>(a, list, count, static_cast<unsigned char *>(scratch), slot_bytes,
                                                 nw);
    note_launch();
}

void launch_num_huge(const NumArgs &a, const int32_t *list, const int64_t *count, int slots, void *scratch,
                     cudaStream_t s) {
    const size_t slot_bytes = bitmap_stride(a.A.nrows);
    const int64_t nw = bitmap_words(a.A.nrows);
    const size_t smem = (size_t)l2_words(nw) * sizeof(unsigned);
    cudaFuncSetAttribute(k_num_huge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    NumArgs b = a;
    if (a.cutp) {
        b.cutp = a.cutp + (int64_t)7 * kCutSlotsPerLaunch;
        b.cut_used = a.cut_used + 7;
    }
    k_num_huge<<<slots, kHugeThreads, smem, s>>>(b, list, count, static_cast<unsigned char *>(scratch), slot_bytes,
                                                 nw);
    note_launch();
}

}  // namespace rig

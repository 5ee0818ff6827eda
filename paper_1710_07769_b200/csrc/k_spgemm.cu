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
//  * mid rows (k_midrow.cu): window + sorted far runs, see there.
//  * huge path (one CTA per row): warp w owns the keys with (j/32) % W == w
//    and walks the whole product stream in order, so again every chain runs in
//    ascending k; the dense accumulator's bitmap yields j-sorted output.
#include "common.cuh"

#include <algorithm>

namespace rig {

static int g_sms_cache = 0;

// ======================================================== merge path
// One thread per row i.  The row's R column runs (column k of A_hat^T, rows j
// ascending) are merged; for the current minimum j the runs holding it are
// folded in ascending k: c_ij = fma(a_ik, a_jk, c_ij) -- the ordered chain.
// IdxT: int32 CSC offsets when nnz < 2^31 (fewer registers), else int64.
// Columns end in an INT_MAX sentinel (csc_begin), so a run needs no end bound.
// The same merge at width R for a row of len <= R entries (runs t >= len are
// empty): a warp runs ONE width -- its longest merge row's -- instead of the
// lanes of different lengths running their instantiations one after another.
template <int R, typename IdxT>
__device__ __forceinline__ int64_t sym_merge_row_w(const Csr &A, const Csc &T, int64_t s, int len, int2 *qs,
                                                   int64_t *f_out) {
    int32_t h[R];
    IdxT q[R];
    int64_t f = 0;
    int32_t cl[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        q[t] = 0;
        cl[t] = 0;
        if (t < len) {
            const int k = A.ci[s + t];
            const int64_t c0 = T.cp[k], c1 = T.cp[k + 1];
            q[t] = (IdxT)(c0 + k);
            cl[t] = (int32_t)min(c1 - c0, (int64_t)INT32_MAX);
            f += c1 - c0;
        }
    }
    *f_out = f;
    if (f > kMergeMaxF) return -1;
    if (qs) {
#pragma unroll
        for (int t = 0; t < R; ++t)
            if (t < len) qs[s + t] = make_int2((int32_t)q[t], cl[t]);
    }
#pragma unroll
    for (int t = 0; t < R; ++t) h[t] = t < len ? T.ri[q[t]] : INT_MAX;
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

template <int R, typename IdxT>
__device__ __forceinline__ int64_t sym_merge_row(const Csr &A, const Csc &T, int64_t s, int2 *qs = nullptr,
                                                 int64_t *f_out = nullptr) {
    int32_t h[R];
    IdxT q[R];
    int64_t f = 0;
    int32_t cl[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int k = A.ci[s + t];
        const int64_t c0 = T.cp[k], c1 = T.cp[k + 1];
        q[t] = (IdxT)(c0 + k);
        cl[t] = (int32_t)min(c1 - c0, (int64_t)INT32_MAX);
        f += c1 - c0;
    }
    if (f_out) *f_out = f;
    if (f > kMergeMaxF) return -1;
    if (qs) {  // runs for the numeric pass (saves it the col_ptr gathers)
#pragma unroll
        for (int t = 0; t < R; ++t) qs[s + t] = make_int2((int32_t)q[t], cl[t]);
    }
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
                                              double *ow, int64_t ub, CutSum &cut, int32_t pi) {
    int32_t h[R];
    IdxT q[R];
    double av[R], hv[R];
    if (a.qs) {  // run starts from the analysis (int32 offsets only)
#pragma unroll
        for (int t = 0; t < R; ++t) {
            q[t] = (IdxT)a.qs[s + t].x;
            av[t] = a.A.v[s + t];
        }
        if ((int64_t)q[0] < 0) return;  // not a merge row
    } else {
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
    }
#pragma unroll
    for (int t = 0; t < R; ++t) {
        h[t] = a.T.ri[q[t]];
        hv[t] = a.T.vt[q[t]];
    }
    int64_t o = 0;
    // fused cut, one output behind: the part[] load of a kept edge j > i is
    // issued when the edge is emitted and consumed at the next emission, so
    // its latency overlaps a merge step instead of stalling it
    int32_t pend_pj = pi;
    double pend_w = 0.0;
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
                    if (pend_pj != pi) cut.add(pend_w);
                    pend_pj = a.part[m];
                    pend_w = w;
                }
            }
        }
    }
    if (a.part) {
        if (pend_pj != pi) cut.add(pend_w);
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
    CutSum cut;
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
            }
            switch (len) {
                case 0:
                    if (a.diag) a.diag[r] = 0.0;
                    break;
                case 1: num_merge_row<1, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 2: num_merge_row<2, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 3: num_merge_row<3, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 4: num_merge_row<4, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 5: if constexpr (RMAX >= 5) num_merge_row<5, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 6: if constexpr (RMAX >= 6) num_merge_row<6, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 7: if constexpr (RMAX >= 7) num_merge_row<7, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 8: if constexpr (RMAX >= 8) num_merge_row<8, IdxT>(a, i, r, s, oc, ow, ub, cut, pi); break;
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
    }
}

// ======================================================== pair kernel
// The merge path with two lanes per row.  A warp takes 16 consecutive rows:
// lane q (< 16) merges row q's keys j < i ascending from the run starts, lane
// q + 16 its keys j >= i descending from the run ends.  Every run of row i
// (column k with a_ik != 0) contains i itself, so the ascending lane stops
// when its minimum reaches i and the descending lane stops after processing
// i (the diagonal): no split positions are needed, and each lane walks about
// half of the row.  For every key the runs holding it are folded in ascending
// k whichever direction the keys are visited in, so each c_ij is exactly the
// R4 chain.  Both lanes run one instruction stream (no divergence): the
// descending lane sees each key as key ^ ~0 (order reversed) and takes the
// minimum like the ascending one.  Runs come from the analysis (qs: start,
// length).  Output goes through a per-warp shared-memory stage (swizzled) and
// is streamed out coalesced; the descending lane fills its row from the end.
// RIG_PAIR_THREADS / RIG_PAIR_MINB (experiments, tools/build_variant.sh): CTA
// size and a register budget fitted to RIG_PAIR_MINB CTAs per SM.  The
// default leaves registers to ptxas (96 for R = 7): more warps only raised
// the L1 miss rate of the run gathers, which bound this kernel (measured).
#ifndef RIG_PAIR_THREADS
#define RIG_PAIR_THREADS 128
#endif
#ifdef RIG_PAIR_MINB
#define RIG_PAIR_BOUNDS __launch_bounds__(RIG_PAIR_THREADS, RIG_PAIR_MINB)
#else
#define RIG_PAIR_BOUNDS __launch_bounds__(RIG_PAIR_THREADS)
#endif
constexpr int kPairThreads = RIG_PAIR_THREADS;
constexpr int kPairWarps = kPairThreads / 32;
constexpr int kPairRows = 16;

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];\n" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_s32(unsigned a, int v) { asm volatile("st.shared.s32 [%0], %1;\n" ::"r"(a), "r"(v)); }
__device__ __forceinline__ void sts_f64(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v)); }

// Output stage index swizzle: entry e of the tile goes to e ^ ((e >> 5) & 31),
// a permutation inside each aligned block of 32 entries.  Rows of equal
// length would otherwise put every lane's n-th entry in the same few banks;
// the flush reads aligned blocks of 32, conflict-free either way.
__device__ __forceinline__ unsigned out_swz(unsigned e) { return e ^ ((e >> 5) & 31u); }

template <int N>
__device__ __forceinline__ int tree_min(const int (&h)[N]) {
    int v[N];
#pragma unroll
    for (int t = 0; t < N; ++t) v[t] = h[t];
#pragma unroll
    for (int w = 1; w < N; w <<= 1) {
#pragma unroll
        for (int t = 0; t + w < N; t += 2 * w) v[t] = min(v[t], v[t + w]);
    }
    return v[0];
}

#ifndef RIG_PAIR_WARP_DISPATCH
#define RIG_PAIR_WARP_DISPATCH 1  // measured: configs 2-4 numeric 3-5 % faster than per-lane widths
#endif
#ifndef RIG_PAIR_LOOKAHEAD
#define RIG_PAIR_LOOKAHEAD 0  // measured: 1 (next key loaded one advance ahead) is 2-5 % slower on configs 2-3
#endif
// Output of a half row: the swizzled shared stage (tile index e, stepping +-1).
struct OutStage {
    unsigned oc0, ow0, e, step;
    __device__ __forceinline__ void put(int j, double w) {
        const unsigned x = out_swz(e);
        sts_s32(oc0 + 4 * x, j);
        sts_f64(ow0 + 8 * x, w);
        e += step;
    }
};
// One half row.  q0[t]: CSC position of run t's first (ascending) or last
// (descending) entry, or -1 for an empty run (t >= len).  Kept entries go to
// `out` in the lane's direction.  CUT: the descending lane's kept edges
// (j > i) with part[j] != pi go to `cut`.  Returns the count.
template <int R, bool CUT = true, class Out>
__device__ __forceinline__ int pair_half_row(const NumArgs &a, bool desc, int64_t i, int64_t r, const int *q0,
                                             const double *av0, Out &out, CutSum &cut, int32_t pi) {
    int h[R], q[R];
    double av[R], hv[R];
#if RIG_PAIR_LOOKAHEAD
    int h2[R];  // each run's NEXT key, loaded one advance ahead: the min of a
                // step never waits on the load issued by the step before it
#endif
    const int xm = desc ? -1 : 0;
    const int step = desc ? -1 : 1;
#pragma unroll
    for (int t = 0; t < R; ++t) {
        q[t] = q0[t];
        av[t] = av0[t];
        h[t] = INT_MAX;
        hv[t] = 0.0;
#if RIG_PAIR_LOOKAHEAD
        h2[t] = INT_MAX;
#endif
        if (q[t] >= 0) {
            h[t] = a.T.ri[q[t]] ^ xm;
            hv[t] = a.T.vt[q[t]];
#if RIG_PAIR_LOOKAHEAD
            h2[t] = a.T.ri[q[t] + step] ^ xm;
#endif
        }
    }
    const int ik = (int)i ^ xm;
    const bool cut_on = CUT && desc && a.part;
    int o = 0;
    int32_t pend_pj = pi;
    double pend_w = 0.0;
    while (true) {
        const int m = tree_min<R>(h);
        if (m == ik && !desc) break;  // every run holds i: no key < i is left
        double acc = +0.0;
#pragma unroll
        for (int t = 0; t < R; ++t) {
            if (h[t] == m) {  // runs visited in ascending k: the ordered chain
                acc = __fma_rn(av[t], hv[t], acc);
                q[t] += step;  // ascending lanes stop at i, descending ones
                               // at i too: a run is never left
#if RIG_PAIR_LOOKAHEAD
                h[t] = h2[t];
                h2[t] = a.T.ri[q[t] + step] ^ xm;  // at most two past the run (readable pads / sentinels)
#else
                h[t] = a.T.ri[q[t]] ^ xm;
#endif
                hv[t] = a.T.vt[q[t]];
            }
        }
        if (m == ik) {  // descending lane: the diagonal comes last
            if (a.diag) a.diag[r] = acc;
            break;
        }
        const double w = fabs(acc);
        if (w > a.tol) {
            const int j = m ^ xm;
            out.put(j, w);
            ++o;
            if (cut_on) {  // j > i: each undirected edge counted once
                if (pend_pj != pi) cut.add(pend_w);
                pend_pj = a.part[j];
                pend_w = w;
            }
        }
    }
    if (cut_on) {
        if (pend_pj != pi) cut.add(pend_w);
    }
    return o;
}

template <int RMAX, bool CUT = true, class Out>
__device__ __forceinline__ int pair_half_row_r(int len, const NumArgs &a, bool desc, int64_t i, int64_t r,
                                               const int *q0, const double *av0, Out &out, CutSum &cut,
                                               int32_t pi) {
    if (len <= 2) return pair_half_row<2, CUT>(a, desc, i, r, q0, av0, out, cut, pi);
    if (RMAX > 4 && len <= 4) return pair_half_row<4, CUT>(a, desc, i, r, q0, av0, out, cut, pi);
    return pair_half_row<RMAX, CUT>(a, desc, i, r, q0, av0, out, cut, pi);
}

// Rows whose output does not fit the stage are merged by num_merge_row with
// direct global stores (the ascending lane; its partner idles).
template <int RMAX>
__global__ void RIG_PAIR_BOUNDS k_num_pair(NumArgs a) {
    extern __shared__ __align__(16) unsigned char pair_smem[];
    const int cap = a.stage_cap;
    const int w = threadIdx.x >> 5, l = lane_id();
    const int qr = l & (kPairRows - 1);
    const bool desc = l >= kPairRows;
    double *st_wp = reinterpret_cast<double *>(pair_smem) + (size_t)w * cap;
    int32_t *st_cp = reinterpret_cast<int32_t *>(reinterpret_cast<double *>(pair_smem) + (size_t)kPairWarps * cap) +
                     (size_t)w * cap;
    const unsigned oc0 = smem_u32(st_cp), ow0 = smem_u32(st_wp);
    const int64_t nloc = a.re - a.rb;
    const int64_t ntiles = (nloc + kPairRows - 1) / kPairRows;
    CutSum cut;
    for (int64_t tile = (int64_t)blockIdx.x * kPairWarps + w; tile < ntiles; tile += (int64_t)gridDim.x * kPairWarps) {
        const int64_t r0 = tile * kPairRows;
        const int rows = (int)min((int64_t)kPairRows, nloc - r0);
        const int64_t r = r0 + qr;
        const int64_t g0 = a.gptr[r0];
        const int64_t span_out = a.gptr[r0 + rows] - g0;
        const bool staged = span_out <= cap;
        const int64_t i = a.rb + r;
        int64_t s = 0, gr = 0, ub = 0;
        int len = 0;
        bool mrow = false;
        int32_t pi = 0;
        int qv[RMAX];
        double av[RMAX];
        if (qr < rows) {
            s = a.A.rp[i];
            len = (int)min(a.A.rp[i + 1] - s, (int64_t)kMergeMaxLen + 1);
            gr = a.gptr[r];
            ub = a.gptr[r + 1] - gr;
            if (a.part) {
                pi = a.part[i];
            }
        }
        // the row's runs and values, loaded before the merge-row test (run 0's
        // start is -1 off the merge path) so they cost no extra round trip
        const int lq = (len >= 1 && len <= RMAX) ? len : 0;
#pragma unroll
        for (int t = 0; t < RMAX; ++t) {
            qv[t] = -1;
            av[t] = 0.0;
            if (t < lq) {  // streamed: read once
                const int2 run = __ldcs(a.qs + s + t);
                if (t == 0) mrow = run.x >= 0;
                qv[t] = desc ? run.x + run.y - 1 : run.x;
                av[t] = __ldcs(a.A.v + s + t);
            }
        }
        int o = 0;
#if RIG_PAIR_WARP_DISPATCH
        // merge width chosen per warp (the tile's longest merge row): one
        // instantiation runs, instead of the lanes of different widths
        // running theirs one after another (mixed lengths: power-law rows)
        const int wlen = (int)__reduce_max_sync(kFull, (unsigned)((mrow && staged) ? len : 0));
#else
        const int wlen = len;
#endif
        if (mrow && staged) {
            const unsigned ob = (unsigned)(gr - g0) + (desc ? (unsigned)(ub - 1) : 0u);
            OutStage out{oc0, ow0, ob, desc ? 0xffffffffu : 1u};
            o = pair_half_row_r<RMAX>(wlen, a, desc, i, r, qv, av, out, cut, pi);
        } else if (mrow && !desc) {  // output beyond the stage: direct global stores
            int32_t *oc = a.gcol + gr;
            double *ow = a.gw + gr;
            switch (len) {
                case 1: num_merge_row<1, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 2: num_merge_row<2, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 3: num_merge_row<3, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 4: num_merge_row<4, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 5: if constexpr (RMAX >= 5) num_merge_row<5, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 6: if constexpr (RMAX >= 6) num_merge_row<6, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 7: if constexpr (RMAX >= 7) num_merge_row<7, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                case 8: if constexpr (RMAX >= 8) num_merge_row<8, int32_t>(a, i, r, s, oc, ow, ub, cut, pi); break;
                default: break;
            }
        } else if (qr < rows && len == 0 && !desc) {
            if (a.diag) a.diag[r] = 0.0;
        }
        if (!staged) continue;
        // dropped entries (|c| <= tol or exact zero): the descending half moves
        // down behind the ascending half; the tail becomes holes
        const int o_asc = __shfl_sync(kFull, o, qr);
        if (desc && mrow && o_asc + o < ub) {
            const unsigned base = (unsigned)(gr - g0);
            for (int t = 0; t < o; ++t) {
                const unsigned src = out_swz(base + (unsigned)(ub - o + t));
                const unsigned dst = out_swz(base + (unsigned)(o_asc + t));
                sts_s32(oc0 + 4 * dst, lds_s32(oc0 + 4 * src));
                sts_f64(ow0 + 8 * dst, lds_f64(ow0 + 8 * src));
            }
            for (int64_t t = o_asc + o; t < ub; ++t) sts_s32(oc0 + 4 * out_swz(base + (unsigned)t), -1);
            atomicOr(a.holes, 1);
        }
        __syncwarp();
        // slots of rows off the merge path are garbage here: k_copy_rows
        // places those rows afterwards
        for (int64_t t = l; t < span_out; t += 32) {
            const unsigned e = out_swz((unsigned)t);
            __stcs(a.gcol + g0 + t, lds_s32(oc0 + 4 * e));  // streamed: keeps the CSC gathers in L2
            __stcs(a.gw + g0 + t, lds_f64(ow0 + 8 * e));
        }
        __syncwarp();  // the stage is reused by the next tile
    }
    if (a.part) {  // fused a7: per-CTA partial of the cut
        const double v = block_tree_sum<kPairThreads>(cut.value());
        if (threadIdx.x == 0) {
            a.cutp[blockIdx.x] = v;
            if (blockIdx.x == 0) *a.cut_used = (int)gridDim.x;
        }
    }
}

static int sms() {
    if (!g_sms_cache) g_sms_cache = num_sms();
    return g_sms_cache;
}

// a3 + a4 fused for the merge path: per row, f_i = sum of column lengths;
// merge-path rows get their structural nnz(C_i) right away, the others are
// binned by ceil(log2(2 f_i)): the mid bins go to the mid-row kernel (k_row_win in temp mode), the
// huge bin (f_i > 2048) to the wide-window / global-far-list / CTA-per-row chain.
// WW: merge width per warp (the warp's longest merge row) instead of per lane,
// for shards whose row lengths vary inside a warp (power-law rows: every lane
// length ran its instantiation in turn); 3 CTAs per SM leave it unspilled.
// Measured: config 4 analysis 0.404 -> 0.268 ms; on stencils (uniform rows)
// per lane is faster (config 3 0.685 vs 0.708 ms), so the host picks.  Per
// lane at 4 CTAs per SM (64 registers, the width it was tuned at; 96 unbounded:
// config 3 0.685 -> 0.852 ms).
template <typename IdxT, bool WW>
__global__ void __launch_bounds__(kMergeThreads, WW ? 3 : 4) k_analyze_sym(SymArgs a, uint8_t *bin8, DevCounters *ctr) {
    const int64_t nloc = a.re - a.rb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t local = 0, nnzr = 0, maxf = 0, slots = 0;
    int maxlen = 0;
    // per-thread bin counts, two 32-bit counters per register (bins 0..7;
    // a thread sees at most nloc / stride rows, far below 2^32)
    unsigned long long pc0 = 0, pc1 = 0, pc2 = 0, pc3 = 0;
    const int lane = lane_id();
    // warp-uniform trip count: rows longer than kLongRow get f_i from the whole
    // warp (a thread walking a 5000-entry row would hold its CTA back)
    constexpr int64_t kLongRow = 64;
    for (int64_t rbase = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); rbase < nloc; rbase += stride) {
        const int64_t r = rbase + lane;
        const bool valid = r < nloc;
        const int64_t i = a.rb + r;
        int64_t s = 0, e = 0;
        if (valid) {
            s = a.A.rp[i];
            e = a.A.rp[i + 1];
        }
        const bool longrow = e - s > kLongRow;
        int64_t fi = 0;
        // rows of <= kMergeMaxLen entries get f_i from their merge count below
        if (!longrow && e - s > kMergeMaxLen) {
            for (int64_t p0 = s; p0 < e; p0 += 8) {  // 8 independent gathers in flight
                int k[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) k[u] = p0 + u < e ? a.A.ci[p0 + u] : -1;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (k[u] >= 0) fi += a.T.cp[k[u] + 1] - a.T.cp[k[u]];
            }
        }
        for (unsigned lm = __ballot_sync(kFull, longrow); lm; lm &= lm - 1) {
            const int u = __ffs(lm) - 1;
            const int64_t su = __shfl_sync(kFull, s, u), eu = __shfl_sync(kFull, e, u);
            int64_t part = 0;
            for (int64_t p = su + lane; p < eu; p += 32) {
                const int k = a.A.ci[p];
                part += a.T.cp[k + 1] - a.T.cp[k];
            }
            part = warp_sum(part);
            if (lane == u) fi = part;
        }
        const int len = valid ? (int)min(e - s, (int64_t)kMergeMaxLen + 1) : 0;
        int64_t c = len == 0 ? 0 : -1;  // merge count (an empty row: 0); -1: off the merge path
        if constexpr (WW) {
            // merge width per warp: the longest merge row of the warp (rows of
            // <= 8 entries: f_i and, if small enough, the count in one pass)
            const int wl = (int)__reduce_max_sync(kFull, (unsigned)(len <= kMergeMaxLen ? len : 0));
            if (len >= 1 && len <= kMergeMaxLen) {
                switch (wl) {
                    case 1: c = sym_merge_row_w<1, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    case 2: c = sym_merge_row_w<2, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    case 3: c = sym_merge_row_w<3, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    case 4: c = sym_merge_row_w<4, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    case 5: c = sym_merge_row_w<5, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    case 6: c = sym_merge_row_w<6, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    case 7: c = sym_merge_row_w<7, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                    default: c = sym_merge_row_w<8, IdxT>(a.A, a.T, s, len, a.qs, &fi); break;
                }
            }
        } else {
            if (!valid) continue;
            switch (len) {  // rows of <= 8 entries: f_i and, if small enough, the count in one pass
                case 1: c = sym_merge_row<1, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 2: c = sym_merge_row<2, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 3: c = sym_merge_row<3, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 4: c = sym_merge_row<4, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 5: c = sym_merge_row<5, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 6: c = sym_merge_row<6, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 7: c = sym_merge_row<7, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                case 8: c = sym_merge_row<8, IdxT>(a.A, a.T, s, a.qs, &fi); break;
                default: break;
            }
        }
        if (!valid) continue;
        nnzr += e - s;
        local += fi;
        if (len <= kMergeMaxLen && c >= 0) {
            maxlen = max(maxlen, len);
            a.nnzc[r] = c;
            a.fnm[r] = 0;
            bin8[r] = kBinNone;
        } else {
            const int64_t m2 = 2 * (fi > 1 ? fi : 1);
            int lg = 64 - __clzll(m2 - 1);
            if (lg < kSymBinMinLog) lg = kSymBinMinLog;
            const int b = lg > kSymBinMaxLog ? kNumSymBins : lg - kSymBinMinLog;
            bin8[r] = (uint8_t)b;
            if (a.qs && e - s <= kMergeMaxLen) a.qs[s] = make_int2(-1, 0);  // the merge kernel skips it
            a.fnm[r] = fi - (e - s);  // >= its off-diagonal entries: temporary slots
            slots += fi - (e - s);
            maxf = max(maxf, fi);
            const unsigned long long inc = 1ull << (32 * (b & 1));
            pc0 += (b >> 1) == 0 ? inc : 0ull;
            pc1 += (b >> 1) == 1 ? inc : 0ull;
            pc2 += (b >> 1) == 2 ? inc : 0ull;
            pc3 += (b >> 1) == 3 ? inc : 0ull;
        }
    }
    // CTA reduction, then one atomic per counter per CTA
    constexpr int W = kMergeThreads / 32;
    __shared__ unsigned long long red[W][8];
    __shared__ int redmax[W];
    const unsigned long long vals[8] = {warp_sum(pc0), warp_sum(pc1), warp_sum(pc2), warp_sum(pc3),
                                        (unsigned long long)warp_sum(local), (unsigned long long)warp_sum(nnzr),
                                        (unsigned long long)__reduce_max_sync(kFull, (unsigned)min(maxf, (int64_t)UINT_MAX)),
                                        (unsigned long long)warp_sum(slots)};
    maxlen = __reduce_max_sync(kFull, maxlen);
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) red[w][q] = vals[q];
        redmax[w] = maxlen;
    }
    __syncthreads();
    if (threadIdx.x < 9) {
        const int q = threadIdx.x;
        unsigned long long t = 0;
        int mx = 0;
        for (int k = 0; k < W; ++k) {
            if (q < 6 || q == 7) t += red[k][q];
            if (q == 6) t = max(t, red[k][q]);
            mx = max(mx, redmax[k]);
        }
        if (q < 4) {  // bin counts: two 32-bit halves per word
            const unsigned long long lo = t & 0xffffffffull, hi = t >> 32;
            if (lo) atomicAdd((unsigned long long *)&ctr->sym_count[2 * q], lo);
            if (hi) atomicAdd((unsigned long long *)&ctr->sym_count[2 * q + 1], hi);
            if (lo + hi) atomicAdd((unsigned long long *)&ctr->n_mid, lo + hi);
        } else if (q == 4) {
            if (t) atomicAdd((unsigned long long *)&ctr->products, t);
        } else if (q == 5) {
            if (t) atomicAdd((unsigned long long *)&ctr->nnz_rows, t);
        } else if (q == 6) {
            if (t) atomicMax((unsigned long long *)&ctr->max_f, t);
        } else if (q == 7) {
            if (t) atomicAdd((unsigned long long *)&ctr->mid_slots, t);
        } else if (mx) {
            atomicMax(&ctr->max_len, mx);
        }
    }
}

void launch_analyze_sym(const SymArgs &a, uint8_t *bin8, DevCounters *ctr, bool warp_width, cudaStream_t s) {
    const int64_t nloc = a.re - a.rb;
    int64_t g = (nloc + kMergeThreads - 1) / kMergeThreads;
    g = g < 1 ? 1 : (g > (int64_t)sms() * 16 ? (int64_t)sms() * 16 : g);
    const bool i32 = csc_fits_i32(a.A);
    if (warp_width && i32)
        k_analyze_sym<int32_t, true><<<(unsigned)g, kMergeThreads, 0, s>>>(a, bin8, ctr);
    else if (warp_width)
        k_analyze_sym<int64_t, true><<<(unsigned)g, kMergeThreads, 0, s>>>(a, bin8, ctr);
    else if (i32)
        k_analyze_sym<int32_t, false><<<(unsigned)g, kMergeThreads, 0, s>>>(a, bin8, ctr);
    else
        k_analyze_sym<int64_t, false><<<(unsigned)g, kMergeThreads, 0, s>>>(a, bin8, ctr);
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
        // per device (context): set before every launch (cheap), never cached in a static
        cudaFuncSetAttribute(k_num_merge<RMAX, IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kMergeWarps * kMaxStageCap * (sizeof(double) + sizeof(int32_t))));
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
    if (csc_fits_i32(a.A))
        launch_merge_r<int32_t>(maxlen, &a, nullptr, s);
    else
        launch_merge_r<int64_t>(maxlen, &a, nullptr, s);
}

template <int RMAX>
static void launch_pair_t(const NumArgs &na, cudaStream_t s) {
    const size_t smem = (size_t)kPairWarps * (size_t)na.stage_cap * (sizeof(double) + sizeof(int32_t));
    // per device (context): set before every launch, never cached in a static
    cudaFuncSetAttribute(k_num_pair<RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)kPairWarps * kMaxStageCap * (sizeof(double) + sizeof(int32_t))));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_num_pair<RMAX>, kPairThreads, smem);
    if (per_sm < 1) per_sm = 1;
    // resident CTAs per SM (grid-stride kernel): RIG_PAIR_CTAS caps them
    // (measured: capping below the occupancy limit is slower on configs 2-4)
    static const int cap_sm = [] {
        const char *e = getenv("RIG_PAIR_CTAS");
        return e ? atoi(e) : 0;
    }();
    if (cap_sm > 0 && per_sm > cap_sm) per_sm = cap_sm;
    const int64_t nloc = na.re - na.rb;
    const int64_t ntiles = (nloc + kPairRows - 1) / kPairRows;
    int64_t g = (ntiles + kPairWarps - 1) / kPairWarps;
    const int64_t gmax = std::min<int64_t>((int64_t)sms() * per_sm, kCutSlotsPerLaunch);
    g = g < 1 ? 1 : (g > gmax ? gmax : g);
    k_num_pair<RMAX><<<(unsigned)g, kPairThreads, smem, s>>>(na);
    note_launch();
}

void launch_num_merge(const NumArgs &a, int maxlen, cudaStream_t s) {
    if (a.qs) {  // int32 CSC offsets and runs from the analysis
        switch (maxlen <= 4 ? 4 : maxlen) {
            case 4: launch_pair_t<4>(a, s); break;
            case 5: launch_pair_t<5>(a, s); break;
            case 6: launch_pair_t<6>(a, s); break;
            case 7: launch_pair_t<7>(a, s); break;
            default: launch_pair_t<8>(a, s); break;
        }
        return;
    }
    if (csc_fits_i32(a.A))
        launch_merge_r<int32_t>(maxlen, nullptr, &a, s);
    else
        launch_merge_r<int64_t>(maxlen, nullptr, &a, s);
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

// Row slots of the huge path: each is a dense accumulator over all rows plus
// a bitmap, so slots cost memory.  With huge rows present (heavy-tailed
// matrices, whose long mid rows also defer) 8 per SM measured fastest on
// config 4 (huge + deferred rows: 4.3 -> 2.9 ms against 2 per SM); otherwise
// only the odd deferred row comes here and 2 per SM do.  Within a budget of
// RIG_HUGE_BUDGET_GB (24) and a quarter of the free device memory.
#ifndef RIG_HUGE_BUDGET_GB
#define RIG_HUGE_BUDGET_GB 24
#endif
#ifndef RIG_HUGE_PER_SM
#define RIG_HUGE_PER_SM 8
#endif
int huge_slots_rw(int64_t nrows, int64_t n_reach, int64_t per_sm) {
    const size_t per = huge_scratch_bytes(nrows, 1, true);
    // budget from the device's TOTAL memory (fixed per device): a budget that
    // followed the current free memory would change the workspace size from
    // build to build and defeat the workspace cache (a regrow costs ms)
    static size_t quarter[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!quarter[dev]) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        quarter[dev] = tot / 4 ? tot / 4 : 1;
    }
    const size_t bud = std::min(((size_t)RIG_HUGE_BUDGET_GB << 30), quarter[dev]);
    int64_t s = std::min<int64_t>(per_sm * (int64_t)sms(), n_reach);
    s = std::min<int64_t>(s, (int64_t)(bud / (per ? per : 1)));
    return (int)std::max<int64_t>(s, 1);
}

int huge_slots(int64_t nrows, int64_t n_huge, bool heavy) {
    const size_t per = huge_scratch_bytes(nrows, 1, true);
    static size_t free_q = 0;
    if (!free_q) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        free_q = fr / 4 ? fr / 4 : 1;
    }
    const size_t bud = std::min(((size_t)RIG_HUGE_BUDGET_GB << 30), free_q);
    int64_t budget = (int64_t)bud / (int64_t)(per ? per : 1);
    int64_t s = (heavy ? RIG_HUGE_PER_SM : 2) * (int64_t)sms();
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

// Numeric: the row's products are enumerated 512 at a time (one 32-product
// sub-chunk per warp) and routed, in product order, into shared-memory queues
// of their owner warp ((j >> 5) % 16).  Each owner then applies its queue in
// order (ordered __match_any_sync chains) to the dense accumulator, so every
// chain runs in ascending k and each product is handled once.
__global__ void __launch_bounds__(kHugeThreads) k_num_huge(MidArgs a, unsigned char *scratch, size_t slot_bytes,
                                                           int64_t nwords) {
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
    const int64_t n = *a.count;
    for (int64_t idx = blockIdx.x; idx < n; idx += gridDim.x) {
        const int64_t i = a.list[idx];
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
        const int64_t g0 = a.toff[r];  // temporary slot of the row
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
                        a.tcol[pos] = (int32_t)j;
                        a.tw[pos] = fabs(c);
                        ++pos;
                    }
                }
                bm[w1] = 0u;
            }
            if (t2 < nw2) l2[t2] = 0u;
            o += tot;
            __syncthreads();
        }
        if (tid == 0) a.cnt[r] = o + 1;  // exact kept count (+1: the scan subtracts the diagonal)
        __syncthreads();
    }
}

void launch_num_huge(const MidArgs &a, int slots, void *scratch, cudaStream_t s) {
    const size_t slot_bytes = bitmap_stride(a.A.nrows);
    const int64_t nw = bitmap_words(a.A.nrows);
    const size_t smem = (size_t)l2_words(nw) * sizeof(unsigned);
    cudaFuncSetAttribute(k_num_huge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_num_huge<<<slots, kHugeThreads, smem, s>>>(a, static_cast<unsigned char *>(scratch), slot_bytes, nw);
    note_launch();
}

}  // namespace rig

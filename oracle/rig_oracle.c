/*
 * rig_oracle.c -- CPU ORACLE for the row inner-product graph (G_RIP) and its
 * cutsize.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1710_07769_b200/) never links, imports or calls it,
 * and shares no code, header, table or helper with it.
 *
 * It is the plain definition written out, in the paper's order:
 *
 *   PAPER.md:293-301  (§2.1, eq. E)    edge (v_i,v_j) iff r_i r_j^T != 0
 *   PAPER.md:310-315  (§2.1, eq14)     cost(v_i,v_j) = |r_i r_j^T|
 *   PAPER.md:317-318  (§2.1)           optional prescaling of rows to unit 2-norm
 *   PAPER.md:321-325, 351-352 (§2.1)   G_RIP == graph of C = A A^T, diagonal ignored
 *   PAPER.md:560-562  (§2.3)           C computed by basic (Gustavson) SpGEMM
 *   PAPER.md:393-405, 1150-1154 (§2.2, eq. partcut)
 *                                      cutsize(Pi) = sum of costs of cut edges
 *   PAPER.md:506-519  (§2.2, eq. ip_km) inter-block inner products (f2)
 *   PAPER.md:572-576  (§2.3)           dense-column sparsification A~ (f1)
 *   PAPER.md:611      (§2.3)           integer edge weights ceil(alpha*cost) (f1)
 *
 * Readings where the paper is silent:
 *   - ordering contract: for each (i,j), c_ij = fma-chain over the shared
 *     columns k in ASCENDING k, starting from +0.0 (c2 #4);
 *   - scaling: ss = ascending-k fma chain of a_ik^2 from +0.0, nrm = sqrt(ss)
 *     (IEEE correctly rounded), a_hat = a / nrm (IEEE division) (c2 #5);
 *   - an edge is kept iff j != i and |c_ij| > drop_tol (strict), c2 #1-#3;
 *   - cutsize sums each undirected cut edge once (stored j > i), Neumaier
 *     compensated (c2 #8-#9).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp (no DAZ/FTZ); fma()
 * is the C99 correctly-rounded fused multiply-add.  OpenMP only runs row
 * chunks of orc_build concurrently (orc_build_par, SURVEY.md §8(c) c1 step
 * 6): every row is computed by the same code, so the result is identical for
 * any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_INVALID (-1)
#define ORC_ERR_ZERO_ROW (-3)
#define ORC_ERR_NONFINITE (-4)
#define ORC_ERR_NOMEM (-5)

/* Row scaling to unit 2-norm, PAPER.md:317-318 (§2.1) and PAPER.md:628
 * (§3.1: "row scaling on A to have 2-norm equal to exactly one").
 * out may alias val.  Returns ORC_ERR_ZERO_ROW for an all-zero / empty row
 * and ORC_ERR_NONFINITE when a value or a norm is not finite. */
int orc_scale_rows(int64_t nrows, const int64_t *row_ptr, const double *val,
                   double *out, double *norms /* may be NULL */) {
    for (int64_t i = 0; i < nrows; ++i) {
        double ss = +0.0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            if (!isfinite(val[p])) return ORC_ERR_NONFINITE;
            ss = fma(val[p], val[p], ss);
        }
        if (!isfinite(ss)) return ORC_ERR_NONFINITE;
        if (ss == 0.0) return ORC_ERR_ZERO_ROW;
        double nrm = sqrt(ss);
        if (norms) norms[i] = nrm;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) out[p] = val[p] / nrm;
    }
    return ORC_OK;
}

/* Column access to A (CSC of A == CSR of A^T), required by Gustavson's
 * row-by-row SpGEMM.  Stable counting sort: rows ascend
 * within each column. */
int orc_transpose(int64_t nrows, int64_t ncols, const int64_t *row_ptr,
                  const int32_t *col_idx, const double *val, int64_t *col_ptr,
                  int32_t *row_idx, double *valT) {
    for (int64_t k = 0; k <= ncols; ++k) col_ptr[k] = 0;
    int64_t nnz = row_ptr[nrows];
    for (int64_t p = 0; p < nnz; ++p) {
        if (col_idx[p] < 0 || col_idx[p] >= ncols) return ORC_ERR_INVALID;
        col_ptr[col_idx[p] + 1] += 1;
    }
    for (int64_t k = 0; k < ncols; ++k) col_ptr[k + 1] += col_ptr[k];
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncols > 0 ? ncols : 1));
    if (!next) return ORC_ERR_NOMEM;
    for (int64_t k = 0; k < ncols; ++k) next[k] = col_ptr[k];
    for (int64_t i = 0; i < nrows; ++i) {
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            int64_t q = next[col_idx[p]]++;
            row_idx[q] = (int32_t)i;
            valT[q] = val[p];
        }
    }
    free(next);
    return ORC_OK;
}

/* Intermediate products of Gustavson's A A^T for row i: f_i = sum over k in
 * row i of nnz(column k).  Total P = sum_k nnz(col k)^2. */
int64_t orc_row_products(int64_t nrows, const int64_t *row_ptr, const int32_t *col_idx,
                         const int64_t *col_ptr, int64_t *f /* may be NULL */) {
    int64_t total = 0;
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t fi = 0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            fi += col_ptr[col_idx[p] + 1] - col_ptr[col_idx[p]];
        if (f) f[i] = fi;
        total += fi;
    }
    return total;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* G_RIP rows [row_begin, row_end) from the (already scaled, if requested)
 * CSR of A and its CSC, by dense-accumulator Gustavson SpGEMM (PAPER.md:
 * 560-562), keeping off-diagonal entries with |c_ij| > drop_tol as edges with
 * cost |c_ij|.
 *
 * Outputs (malloc'ed here, released with orc_free):
 *   *g_row_ptr  int64[nloc+1]  (local, starts at 0)
 *   *g_col      int32[nnz]     ascending per row
 *   *g_w        double[nnz]    |c_ij|
 * Optional caller arrays (length nloc, may be NULL):
 *   diag[]   c_ii (0.0 when row i is empty)
 *   nnzc[]   structural nnz of row i of C including the diagonal
 */
int orc_build(int64_t nrows, int64_t ncols, const int64_t *row_ptr,
              const int32_t *col_idx, const double *val, const int64_t *col_ptr,
              const int32_t *row_idx, const double *valT, double drop_tol,
              int64_t row_begin, int64_t row_end, int64_t **g_row_ptr,
              int32_t **g_col, double **g_w, int64_t *g_nnz, double *diag,
              int64_t *nnzc) {
    (void)ncols;
    if (row_begin < 0 || row_end > nrows || row_begin > row_end) return ORC_ERR_INVALID;
    if (!(drop_tol >= 0.0)) return ORC_ERR_INVALID;
    int64_t nloc = row_end - row_begin;
    int64_t cap = 1024, len = 0;
    double *acc = (double *)malloc(sizeof(double) * (size_t)(nrows > 0 ? nrows : 1));
    int64_t *mark = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nrows > 0 ? nrows : 1));
    int32_t *touched = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nrows > 0 ? nrows : 1));
    int64_t *rp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nloc + 1));
    int32_t *gc = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    double *gw = (double *)malloc(sizeof(double) * (size_t)cap);
    if (!acc || !mark || !touched || !rp || !gc || !gw) {
        free(acc); free(mark); free(touched); free(rp); free(gc); free(gw);
        return ORC_ERR_NOMEM;
    }
    for (int64_t j = 0; j < nrows; ++j) mark[j] = -1;
    rp[0] = 0;
    for (int64_t i = row_begin; i < row_end; ++i) {
        int64_t nt = 0;
        /* row i of C: for k in row i (ascending), for j in column k */
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            int32_t k = col_idx[p];
            double a_ik = val[p];
            for (int64_t q = col_ptr[k]; q < col_ptr[k + 1]; ++q) {
                int32_t j = row_idx[q];
                if (mark[j] != i) {
                    mark[j] = i;
                    acc[j] = +0.0;
                    touched[nt++] = j;
                }
                acc[j] = fma(a_ik, valT[q], acc[j]);
            }
        }
        qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
        if (diag) diag[i - row_begin] = 0.0;
        if (nnzc) nnzc[i - row_begin] = nt;
        for (int64_t t = 0; t < nt; ++t) {
            int32_t j = touched[t];
            double c = acc[j];
            if (j == i) {
                if (diag) diag[i - row_begin] = c;
                continue;
            }
            double w = fabs(c);
            if (!(w > drop_tol)) continue;
            if (len == cap) {
                cap *= 2;
                int32_t *nc = (int32_t *)realloc(gc, sizeof(int32_t) * (size_t)cap);
                if (nc) gc = nc;
                double *nw = (double *)realloc(gw, sizeof(double) * (size_t)cap);
                if (nw) gw = nw;
                if (!nc || !nw) {
                    free(acc); free(mark); free(touched); free(rp); free(gc); free(gw);
                    return ORC_ERR_NOMEM;
                }
            }
            gc[len] = j;
            gw[len] = w;
            ++len;
        }
        rp[i - row_begin + 1] = len;
    }
    free(acc);
    free(mark);
    free(touched);
    *g_row_ptr = rp;
    *g_col = gc;
    *g_w = gw;
    *g_nnz = len;
    return ORC_OK;
}

void orc_free(void *p) { free(p); }

/* orc_build over rows [row_begin, row_end) in contiguous row chunks run by
 * `nthreads` OpenMP threads (each chunk: its own dense accumulator), outputs
 * concatenated in row order.  Same outputs as orc_build, bit for bit. */
int orc_build_par(int64_t nrows, int64_t ncols, const int64_t *row_ptr,
                  const int32_t *col_idx, const double *val, const int64_t *col_ptr,
                  const int32_t *row_idx, const double *valT, double drop_tol,
                  int64_t row_begin, int64_t row_end, int nthreads, int64_t **g_row_ptr,
                  int32_t **g_col, double **g_w, int64_t *g_nnz, double *diag,
                  int64_t *nnzc) {
    if (row_begin < 0 || row_end > nrows || row_begin > row_end) return ORC_ERR_INVALID;
    if (nthreads < 1) nthreads = 1;
    int64_t nloc = row_end - row_begin;
    int64_t nch = (int64_t)nthreads * 4;
    if (nch > nloc) nch = nloc > 0 ? nloc : 1;
    int64_t **rps = (int64_t **)calloc((size_t)nch, sizeof(int64_t *));
    int32_t **gcs = (int32_t **)calloc((size_t)nch, sizeof(int32_t *));
    double **gws = (double **)calloc((size_t)nch, sizeof(double *));
    int64_t *cnt = (int64_t *)calloc((size_t)nch, sizeof(int64_t));
    int *st = (int *)calloc((size_t)nch, sizeof(int));
    int64_t *rp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nloc + 1));
    if (!rps || !gcs || !gws || !cnt || !st || !rp) {
        free(rps); free(gcs); free(gws); free(cnt); free(st); free(rp);
        return ORC_ERR_NOMEM;
    }
    #pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t a = row_begin + nloc * c / nch, b = row_begin + nloc * (c + 1) / nch;
        st[c] = orc_build(nrows, ncols, row_ptr, col_idx, val, col_ptr, row_idx, valT, drop_tol, a, b,
                          &rps[c], &gcs[c], &gws[c], &cnt[c], diag ? diag + (a - row_begin) : NULL,
                          nnzc ? nnzc + (a - row_begin) : NULL);
    }
    int err = ORC_OK;
    int64_t total = 0;
    for (int64_t c = 0; c < nch; ++c) {
        if (st[c] && !err) err = st[c];
        total += cnt[c];
    }
    int32_t *gc = NULL;
    double *gw = NULL;
    if (!err) {
        gc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(total > 0 ? total : 1));
        gw = (double *)malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
        if (!gc || !gw) err = ORC_ERR_NOMEM;
    }
    if (!err) {
        int64_t off = 0;
        rp[0] = 0;
        for (int64_t c = 0; c < nch; ++c) {
            int64_t a = nloc * c / nch, b = nloc * (c + 1) / nch;
            for (int64_t r = a; r < b; ++r) rp[r + 1] = off + rps[c][r - a + 1];
            memcpy(gc + off, gcs[c], sizeof(int32_t) * (size_t)cnt[c]);
            memcpy(gw + off, gws[c], sizeof(double) * (size_t)cnt[c]);
            off += cnt[c];
        }
    }
    for (int64_t c = 0; c < nch; ++c) {
        free(rps[c]); free(gcs[c]); free(gws[c]);
    }
    free(rps); free(gcs); free(gws); free(cnt); free(st);
    if (err) {
        free(rp); free(gc); free(gw);
        return err;
    }
    *g_row_ptr = rp;
    *g_col = gc;
    *g_w = gw;
    *g_nnz = total;
    return ORC_OK;
}

/* Neumaier-compensated summation step. */
static void neumaier(double *s, double *c, double x) {
    double t = *s + x;
    if (fabs(*s) >= fabs(x))
        *c += (*s - t) + x;
    else
        *c += (x - t) + *s;
    *s = t;
}

/* cutsize(Pi) = sum of cost(v_i,v_j) over cut edges (§2.2;
 * PAPER.md:1150-1154, eq. partcut), each undirected edge counted once
 * (stored (i,j) with j > i).  Also returns the total edge weight and the
 * intra-block weight (the identity cut = total - intra is a test pin).
 * Rows are [row_begin, row_begin + nloc) of the global graph; part has the
 * global length.  Returns ORC_ERR_INVALID if a part id is outside [0, K). */
int orc_cutsize(int64_t nloc, int64_t row_begin, const int64_t *g_row_ptr,
                const int32_t *g_col, const double *g_w, int64_t n_global,
                const int32_t *part, int32_t K, double *cut, double *total,
                double *intra) {
    for (int64_t v = 0; v < n_global; ++v)
        if (part[v] < 0 || part[v] >= K) return ORC_ERR_INVALID;
    double sc = 0.0, cc = 0.0, st = 0.0, ct = 0.0, si = 0.0, ci = 0.0;
    for (int64_t r = 0; r < nloc; ++r) {
        int64_t i = row_begin + r;
        for (int64_t e = g_row_ptr[r]; e < g_row_ptr[r + 1]; ++e) {
            int64_t j = g_col[e];
            if (j <= i) continue;
            neumaier(&st, &ct, g_w[e]);
            if (part[i] != part[j])
                neumaier(&sc, &cc, g_w[e]);
            else
                neumaier(&si, &ci, g_w[e]);
        }
    }
    *cut = sc + cc;
    if (total) *total = st + ct;
    if (intra) *intra = si + ci;
    return ORC_OK;
}

/* ---------------------------------------------------------------- f2
 * Inter-block inner-product matrix of a K-way block-row partition
 * (eq. ip_km):
 *   ip_km = sum over r_i in R_k, r_j in R_m of |r_i r_j^T| = sum |c_ij|, k != m,
 * i.e. the sum of the stored graph weights w_ij of edges with part[i] = k and
 * part[j] = m (both orientations are stored, so ip is symmetric), and the
 * part weights (eq16 and 1141-1146 eq. Wk):
 *   W_k = sum over v_i in V_k of w(v_i), w(v_i) = 1 or nnz(r_i).
 * ip[K*K] (row-major, diagonal 0) is summed per cell with Neumaier
 * compensation over the rows in ascending order; W[K] counts exactly.
 * a_row_ptr: A's row pointers for nnz weights, or NULL for unit weights.
 * Rows are [row_begin, row_begin + nloc) of the global graph. */
int orc_ip_matrix(int64_t nloc, int64_t row_begin, const int64_t *g_row_ptr, const int32_t *g_col,
                  const double *g_w, int64_t n_global, const int32_t *part, int32_t K,
                  const int64_t *a_row_ptr, double *ip, int64_t *W) {
    for (int64_t v = 0; v < n_global; ++v)
        if (part[v] < 0 || part[v] >= K) return ORC_ERR_INVALID;
    double *comp = (double *)calloc((size_t)K * (size_t)K, sizeof(double));
    if (!comp) return ORC_ERR_NOMEM;
    memset(ip, 0, sizeof(double) * (size_t)K * (size_t)K);
    memset(W, 0, sizeof(int64_t) * (size_t)K);
    for (int64_t r = 0; r < nloc; ++r) {
        const int64_t i = row_begin + r;
        const int32_t k = part[i];
        W[k] += a_row_ptr ? a_row_ptr[i + 1] - a_row_ptr[i] : 1;
        for (int64_t e = g_row_ptr[r]; e < g_row_ptr[r + 1]; ++e) {
            const int32_t m = part[g_col[e]];
            if (m == k) continue;
            neumaier(&ip[(int64_t)k * K + m], &comp[(int64_t)k * K + m], g_w[e]);
        }
    }
    for (int64_t c = 0; c < (int64_t)K * K; ++c) ip[c] += comp[c];
    free(comp);
    return ORC_OK;
}

/* ---------------------------------------------------------------- f1
 * Dense-column threshold (§2.3): a column is dense if it holds
 * more than sqrt(n) nonzeros, and a dense column keeps its sqrt(n) largest
 * entries.  Reading R20: the kept count
 * is T = ceil(sqrt(n)), the smallest integer t with t*t >= n, n = nrows;
 * "nnz > sqrt(n)" and "nnz > T" select the same columns to shrink, since a
 * column with nnz <= T keeps all of its entries either way. */
int64_t orc_dense_threshold(int64_t n) {
    int64_t t = 0;
    while (t * t < n) ++t;
    return t;
}

typedef struct {
    double mag;
    int32_t row;
    int64_t pos; /* position in the CSR */
} orc_entry;

/* (|value| descending, row ascending): ties go to the lower row */
static int cmp_entry(const void *a, const void *b) {
    const orc_entry *x = (const orc_entry *)a, *y = (const orc_entry *)b;
    if (x->mag != y->mag) return x->mag > y->mag ? -1 : 1;
    return (x->row > y->row) - (x->row < y->row);
}

/* A~ from A (§2.3): every column with more than T nonzeros
 * keeps the T entries of largest absolute value (ties: lower row), every
 * other column is unchanged.  Values are copied, not re-normalised (reading
 * R21: A~ is extracted from the already scaled A; SPEC.md:242 open question).
 * Output CSR (rows ascending, columns ascending within a row, as the input)
 * into caller arrays of capacity nnz(A); *nnz_out = nnz(A~). */
int orc_sparsify(int64_t nrows, int64_t ncols, const int64_t *row_ptr, const int32_t *col_idx,
                 const double *val, int64_t *out_row_ptr, int32_t *out_col, double *out_val,
                 int64_t *nnz_out) {
    const int64_t T = orc_dense_threshold(nrows);
    const int64_t nnz = row_ptr[nrows];
    int64_t *col_ptr = (int64_t *)calloc((size_t)ncols + 1, sizeof(int64_t));
    orc_entry *ent = (orc_entry *)malloc(sizeof(orc_entry) * (size_t)(nnz > 0 ? nnz : 1));
    unsigned char *keep = (unsigned char *)malloc((size_t)(nnz > 0 ? nnz : 1));
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncols > 0 ? ncols : 1));
    if (!col_ptr || !ent || !keep || !next) {
        free(col_ptr); free(ent); free(keep); free(next);
        return ORC_ERR_NOMEM;
    }
    for (int64_t p = 0; p < nnz; ++p) {
        if (col_idx[p] < 0 || col_idx[p] >= ncols) {
            free(col_ptr); free(ent); free(keep); free(next);
            return ORC_ERR_INVALID;
        }
        col_ptr[col_idx[p] + 1] += 1;
    }
    for (int64_t k = 0; k < ncols; ++k) col_ptr[k + 1] += col_ptr[k];
    for (int64_t k = 0; k < ncols; ++k) next[k] = col_ptr[k];
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            orc_entry e = {fabs(val[p]), (int32_t)i, p};
            ent[next[col_idx[p]]++] = e;
        }
    for (int64_t p = 0; p < nnz; ++p) keep[p] = 1;
    for (int64_t k = 0; k < ncols; ++k) {
        const int64_t len = col_ptr[k + 1] - col_ptr[k];
        if (len <= T) continue;
        qsort(ent + col_ptr[k], (size_t)len, sizeof(orc_entry), cmp_entry);
        for (int64_t q = col_ptr[k] + T; q < col_ptr[k + 1]; ++q) keep[ent[q].pos] = 0;
    }
    int64_t o = 0;
    out_row_ptr[0] = 0;
    for (int64_t i = 0; i < nrows; ++i) {
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
            if (keep[p]) {
                out_col[o] = col_idx[p];
                out_val[o] = val[p];
                ++o;
            }
        out_row_ptr[i + 1] = o;
    }
    *nnz_out = o;
    free(col_ptr); free(ent); free(keep); free(next);
    return ORC_OK;
}

/* Integer edge weights for the partitioner (§2.3):
 *   wgt(v_i,v_j) = ceil(alpha * cost(v_i,v_j)),  alpha a positive integer.
 * Exact: w = m * 2^e with m a 53-bit integer (frexp), so alpha * w =
 * (alpha * m) * 2^e with alpha * m exact in 128-bit integers; the ceiling is
 * a shift (e >= 0) or a rounded-up division by 2^-e (e < 0).  Requires
 * 1 <= alpha <= 2^53 and w >= 0 finite; ORC_ERR_INVALID otherwise or if a
 * result exceeds 2^62. */
int orc_int_weights(int64_t n, const double *w, int64_t alpha, int64_t *wgt) {
    if (alpha < 1 || alpha > ((int64_t)1 << 53)) return ORC_ERR_INVALID;
    for (int64_t e = 0; e < n; ++e) {
        const double x = w[e];
        if (!(x >= 0.0) || !isfinite(x)) return ORC_ERR_INVALID;
        if (x == 0.0) {
            wgt[e] = 0;
            continue;
        }
        int ex;
        const double fr = frexp(x, &ex);             /* x = fr * 2^ex, fr in [0.5, 1) */
        const int64_t m = (int64_t)ldexp(fr, 53);     /* exact: x = m * 2^(ex - 53) */
        const int sh = ex - 53;
        const unsigned __int128 prod = (unsigned __int128)(uint64_t)alpha * (uint64_t)m;
        unsigned __int128 q;
        if (sh >= 0) {
            if (sh > 62) return ORC_ERR_INVALID;
            q = prod << sh;
            if ((q >> sh) != prod) return ORC_ERR_INVALID;
        } else if (-sh >= 127) {
            q = 1; /* 0 < alpha * x < 1 */
        } else {
            const unsigned __int128 d = (unsigned __int128)1 << (-sh);
            q = prod / d + (prod % d != 0);
        }
        if (q > ((unsigned __int128)1 << 62)) return ORC_ERR_INVALID;
        wgt[e] = (int64_t)q;
    }
    return ORC_OK;
}

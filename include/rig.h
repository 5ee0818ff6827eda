/*
 * rig.h -- C ABI of librig, the B200 (sm_100a) builder of the row
 * inner-product graph G_RIP of a sparse matrix A and the cutsize of a K-way
 * block-row partition (arXiv 1710.07769, "row inner-product graph model").
 *
 * What the calls compute (PAPER.md = /root/reference/PAPER.md):
 *   - G_RIP(A): one vertex per row r_i; an edge (v_i,v_j) iff r_i r_j^T != 0
 *     (§2.1, eq. for E) with cost |r_i r_j^T| (PAPER.md:
 *     310-315, eq14).  It is the off-diagonal pattern and |values| of
 *     C = A A^T, computed by Gustavson SpGEMM
 *     (§2.3).  Rows may first be scaled to unit 2-norm so
 *     costs are |cosines|.
 *   - cutsize(Pi) = sum of costs of cut edges = interIP(Pi) (PAPER.md:393-405,
 *     §2.2, eq. partcut).
 *
 * Arithmetic contract (readings R1-R9), identical to the CPU
 * oracle in oracle/ so structure and weights match bit for bit:
 *   - scaling: ss_i = fma-chain of a_ik^2 over ascending k from +0.0,
 *     nrm_i = sqrt_rn(ss_i), a_hat_ik = a_ik /_rn nrm_i;
 *   - c_ij = fma-chain of a_hat_ik * a_hat_jk over the shared columns k in
 *     ascending k, starting from +0.0;
 *   - edge (i,j) kept iff j != i and |c_ij| > drop_tol (strict);
 *   - the graph is stored symmetric (both (i,j) and (j,i)), columns
 *     ascending within each row.
 *
 * Conventions for every call:
 *   - All matrix / graph / partition pointers are DEVICE pointers on the
 *     current CUDA device, except in rig_build_host (HOST pointers).
 *   - Index types: row pointers int64, column / row indices int32, values and
 *     weights float64, part ids int32.
 *   - Input CSR must be canonical (row_ptr[0]=0, non-decreasing,
 *     row_ptr[nrows]=nnz, columns strictly increasing per row and in
 *     [0, ncols)); pass RIG_FLAG_VALIDATE to have it checked on the device.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *     enqueued on it; inputs are borrowed and must stay valid until the
 *     stream has passed the call.
 *   - Every call returns RIG_OK (0) or a negative RIG_ERR_* code; the message
 *     of the last failure on the calling thread is rig_last_error().  No C++
 *     exception crosses the ABI.  Asynchronous kernel faults surface at the
 *     next synchronising call as RIG_ERR_CUDA.
 */
#ifndef RIG_H_
#define RIG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define RIG_OK 0
#define RIG_ERR_INVALID (-1)      /* null pointer, bad size/range, drop_tol < 0 or NaN, capacity too small */
#define RIG_ERR_NONCANONICAL (-2) /* RIG_FLAG_VALIDATE found a non-canonical CSR */
#define RIG_ERR_ZERO_ROW (-3)     /* scale_rows = 1 and a row is empty / all zero */
#define RIG_ERR_NONFINITE (-4)    /* a value or a row norm is Inf/NaN (checked when scaling or validating) */
#define RIG_ERR_NOMEM (-5)        /* device or host allocation failed */
#define RIG_ERR_CUDA (-6)         /* a CUDA runtime error; message holds cudaGetErrorString */

/* ---- flags ------------------------------------------------------------- */
#define RIG_FLAG_VALIDATE 0x1u /* a0: check canonical CSR and finite values on the device */
#define RIG_FLAG_DIAG 0x2u     /* also return diag[i] = c_ii (0 for an empty row) */
/* f1: build the sparsified graph G~_RIP = graph of A~ A~^T (PAPER.md:572-579,
 * §2.3) instead: every column of A_hat with more than T = ceil(sqrt(nrows))
 * nonzeros keeps its T entries of largest |a_hat| (ties: the lower row;
 * DESIGN.md readings R20-R21; no re-normalisation after the cut).  Costs one
 * extra host synchronisation (the size of A~), and the whole A~ is formed on
 * every rank (columns are global).  Without dense columns the graph equals
 * the one built without the flag. */
#define RIG_FLAG_SPARSIFY 0x4u

typedef void *rig_stream_t; /* a cudaStream_t */

#if defined(__GNUC__)
#define RIG_API __attribute__((visibility("default")))
#else
#define RIG_API
#endif

/* Sparse A (nrows x ncols), canonical CSR. */
typedef struct {
    int64_t nrows, ncols, nnz;
    const int64_t *row_ptr; /* [nrows+1] */
    const int32_t *col_idx; /* [nnz] */
    const double *val;      /* [nnz] */
} rig_csr_t;

/* G_RIP rows [row_begin, row_begin + n) as symmetric CSR (local row_ptr
 * starting at 0, global column ids).  w[e] = |c_ij| > drop_tol, j != i. */
typedef struct {
    int64_t n, nnz;
    int64_t *row_ptr; /* [n+1] */
    int32_t *col_idx; /* [nnz] ascending within each row */
    double *w;        /* [nnz] */
    double *diag;     /* [n] c_ii, or NULL (RIG_FLAG_DIAG not given) */
} rig_graph_t;

typedef struct rig_plan rig_plan_t;

/* ---- simple API: library-owned output ---------------------------------- */

/* Build G_RIP(A) for all rows (steps a0-a6 of DESIGN.md §2).
 *   A          device CSR (borrowed).
 *   scale_rows 1: scale rows to unit 2-norm first; 0: use A as is.
 *   drop_tol   >= 0; an off-diagonal entry is an edge iff |c_ij| > drop_tol.
 *   flags      RIG_FLAG_VALIDATE | RIG_FLAG_DIAG | RIG_FLAG_SPARSIFY.
 *   out        filled with device arrays allocated by the library (stream-
 *              ordered on `stream`); release them with rig_graph_free.
 *              col_idx / w are allocated with the capacity bound
 *              sum_i (f_i - len_i) (f_i: products of row i) >= out->nnz.
 * Synchronises `stream` to size allocations and to read the graph nnz: twice
 * in general, once when every row takes the merge path (the decision and the
 * bound come from the column histogram while the transpose runs, DESIGN.md
 * §4.5); device-side errors are reported at that synchronisation. */
RIG_API int rig_build(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, rig_graph_t *out,
              rig_stream_t stream);

/* Release the arrays of a graph returned by rig_build / rig_build_rows / rig_build_cut;
 * zeroes *g.  NULL arrays are ignored. */
RIG_API int rig_graph_free(rig_graph_t *g, rig_stream_t stream);

/* Same as rig_build restricted to rows [row_begin, row_end) of C (one shard
 * of a multi-GPU build).  A is the FULL matrix (replicated);
 * out->row_ptr is local (starts at 0); column ids are global. */
RIG_API int rig_build_rows(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t row_begin,
                   int64_t row_end, rig_graph_t *out, rig_stream_t stream);

/* Build + score in one call (the whole hot path): rig_build_rows
 * for rows [row_begin, row_end), then the cutsize of `part` (device int32
 * [A->nrows], ids in [0, K)) over those rows into cut_dev[0] (device double),
 * enqueued behind the numeric pass before the final synchronisation.
 * Multi-GPU: each rank passes its shard and allreduces cut_dev. */
RIG_API int rig_build_cut(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t row_begin,
                          int64_t row_end, const int32_t *part, int32_t K, rig_graph_t *out, double *cut_dev,
                          rig_stream_t stream);

/* ---- staged API: caller-owned output (estimate -> allocate -> compute) --- */

/* Runs steps a0-a4 for rows [row_begin, row_end): validation, scaling,
 * transpose, flop count, the merge rows' symbolic pass and the lists of the
 * other rows.  Synchronises once. */
RIG_API int rig_plan_create(const rig_csr_t *A, int scale_rows, double drop_tol, uint32_t flags, int64_t row_begin,
                    int64_t row_end, rig_plan_t **plan, rig_stream_t stream);

/* nnz_upper: graph capacity needed, the bound sum_i (f_i - len_i) >= the
 * shard's off-diagonal nnz (every row i of A meets itself in each of its
 * len_i columns); products: Gustavson intermediate products of the shard
 * (sum f_i); workspace_bytes: device bytes rig_plan_execute needs in
 * `workspace` (0: internal temporaries are stream-ordered allocations). */
RIG_API int rig_plan_query(const rig_plan_t *plan, int64_t *nnz_upper, int64_t *products, size_t *workspace_bytes);

/* Steps a5-a6 into caller arrays: out->row_ptr [n+1], out->col_idx and
 * out->w with capacity >= nnz_upper, out->diag [n] or NULL.  `workspace`
 * must hold workspace_bytes (may be NULL if that is 0).  Sets out->n and
 * out->nnz.  Synchronises once (to read the nnz; again only if a merge row
 * dropped an entry by value and the graph is compacted). */
RIG_API int rig_plan_execute(rig_plan_t *plan, void *workspace, rig_graph_t *out, rig_stream_t stream);

RIG_API int rig_plan_destroy(rig_plan_t *plan);

/* ---- multi-GPU helper -------------------------------------------------- */

/* Flop-balanced contiguous split of the rows of C into `parts` shards:
 * split[0]=0, split[parts]=nrows, split[g] = first row whose inclusive
 * prefix of products f_i reaches ceil(g*P/parts).
 * `split` is a HOST array of parts+1 entries.  Deterministic: every rank
 * computes the same split.  Synchronises. */
RIG_API int rig_row_split(const rig_csr_t *A, int32_t parts, int64_t *split, rig_stream_t stream);

/* ---- cutsize ----------------------------------------------------------- */

/* cut_dev[0] = sum over stored edges (i,j) of g with j > i and
 * part[i] != part[j] of w_ij, i = row_begin + local row.
 * part: device int32[n_global] with values in [0, K); an out-of-range id
 * makes cut_dev[0] = NaN.  Deterministic for a fixed graph.  Fully
 * asynchronous (no host sync).  Multi-GPU: allreduce cut_dev outside. */
RIG_API int rig_cutsize(const rig_graph_t *g, int64_t row_begin, int64_t n_global, const int32_t *part, int32_t K,
                double *cut_dev, rig_stream_t stream);

/* ---- partition quality ------------------------------ */

/* Inter-block inner-product matrix of a K-way block-row partition
 * (eq. ip_km): ip_km = sum of |c_ij| = w_ij over stored
 * edges with part[i] = k != m = part[j] (symmetric; sum_{k<m} ip_km =
 * cutsize), and part weights (eq16, 1141-1146 eq. Wk):
 * W_k = sum of w(v_i) over rows i of part k, w(v_i) = nnz(r_i) when
 * a_row_ptr (device, A's row pointers) is given, else 1.
 *   acc  device int64 [4*K*K + 1], ZEROED by the caller: every weight is added
 *        exactly as four 32-bit limbs of trunc(w * 2^64) in separate 64-bit
 *        counters (integer sums: order-independent and deterministic); the
 *        last element is an error flag (part id outside [0, K), or a weight
 *        outside [0, 2^63)).
 *   W    device int64 [K], ZEROED by the caller.
 * Rows of g are [row_begin, row_begin + g->n) of the global graph.
 * Accumulates, asynchronously.  Multi-GPU: allreduce acc and W (int64 sums)
 * before rig_partition_ip_finalize. */
RIG_API int rig_partition_ip(const rig_graph_t *g, int64_t row_begin, int64_t n_global, const int32_t *part,
                             int32_t K, const int64_t *a_row_ptr, int64_t *acc, int64_t *W, rig_stream_t stream);

/* HOST function: ip_host[K*K] (row-major, zero diagonal) from a host copy of
 * acc: each cell's fixed-point sum converted to double (one correctly
 * rounded conversion while the sum fits 2^63).  RIG_ERR_INVALID if the error
 * flag is set. */
RIG_API int rig_partition_ip_finalize(const int64_t *acc_host, int32_t K, double *ip_host);

/* ---- steps next to the path ------------------------ */

/* A~ alone: the (optionally row-scaled, as in rig_build)
 * matrix with every column holding more than T = ceil(sqrt(nrows)) nonzeros
 * cut to its T largest |values| (ties: the lower row).  out receives
 * library-owned DEVICE arrays (one allocation, stream-ordered) in canonical
 * CSR, values bit-identical to A_hat's; release with rig_csr_free.  flags:
 * RIG_FLAG_VALIDATE or 0.  Synchronises. */
RIG_API int rig_sparsify(const rig_csr_t *A, int scale_rows, uint32_t flags, rig_csr_t *out, rig_stream_t stream);
RIG_API int rig_csr_free(rig_csr_t *A, rig_stream_t stream);

/* Integer edge weights for a partitioner:
 * wgt[e] = ceil(alpha * w[e]) exactly (no rounding of the product), for
 * device arrays w [n] and wgt [n]; 1 <= alpha <= 2^53 (else RIG_ERR_INVALID).
 * An element with w < 0, w not finite, or a result beyond 2^62 gets -1.
 * Costs in (0, 1] (scaled rows) give weights in [1, alpha].  Asynchronous. */
RIG_API int rig_int_weights(const double *w, int64_t n, int64_t alpha, int64_t *wgt, rig_stream_t stream);

/* ---- f4: first stage of a multilevel partitioner ----- */

/* Coarse graph of one coarsening step: library-owned DEVICE arrays (one
 * allocation, stream-ordered), released with rig_coarse_free. */
typedef struct {
    int64_t n;        /* coarse vertices */
    int64_t nnz;      /* stored coarse edges (both directions) */
    int64_t *row_ptr; /* [n+1] */
    int32_t *col_idx; /* [nnz] coarse ids, ascending per row */
    int64_t *wgt;     /* [nnz] summed fine edge weights */
    int64_t *vwgt;    /* [n] summed fine vertex weights */
    int32_t *cmap;    /* [n_fine] coarse id of every fine vertex */
} rig_coarse_t;

/* Heavy-edge matching on a symmetric graph with int64 edge weights (the
 * METIS input of PAPER.md:609-613: rig_int_weights of G_RIP), all DEVICE
 * arrays: row_ptr [n+1], col [nnz] (no self loops), wgt [nnz]; match [n]
 * receives each vertex's partner or -1.  DESIGN.md R23: in each of `rounds`
 * rounds every unmatched vertex picks its heaviest unmatched neighbour (ties:
 * the smaller index) and mutual picks match.  Asynchronous. */
RIG_API int rig_hem_match(const int64_t *row_ptr, const int32_t *col, const int64_t *wgt, int64_t n,
                          int32_t rounds, int32_t *match, rig_stream_t stream);

/* One coarsening step (R24-R25): matched pairs and unmatched
 * vertices become coarse vertices numbered by their smaller member; coarse
 * edge weights sum the fine edges between the groups (the contracted edges
 * vanish); vwgt [n] (DEVICE, may be NULL: unit weights) are summed.  Integer
 * sums: exact.  Synchronises three times (coarse size, temporary size, coarse nnz). */
RIG_API int rig_coarsen(const int64_t *row_ptr, const int32_t *col, const int64_t *wgt, const int64_t *vwgt,
                        int64_t n, const int32_t *match, rig_coarse_t *out, rig_stream_t stream);
RIG_API int rig_coarse_free(rig_coarse_t *c, rig_stream_t stream);

/* ---- end-to-end from host memory --------------------------------------- */

/* Host-to-host convenience for the whole path: copies A (HOST CSR) and part
 * (HOST, may be NULL) to the device, builds G_RIP, computes the cutsize, and
 * copies the graph into the caller's HOST arrays out_host->row_ptr [nrows+1],
 * col_idx / w (capacity entries each) and diag ([nrows], only with
 * RIG_FLAG_DIAG).  If capacity is too small, returns RIG_ERR_INVALID with
 * out_host->nnz set to the required capacity.  *cut_host receives the cutsize
 * (NaN when part is NULL).  Pinned host memory gives full PCIe bandwidth. */
RIG_API int rig_build_host(const rig_csr_t *A_host, int scale_rows, double drop_tol, uint32_t flags,
                   const int32_t *part_host, int32_t K, rig_graph_t *out_host, int64_t capacity, double *cut_host,
                   rig_stream_t stream);

/* ---- diagnostics ------------------------------------------------------- */

/* Per-pass device timing.  While enabled, every pass of rig_build /
 * rig_plan_* / rig_cutsize records a CUDA event pair on the stream it runs
 * on.  rig_profile_read waits for those events and returns, per pass id in
 * [0, RIG_NPASS), the summed milliseconds and the number of occurrences since
 * the previous read (then clears them).  Pass names: rig_pass_name. */
/* The simple API (rig_build*, rig_build_host) keeps its internal work
 * buffers in a grow-only cache per calling thread, device and stream, reused
 * in stream order by the next build.  rig_trim releases the calling thread's
 * cache (stream-ordered frees). */
RIG_API int rig_trim(void);

#define RIG_NPASS 13
RIG_API int rig_profile_enable(int on);
RIG_API int rig_profile_read(double *ms, int64_t *count);
RIG_API const char *rig_pass_name(int pass);

RIG_API const char *rig_last_error(void);
/* Number of kernels this library has launched since it was loaded. */
RIG_API uint64_t rig_launch_count(void);
RIG_API const char *rig_version(void);
/* Numeric path taken by the calling thread's last a5-a6 pass (diagnostics,
 * bench labels): "merge" (every row on the k-way merge path, k_num_pair),
 * "rowwin" (no row on the merge path: k_row_win, look-back placement) or
 * "mixed" (merge rows + mid-row passes + placement copy); "" before any
 * build.  Thread-local; the pointer stays valid until the thread's next build. */
RIG_API const char *rig_last_path(void);
/* Measurement only (north star "L2 hit rate on the A^T
 * gathers"): runs a0-a4 on A (device CSR) and then k_gather_probe, the
 * numeric pass's gather loop (warp per row, ascending rows, every column k
 * of each row read from the CSC of A_hat) with no accumulation and no
 * writes, so ncu's L2/DRAM counters of that kernel are the gathers' own.
 * *checksum_host (may be NULL) receives a checksum of the gathered data.
 * Synchronises the stream. */
/* Measurement: the current device's stream-ordered memory pool (which holds
 * every library allocation: workspaces, library-owned graphs) -- bytes in use
 * now and the high-water mark since the last reset (reset = 1 clears it
 * after reading). */
RIG_API int rig_mem_stats(uint64_t *used_now, uint64_t *used_high, int reset);
RIG_API int rig_gather_probe(const rig_csr_t *A, int scale_rows, double *checksum_host, rig_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* RIG_H_ */

/*
 * include/msk.h -- C-ABI of libmsk, the B200-native (sm_100a, FP64) hot path
 * of Lot & Rieger's monolithic kernel-based multiscale method
 * (arXiv 2503.04914; /root/reference/PAPER.md cited as P:<line>).
 *
 * The problem: reconstruct f : Omega in R^d
 * -> R from samples f^{(l)} = f|_{X_l} on a hierarchy X_1, ..., X_L with
 * per-level support radii delta_l and a Wendland function phi_{d,k}.  The
 * coefficients alpha^{(l)} solve the block-lower-triangular system
 * T_L alpha = f (eq:bigt), i.e. for l = 1..L
 *     A_l alpha^{(l)} = f^{(l)} - sum_{k<l} B_{lk} alpha^{(k)}      (eq:mas P:287)
 * with A_l = (Phi_{delta_l}(x_i^{(l)} - x_j^{(l)})),
 *      B_{lk} = (Phi_{delta_k}(x_i^{(l)} - x_j^{(k)}))  (column level's delta,
 *      P:276, reading C-1),
 *      Phi_delta(x) = delta^{-d} phi_{d,k}(||x||_2 / delta)   (eq:kernelscaling P:67).
 * The library solves it as the paper does, through the split
 * D_L alpha = beta, T'_L beta = f (eq:split P:585-591): an L-sweep Jacobi
 * iteration on T'_L (Theorem jacobi, Algorithm 2) and
 * block-diagonal conjugate gradients on the SPD A_l (Theorem cg P:603-661,
 * Algorithm 1).  The approximant is
 *     f_L(x) = sum_l sum_n alpha_n^{(l)} Phi_{delta_l}(x - x_n^{(l)})  (eq:fapproximation P:295).
 *
 * Conventions common to every entry point
 * ---------------------------------------
 * - Every pointer to bulk data (points, f, alpha, x, s, v, y) may be HOST or
 *   DEVICE memory (on the context's device); the library detects which with
 *   cudaPointerGetAttributes and copies host data through its own stream.
 *   Small parameter arrays marked [host] must be host memory.
 * - Points are row-major n x d FP64 ("x-major": x, y[, z] of point 0, then
 *   point 1, ...).  Vectors are FP64 in the CALLER's point order.
 * - All calls are synchronous with respect to the host: on return every
 *   output is written and the context stream is idle.
 * - The caller owns every buffer it passes; the library deep-copies inputs
 *   it keeps (points, delta, q).  Handles are opaque, not thread-safe, and
 *   destroyed explicitly.  Distinct handles are independent.
 * - Every call returns an msk_status.  No C++ exception crosses the ABI.
 *   On error the outputs are unspecified and msk_last_error() (thread-local,
 *   valid until the next call on the same thread) names the cause.
 * - There is no CPU fallback: if no CUDA device is usable every call that
 *   needs one fails with MSK_ERR_CUDA.
 */
#ifndef MSK_H
#define MSK_H

#include <stdint.h>

#if defined(__GNUC__)
#define MSK_API __attribute__((visibility("default")))
#else
#define MSK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MSK_OK = 0,
    MSK_ERR_INVALID = 1,  /* bad argument: d not in {2,3}; L<1 or L>16; n[l]<1; delta<=0 or
                             non-finite; k not in {0,1,2}; duplicate points in a level
                             (q_l = 0 => A_l singular); tol not in (0,1); null pointer */
    MSK_ERR_NOMEM = 2,    /* device allocation failed */
    MSK_ERR_CUDA = 3,     /* CUDA runtime error (includes: no device) */
    MSK_ERR_NCCL = 4,     /* NCCL unavailable or an NCCL call failed (multi-GPU context) */
    MSK_ERR_NOCONV = 5,   /* CG reached max_iter; msk_last_error names level and residual */
    MSK_ERR_STATE = 6     /* call out of order (e.g. msk_solve before msk_assemble) */
} msk_status;

/* msk_hierarchy_create flags */
#define MSK_FLAG_NONE 0u
#define MSK_FLAG_DIST_ALL 1u /* distributed context: partition every level that has at least world
                                row chunks (default: the levels whose CG iteration a latency model
                                says gets faster split over the ranks -- bytes per iteration vs a
                                ~15 us floor plus the partitioned path's barriers, DESIGN.md §10;
                                on C3 the 1.25M- and 1e7-point levels; the others are solved
                                redundantly on every rank) */
#define MSK_FLAG_MATRIX_FREE 2u /* a3 matrix-free: A_l is never stored;
                                   every CG SpMV evaluates Phi on the fly over the level's cell list,
                                   visiting the columns in the stored CSR order, so alpha is
                                   BIT-IDENTICAL to the assembled solve (both schedules).
                                   msk_assemble(T > 0) and msk_cg_level are MSK_ERR_INVALID /
                                   MSK_ERR_STATE on such a hierarchy */

#define MSK_FLAG_OUTPUT_LOCAL 4u /* distributed context: msk_evaluate writes only the values of this
                                    rank's share of the (spatially sorted) evaluation points and skips
                                    their all-gather (perf runs that consume s_L rank-locally); alpha is
                                    complete either way.  No effect on one GPU or in the emulation */

/* msk_solve schedules */
#define MSK_SCHED_PRUNED 0u  /* Algorithm 2 with each inner solve t^{(l)} = A_l^{-1} beta^{(l)} done
                                once, when beta^{(l)} is final; beta bit-identical to LITERAL */
#define MSK_SCHED_LITERAL 1u /* Algorithm 2 as printed: L sweeps x (L-1) inner solves, then the
                                block-diagonal CG on all levels */

#define MSK_MAX_LEVELS 16

typedef struct msk_ctx msk_ctx;
typedef struct msk_hierarchy msk_hierarchy;

/* Per-solve report (msk_solve, nullable). */
typedef struct {
    int32_t L;
    int32_t jacobi_sweeps;                  /* L for LITERAL; 0 for PRUNED (lazy sweeps)        */
    int32_t cg_iters[MSK_MAX_LEVELS];       /* iterations of the solve that produced alpha_l    */
    int32_t inner_iters[MSK_MAX_LEVELS];    /* sum of inner Jacobi CG iterations per level      */
    double rel_res[MSK_MAX_LEVELS];         /* final recurrence ||r||/||b|| per level           */
    double nnz_cg;                          /* Wendland nonzeros read by CG SpMVs               */
    double nnz_gather;                      /* Wendland nonzeros evaluated by the B products    */
    double bytes_cg;                        /* algorithmic HBM bytes of the CG launches         */
    double t_cg_ms;                         /* device time of the CG launches (CUDA events)     */
    double t_gather_ms;                     /* device time of the B-product launches            */
    double t_total_ms;                      /* device time of the whole call                    */
    double t_cg_level_ms[MSK_MAX_LEVELS];   /* device time of the CG launch(es) per level       */
    double bytes_cg_level[MSK_MAX_LEVELS];  /* algorithmic bytes of those launches              */
    int32_t launches;                       /* kernels launched by the call                     */
    double kappa_est[MSK_MAX_LEVELS];       /* condition number of A_l estimated from the CG
                                               coefficients of the solve that produced alpha_l
                                               (extreme eigenvalues of the Lanczos tridiagonal,
                                               Sturm bisection on the host); 0 if no iteration */
} msk_solve_info;

/* Per-hierarchy facts (msk_hierarchy_info). */
typedef struct {
    int32_t d, L, k;
    int64_t n[MSK_MAX_LEVELS];
    int64_t nnz_A[MSK_MAX_LEVELS];          /* nnz of assembled A_l (0 before msk_assemble)     */
    int64_t ncells[MSK_MAX_LEVELS];         /* cells of level l's uniform grid                  */
    double delta[MSK_MAX_LEVELS];
    double q[MSK_MAX_LEVELS];               /* given, or 1/2 min pair distance        */
    double t_create_ms, t_assemble_ms;      /* device time of the last create / assemble        */
    int32_t launches_create, launches_assemble;
} msk_hierarchy_info;

/* Per-evaluation report (msk_evaluate_ex, nullable). */
typedef struct {
    double nnz;                             /* Wendland nonzeros evaluated                      */
    double t_sort_ms, t_eval_ms, t_total_ms;
    int32_t launches;
} msk_eval_info;

/* ---------------------------------------------------------------- context */

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t of
 * that device to enqueue on, or NULL to let the library create its own.
 * Distribution (north_star: levels partitioned across the GPUs of one box by
 * spatially sorted row blocks, halo exchange + reductions over NCCL):
 *   world_size == 1: rank 0, nccl_unique_id NULL (single GPU);
 *   world_size in 2..16, 0 <= rank < world_size, nccl_unique_id = the 128-byte
 *     ncclUniqueId from msk_nccl_unique_id on rank 0 (broadcast by the caller,
 *     e.g. with torch.distributed): one partition per rank over NCCL (the
 *     libnccl already loaded by the process is used; the environment variable
 *     MSK_NCCL_LIBRARY=<path> names another library exporting the same NCCL
 *     entry points instead -- the tests' in-process shim for ranks that are
 *     threads of one process, tests/nccl_shim);
 *   world_size in 2..16, rank == -1, nccl_unique_id NULL: single-process
 *     emulation -- all world_size partitions run on this device and exchange
 *     through device copies (used to test the partitioned path on one GPU).
 * Every rank must pass identical inputs to every later call. */
MSK_API msk_status msk_ctx_create(int device, void *cuda_stream, int rank, int world_size,
                          const void *nccl_unique_id, msk_ctx **out);
MSK_API void msk_ctx_destroy(msk_ctx *ctx);

/* out [host, 128 bytes]: a fresh ncclUniqueId (call on rank 0 only). */
MSK_API msk_status msk_nccl_unique_id(void *out);

/* Host-only row partition of a level of n points over `world` partitions:
 * bounds [host, world+1] with partition r owning spatial rows
 * [bounds[r], bounds[r+1]); boundaries fall on whole reduction chunks (DESIGN.md
 * §Multi-GPU), so per-chunk partial sums are identical for every world size. */
MSK_API msk_status msk_partition_rows(int64_t n, int world, int64_t *bounds);

/* Host-only halo plan of partition `rank` for one partitioned level:
 * rows [host, world+1] from msk_partition_rows; hlo/hhi [host, world]: the
 * column range [hlo[s], hhi[s]) referenced by partition s's rows (its own rows
 * included).  Outputs [host, world each]: partition `rank` sends its rows
 * [send_lo[s], send_hi[s]) of p to s and receives rows [recv_lo[s],
 * recv_hi[s]) from s before every SpMV (empty ranges have lo == hi; s == rank
 * is always empty). */
MSK_API msk_status msk_halo_plan(int world, int rank, const int64_t *rows, const int64_t *hlo,
                                 const int64_t *hhi, int64_t *send_lo, int64_t *send_hi, int64_t *recv_lo,
                                 int64_t *recv_hi);

/* ------------------------------------------------------------- hierarchy */

/* a0 + a1: ingest the hierarchy X_1..X_L (Assumption pointset P:87-114) and
 * build one uniform-grid cell list per level (cell side >= delta_l; points
 * stably sorted by (cell key, original index)).
 *   d            2 or 3.
 *   L            1..16 levels, coarse to fine.
 *   n [host]     L point counts, each in 1 .. 2^31 - 2 (an empty level has no
 *                interpolant: MSK_ERR_INVALID).
 *   points       L pointers, each n[l] x d row-major FP64 (host or device).
 *   delta [host] L support radii delta_l > 0 (eq:deltadef P:105-107: nu h_l).
 *   q [host]     L separation values (used only by thresholding), or
 *                NULL: computed exactly as 1/2 min distance: from
 *                the pattern pass when the closest pair lies within delta_l,
 *                else by a widening cell search (a one-point level: delta_l/2).
 *   wendland_k   0, 1 or 2: phi_{d,k} (reading C-3).
 *   flags        MSK_FLAG_NONE, or an OR of MSK_FLAG_DIST_ALL, MSK_FLAG_MATRIX_FREE,
 *                MSK_FLAG_OUTPUT_LOCAL.
 * Duplicate points within one level => MSK_ERR_INVALID. */
MSK_API msk_status msk_hierarchy_create(msk_ctx *ctx, int d, int L, const int64_t *n,
                                const double *const *points, const double *delta,
                                const double *q, int wendland_k, uint32_t flags,
                                msk_hierarchy **out);
MSK_API void msk_hierarchy_destroy(msk_hierarchy *h);

/* Facts about the hierarchy (sizes, nnz, timings of the last create/assemble). */
MSK_API msk_status msk_hierarchy_info_get(const msk_hierarchy *h, msk_hierarchy_info *info);

/* a2 (+ a6): assemble the level matrices A_l in CSR (pattern r^2 <
 * delta_l^2, strict, bit-exact; values Phi_{delta_l}).  Any (re-)assembly resets
 * the solve state (msk_evaluate needs a new msk_solve); a failed one leaves the
 * hierarchy unassembled (msk_solve => MSK_ERR_STATE).
 *   T <= 0: exact mode; the B_{kl} stay matrix-free and msk_solve runs the
 *           exact Jacobi of Algorithm 2 (inner CG solves).
 *   T > 0:  additionally build the thresholded factor M~(T) (eq:perturbedmatrix
 *           P:846-861): X~_{kl}[j,i] = chi_i^{(l)}(x_j^{(k)}) kept iff
 *           ||x_j^{(k)} - x_i^{(l)}||^2 < (T q_l)^2 (coarse level's q,
 *           strict; reading C-5), with the Lagrange coefficients
 *           A_l^{-1} e_i (eq:chi P:373-377) solved by CG to relative residual
 *           lagrange_tol in (0,1).  msk_solve then runs the Jacobi sweep with
 *           the stored factor (eq:perturbed_split P:865-869).  Cost grows
 *           like sum_l N(l)^2 (one solve per coarse column).  In a
 *           distributed context the factor build is replicated on every rank
 *           (the partitioned column levels keep their full A_l for it); the
 *           Jacobi runs on the owned rows of the partitioned levels and their
 *           CG is the partitioned CG (bit-identical to one GPU).
 * Non-convergence of a Lagrange solve => MSK_ERR_NOCONV. */
MSK_API msk_status msk_assemble(msk_hierarchy *h, double T, double lagrange_tol);

/* The T sweep of one factor build: every stored entry keeps
 * the smallest integer t with ||x_j - x_i||^2 < (t q_l)^2 (reading C-5 recipe),
 * so a factor built at T also serves every integer T' in [1, floor(T)] (at
 * most 24): msk_set_threshold(h, T') makes msk_solve, msk_m_norm_ex and
 * msk_export_factor use exactly the entries a fresh msk_assemble(T') would
 * store, with the same values (the Lagrange functions do not depend on T) and
 * in the same order -- bit-identical results.  T' == the build's T restores all
 * entries.  MSK_ERR_STATE without a factor, MSK_ERR_INVALID for another T'. */
MSK_API msk_status msk_set_threshold(msk_hierarchy *h, double T);

/* msk_assemble with local-patch Lagrange functions for
 * the coarse levels with more than patch_min_n points (patch_R > 0): the
 * coefficients of chi_i^(l) solve A_l restricted to the patch
 * {x_h : ||x_h - x_i^(l)|| < patch_R q_l} (zero outside; Lagrange functions
 * decay exponentially away from x_i, Lemma lagrangedecay), one CTA
 * and one shared-memory system per column, so the build costs O(N(l)) instead
 * of O(N(l)^2).  An approximation of the exact factor: the error at the stored
 * entries falls with patch_R - T.  patch_R <= 0: exactly
 * msk_assemble.  A patch whose workspace does not fit in one CTA's shared
 * memory runs from a per-CTA slice of a global workspace (slower: the vectors
 * then live in L2); a patch workspace above 1 GiB => MSK_ERR_INVALID (reduce
 * patch_R).  On any error the hierarchy is left unassembled (msk_solve =>
 * MSK_ERR_STATE until the next successful msk_assemble). */
MSK_API msk_status msk_assemble_ex(msk_hierarchy *h, double T, double lagrange_tol, double patch_R,
                           int64_t patch_min_n);

/* a3-a5, a8: solve T_L alpha = f (eq:bigt) through eq:split.
 *   f      L pointers to f^{(l)} (n[l] FP64, caller order, host or device).
 *   tol    relative CG tolerance in (0,1): stop when ||r||_2 <= tol ||b||_2
 *          per level (reading C-9); inner Jacobi solves use tol/10 (C-10).
 *   max_iter  CG iteration cap per solve (>= 1).
 *   schedule  MSK_SCHED_PRUNED or MSK_SCHED_LITERAL.
 *   alpha  L pointers to caller-owned outputs alpha^{(l)} (n[l] FP64, caller
 *          order, host or device).
 *   info   nullable report.
 * Requires msk_assemble.  A zero right-hand side gives alpha = 0 after 0
 * iterations.  Non-convergence => MSK_ERR_NOCONV ("level l: rel. residual r
 * after k iterations"). */
MSK_API msk_status msk_solve(msk_hierarchy *h, const double *const *f, double tol, int32_t max_iter,
                     uint32_t schedule, double *const *alpha, msk_solve_info *info);

/* a9: s_j = f_L(x_j) = sum_l sum_n alpha_n^{(l)} Phi_{delta_l}(x_j - x_n^{(l)})
 * (eq:fapproximation P:293-296) for m points x (m x d row-major, host or
 * device), using the alpha of the last successful msk_solve.  s: m FP64
 * (host or device).  m = 0 is allowed.  MSK_ERR_STATE before msk_solve. */
MSK_API msk_status msk_evaluate(msk_hierarchy *h, int64_t m, const double *x, double *s);
MSK_API msk_status msk_evaluate_ex(msk_hierarchy *h, int64_t m, const double *x, double *s,
                           msk_eval_info *info);

/* ----------------------------------- truncation diagnostics (§8(f) NEXT-2) */

/* ||M_L||_2 (Figure 1; M = id - T'_L, lower blocks -X_kl =
 * -B_kl A_l^{-1}, reading C-7) by power iteration on M^T M with M and M^T
 * applied matrix-free (A_l^{-1}: CG at cg_tol; B_kl, B_kl^T: kernel sums).
 * Stops when the estimate changes by <= rel_tol relative, or after max_iter
 * iterations (*iters reports the count; nullable).  The estimate increases
 * towards ||M||_2 from below.  Requires msk_assemble (assembled A_l, one GPU);
 * L = 1 gives 0. */
MSK_API msk_status msk_m_norm(msk_hierarchy *h, int32_t max_iter, double rel_tol, double cg_tol, double *norm,
                      int32_t *iters);
/* which = 0: ||M_L||_2 (as msk_m_norm); which = 2: ||M~_L(T)||_2 of the stored
 * factor alone (the max(||M||, ||M~||) of the corrected Lemma pert1 bound,
 * DESIGN.md reading C-22); which = 1: ||M_L - M~_L(T)||_2 with the
 * stored thresholded factor of the last msk_assemble(T > 0) (Figure 2,
 * M - M~ = -(X - X~), X~ applied from the stored CSR and its
 * transpose; MSK_ERR_STATE without a factor).  The transposed product sums a
 * column's entries in the order of an atomic fill: reproducible to rounding,
 * not bit for bit (a diagnostic, not the solve path). */
MSK_API msk_status msk_m_norm_ex(msk_hierarchy *h, int32_t which, int32_t max_iter, double rel_tol,
                         double cg_tol, double *norm, int32_t *iters);

/* ------------------------------------------- multi-RHS */

/* Solve the multiscale system (eq:mas P:284-290, PRUNED schedule as msk_solve)
 * for nrhs right-hand sides at once.  f[l]: n[l] x nrhs row-major (f[l][i*nrhs
 * + r] = sample of function r at x_i^(l)), [host] or [dev]; alpha[l]: n[l] x
 * nrhs, caller-owned, same layout.  Columns are processed in groups of 4 (the
 * tail 2 or 4, zero-padded): every CSR piece and every kernel evaluation of the
 * B products serves the whole group, so the HBM traffic per right-hand side
 * falls.  Every column is bit-identical to msk_solve with that column alone.
 * iters: nullable, [L * nrhs] (iters[l*nrhs + r]).  t_ms: nullable, device
 * time.  Requirements: exact mode (msk_assemble with T <= 0), assembled A_l (not
 * MSK_FLAG_MATRIX_FREE), one GPU (world 1), else MSK_ERR_INVALID.  Keeps the
 * coefficients for msk_evaluate_multi.  MSK_ERR_NOCONV names level and rhs. */
MSK_API msk_status msk_solve_multi(msk_hierarchy *h, int32_t nrhs, const double *const *f, double tol,
                           int32_t max_iter, double *const *alpha, int32_t *iters, double *t_ms);

/* s[i*nrhs + r] = f_L of right-hand side r at x_i (eq:fapproximation P:293-296)
 * from the last msk_solve_multi; x: m x d, s: m x nrhs ([host] or [dev]).
 * MSK_ERR_STATE before msk_solve_multi. */
MSK_API msk_status msk_evaluate_multi(msk_hierarchy *h, int64_t m, const double *x, double *s);

/* ----------------------------------------- row-level entry points (tests) */

/* Sparsity pattern (and optionally values) of block B_{row_level,col_level}
 * (row_level >= col_level; row_level == col_level gives A_l), in CALLER
 * indices with ascending columns.  row_ptr [host]: n[row_level]+1 int64,
 * always written.  col [host] / val [host]: nnz entries, or NULL to query
 * nnz (= row_ptr[n]) first.  0-based levels.  Pattern r^2 < delta_col^2 is
 * bit-exact (reading C-4). */
MSK_API msk_status msk_export_block(msk_hierarchy *h, int row_level, int col_level, int64_t *row_ptr,
                            int32_t *col, double *val);

/* Entries of the thresholded factor block X~_{row_level,col_level}(T)
 * (eq:perturbedmatrix P:846-861; 0 <= col_level < row_level) built by the last
 * msk_assemble(T > 0), in CALLER indices with ascending columns: row_ptr
 * [host] n[row_level]+1, col / val [host] nnz or NULL (query), T_out
 * (nullable) the T it was built for.  MSK_ERR_STATE without a factor. */
MSK_API msk_status msk_export_factor(msk_hierarchy *h, int row_level, int col_level, int64_t *row_ptr,
                                     int32_t *col, double *val, double *T_out);

/* Cell list of level l [host outputs]: perm (n[l] int32, sorted position ->
 * caller index), cell_start (ncells+1 int32), cell_key (n[l] int64, key of
 * each sorted point), origin lo (d doubles), cell side, grid dims (d int64).
 * Any output may be NULL. */
MSK_API msk_status msk_export_cells(msk_hierarchy *h, int level, int32_t *perm, int32_t *cell_start,
                            int64_t *cell_key, double *lo, double *cell, int64_t *dims);

/* The exact grid of level l (a1; reading C-26): origin lo [host] d doubles,
 * inv_cell [host] d doubles -- the FP64 factors of the key map per axis, so a
 * point's cell coordinate along axis a is floor((x_a - lo_a) * inv_cell[a])
 * with one rounded subtraction and one rounded multiplication (no FMA, reading
 * C-4), clamped to [0, dims_a - 1]; the last axis has cells zf times thinner
 * (inv_cell[d-1] = zf inv_cell[0], zf a power of two) -- and dims [host] d
 * int64.  Any output may be NULL.  MSK_ERR_INVALID for a bad level. */
MSK_API msk_status msk_export_grid(msk_hierarchy *h, int level, double *lo, double *inv_cell, int64_t *dims);

/* y = B_{row_level,col_level} v (a3).  row_level == col_level uses the
 * assembled A_l (CSR SpMV kernel; requires msk_assemble), row_level >
 * col_level the matrix-free kernel.  v: n[col_level], y: n[row_level], caller
 * order, host or device.  t_ms (nullable): device time of the kernel launch. */
MSK_API msk_status msk_apply_block(msk_hierarchy *h, int row_level, int col_level, const double *v,
                           double *y, double *t_ms);

/* a4 on one level: x = A_l^{-1} b by the library's CG (x0 = 0), caller order,
 * host or device.  iters / rel_res / t_ms nullable. */
MSK_API msk_status msk_cg_level(msk_hierarchy *h, int level, const double *b, double *x, double tol,
                        int32_t max_iter, int32_t *iters, double *rel_res, double *t_ms);

/* Thread-local description of the last error ("" if none). */
MSK_API const char *msk_last_error(void);

/* Library version string. */
MSK_API const char *msk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MSK_H */

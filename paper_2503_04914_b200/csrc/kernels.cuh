// kernels.cuh -- host-side launchers of the libmsk CUDA kernels.
#pragma once
#include "common.cuh"

namespace msk {

// ---- scan.cu
void exclusive_scan_i32(const int32_t *in, int64_t n, int32_t *out, cudaStream_t st, int *launches);
void exclusive_scan_i64(const int32_t *in, int64_t n, int64_t *out, cudaStream_t st, int *launches);

// ---- celllist.cu  (a1)
// Build the cell list of one point set: keys, counting sort by key with ties
// broken by original index (if stable), SoA coordinates in sorted order.
//   pts_rm   device, n x d row-major (caller order)
//   perm     out, n: sorted position -> caller index
//   xs       out, d arrays of n (SoA, sorted order)
//   cell_start out, ncells + 1
//   keys     out (nullable), n: key of each sorted point
struct CellListOut {
    int32_t *perm;
    double *xs[3];
    int32_t *cell_start;
    int64_t *keys;
};
void build_cell_list(int d, int64_t n, const double *pts_rm, const Grid &g, bool stable,
                     const CellListOut &out, cudaStream_t st, int *launches);

// ---- assemble.cu  (a2)
// Row counts of A_l (or of a rectangular block rows x cols when rows != cols)
// and the minimum off-diagonal squared distance / duplicate flag.
void count_pattern(int d, const LevelView &rows, const LevelView &cols, bool same, int32_t *cnt,
                   unsigned long long *min_r2_bits, cudaStream_t st, int *launches,
                   int64_t row0 = 0);
// Fill CSR columns (column spatial index) and values Phi_{delta_col}.
void fill_pattern(int d, int k, const LevelView &rows, const LevelView &cols,
                  const int64_t *row_ptr, int32_t *col, double *val, cudaStream_t st,
                  int *launches);

// ---- gather.cu  (a3 matrix-free, a5 B products, a9 evaluation)
// out[i] = (base ? base[base_perm ? base_perm[i] : i] : 0)
//          + sign * sum_{l in levels} scale_l sum_n phi(r/delta_l) coef_l[n]
// for target points tx (SoA, nt).  If out_perm: writes out[out_perm[i]].
// hits (nullable): adds the number of (target, source) pairs inside support.
struct GatherArgs {
    int d, k;
    int64_t nt;
    const double *tx[3];
    int nlev;
    LevelView lev[kMaxLevels];
    const double *base;
    const int32_t *base_perm;
    double sign;
    double *out;
    const int32_t *out_perm;
    unsigned long long *hits;
};
void gather(const GatherArgs &a, cudaStream_t st, int *launches);
// true unless MSK_GATHER_WARP is set: the per-thread matrix-free kernels (default)
// instead of the warp-cooperative ones (wscan.cuh)
bool gather_v1();
// multi-RHS kernel sums (msk_solve_multi / msk_evaluate_multi): R coefficient
// columns per source level (spatial rows, row stride ldc); per column the same
// arithmetic, in the same order, as gather() -- bit-identical to R single runs.
struct GatherMArgs {
    int d, k, R;
    int64_t nt;
    const double *tx[3];
    int nlev;
    LevelView lev[kMaxLevels];   // cells, .rec (coordinates), .frec
    const double *coef[kMaxLevels];
    int64_t ldc;
    const double *base;          // optional: base[(perm ? perm[i] : i) * ldb + bcol0 + r], r < bcols
    const int32_t *base_perm;
    int64_t ldb;
    int bcol0, bcols;
    double sign;
    double *out;                 // out[(perm ? perm[i] : i) * ldo + ocol0 + r], r < wcols
    const int32_t *out_perm;
    int64_t ldo;
    int ocol0, wcols;
    unsigned long long *hits;
};
void gather_multi(const GatherMArgs &a, cudaStream_t st, int *launches);
// transposed B products (msk_m_norm): for target points x_i of level l,
// out_i = sum_{k in srcs} sum_{j: r < delta_l} delta_l^-d phi(r / delta_l) y_k[j]
// = sum_k (B_kl^T y_k)_i, the sources enumerated in level k's grid with a reach
// of `reach[k]` cells (delta_l spans several cells of a finer level).
struct GatherTArgs {
    int d, k;
    int64_t nt;
    const double *tx[3];
    double delta2, inv_delta, scale;   // of the TARGET level l (column level of B_kl)
    int nsrc;
    LevelView src[kMaxLevels];         // SoA coordinates + cells of level k
    const double *y[kMaxLevels];       // spatial order
    int reach[kMaxLevels];
    double *out;                       // spatial order of the targets
};
void gather_t(const GatherTArgs &a, cudaStream_t st, int *launches);
// deterministic dot product of n doubles (one block-reduction tree; host result)
double dev_dot(const double *a, const double *b, int64_t n, double *scratch, cudaStream_t st);
void dev_scale(double *v, double s, int64_t n, cudaStream_t st);
// rec[i] = (x, y, z, coef) (2-D: (x, y, coef, 0)) from SoA xs (d arrays of n)
void pack_records(int64_t n, int d, const double *xs, const double *coef, double4 *rec,
                  cudaStream_t st, int *launches);
// frec[i] = float(x - lo) per axis (prefilter coordinates)
void pack_frecords(int64_t n, int d, const double *xs, const double *lo, float4 *frec, cudaStream_t st,
                   int *launches);
float prefilter_threshold(double delta, double M, int d);

// ---- cg.cu  (a4 / a8 block-diagonal CG, fused SpMV + reductions)
struct CGLevelArgs {
    int64_t n;
    int64_t nnz;
    const int64_t *row_ptr;
    const int32_t *col;
    const double *val;
    const double *b;          // spatial order
    const double *b_src;      // if set: b[i] = b_src[b_perm[i]] gathered at init (caller order)
    const int32_t *b_perm;
    double *x, *r, *p, *q;    // spatial order, n each
    double *x_out;            // optional: x_out[x_perm[i]] = x[i] at the end
    const int32_t *x_perm;
    double tol2;              // tol^2
    int max_iter;
    int nblocks;              // CTAs for this level (filled by launcher)
    int block_begin;
    int chunk_tiles;          // tiles per reduction chunk (filled by launcher, function of n)
    double *partials;         // 3 * nblocks doubles (filled by launcher)
    unsigned long long *barrier;
    int *out_iters;           // device
    double *out_rr;           // device: final rr, bb
    int *out_status;          // device: 0 ok, 1 noconv
    unsigned long long *dbg;  // optional: 6 phase times (ns) of CTA 0 (spmv, bar1, r, bar2, -, -)
    double *coef;             // optional: CG scalars (alpha_k, beta_k) of iterations k < coef_cap
    int coef_cap;             //   (Lanczos tridiagonal -> kappa estimate, msk_solve_info.kappa_est)
    // optional 16-bit columns (cg.cu col16_build): entry -> (window << 14 | offset), the
    // column = cbase[chunk].{x,y,z,w}[window] + offset; k_cg streams these instead of col
    const uint16_t *col16;
    const int4 *cbase;        // per reduction chunk (chunk_tiles * 256 rows): 4 window bases
    const int4 *clen;         //   and the extents the chunk's columns span (L2 prefetch of r), or null
};
// ---- multi-RHS CG (msk_solve_multi; cg.cu): one level, R right-hand sides
// with their own scalars; per column the arithmetic of k_cg (bit-identical to
// R single solves).  Vectors are [n][R] row-major in spatial order.
struct CGRArgs {
    int64_t n, nnz;
    const int64_t *row_ptr;
    const int32_t *col;
    const double *val;
    const double *b;             // spatial [n][R], or null: b_src (caller order) below
    const double *b_src;         // b_src[b_perm[i] * ldb + col0 + r], r < nvalid (else 0)
    const int32_t *b_perm;
    int64_t ldb;
    int col0, nvalid;
    double *x;                   // spatial, row stride ldx
    int64_t ldx;
    double *r, *p, *q;           // spatial [n][R]
    double *x_out;               // optional: x_out[x_perm[i] * ldo + col0 + r] = x[i][r], r < nvalid
    const int32_t *x_perm;
    int64_t ldo;
    double tol2;
    int max_iter;
    int *out_iters;              // R
    double *out_rr;              // 2R: final rr, bb per column
    int *out_status;             // R
};
void cg_multi(const CGRArgs &a, int R, cudaStream_t st, int *launches);

// ---- distributed CG (partitioned levels; cg.cu)
constexpr int kMaxParts = 16;
struct DistCGScalars {
    double bb, rr, pq, alpha, beta;
    int it, active, status, pad;
};
struct DistCGArgs {
    CGLevelArgs L;             // n, tol2, max_iter, chunk_tiles, vectors (full length, owned rows
                               // valid), row_ptr indexed by GLOBAL row (local storage - lo), col/val local
    int64_t c0, c1, nchunks;   // owned chunks [c0, c1) of nchunks
    double *part_send;         // indexed by chunk (the owned chunks are written)
    const double *part_recv;   // gw == 0: nchunks partials by chunk; gw > 0: the all-gathered
                               // blocks, chunk c of rank r at r * gcmax + c - gc0[r]
    DistCGScalars *sc;
    int gw;
    int64_t gcmax;
    int64_t gc0[kMaxParts + 1];
};
struct DistPtrs {
    const double *p[kMaxParts];
};
int cg_chunk_tiles(int64_t n);
void dcg_init(const DistCGArgs &a, cudaStream_t st);
void dcg_spmv(const DistCGArgs &a, cudaStream_t st);
void dcg_rupd(const DistCGArgs &a, cudaStream_t st);
void dcg_xfin(const DistCGArgs &a, cudaStream_t st);
// matrix-free pass 1 of the CG iteration (MSK_FLAG_MATRIX_FREE): w = A r with
// A's entries evaluated on the fly over V's cell list, then the k_cg epilogue
void dcg_mf_spmv(const DistCGArgs &a, const LevelView &v, int d, int k, cudaStream_t st);
// [lo, hi] of the column indices hit by rows (exact test): halo of a matrix-free partition
void hit_range(int d, const LevelView &rows, const LevelView &cols, unsigned long long *mm, cudaStream_t st);
double min_r2_reach(int d, const LevelView &v, int m, cudaStream_t st);
void dcg_scalar(const DistCGArgs &a, int mode, cudaStream_t st);
void sum_arrays(int W, const DistPtrs &srcs, double *dst, int64_t n, cudaStream_t st);
void col_minmax(int64_t nnz, const int32_t *col, unsigned long long *mm, cudaStream_t st);

// Run independent CGs on several levels in one cooperative launch.
// CSR arrays must be 16-byte aligned and padded: row_ptr n+3 entries,
// col nnz+4, val nnz+2 (bulk copies round their extents to 16 bytes).
int cg_max_resident_blocks();
// 16-bit column encoding of a level's CSR per reduction chunk (k_cg's 10 B/nnz
// stream): returns false (and writes nothing usable) when some chunk's columns
// need more than 4 windows of 2^14 indices
bool col16_build(int64_t n, const int64_t *row_ptr, const int32_t *col, uint16_t *col16, int4 *cbase,
                 int4 *clen, cudaStream_t st);

// ---- partitioned CG over peer memory (cg.cu k_pcg): the
// whole CG of a row-partitioned level in ONE persistent launch per rank.
// Chunk partials and halo rows of r are STORED into the peers' buffers (NVLink
// peer pointers, IPC-mapped; or, in the single-GPU emulation, the other
// partitions' buffers), and the ranks meet in a device-side barrier on
// counters in each rank's memory (release/acquire at system scope) -- no host
// round trip, no NCCL call, no launch per phase.  Same chunk partials and the
// same fixed-order sums as k_cg => bit-identical to the single-GPU solve.
struct PeerRank {
    double *x, *r, *p, *q;      // this rank's vectors (global row index space; owned rows, r also its halo)
    double *part;               // 3 * nchunks chunk partials (every rank pushes its chunks into every copy)
    double *alpha;              // full-length result (every rank pushes its owned x)
    unsigned long long *xcnt;   // cross-rank arrival counter (every rank adds 1 per barrier; never reset)
    unsigned long long *nbar;   // barriers completed by earlier launches (this rank's copy)
    unsigned long long *gbar;   // this rank's group-barrier counter (own CTAs; zeroed before the launch)
    const int64_t *row_ptr;     // owned rows' CSR, indexed by global row
    const int32_t *col;
    const double *val;
    int64_t c0, c1;             // owned chunks [c0, c1)
    int64_t hlo, hhi;           // rows this rank's SpMV reads (owned rows and halo)
    int64_t slo, shi;           // owned rows some peer reads (the union of the send ranges)
};
struct PeerCGArgs {
    CGLevelArgs L;              // n, nnz, b / b_src / b_perm, tol2, max_iter, chunk_tiles, out_*, coef
    int64_t nchunks;
    int W;                      // ranks
    int rank;                   // this process's rank, or -1: emulation (all ranks in one launch,
                                // rank = blockIdx.x / nb)
    int nb;                     // CTAs per rank
    PeerRank R[kMaxParts];      // every rank's buffers as addressed from this process
};
// variant (piece capacity) and co-resident CTAs of k_pcg for a level
int pcg_resident_blocks(double nnz, double rows);
void pcg_launch(const PeerCGArgs &a, cudaStream_t st);
void cg_batched(CGLevelArgs *levels, int nlev, cudaStream_t st, int *launches);
void spmv_csr(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *val,
              const double *v, double *y, cudaStream_t st, int *launches);

// ---- thresh.cu  (a6 / a7 thresholded factor)
constexpr int kMaxTBucket = 24;
struct ThreshPatternArgs {
    int d;
    int64_t nt;                     // target rows (points of one finer level, spatial order)
    const double *tx[3];
    int nlev;                       // coarse levels 0..nlev-1
    LevelView lev[kMaxLevels];
    double R2[kMaxLevels];          // (T q_l)^2
    int reach[kMaxLevels];          // cells per axis covering T q_l
    int64_t col_off[kMaxLevels];    // global column offset of level l
    const int64_t *row_ptr;         // fill: row pointers of these rows
    int32_t *cnt;                   // count: output
    int32_t *col;                   // fill: output (global columns)
    // fill: distance bucket of each entry, the smallest integer t in 1..nb with
    // r^2 < (t q_l)^2 (tq2[l][t-1], same rounding recipe as R2), else nb + 1
    uint8_t *bucket;
    int nb;
    double tq2[kMaxLevels][kMaxTBucket];
};
void thresh_count(const ThreshPatternArgs &a, cudaStream_t st, int *launches);
void thresh_fill(const ThreshPatternArgs &a, cudaStream_t st, int *launches);
// transpose index of the factor pattern: for each coarse column c (global),
// positions cpos[cptr[c]..cptr[c+1]) of its entries, their rows crow and ccol = c
void thresh_csc(int64_t nrows_total, int64_t row0, int64_t nnz, int64_t ncols, const int64_t *row_ptr,
                const int32_t *col, int64_t *cptr, int64_t *cpos, int32_t *crow, int32_t *ccol,
                cudaStream_t st, int *launches);
struct CGMultiArgs {
    int64_t n, ncols;               // A_l size; columns to solve (= n)
    const int64_t *row_ptr;
    const int32_t *col;
    const double *val;
    double tol2;
    int max_iter;
    int64_t batch0, nbatches;       // batches (of 32 columns) of this launch start at batch0
    double *ws;                     // per CTA: X, R, P, Q (n x 32 each, row-major)
    int *fail;                      // device counter of batches that hit max_iter
    int *max_iters;                 // device max of iterations
};
void thresh_cg_multi(const CGMultiArgs &a, int nblocks, cudaStream_t st, int *launches);
struct ThreshValueArgs {
    int d, k, L;
    int64_t pos0, pos1;             // CSC positions of this round's columns
    const int64_t *cpos;
    const int32_t *crow;
    const int64_t *cptr;            // CSC column starts (global coarse columns)
    int64_t c_lo, c_hi;             // global columns of this round: positions [cptr[c_lo], cptr[c_hi])
    int32_t col_off;                // global column offset of the coarse level
    int64_t first_col;              // first (level-local) column of this round
    int64_t lev_off[kMaxLevels + 1];
    const double *lev_xs[kMaxLevels];
    int64_t lev_n[kMaxLevels];
    LevelView Lv;                   // the coarse level
    const double *ws;               // the round's CG workspaces (X first)
    double *val;                    // factor values (output)
};
void thresh_values(const ThreshValueArgs &a, cudaStream_t st, int *launches);
// Local-patch Lagrange functions: for coarse column i of level
// l, c = A_P^{-1} e_i on the patch P = {h : |x_h - x_i| < rho} (A_l restricted
// to P), chi~_i = sum_{h in P} c_h Phi_l(. - x_h), written at the column's
// stored entries.  One CTA per column, patch system in shared memory.
struct PatchArgs {
    int d, k, L;
    int64_t ncols;                  // columns of level l processed (0 .. ncols-1)
    double rho2;                    // patch radius^2 (no-FMA test, reading C-4 recipe)
    int reach;                      // cells of level l's grid spanned by rho
    int pmax, nnzmax;               // shared-memory capacity (points, local entries)
    int nq;                         // patch columns of the box, (2 reach + 1)^(d-1)
    LevelView Lv;                   // the coarse level (cells, SoA coordinates)
    const int64_t *row_ptr;         // A_l (spatial)
    const int32_t *col;
    const double *val;
    double tol2;                    // lagrange_tol^2 (||e_i|| = 1)
    int max_iter;
    // stored entries (CSC over the global coarse columns)
    const int64_t *cptr;            // indexed by global column col_off + i
    const int64_t *cpos;
    const int32_t *crow;
    int64_t col_off;
    int64_t lev_off[kMaxLevels + 1];
    const double *lev_xs[kMaxLevels];
    int64_t lev_n[kMaxLevels];
    double *val_out;                // factor values
    int *fail;                      // [0] CG failures, [1] patch overflows, [2] max iterations, [3] max patch
};
// max patch size over the columns (count pass, exact test) into pmax_out[0] and the max
// sum of the members' row lengths of A_l (rowcnt; bounds the patch-local entries) into [1]
void patch_count(const PatchArgs &a, const int32_t *rowcnt, int *pmax_out, cudaStream_t st);
void patch_lagrange(const PatchArgs &a, size_t smem, cudaStream_t st, int *launches);
size_t patch_smem_bytes(int pmax, int nnzmax, int nq);
// out[g] = base[g] - sum_p val[p] v[col[p]] for global rows g in [r0, r1)
// bucket/tmax (optional): only entries with bucket <= tmax take part (the T sweep)
void csc_spmv_add(int64_t ncols, const int64_t *cptr, const int64_t *cpos, const int32_t *crow, const double *val,
                  const double *u, double *out, cudaStream_t st, const uint8_t *bucket = nullptr, int tmax = 255);
void thresh_residual(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col, const double *val,
                     const double *base, const double *v, double *out, cudaStream_t st, int *launches,
                     const uint8_t *bucket = nullptr, int tmax = 255);
// number of entries with bucket <= tmax (device count, host result)
int64_t bucket_count(const uint8_t *bucket, int64_t nnz, int tmax, cudaStream_t st);

// ---- misc.cu
// mm[0..2] = ordered keys of per-axis minima (init ~0), mm[3..5] maxima (init 0)
void minmax_points(int64_t n, int d, const double *pts, unsigned long long *mm, cudaStream_t st,
                   int *launches);
double ord_key_to_double(unsigned long long k);
int64_t sum_i32(const int32_t *v, int64_t n, cudaStream_t st);
void permute_gather(int64_t n, const double *src, const int32_t *perm, double *dst,
                    cudaStream_t st, int *launches);  // dst[i] = src[perm[i]]
void permute_scatter(int64_t n, const double *src, const int32_t *perm, double *dst,
                     cudaStream_t st, int *launches);  // dst[perm[i]] = src[i]

}  // namespace msk

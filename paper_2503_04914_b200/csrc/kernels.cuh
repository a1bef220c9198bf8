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
                   unsigned long long *min_r2_bits, cudaStream_t st, int *launches);
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
};
// Run independent CGs on several levels in one cooperative launch.
// CSR arrays must be 16-byte aligned and padded: row_ptr n+3 entries,
// col nnz+4, val nnz+2 (bulk copies round their extents to 16 bytes).
int cg_max_resident_blocks();
void cg_batched(CGLevelArgs *levels, int nlev, cudaStream_t st, int *launches);
void spmv_csr(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *val,
              const double *v, double *y, cudaStream_t st, int *launches);

// ---- misc.cu
// mm[0..2] = ordered keys of per-axis minima (init ~0), mm[3..5] maxima (init 0)
void minmax_points(int64_t n, int d, const double *pts, unsigned long long *mm, cudaStream_t st,
                   int *launches);
double ord_key_to_double(unsigned long long k);
void permute_gather(int64_t n, const double *src, const int32_t *perm, double *dst,
                    cudaStream_t st, int *launches);  // dst[i] = src[perm[i]]
void permute_scatter(int64_t n, const double *src, const int32_t *perm, double *dst,
                     cudaStream_t st, int *launches);  // dst[perm[i]] = src[i]

}  // namespace msk

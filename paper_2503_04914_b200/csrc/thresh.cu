// thresh.cu -- a6/a7: the thresholded lower factor M~(T) (eq:perturbedmatrix
// P:846-861) and its Jacobi sweep (eq:perturbed_split P:865-869).
//
// X~_{kl}[j,i] = chi_i^{(l)}(x_j^{(k)}) if ||x_j^{(k)} - x_i^{(l)}|| < T q_l, else 0
// (coarse column level's q, strict, reading C-5), where the Lagrange function
// chi_i^{(l)} = sum_h c_i[h] Phi_{delta_l}(. - x_h^{(l)}) has c_i = A_l^{-1} e_i
// (eq:chi P:373-377).  Build (column approach):
//   1. pattern (bit-exact geometric predicate) of all blocks, one CSR whose
//      rows are the points of levels >= 2 and whose columns are global
//      (level-major, spatial) indices of the coarse levels;
//   2. its transpose index (positions grouped by column);
//   3. for each coarse level, batches of 32 Lagrange columns solved by a
//      multi-RHS CG, one CTA per batch (SpMM with lane = right-hand side),
//      many batches concurrently;
//   4. each stored entry evaluated as chi_i(x_j) from the batch's coefficients.
// The Jacobi sweep then is a CSR SpMV per target level (no inner solves).
#include <vector>

#include <stdlib.h>

#include "kernels.cuh"
#include "neighbors.cuh"

namespace msk {

namespace {
constexpr int NT = 256;
constexpr int NWM = NT / 32;
#ifndef MSK_PATCH_EC
#define MSK_PATCH_EC 6  // CSR entries per row kept in registers by the patch CG
#endif
#ifndef MSK_MERGE_PF
#define MSK_MERGE_PF 12  // columns per row loaded up front by the patch-local CSR merge
#endif
#ifndef MSK_PATCH_REGC
#define MSK_PATCH_REGC 1
#endif

template <int D>
__global__ void __launch_bounds__(NT) k_tcount(ThreshPatternArgs a) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= a.nt) return;
    double x[3];
#pragma unroll
    for (int t = 0; t < D; ++t) x[t] = a.tx[t][i];
    int c = 0;
    for (int l = 0; l < a.nlev; ++l) {
        const LevelView &L = a.lev[l];
        const double R2 = a.R2[l];
        for_each_range_m<D>(L, x, a.reach[l], [&](int b, int e) {
            for (int j = b; j < e; ++j) {
                double y[3];
#pragma unroll
                for (int t = 0; t < D; ++t) y[t] = L.x[t][j];
                if (dist2_nofma<D>(x, y) < R2) ++c;
            }
        });
    }
    a.cnt[i] = c;
}

template <int D>
__global__ void __launch_bounds__(NT) k_tfill(ThreshPatternArgs a) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= a.nt) return;
    double x[3];
#pragma unroll
    for (int t = 0; t < D; ++t) x[t] = a.tx[t][i];
    int64_t p = a.row_ptr[i];
    for (int l = 0; l < a.nlev; ++l) {
        const LevelView &L = a.lev[l];
        const double R2 = a.R2[l];
        const int32_t off = (int32_t)a.col_off[l];
        for_each_range_m<D>(L, x, a.reach[l], [&](int b, int e) {
            for (int j = b; j < e; ++j) {
                double y[3];
#pragma unroll
                for (int t = 0; t < D; ++t) y[t] = L.x[t][j];
                const double r2 = dist2_nofma<D>(x, y);
                if (r2 < R2) {
                    if (a.bucket) {
                        int t = 1;
                        while (t <= a.nb && !(r2 < a.tq2[l][t - 1])) ++t;
                        a.bucket[p] = (uint8_t)t;
                    }
                    a.col[p++] = off + j;
                }
            }
        });
    }
}

__global__ void k_csc_count(int64_t nnz, const int32_t *__restrict__ col, int32_t *__restrict__ ccnt) {
    int64_t p = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (p < nnz) atomicAdd(&ccnt[col[p]], 1);
}

__global__ void k_csc_fill(int64_t nrows, int64_t row0, const int64_t *__restrict__ row_ptr,
                           const int32_t *__restrict__ col, const int64_t *__restrict__ cptr,
                           int32_t *__restrict__ cur, int64_t *__restrict__ cpos,
                           int32_t *__restrict__ crow) {
    int64_t r = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (r >= nrows) return;
    const int64_t g = row0 + r;
    for (int64_t p = row_ptr[g]; p < row_ptr[g + 1]; ++p) {
        const int32_t c = col[p];
        const int64_t pos = cptr[c] + atomicAdd(&cur[c], 1);
        cpos[pos] = p;
        crow[pos] = (int32_t)g;
    }
}

// The same two passes row by row with warp-aggregated atomics: the lanes of a
// warp hold neighbouring rows, whose t-th entries mostly fall into the same
// coarse column (a coarse column collects thousands of entries), so one
// atomic per distinct column and warp step replaces one per entry.
// FILL = false: counts only.  (The order inside a column stays arbitrary, as
// with k_csc_fill: every consumer indexes by cpos.)
template <bool FILL>
__global__ void k_csc_agg(int64_t nrows, int64_t row0, const int64_t *__restrict__ row_ptr,
                          const int32_t *__restrict__ col, const int64_t *__restrict__ cptr,
                          int32_t *__restrict__ cur, int64_t *__restrict__ cpos, int32_t *__restrict__ crow) {
    const int64_t r = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t g = row0 + r;
    int64_t p = r < nrows ? row_ptr[g] : 0;
    const int64_t pe = r < nrows ? row_ptr[g + 1] : 0;
    while (__any_sync(0xffffffffu, p < pe)) {
        const bool act = p < pe;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        if (act) {
            const int32_t c = col[p];
            const unsigned grp = __match_any_sync(am, c);
            const int leader = __ffs(grp) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&cur[c], __popc(grp));
            if (FILL) {
                base = __shfl_sync(grp, base, leader);
                const int64_t pos = cptr[c] + base + __popc(grp & ((1u << lane) - 1u));
                cpos[pos] = p;
                crow[pos] = (int32_t)g;
            }
            ++p;
        }
    }
}

// Multi-RHS CG, one CTA per batch of 32 columns of A_l (lane = right-hand
// side e_{i0+lane}).  Every column runs the CG of reading C-9 (x0 = 0,
// ||r|| <= tol ||e_i|| = tol) and is frozen once converged; reductions are
// per lane over rows in a fixed order (warp w owns rows w, w + 8, ...; warps
// summed in order), so a column's result does not depend on the batch.
__global__ void __launch_bounds__(NT) k_cgm(CGMultiArgs a) {
    __shared__ double red[NWM][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t batch = a.batch0 + blockIdx.x;
    if (batch >= a.nbatches) return;
    const int64_t n = a.n;
    const int64_t i0 = batch * 32;
    const int64_t stride = (int64_t)n * 32;
    double *X = a.ws + (int64_t)blockIdx.x * 4 * stride;
    double *R = X + stride, *P = R + stride, *Q = P + stride;
    const int64_t mycol = i0 + lane;
    const bool valid = mycol < a.ncols;
    for (int64_t h = w; h < n; h += NWM) {
        double e = (valid && h == mycol) ? 1.0 : 0.0;
        X[h * 32 + lane] = 0.0;
        R[h * 32 + lane] = e;
        P[h * 32 + lane] = e;
    }
    double rr = valid ? 1.0 : 0.0;
    int it = 0;
    __syncthreads();
    for (;;) {
        const bool active = rr > a.tol2;  // ||e_i||^2 = 1
        if (!__syncthreads_or(active)) break;
        if (it >= a.max_iter) {
            if (threadIdx.x == 0) atomicAdd(a.fail, 1);
            break;
        }
        // Q = A P, pq = P.Q per column
        double pq = 0.0;
        for (int64_t h = w; h < n; h += NWM) {
            double acc = 0.0;
            for (int64_t k = a.row_ptr[h]; k < a.row_ptr[h + 1]; ++k)
                acc += a.val[k] * P[(int64_t)a.col[k] * 32 + lane];
            Q[h * 32 + lane] = acc;
            pq += P[h * 32 + lane] * acc;
        }
        red[w][lane] = pq;
        __syncthreads();
        pq = 0.0;
#pragma unroll
        for (int t = 0; t < NWM; ++t) pq += red[t][lane];
        const double alpha = active ? rr / pq : 0.0;
        double rn = 0.0;
        for (int64_t h = w; h < n; h += NWM) {
            double rv = R[h * 32 + lane] - alpha * Q[h * 32 + lane];
            R[h * 32 + lane] = rv;
            rn += rv * rv;
        }
        __syncthreads();  // red[] reuse
        red[w][lane] = rn;
        __syncthreads();
        rn = 0.0;
#pragma unroll
        for (int t = 0; t < NWM; ++t) rn += red[t][lane];
        const double beta = active ? rn / rr : 0.0;
        for (int64_t h = w; h < n; h += NWM) {
            const double pv = P[h * 32 + lane];
            X[h * 32 + lane] += alpha * pv;
            P[h * 32 + lane] = R[h * 32 + lane] + beta * pv;
        }
        if (active) rr = rn;
        ++it;
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(a.max_iters, it);
}

// val[p] = chi_i(x_j) for the stored entries of the columns solved in this
// round: sum_h X[h][r] Phi_{delta_l}(x_j - x_h), h over level l neighbours.
template <int D, int K>
__global__ void __launch_bounds__(NT) k_tvalues(ThreshValueArgs a) {
    const int64_t t = a.pos0 + (int64_t)blockIdx.x * NT + threadIdx.x;
    if (t >= a.pos1) return;
    const int64_t g = a.crow[t];                 // global row (point of a finer level)
    // column of CSC position t: the largest global column c in [c_lo, c_hi) with
    // cptr[c] <= t (empty columns share their start with the next one)
    int64_t lo = a.c_lo, hi = a.c_hi;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.cptr[mid] <= t) lo = mid; else hi = mid;
    }
    const int32_t c = (int32_t)(lo - a.col_off);  // column inside level l
    int k = 0;
    while (k + 1 < a.L && g >= a.lev_off[k + 1]) ++k;
    const int64_t j = g - a.lev_off[k];
    double x[3];
#pragma unroll
    for (int q = 0; q < D; ++q) x[q] = a.lev_xs[k][(int64_t)q * a.lev_n[k] + j];
    const int64_t rel = (int64_t)c - a.first_col;
    const double *Xs = a.ws + (rel / 32) * 4 * (int64_t)a.Lv.n * 32;
    const int r = (int)(rel % 32);
    const LevelView &L = a.Lv;
    const double d2 = L.delta2, inv = L.inv_delta;
    double s = 0.0;
    for_each_range<D>(L, x, [&](int b, int e) {
        for (int h = b; h < e; ++h) {
            double y[3];
#pragma unroll
            for (int q = 0; q < D; ++q) y[q] = L.x[q][h];
            const double r2 = dist2_nofma<D>(x, y);
            if (r2 < d2) s = fma(wendland<K>(sqrt(r2) * inv), Xs[(int64_t)h * 32 + r], s);
        }
    });
    a.val[a.cpos[t]] = L.scale * s;
}

__global__ void k_csc_col(int64_t ncols, const int64_t *__restrict__ cptr, int32_t *__restrict__ ccol) {
    int64_t c = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (c >= ncols) return;
    for (int64_t p = cptr[c]; p < cptr[c + 1]; ++p) ccol[p] = (int32_t)c;
}

// out[g] = base[g] - sum_p val[p] v[col[p]] for global rows g in [r0, r1)
__global__ void __launch_bounds__(NT) k_tresidual(int64_t r0, int64_t r1, const int64_t *__restrict__ row_ptr,
                                                  const int32_t *__restrict__ col, const double *__restrict__ val,
                                                  const double *base, const double *v, double *out,
                                                  const uint8_t *__restrict__ bucket, int tmax) {
    const int64_t g = r0 + (int64_t)blockIdx.x * NT + threadIdx.x;
    if (g >= r1) return;
    double s = 0.0;
    for (int64_t p = row_ptr[g]; p < row_ptr[g + 1]; ++p)
        if (!bucket || bucket[p] <= tmax) s += val[p] * v[col[p]];
    out[g] = base[g] - s;
}

__global__ void k_bucket_count(const uint8_t *__restrict__ b, int64_t n, int tmax, unsigned long long *out) {
    __shared__ long long sm[NT / 32 + 1];
    long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
        c += b[i] <= tmax;
    c = block_sum_ll<NT>(c, sm);
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)c);
}
// out[c] += sum over column c's entries of val[cpos[k]] * u[crow[k]] (transposed SpMV)
__global__ void __launch_bounds__(NT) k_csc_spmv_add(int64_t ncols, const int64_t *__restrict__ cptr,
                                                     const int64_t *__restrict__ cpos,
                                                     const int32_t *__restrict__ crow,
                                                     const double *__restrict__ val, const double *__restrict__ u,
                                                     double *__restrict__ out, const uint8_t *__restrict__ bucket,
                                                     int tmax) {
    const int64_t c = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (c >= ncols) return;
    double s = 0.0;
    for (int64_t k = cptr[c]; k < cptr[c + 1]; ++k)
        if (!bucket || bucket[cpos[k]] <= tmax) s = fma(val[cpos[k]], u[crow[k]], s);
    out[c] += s;
}

// ---------------------------------------------------------------------------
// Local-patch Lagrange functions (PatchArgs, kernels.cuh).
//
// A CTA owns coarse column i of level l:
//  1. patch P = level-l points with |x_h - x_i|^2 < rho^2, enumerated over the
//     nq <= (2m+1)^(d-1) z-columns of cells around x_i in increasing key order
//     (the "patch columns" of the box), so the global ids pid[] come out
//     ascending; per patch column its id range [cb, ce) and member range
//     [ccnt[q], ccnt[q+1]) are kept, per member its column pq[];
//  2. local CSR of A_P: row r of A_l restricted to the members.  A_l's
//     neighbours of a point lie in the 3^(d-1) columns around its own, which
//     are visited in ascending order (a binary search for the row's first id
//     in each, then a monotone member pointer); values copied;
//  3. CG on A_P c = e_i (x0 = 0, stop ||r|| <= lagrange_tol, reading C-9),
//     vectors in shared memory, in the single-reduction form of k_cg (q = A r
//     + beta q by recurrence: one fixed-order block reduction of r.r and r.Ar
//     per iteration); patches of <= 3 NT points keep the first MSK_PATCH_EC
//     entries of each thread row in registers;
//  4. for each stored entry (fine point x_j) of column i:
//     chi~_i(x_j) = delta_l^-d sum_{h in P, r < delta_l} phi(r/delta_l) c_h,
//     h ascending (the order of k_tvalues), visiting only the members in the
//     3^(d-1) patch columns and z window around x_j (members' coordinates
//     and last-axis cells staged in shared memory after the CG).
size_t patch_smem_bytes_impl(int pmax, int nnzmax, int nq) {
    size_t b = 0;
    b += sizeof(int32_t) * (size_t)pmax;          // pid
    b += sizeof(int32_t) * (size_t)(pmax + 1);    // prow (row slots: starts)
    b += sizeof(int32_t) * (size_t)pmax;          // pcnt (entries per row slot)
    b += sizeof(uint16_t) * (size_t)pmax;         // pq (patch column of each member)
    b = (b + 15) & ~(size_t)15;
    b += sizeof(double) * 5 * (size_t)pmax;       // x r p s w
    b += sizeof(double) * ((size_t)nnzmax + 1);   // pval (+ a zero sentinel)
    b += sizeof(uint16_t) * ((size_t)nnzmax + 1); // pcol (patch-local, < 65536 points)
    b = (b + 15) & ~(size_t)15;
    b += sizeof(int32_t) * (3 * (size_t)nq + 1);  // ccnt (member starts), cb, ce (id ranges)
    return b + 64;
}

template <int D>
__device__ __forceinline__ void patch_columns(const LevelView &L, const double *x, int m, int64_t c[3],
                                              int64_t &x0, int64_t &x1, int64_t &y0, int64_t &y1,
                                              int64_t &z0, int64_t &z1) {
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = cell_coord(L.g, a, x[a]);
    const int la = D - 1;
    const int64_t mz = (int64_t)m * L.g.zf;  // thin last-axis cells
    z0 = c[la] - mz < 0 ? 0 : c[la] - mz;
    z1 = c[la] + mz >= L.g.dim[la] ? L.g.dim[la] - 1 : c[la] + mz;
    x0 = c[0] - m < 0 ? 0 : c[0] - m;
    x1 = c[0] + m >= L.g.dim[0] ? L.g.dim[0] - 1 : c[0] + m;
    if (D == 3) {
        y0 = c[1] - m < 0 ? 0 : c[1] - m;
        y1 = c[1] + m >= L.g.dim[1] ? L.g.dim[1] - 1 : c[1] + m;
    } else {
        y0 = 0;
        y1 = 0;
    }
}

// range of the q-th z-column (row-major over (ix, iy)); empty if z0 > z1
template <int D>
__device__ __forceinline__ void patch_range(const LevelView &L, int q, int64_t x0, int64_t y0, int64_t y1,
                                            int64_t z0, int64_t z1, int &b, int &e) {
    const int64_t ny = y1 - y0 + 1;
    const int64_t ix = x0 + q / ny, iy = y0 + q % ny;
    const int64_t kb = D == 3 ? (ix * L.g.dim[1] + iy) * L.g.dim[2] : ix * L.g.dim[1];
    b = L.cell_start[kb + z0];
    e = L.cell_start[kb + z1 + 1];
}

// per column: the patch size and the sum of its members' row lengths in A_l
// (an upper bound of the patch-local nonzeros) -> maxima in pmax_out[0], [1]
template <int D>
__global__ void __launch_bounds__(NT) k_patch_count(PatchArgs a, const int32_t *__restrict__ rowcnt,
                                                    int *pmax_out) {
    const int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= a.ncols) return;
    const LevelView &L = a.Lv;
    double x[3];
#pragma unroll
    for (int t = 0; t < D; ++t) x[t] = L.x[t][i];
    int cnt = 0;
    long long nz = 0;
    for_each_range_m<D>(L, x, a.reach, [&](int b, int e) {
        for (int h = b; h < e; ++h) {
            double y[3];
#pragma unroll
            for (int t = 0; t < D; ++t) y[t] = L.x[t][h];
            if (dist2_nofma<D>(x, y) < a.rho2) {
                ++cnt;
                nz += rowcnt[h];
            }
        }
    });
    atomicMax(pmax_out, cnt);
    atomicMax(pmax_out + 1, (int)(nz < 0x7fffffffll ? nz : 0x7fffffffll));
}

// the patch kernel's CTA size (rows per thread in the CG: RC for patches of
// at most RC x PNT points with the register cache)
#ifndef MSK_PNT
#define MSK_PNT 384  // 384: C4F level-4 patches 723 -> 714 ms, levels 2/3 43/120 -> 34/112 ms (512: 828)
#endif
constexpr int PNT = MSK_PNT;
constexpr int RC = PNT >= 384 ? 2 : 3;
// exclusive block scan of cnt[0..n) in shared memory (n <= PNT * k), result in place; returns the total
__device__ __forceinline__ int block_scan_excl(int32_t *cnt, int n, int32_t *tmp /* PNT */) {
    const int tid = threadIdx.x;
    const int per = (n + PNT - 1) / PNT;
    int s = 0;
    for (int k = 0; k < per; ++k) {
        const int idx = tid * per + k;
        if (idx < n) s += cnt[idx];
    }
    tmp[tid] = s;
    __syncthreads();
    if (tid == 0) {
        int run = 0;
        for (int t = 0; t < PNT; ++t) {
            const int v = tmp[t];
            tmp[t] = run;
            run += v;
        }
        tmp[PNT] = run;
    }
    __syncthreads();
    int run = tmp[tid];
    for (int k = 0; k < per; ++k) {
        const int idx = tid * per + k;
        if (idx < n) {
            const int v = cnt[idx];
            cnt[idx] = run;
            run += v;
        }
    }
    const int total = tmp[PNT];
    __syncthreads();
    return total;
}

// one column; `base` = the CTA's workspace (shared memory, or a global slice
// for patches that do not fit); every early return is CTA-uniform
template <int D, int K>
__device__ __forceinline__ void patch_column(const PatchArgs &a, int64_t i, unsigned char *base) {
    __shared__ double red[2 * (PNT / 32)];  // r.r and r.Ar warp partials
    __shared__ int32_t tmp[PNT + 1];
    const int tid = threadIdx.x;
    const LevelView &L = a.Lv;
    const int pmax = a.pmax, nq = a.nq;
    // byte offsets from base (base is 16-byte aligned; no integer round trip of
    // the pointers, so a shared-memory base keeps shared addressing)
    const size_t o_prow = sizeof(int32_t) * (size_t)pmax, o_pcnt = o_prow + sizeof(int32_t) * (size_t)(pmax + 1);
    const size_t o_pq = o_pcnt + sizeof(int32_t) * (size_t)pmax;
    const size_t o_x = (o_pq + sizeof(uint16_t) * (size_t)pmax + 15) & ~(size_t)15;
    const size_t o_pcol = o_x + sizeof(double) * (5 * (size_t)pmax + (size_t)a.nnzmax + 1);
    const size_t o_ccnt = (o_pcol + sizeof(uint16_t) * ((size_t)a.nnzmax + 1) + 15) & ~(size_t)15;
    int32_t *pid = reinterpret_cast<int32_t *>(base);
    int32_t *prow = reinterpret_cast<int32_t *>(base + o_prow);
    int32_t *pcnt = reinterpret_cast<int32_t *>(base + o_pcnt);
    uint16_t *pq = reinterpret_cast<uint16_t *>(base + o_pq);
    double *X = reinterpret_cast<double *>(base + o_x);
    double *Rv = X + pmax, *P = Rv + pmax, *S = P + pmax, *W = S + pmax;
    double *pval = W + pmax;
    uint16_t *pcol = reinterpret_cast<uint16_t *>(base + o_pcol);
    int32_t *ccnt = reinterpret_cast<int32_t *>(base + o_ccnt);  // nq + 1 member starts
    int32_t *cb = ccnt + nq + 1, *ce = cb + nq;                   // per patch column: global id range
    double xc[3];
#pragma unroll
    for (int t = 0; t < D; ++t) xc[t] = L.x[t][i];
    // ---- 1. patch points, ascending global id
    int64_t c[3], x0, x1, y0, y1, z0, z1;
    patch_columns<D>(L, xc, a.reach, c, x0, x1, y0, y1, z0, z1);
    const int nyb = (int)(y1 - y0 + 1);  // 1 in 2-D
    const int ncolz = (int)((x1 - x0 + 1) * nyb);
    if (ncolz > nq) {
        if (tid == 0) atomicAdd(&a.fail[1], 1);
        return;
    }
    for (int q = tid; q < ncolz; q += PNT) {
        int b, e, n = 0;
        patch_range<D>(L, q, x0, y0, y1, z0, z1, b, e);
        for (int h = b; h < e; ++h) {
            double y[3];
#pragma unroll
            for (int t = 0; t < D; ++t) y[t] = L.x[t][h];
            if (dist2_nofma<D>(xc, y) < a.rho2) ++n;
        }
        ccnt[q] = n;
        cb[q] = b;
        ce[q] = e;
    }
    __syncthreads();
    const int np = block_scan_excl(ccnt, ncolz, tmp);
    if (np > pmax) {
        if (tid == 0) atomicAdd(&a.fail[1], 1);
        return;
    }
    if (tid == 0) ccnt[ncolz] = np;
    for (int q = tid; q < ncolz; q += PNT) {
        int w = ccnt[q];
        const int b = cb[q], e = ce[q];
        for (int h = b; h < e; ++h) {
            double y[3];
#pragma unroll
            for (int t = 0; t < D; ++t) y[t] = L.x[t][h];
            if (dist2_nofma<D>(xc, y) < a.rho2) {
                MSK_DASSERT(w < np && (q + 1 == ncolz || w < ccnt[q + 1]));
                pid[w] = h;
                pq[w] = (uint16_t)q;
                ++w;
            }
        }
    }
    __syncthreads();
    if (tid == 0) atomicMax(&a.fail[3], np);
    // ---- 2. local CSR of A restricted to the patch, in one pass: row r gets a
    // slot of its full A_l row length (the slots fit: the workspace is sized by
    // the largest sum of the members' row lengths), pcnt[r] of them are used
    for (int r0 = tid; r0 < np; r0 += 4 * PNT) {  // four rows' pointer loads in flight
        int64_t b4[4], e4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = r0 + u * PNT;
            const int32_t g = r < np ? pid[r] : 0;
            b4[u] = r < np ? a.row_ptr[g] : 0;
            e4[u] = r < np ? a.row_ptr[g + 1] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (r0 + u * PNT < np) prow[r0 + u * PNT] = (int32_t)(e4[u] - b4[u]);
    }
    __syncthreads();
    int nslot = 0;
    {
        nslot = block_scan_excl(prow, np, tmp);
        if (tid == 0) prow[np] = nslot;
    }
    if (nslot > a.nnzmax) {
        if (tid == 0) atomicAdd(&a.fail[1], 1);
        return;
    }
    const int nnz_sent = a.nnzmax;  // zero entry read by finished rows in the CG's SpMV
    if (tid == 0) {
        pval[nnz_sent] = 0.0;
        pcol[nnz_sent] = 0;
    }
    constexpr int NS = D == 3 ? 9 : 3;  // neighbour columns (dx, dy) in ascending key order
    for (int r = tid; r < np; r += PNT) {
        const int32_t g = pid[r];
        const int q = pq[r], qx = q / nyb, qy = q - qx * nyb;
        int w = prow[r];
        int s = -1, m = 0, mend = 0;
        int32_t lo = 0, hi = 0;  // the current column's id range
        bool fresh = true;       // no member of the current column looked at yet
        auto next = [&]() {
            while (++s < NS) {
                const int ax = qx + s / (NS / 3) - 1, ay = D == 3 ? qy + s % 3 - 1 : 0;
                if (ax < 0 || ax > (int)(x1 - x0) || ay < 0 || ay >= nyb) continue;
                const int cq = ax * nyb + ay;
                m = ccnt[cq];
                mend = ccnt[cq + 1];
                lo = cb[cq];
                hi = ce[cq];
                fresh = true;
                return true;
            }
            return false;
        };
        bool have = next();
        const int64_t kr0 = a.row_ptr[g], kr1 = a.row_ptr[g + 1];
        // the row's first MSK_MERGE_PF columns loaded together (one round trip
        // instead of one per entry), the rest as before
        constexpr int PF = MSK_MERGE_PF;
        int32_t cpf[PF];
#pragma unroll
        for (int t = 0; t < PF; ++t) cpf[t] = kr0 + t < kr1 ? a.col[kr0 + t] : 0;
        for (int64_t k = kr0; have && k < kr1; ++k) {  // ascending columns
            int32_t cc = 0;
#pragma unroll
            for (int t = 0; t < PF; ++t)
                if (k - kr0 == t) cc = cpf[t];
            if (k - kr0 >= PF) cc = a.col[k];
            while (have && cc >= hi) have = next();
            if (!have || cc < lo) continue;
            if (fresh) {  // the first id of this column: binary search (tens of members per column)
                int h2 = mend;
                while (m < h2) {
                    const int mid = (m + h2) >> 1;
                    if (pid[mid] < cc) m = mid + 1; else h2 = mid;
                }
                fresh = false;
            }
            while (m < mend && pid[m] < cc) ++m;  // then a few steps per id
            if (m < mend && pid[m] == cc) {
                MSK_DASSERT(m < np && w < prow[r] + (int)(a.row_ptr[g + 1] - a.row_ptr[g]) && w < a.nnzmax);
                pcol[w] = (uint16_t)m;
                pval[w] = a.val[k];
                ++w;
            }
        }
        pcnt[r] = w - prow[r];
    }
    // ---- 3. CG on A_P c = e_center, single-reduction form (as k_cg): per
    // iteration w = A r, then r.r and r.w in ONE block reduction, then
    // p = r + beta p, s = w + beta s (= A p), x += alpha p, r -= alpha s
    int ctr = -1;
    {
        const int q = (int)((c[0] - x0) * nyb + (D == 3 ? c[1] - y0 : 0));  // the centre's own column
        for (int m = ccnt[q]; m < ccnt[q + 1]; ++m)
            if (pid[m] == (int32_t)i) ctr = m;
        MSK_DASSERT(q >= 0 && q < ncolz && ctr >= 0);
    }
    __syncthreads();
    for (int r = tid; r < np; r += PNT) {
        X[r] = 0.0;
        Rv[r] = r == ctr ? 1.0 : 0.0;
        P[r] = 0.0;
        S[r] = 0.0;
    }
    double rr_prev = 1.0, alpha = 0.0;
    int it = 0;
    __syncthreads();
    // patches of at most 3 PNT points (CTA-uniform): the first EC entries of each
    // of the thread's three rows live in registers for the whole CG, so an
    // entry costs one shared-memory load (the gathered r) instead of three
    constexpr int EC = MSK_PATCH_EC;
    const bool regc = MSK_PATCH_REGC && np <= RC * PNT;
    double ev[RC][EC];
    int ecl[RC][EC], nrow[RC], kb3[RC];
#pragma unroll
    for (int u = 0; u < RC; ++u) {
        const int r = tid + u * PNT;
        nrow[u] = regc && r < np ? pcnt[r] : 0;
        kb3[u] = regc && r < np ? prow[r] : 0;
#pragma unroll
        for (int t = 0; t < EC; ++t) {
            const bool in = t < nrow[u];
            ev[u][t] = in ? pval[kb3[u] + t] : 0.0;
            ecl[u][t] = in ? (int)pcol[kb3[u] + t] : 0;
        }
    }
    for (;;) {
        double vrr = 0.0, vrw = 0.0;
        if (regc) {
            double acc[RC];
#pragma unroll
            for (int u = 0; u < RC; ++u) acc[u] = 0.0;
#pragma unroll
            for (int t = 0; t < EC; ++t)
#pragma unroll
                for (int u = 0; u < RC; ++u)
                    if (t < nrow[u]) acc[u] = fma(ev[u][t], Rv[ecl[u][t]], acc[u]);
            int n = 0;
#pragma unroll
            for (int u = 0; u < RC; ++u) n = max(n, nrow[u]);
            for (int t = EC; t < n; ++t)
#pragma unroll
                for (int u = 0; u < RC; ++u)
                    if (t < nrow[u]) {
                        const int k = kb3[u] + t;
                        acc[u] = fma(pval[k], Rv[pcol[k]], acc[u]);
                    }
#pragma unroll
            for (int u = 0; u < RC; ++u) {
                const int r = tid + u * PNT;
                if (r < np) {
                    W[r] = acc[u];
                    const double rv = Rv[r];
                    vrr += rv * rv;
                    vrw += rv * acc[u];
                }
            }
        }
        // a thread's rows rb, rb + PNT, rb + 2 PNT as three independent chains
        // (the loads of all three in flight; each row still sums in ascending
        // k); a finished row reads the zero sentinel entry at nnzmax
        for (int rb = tid; !regc && rb < np; rb += 3 * PNT) {
            int kk[3], ke[3];
            double acc[3] = {0.0, 0.0, 0.0};
            int n = 0;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int r = rb + u * PNT;
                kk[u] = r < np ? prow[r] : 0;
                ke[u] = r < np ? kk[u] + pcnt[r] : 0;
                n = max(n, ke[u] - kk[u]);
            }
            for (int t = 0; t < n; ++t) {
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int k = kk[u] + t < ke[u] ? kk[u] + t : nnz_sent;
                    MSK_DASSERT(k <= a.nnzmax && pcol[k] < np);
                    acc[u] = fma(pval[k], Rv[pcol[k]], acc[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int r = rb + u * PNT;
                if (r < np) {
                    W[r] = acc[u];
                    const double rv = Rv[r];
                    vrr += rv * rv;
                    vrw += rv * acc[u];
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            vrr += __shfl_xor_sync(0xffffffffu, vrr, o);
            vrw += __shfl_xor_sync(0xffffffffu, vrw, o);
        }
        if ((tid & 31) == 0) {
            red[tid >> 5] = vrr;
            red[PNT / 32 + (tid >> 5)] = vrw;
        }
        __syncthreads();
        double rr = 0.0, rw = 0.0;
#pragma unroll
        for (int w = 0; w < PNT / 32; ++w) {  // warp order: deterministic
            rr += red[w];
            rw += red[PNT / 32 + w];
        }
        if (rr <= a.tol2) break;
        if (it >= a.max_iter) {
            if (tid == 0) atomicAdd(&a.fail[0], 1);
            break;
        }
        const double beta = it == 0 ? 0.0 : rr / rr_prev;
        alpha = it == 0 ? rr / rw : rr / (rw - beta * rr / alpha);
        rr_prev = rr;
        for (int r = tid; r < np; r += PNT) {
            const double pn = Rv[r] + beta * P[r];
            const double sn = W[r] + beta * S[r];
            P[r] = pn;
            S[r] = sn;
            X[r] += alpha * pn;
            Rv[r] -= alpha * sn;
        }
        __syncthreads();  // r complete before the next w = A r; red[] read before it is rewritten
        ++it;
    }
    if (tid == 0) atomicMax(&a.fail[2], it);
    // the members' coordinates into the CG's dead vectors (every thread left the
    // loop after the same reduction barrier, past its last read of r, p, s):
    // phase 4 reads them from shared memory
    // and each member's last-axis cell relative to the box into pq (dead since
    // phase 2): a column's members are in key order, i.e. ascending in it
    double *cx[3] = {Rv, P, S};
    for (int r = tid; r < np; r += PNT) {
        const int32_t g = pid[r];
#pragma unroll
        for (int u = 0; u < D; ++u) cx[u][r] = L.x[u][g];
        pq[r] = (uint16_t)(cell_coord(L.g, D - 1, cx[D - 1][r]) - z0);
    }
    __syncthreads();
    // ---- 4. values at the stored entries of column i
    const int64_t gc = a.col_off + i;
    const double d2 = L.delta2, inv = L.inv_delta;
    const int la = D - 1;
    const int64_t zf = L.g.zf;
    for (int64_t t = a.cptr[gc] + tid; t < a.cptr[gc + 1]; t += PNT) {
        const int64_t g = a.crow[t];
        int k = 0;
        while (k + 1 < a.L && g >= a.lev_off[k + 1]) ++k;
        const int64_t j = g - a.lev_off[k];
        double xj[3];
#pragma unroll
        for (int q = 0; q < D; ++q) xj[q] = a.lev_xs[k][(int64_t)q * a.lev_n[k] + j];
        int64_t cj[3];
#pragma unroll
        for (int q = 0; q < D; ++q) cj[q] = cell_coord(L.g, q, xj[q]);
        const int64_t zlo = cj[la] - zf > z0 ? cj[la] - zf : z0, zhi = cj[la] + zf < z1 ? cj[la] + zf : z1;
        double s = 0.0;
        if (zlo <= zhi) {
            for (int64_t ix = cj[0] - 1; ix <= cj[0] + 1; ++ix) {
                if (ix < x0 || ix > x1) continue;
                for (int64_t iy = D == 3 ? cj[1] - 1 : 0; iy <= (D == 3 ? cj[1] + 1 : 0); ++iy) {
                    if (D == 3 && (iy < y0 || iy > y1)) continue;
                    const int q = (int)((ix - x0) * nyb + (iy - y0));
                    MSK_DASSERT(q >= 0 && q < ncolz);
                    // the members in cells zlo..zhi of this column, ascending: the first
                    // by a binary search of the column's last-axis cells (large patches
                    // hold tens of members per column), then while in the window
                    const int zl = (int)(zlo - z0), zh = (int)(zhi - z0);
                    int m = ccnt[q], mh = ccnt[q + 1];
                    {
                        int hi2 = mh;
                        while (m < hi2) {
                            const int mid = (m + hi2) >> 1;
                            if ((int)pq[mid] < zl) m = mid + 1; else hi2 = mid;
                        }
                    }
                    for (; m < mh && (int)pq[m] <= zh; ++m) {
                        double y[3];
#pragma unroll
                        for (int u = 0; u < D; ++u) y[u] = cx[u][m];
                        const double r2 = dist2_nofma<D>(xj, y);
                        if (r2 < d2) s = fma(wendland<K>(sqrt(r2) * inv), X[m], s);
                    }
                }
            }
        }
        a.val_out[a.cpos[t]] = L.scale * s;
    }
}

// GWS = false: the workspace is the dynamic shared memory, addressed as such
// (LDS/STS; a pointer that may be either is generic LD/ST with 64-bit
// addresses); GWS = true: a global slice per CTA for patches that do not fit
template <int D, int K, bool GWS>
__global__ void __launch_bounds__(PNT) k_patch(PatchArgs a, unsigned char *gws, size_t gstride) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = GWS ? gws + (size_t)blockIdx.x * gstride : smem_raw;
    for (int64_t i = blockIdx.x; i < a.ncols; i += gridDim.x) {
        patch_column<D, K>(a, i, base);
        __syncthreads();  // the workspace is reused by the next column
    }
}
}  // namespace

size_t patch_smem_bytes(int pmax, int nnzmax, int nq) { return patch_smem_bytes_impl(pmax, nnzmax, nq); }

void patch_count(const PatchArgs &a, const int32_t *rowcnt, int *pmax_out, cudaStream_t st) {
    if (a.ncols <= 0) return;
    if (a.d == 2) k_patch_count<2><<<ceil_div_u(a.ncols, NT), NT, 0, st>>>(a, rowcnt, pmax_out);
    else k_patch_count<3><<<ceil_div_u(a.ncols, NT), NT, 0, st>>>(a, rowcnt, pmax_out);
    MSK_CHECK_LAUNCH();
}

void patch_lagrange(const PatchArgs &a, size_t smem, cudaStream_t st, int *launches) {
    if (a.ncols <= 0) return;
    // a patch that does not fit in shared memory: a global workspace slice per
    // CTA of a persistent grid (slower, L2-resident vectors)
    // the opt-in limit minus the kernel's static shared memory (block reductions)
    int dev = 0, optin = 0;
    MSK_CUDA(cudaGetDevice(&dev));
    MSK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    if (a.d == 2)
        MSK_CUDA(cudaFuncGetAttributes(&fa, a.k == 0 ? k_patch<2, 0, false> : a.k == 1 ? k_patch<2, 1, false> : k_patch<2, 2, false>));
    else
        MSK_CUDA(cudaFuncGetAttributes(&fa, a.k == 0 ? k_patch<3, 0, false> : a.k == 1 ? k_patch<3, 1, false> : k_patch<3, 2, false>));
    const bool global = smem + fa.sharedSizeBytes > (size_t)optin;
    unsigned grid = (unsigned)a.ncols;
    unsigned char *gws = nullptr;
    const size_t stride = (smem + 255) & ~(size_t)255;
    if (global) {
        grid = (unsigned)(a.ncols < 148 * 4 ? a.ncols : 148 * 4);
        MSK_CUDA(cudaMallocAsync((void **)&gws, stride * grid, st));
    }
    const size_t dyn = global ? 0 : smem;
#define MSK_PT(DD, KK)                                                                            \
    do {                                                                                         \
        if (!global) {                                                                           \
            MSK_CUDA(cudaFuncSetAttribute(k_patch<DD, KK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                          (int)smem));                                           \
            k_patch<DD, KK, false><<<grid, PNT, dyn, st>>>(a, gws, stride);                       \
        } else {                                                                                 \
            k_patch<DD, KK, true><<<grid, PNT, dyn, st>>>(a, gws, stride);                        \
        }                                                                                        \
    } while (0)
    if (a.d == 2) {
        if (a.k == 0) MSK_PT(2, 0); else if (a.k == 1) MSK_PT(2, 1); else MSK_PT(2, 2);
    } else {
        if (a.k == 0) MSK_PT(3, 0); else if (a.k == 1) MSK_PT(3, 1); else MSK_PT(3, 2);
    }
#undef MSK_PT
    MSK_CHECK_LAUNCH();
    if (gws) MSK_CUDA(cudaFreeAsync(gws, st));
    if (launches) *launches += 1;
}

void csc_spmv_add(int64_t ncols, const int64_t *cptr, const int64_t *cpos, const int32_t *crow, const double *val,
                  const double *u, double *out, cudaStream_t st, const uint8_t *bucket, int tmax) {
    if (ncols <= 0) return;
    k_csc_spmv_add<<<ceil_div_u(ncols, NT), NT, 0, st>>>(ncols, cptr, cpos, crow, val, u, out, bucket, tmax);
    MSK_CHECK_LAUNCH();
}

int64_t bucket_count(const uint8_t *bucket, int64_t nnz, int tmax, cudaStream_t st) {
    unsigned long long *d = nullptr, h = 0;
    MSK_CUDA(cudaMallocAsync((void **)&d, sizeof(unsigned long long), st));
    MSK_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
    if (nnz > 0) {
        const int64_t nb = (nnz + NT - 1) / NT;
        k_bucket_count<<<(unsigned)(nb < 1184 ? nb : 1184), NT, 0, st>>>(bucket, nnz, tmax, d);
        MSK_CHECK_LAUNCH();
    }
    MSK_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    MSK_CUDA(cudaFreeAsync(d, st));
    return (int64_t)h;
}

void thresh_count(const ThreshPatternArgs &a, cudaStream_t st, int *launches) {
    if (a.nt == 0) return;
    if (a.d == 2) k_tcount<2><<<ceil_div_u(a.nt, NT), NT, 0, st>>>(a);
    else k_tcount<3><<<ceil_div_u(a.nt, NT), NT, 0, st>>>(a);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void thresh_fill(const ThreshPatternArgs &a, cudaStream_t st, int *launches) {
    if (a.nt == 0) return;
    if (a.d == 2) k_tfill<2><<<ceil_div_u(a.nt, NT), NT, 0, st>>>(a);
    else k_tfill<3><<<ceil_div_u(a.nt, NT), NT, 0, st>>>(a);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void thresh_csc(int64_t nrows_total, int64_t row0, int64_t nnz, int64_t ncols, const int64_t *row_ptr,
                const int32_t *col, int64_t *cptr, int64_t *cpos, int32_t *crow, int32_t *ccol,
                cudaStream_t st, int *launches) {
    int32_t *cnt = nullptr;
    MSK_CUDA(cudaMallocAsync((void **)&cnt, sizeof(int32_t) * (size_t)(ncols + 1), st));
    MSK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)(ncols + 1), st));
    static const bool agg = !(getenv("MSK_CSC_AGG") && getenv("MSK_CSC_AGG")[0] == '0');
    if (agg) {  // every entry lies in rows [row0, row0 + nrows_total)
        if (nrows_total) {
            k_csc_agg<false><<<ceil_div_u(nrows_total, NT), NT, 0, st>>>(nrows_total, row0, row_ptr, col, cptr,
                                                                         cnt, cpos, crow);
            MSK_CHECK_LAUNCH();
        }
    } else if (nnz) {
        k_csc_count<<<ceil_div_u(nnz, NT), NT, 0, st>>>(nnz, col, cnt);
        MSK_CHECK_LAUNCH();
    }
    exclusive_scan_i64(cnt, ncols, cptr, st, launches);
    MSK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)(ncols + 1), st));
    if (nrows_total) {
        if (agg)
            k_csc_agg<true><<<ceil_div_u(nrows_total, NT), NT, 0, st>>>(nrows_total, row0, row_ptr, col, cptr, cnt,
                                                                        cpos, crow);
        else
            k_csc_fill<<<ceil_div_u(nrows_total, NT), NT, 0, st>>>(nrows_total, row0, row_ptr, col, cptr, cnt,
                                                                   cpos, crow);
        MSK_CHECK_LAUNCH();
    }
    if (ncols && ccol) {
        k_csc_col<<<ceil_div_u(ncols, NT), NT, 0, st>>>(ncols, cptr, ccol);
        MSK_CHECK_LAUNCH();
    }
    if (launches) *launches += 3;
    MSK_CUDA(cudaFreeAsync(cnt, st));
}

void thresh_cg_multi(const CGMultiArgs &a, int nblocks, cudaStream_t st, int *launches) {
    if (nblocks <= 0) return;
    k_cgm<<<nblocks, NT, 0, st>>>(a);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void thresh_values(const ThreshValueArgs &a, cudaStream_t st, int *launches) {
    const int64_t m = a.pos1 - a.pos0;
    if (m <= 0) return;
#define MSK_TV(DD, KK) k_tvalues<DD, KK><<<ceil_div_u(m, NT), NT, 0, st>>>(a)
    if (a.d == 2) {
        if (a.k == 0) MSK_TV(2, 0); else if (a.k == 1) MSK_TV(2, 1); else MSK_TV(2, 2);
    } else {
        if (a.k == 0) MSK_TV(3, 0); else if (a.k == 1) MSK_TV(3, 1); else MSK_TV(3, 2);
    }
#undef MSK_TV
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void thresh_residual(int64_t r0, int64_t r1, const int64_t *row_ptr, const int32_t *col, const double *val,
                     const double *base, const double *v, double *out, cudaStream_t st, int *launches,
                     const uint8_t *bucket, int tmax) {
    if (r1 <= r0) return;
    k_tresidual<<<ceil_div_u(r1 - r0, NT), NT, 0, st>>>(r0, r1, row_ptr, col, val, base, v, out, bucket, tmax);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

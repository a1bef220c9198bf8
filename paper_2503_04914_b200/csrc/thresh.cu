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

#include "kernels.cuh"
#include "neighbors.cuh"

namespace msk {

namespace {
constexpr int NT = 256;
constexpr int NWM = NT / 32;

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
                if (dist2_nofma<D>(x, y) < R2) a.col[p++] = off + j;
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
    const int32_t c = a.ccol[t] - a.col_off;     // column inside level l
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
                                                  const double *base, const double *v, double *out) {
    const int64_t g = r0 + (int64_t)blockIdx.x * NT + threadIdx.x;
    if (g >= r1) return;
    double s = 0.0;
    for (int64_t p = row_ptr[g]; p < row_ptr[g + 1]; ++p) s += val[p] * v[col[p]];
    out[g] = base[g] - s;
}
// out[c] += sum over column c's entries of val[cpos[k]] * u[crow[k]] (transposed SpMV)
__global__ void __launch_bounds__(NT) k_csc_spmv_add(int64_t ncols, const int64_t *__restrict__ cptr,
                                                     const int64_t *__restrict__ cpos,
                                                     const int32_t *__restrict__ crow,
                                                     const double *__restrict__ val, const double *__restrict__ u,
                                                     double *__restrict__ out) {
    const int64_t c = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (c >= ncols) return;
    double s = 0.0;
    for (int64_t k = cptr[c]; k < cptr[c + 1]; ++k) s = fma(val[cpos[k]], u[crow[k]], s);
    out[c] += s;
}
}  // namespace

void csc_spmv_add(int64_t ncols, const int64_t *cptr, const int64_t *cpos, const int32_t *crow, const double *val,
                  const double *u, double *out, cudaStream_t st) {
    if (ncols <= 0) return;
    k_csc_spmv_add<<<ceil_div_u(ncols, NT), NT, 0, st>>>(ncols, cptr, cpos, crow, val, u, out);
    MSK_CHECK_LAUNCH();
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
    if (nnz) {
        k_csc_count<<<ceil_div_u(nnz, NT), NT, 0, st>>>(nnz, col, cnt);
        MSK_CHECK_LAUNCH();
    }
    exclusive_scan_i64(cnt, ncols, cptr, st, launches);
    MSK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)(ncols + 1), st));
    if (nrows_total) {
        k_csc_fill<<<ceil_div_u(nrows_total, NT), NT, 0, st>>>(nrows_total, row0, row_ptr, col, cptr, cnt,
                                                               cpos, crow);
        MSK_CHECK_LAUNCH();
    }
    if (ncols) {
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
                     const double *base, const double *v, double *out, cudaStream_t st, int *launches) {
    if (r1 <= r0) return;
    k_tresidual<<<ceil_div_u(r1 - r0, NT), NT, 0, st>>>(r0, r1, row_ptr, col, val, base, v, out);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

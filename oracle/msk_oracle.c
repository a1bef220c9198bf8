/*
 * oracle/msk_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load the shared library built from this file.  The
 * product path (paper_2503_04914_b200/, include/, csrc/) never links, loads
 * or calls it, and this file includes nothing from the product path.
 *
 * A plain, slow, obviously-correct FP64 implementation of what the hot path
 * of Lot & Rieger, "Efficiently parallelizable kernel-based multi-scale
 * algorithm" (arXiv 2503.04914, /root/reference/PAPER.md, cited as P:<line>)
 * computes.  Every function cites the passage it follows.  No blocking, no
 * fusion, no reordering beyond the written definition.  Compiled with
 * -ffp-contract=off so that r^2 = ((dx*dx)+dy*dy)+dz*dz is evaluated left to
 * right without FMA (reading C-4).
 *
 * Threads: built as it stands (no -fopenmp) every loop is serial.  The CPU
 * baseline of bench.py also builds it with -fopenmp (-O3 -march=native): the
 * pragmas below then split ROW loops (each row's result written by one
 * thread, in the same order as serially) and elementwise vector updates over
 * threads; every reduction (dot products, row sums) stays serial, so results
 * are bit-identical for any thread count (tests/test_oracle_solvers.py).
 *
 * Functions and their pins (tests/test_oracle_*.py):
 *   mo_phi, mo_kernel ........ closed forms phi(0)=1, phi(1/2)=0.1875,
 *                              phi(1)=0, Phi_2(r=1,d=2)=0.046875, C^{2k}
 *                              smoothness at r=1, positive definiteness.
 *   mo_pattern_bruteforce .... brute force by definition (ground truth).
 *   mo_pattern_grid .......... == brute force (bit-exact), row-count bound
 *                              eq:rowcost, symmetry.
 *   mo_cg, mo_cholesky_solve . identity / zero-rhs special cases, agreement
 *                              with each other and with numpy LU.
 *   mo_sequential ............ == dense LU of T_L (eq:bigt, via
 *                              oracle/dense.py, itself pinned by Figures
 *                              1-3); f in W_1 => alpha=(c,0..0); f_L=f on X_L.
 *   mo_jacobi_literal ........ == mo_sequential (Theorem jacobi, exact after
 *                              L sweeps); start-vector independence.
 *   mo_evaluate .............. alpha=0 => 0; unit alpha => Phi(x-c);
 *                              interpolation f_L = f on X_L.
 *   mo_separation ............ Table 1 q_l values.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* O1  Wendland functions and the scaled kernel                               */
/* ------------------------------------------------------------------------- */

/* phi_{d,k}(r), Wendland's compactly supported functions with
 * l = floor(d/2) + k + 1 (reading C-3; "2 tau = d + 2k + 1",
 * P:1275 "phi_(3,1)(r) = (1-r)_+^4 (4r+1)"):
 *   k=0: (1-r)_+^l
 *   k=1: (1-r)_+^{l+1} ((l+1) r + 1)
 *   k=2: (1-r)_+^{l+2} ((l^2+4l+3) r^2 + (3l+6) r + 3) / 3
 * For d in {2,3} and k=1 this is exactly (1-r)^4 (4r+1).  phi(0)=1. */
double mo_phi(int d, int k, double r)
{
    if (!(r >= 0.0)) return NAN;
    if (r >= 1.0) return 0.0;
    int l = d / 2 + k + 1;
    double s = 1.0 - r;
    if (k == 0) return pow(s, (double)l);
    if (k == 1) return pow(s, (double)(l + 1)) * ((double)(l + 1) * r + 1.0);
    if (k == 2)
        return pow(s, (double)(l + 2)) *
               ((double)(l * l + 4 * l + 3) * r * r + (double)(3 * l + 6) * r + 3.0) / 3.0;
    return NAN;
}

/* squared distance, left to right, no FMA (reading C-4) */
static double dist2(int d, const double *x, const double *y)
{
    double s = 0.0;
    for (int a = 0; a < d; ++a) {
        double t = x[a] - y[a];
        s = s + t * t;
    }
    return s;
}

/* Phi_delta(x - y) = delta^{-d} Phi((x-y)/delta)  (eq:kernelscaling),
 * Phi(x) = phi(||x||_2).  Zero unless r^2 < delta^2 (strict; the value
 * at r = delta is phi(1) = 0 either way, reading C-4). */
double mo_kernel(int d, int k, double delta, const double *x, const double *y)
{
    double r2 = dist2(d, x, y);
    if (!(r2 < delta * delta)) return 0.0;
    return pow(delta, -(double)d) * mo_phi(d, k, sqrt(r2) / delta);
}

/* ------------------------------------------------------------------------- */
/* O2  Neighbour patterns                                                     */
/* ------------------------------------------------------------------------- */

/* Brute force, by definition: row j of X (nr x d), column n of Y (nc x d) is
 * in the pattern iff ||x_j - y_n||^2 < delta^2 (P:274-279 with compact support
 * P:65; strict, reading C-4).  Columns ascending.  If col == NULL only
 * row_ptr is filled.  Returns nnz. */
int64_t mo_pattern_bruteforce(int d, int64_t nr, const double *X, int64_t nc,
                              const double *Y, double delta, int64_t *row_ptr,
                              int32_t *col)
{
    double d2 = delta * delta;
    int64_t nnz = 0;
    for (int64_t j = 0; j < nr; ++j) {
        row_ptr[j] = nnz;
        for (int64_t n = 0; n < nc; ++n) {
            if (dist2(d, X + j * d, Y + n * d) < d2) {
                if (col) col[nnz] = (int32_t)n;
                ++nnz;
            }
        }
    }
    row_ptr[nr] = nnz;
    return nnz;
}

/* A simple bucket grid (qsort + binary search), used to make the oracle
 * usable above ~2e4 points.  Bucket side = delta*(1+1e-9) so a pair with
 * r < delta is never more than one bucket apart.  Pinned bit-exactly to
 * mo_pattern_bruteforce. */
typedef struct { int64_t c[3]; int64_t i; } mo_entry;
typedef struct { int d; double inv; int64_t n; const double *P; mo_entry *e; } mo_grid;

static int cmp_cell(const int64_t *a, const int64_t *b)
{
    for (int t = 0; t < 3; ++t) {
        if (a[t] < b[t]) return -1;
        if (a[t] > b[t]) return 1;
    }
    return 0;
}

static int cmp_entry(const void *pa, const void *pb)
{
    const mo_entry *a = (const mo_entry *)pa, *b = (const mo_entry *)pb;
    int c = cmp_cell(a->c, b->c);
    if (c) return c;
    return (a->i > b->i) - (a->i < b->i);
}

static void grid_cell(const mo_grid *g, const double *x, int64_t *c)
{
    c[0] = c[1] = c[2] = 0;
    for (int a = 0; a < g->d; ++a) c[a] = (int64_t)floor(x[a] * g->inv);
}

static int grid_build(mo_grid *g, int d, int64_t n, const double *P, double delta)
{
    g->d = d;
    g->n = n;
    g->P = P;
    g->inv = 1.0 / (delta * (1.0 + 1e-9));
    g->e = (mo_entry *)malloc(sizeof(mo_entry) * (size_t)(n > 0 ? n : 1));
    if (!g->e) return -1;
    for (int64_t i = 0; i < n; ++i) {
        grid_cell(g, P + i * d, g->e[i].c);
        g->e[i].i = i;
    }
    qsort(g->e, (size_t)n, sizeof(mo_entry), cmp_entry);
    return 0;
}

static void grid_free(mo_grid *g) { free(g->e); g->e = NULL; }

static int64_t grid_lower(const mo_grid *g, const int64_t *key)
{
    int64_t lo = 0, hi = g->n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (cmp_cell(g->e[mid].c, key) < 0) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Collect the indices n with ||x - y_n||^2 < delta^2 into buf (unsorted).
 * Returns count. */
static int64_t grid_query(const mo_grid *g, const double *x, double delta,
                          int64_t *buf)
{
    double d2 = delta * delta;
    int64_t c[3], key[3], cnt = 0;
    grid_cell(g, x, c);
    int rz = g->d == 3 ? 1 : 0;
    for (int64_t ox = -1; ox <= 1; ++ox)
        for (int64_t oy = -1; oy <= 1; ++oy)
            for (int64_t oz = -rz; oz <= rz; ++oz) {
                key[0] = c[0] + ox; key[1] = c[1] + oy; key[2] = c[2] + oz;
                for (int64_t p = grid_lower(g, key);
                     p < g->n && cmp_cell(g->e[p].c, key) == 0; ++p) {
                    int64_t n = g->e[p].i;
                    if (dist2(g->d, x, g->P + n * g->d) < d2) buf[cnt++] = n;
                }
            }
    return cnt;
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Same contract as mo_pattern_bruteforce, computed through the bucket grid.
 * Returns nnz, or -1 on allocation failure. */
int64_t mo_pattern_grid(int d, int64_t nr, const double *X, int64_t nc,
                        const double *Y, double delta, int64_t *row_ptr,
                        int32_t *col)
{
    mo_grid g;
    if (grid_build(&g, d, nc, Y, delta)) return -1;
#ifdef _OPENMP
    /* threaded build: counts per row, a serial prefix, then the rows */
    int fail = 0;
#pragma omp parallel
    {
        int64_t *tb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
        if (!tb) {
#pragma omp atomic write
            fail = 1;
        }
#pragma omp for schedule(dynamic, 1024)
        for (int64_t j = 0; j < nr; ++j)
            row_ptr[j + 1] = tb ? grid_query(&g, X + j * d, delta, tb) : 0;
#pragma omp single
        {
            row_ptr[0] = 0;
            for (int64_t j = 0; j < nr; ++j) row_ptr[j + 1] += row_ptr[j];
        }
        if (col) {
#pragma omp for schedule(dynamic, 1024)
            for (int64_t j = 0; j < nr; ++j) {
                if (!tb) continue;
                int64_t cnt = grid_query(&g, X + j * d, delta, tb);
                qsort(tb, (size_t)cnt, sizeof(int64_t), cmp_i64);
                for (int64_t t = 0; t < cnt; ++t) col[row_ptr[j] + t] = (int32_t)tb[t];
            }
        }
        free(tb);
    }
    grid_free(&g);
    return fail ? -1 : row_ptr[nr];
#endif
    int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
    if (!buf) { grid_free(&g); return -1; }
    int64_t nnz = 0;
    for (int64_t j = 0; j < nr; ++j) {
        row_ptr[j] = nnz;
        int64_t cnt = grid_query(&g, X + j * d, delta, buf);
        if (col) {
            qsort(buf, (size_t)cnt, sizeof(int64_t), cmp_i64);
            for (int64_t t = 0; t < cnt; ++t) col[nnz + t] = (int32_t)buf[t];
        }
        nnz += cnt;
    }
    row_ptr[nr] = nnz;
    free(buf);
    grid_free(&g);
    return nnz;
}

/* O3 values of B_{l2,l1} = (Phi_{l1}(x^{(l2)}_{n2} - x^{(l1)}_{n1})) on a
 * given pattern (the COLUMN level's delta, reading C-1). */
void mo_values(int d, int k, double delta, int64_t nr, const double *X,
               const double *Y, const int64_t *row_ptr, const int32_t *col,
               double *val)
{
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t j = 0; j < nr; ++j)
        for (int64_t p = row_ptr[j]; p < row_ptr[j + 1]; ++p)
            val[p] = mo_kernel(d, k, delta, X + j * d, Y + (int64_t)col[p] * d);
}

/* y = A v for CSR A */
void mo_spmv(int64_t n, const int64_t *row_ptr, const int32_t *col,
             const double *val, const double *v, double *y)
{
#pragma omp parallel for schedule(static, 4096)
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t p = row_ptr[j]; p < row_ptr[j + 1]; ++p) s += val[p] * v[col[p]];
        y[j] = s;
    }
}

/* y_j = sum_n Phi_delta(x_j - y_n) v_n, matrix-free (one block B v). */
int mo_apply(int d, int k, double delta, int64_t nr, const double *X,
             int64_t nc, const double *Y, const double *v, double *out)
{
    mo_grid g;
    if (grid_build(&g, d, nc, Y, delta)) return -1;
    int fail = 0;
#pragma omp parallel
    {
        int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
        if (!buf) {
#pragma omp atomic write
            fail = 1;
        }
#pragma omp for schedule(dynamic, 1024)
        for (int64_t j = 0; j < nr; ++j) {
            if (!buf) continue;
            int64_t cnt = grid_query(&g, X + j * d, delta, buf);
            qsort(buf, (size_t)cnt, sizeof(int64_t), cmp_i64);
            double s = 0.0;
            for (int64_t t = 0; t < cnt; ++t)
                s += mo_kernel(d, k, delta, X + j * d, Y + buf[t] * d) * v[buf[t]];
            out[j] = s;
        }
        free(buf);
    }
    grid_free(&g);
    return fail ? -1 : 0;
}

/* ------------------------------------------------------------------------- */
/* Linear solvers                                                             */
/* ------------------------------------------------------------------------- */

static double dot(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* Conjugate gradients on SPD A (Theorem cg, Algorithm 1
 * P:1501-1535; details reading C-9): x0 = 0, r = b, p = r; stop when
 * ||r||_2 <= tol ||b||_2 (recurrence residual); alpha = r'r / p'Ap;
 * beta = r_new'r_new / r'r.  b = 0 => 0 iterations.  Returns 0, or 1 if
 * max_iter was reached first. */
int mo_cg(int64_t n, const int64_t *row_ptr, const int32_t *col,
          const double *val, const double *b, double *x, double tol,
          int max_iter, int *iters)
{
    double *r = (double *)malloc(sizeof(double) * (size_t)n);
    double *p = (double *)malloc(sizeof(double) * (size_t)n);
    double *q = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; p[i] = b[i]; }
    double bb = dot(n, b, b), rr = bb;
    int it = 0, status = 0;
    if (bb > 0.0) {
        for (;;) {
            if (rr <= tol * tol * bb) break;
            if (it >= max_iter) { status = 1; break; }
            mo_spmv(n, row_ptr, col, val, p, q);
            double alpha = rr / dot(n, p, q);
#pragma omp parallel for schedule(static, 4096)
            for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
#pragma omp parallel for schedule(static, 4096)
            for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
            double rr_new = dot(n, r, r);
            double beta = rr_new / rr;
#pragma omp parallel for schedule(static, 4096)
            for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
            rr = rr_new;
            ++it;
        }
    }
    if (iters) *iters = it;
    free(r); free(p); free(q);
    return status;
}

/* Direct solve of A x = b via dense Cholesky A = L L^T (A SPD).
 * Returns 0, or 2 if A is not numerically positive definite. */
/* dense lower Cholesky factor of CSR A (n x n), or NULL (not SPD / no memory) */
static double *chol_factor(int64_t n, const int64_t *row_ptr, const int32_t *col,
                           const double *val, int *status)
{
    double *A = (double *)calloc((size_t)(n * n > 0 ? n * n : 1), sizeof(double));
    if (!A) { *status = -1; return NULL; }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) A[i * n + col[p]] = val[p];
    for (int64_t j = 0; j < n; ++j) {
        double s = A[j * n + j];
        for (int64_t t = 0; t < j; ++t) s -= A[j * n + t] * A[j * n + t];
        if (!(s > 0.0)) { free(A); *status = 2; return NULL; }
        double ljj = sqrt(s);
        A[j * n + j] = ljj;
        for (int64_t i = j + 1; i < n; ++i) {
            double u = A[i * n + j];
            for (int64_t t = 0; t < j; ++t) u -= A[i * n + t] * A[j * n + t];
            A[i * n + j] = u / ljj;
        }
    }
    *status = 0;
    return A;
}

/* x = (L L^T)^{-1} b with the factor of chol_factor */
static void chol_solve(int64_t n, const double *A, const double *b, double *x)
{
    for (int64_t i = 0; i < n; ++i) {            /* L y = b */
        double s = b[i];
        for (int64_t t = 0; t < i; ++t) s -= A[i * n + t] * x[t];
        x[i] = s / A[i * n + i];
    }
    for (int64_t i = n - 1; i >= 0; --i) {       /* L^T x = y */
        double s = x[i];
        for (int64_t t = i + 1; t < n; ++t) s -= A[t * n + i] * x[t];
        x[i] = s / A[i * n + i];
    }
}

int mo_cholesky_solve(int64_t n, const int64_t *row_ptr, const int32_t *col,
                      const double *val, const double *b, double *x)
{
    int st = 0;
    double *A = chol_factor(n, row_ptr, col, val, &st);
    if (!A) return st;
    chol_solve(n, A, b, x);
    free(A);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Level matrices                                                             */
/* ------------------------------------------------------------------------- */

typedef struct { int64_t n, nnz; int64_t *row_ptr; int32_t *col; double *val; } mo_csr;

static void csr_free(mo_csr *m) { free(m->row_ptr); free(m->col); free(m->val); }

/* A_l = B_{l,l} = (Phi_{delta_l}(x_i - x_j)). */
static int build_A(int d, int k, int64_t n, const double *P, double delta, mo_csr *m)
{
    m->n = n;
    m->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t nnz = mo_pattern_grid(d, n, P, n, P, delta, m->row_ptr, NULL);
    if (nnz < 0) return -1;
    m->nnz = nnz;
    m->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    m->val = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    mo_pattern_grid(d, n, P, n, P, delta, m->row_ptr, m->col);
    mo_values(d, k, delta, n, P, P, m->row_ptr, m->col, m->val);
    return 0;
}

static int solve_level(const mo_csr *A, const double *b, double *x, double tol,
                       int max_iter, int64_t direct_max_n, int *iters)
{
    if (A->n <= direct_max_n) {
        if (iters) *iters = 0;
        return mo_cholesky_solve(A->n, A->row_ptr, A->col, A->val, b, x);
    }
    return mo_cg(A->n, A->row_ptr, A->col, A->val, b, x, tol, max_iter, iters);
}

/* ------------------------------------------------------------------------- */
/* O4  Sequential multiscale residual correction (the plain definition)       */
/* ------------------------------------------------------------------------- */

/* For l = 1..L:  A_l alpha^{(l)} = f^{(l)} - sum_{k<l} B_{l k} alpha^{(k)}
 * (eq:mas; matrix form of P:156-166), B_{lk} with the column
 * level's delta_k (reading C-1).  Levels with N(l) <= direct_max_n are
 * solved by Cholesky, the others by mo_cg at tol.  counters (nullable, 3
 * doubles): [0] nnz of all A_l, [1] sum over CG iterations of nnz(A_l),
 * [2] nonzeros of the B products.  Returns 0, 1 (no convergence), <0 alloc. */
int mo_sequential(int d, int k, int L, const int64_t *n, const double *const *pts,
                  const double *delta, const double *const *f, double tol,
                  int max_iter, int64_t direct_max_n, double *const *alpha,
                  int *iters, double *counters)
{
    double cA = 0.0, cCG = 0.0, cB = 0.0;
    int status = 0;
    for (int l = 0; l < L && status == 0; ++l) {
        double *rhs = (double *)malloc(sizeof(double) * (size_t)n[l]);
        double *tmp = (double *)malloc(sizeof(double) * (size_t)n[l]);
        memcpy(rhs, f[l], sizeof(double) * (size_t)n[l]);
        for (int kk = 0; kk < l; ++kk) {
            mo_apply(d, k, delta[kk], n[l], pts[l], n[kk], pts[kk], alpha[kk], tmp);
            for (int64_t j = 0; j < n[l]; ++j) rhs[j] -= tmp[j];
            if (counters) {
                int64_t *rp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n[l] + 1));
                cB += (double)mo_pattern_grid(d, n[l], pts[l], n[kk], pts[kk], delta[kk], rp, NULL);
                free(rp);
            }
        }
        mo_csr A;
        if (build_A(d, k, n[l], pts[l], delta[l], &A)) { free(rhs); free(tmp); return -1; }
        int it = 0;
        status = solve_level(&A, rhs, alpha[l], tol, max_iter, direct_max_n, &it);
        if (iters) iters[l] = it;
        cA += (double)A.nnz;
        cCG += (double)A.nnz * it;
        csr_free(&A);
        free(rhs);
        free(tmp);
    }
    if (counters) { counters[0] = cA; counters[1] = cCG; counters[2] = cB; }
    return status;
}

/* ------------------------------------------------------------------------- */
/* O5  Evaluation of the approximant                                          */
/* ------------------------------------------------------------------------- */

/* s(x) = f_L(x) = sum_l sum_n alpha_n^{(l)} Phi_l(x - x_n^{(l)})
 * (eq:fapproximation) at m points x (m x d).  Returns 0. */
int mo_evaluate(int d, int k, int L, const int64_t *n, const double *const *pts,
                const double *delta, const double *const *alpha, int64_t m,
                const double *x, double *s)
{
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    for (int64_t j = 0; j < m; ++j) s[j] = 0.0;
    for (int l = 0; l < L; ++l) {
        if (mo_apply(d, k, delta[l], m, x, n[l], pts[l], alpha[l], tmp)) { free(tmp); return -1; }
        for (int64_t j = 0; j < m; ++j) s[j] += tmp[j];
    }
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O6  Monolithic solve, literal Algorithm 2 + Algorithm 1                    */
/* ------------------------------------------------------------------------- */

/* eq:split: T'_L beta = f by the Jacobi iteration
 * beta_{m+1} = f + (id - T'_L) beta_m (eq:jacobi P:678), run for exactly L
 * sweeps from beta_0 (beta0 == NULL means beta_0 = f, reading C-11).
 * (id - T'_L) has blocks -X_{kl} = -B_{kl} A_l^{-1} (reading C-7),
 * applied as in Algorithm 2: t^{(l)} = A_l^{-1} beta^{(l)} for
 * l < L (inner tolerance inner_tol, reading C-10), then
 * beta^{(k)} = f^{(k)} - sum_{l<k} B_{kl} t^{(l)}.  Finally D_L alpha = beta
 * blockwise (eq:blockdiagonal_levelwise P:616) at tol.  beta_out may be NULL. */
int mo_jacobi_literal(int d, int k, int L, const int64_t *n, const double *const *pts,
                      const double *delta, const double *const *f,
                      const double *const *beta0, double tol, double inner_tol,
                      int max_iter, int64_t direct_max_n, double *const *beta_out,
                      double *const *alpha)
{
    mo_csr *A = (mo_csr *)calloc((size_t)L, sizeof(mo_csr));
    double **beta = (double **)calloc((size_t)L, sizeof(double *));
    double **t = (double **)calloc((size_t)L, sizeof(double *));
    int status = 0;
    for (int l = 0; l < L; ++l) {
        if (build_A(d, k, n[l], pts[l], delta[l], &A[l])) return -1;
        beta[l] = (double *)malloc(sizeof(double) * (size_t)n[l]);
        t[l] = (double *)malloc(sizeof(double) * (size_t)n[l]);
        memcpy(beta[l], beta0 ? beta0[l] : f[l], sizeof(double) * (size_t)n[l]);
    }
    for (int sweep = 0; sweep < L && status == 0; ++sweep) {
        for (int l = 0; l + 1 < L && status == 0; ++l)
            status = solve_level(&A[l], beta[l], t[l], inner_tol, max_iter, direct_max_n, NULL);
        for (int kk = 0; kk < L && status == 0; ++kk) {
            double *tmp = (double *)malloc(sizeof(double) * (size_t)n[kk]);
            memcpy(beta[kk], f[kk], sizeof(double) * (size_t)n[kk]);
            for (int l = 0; l < kk; ++l) {
                mo_apply(d, k, delta[l], n[kk], pts[kk], n[l], pts[l], t[l], tmp);
                for (int64_t j = 0; j < n[kk]; ++j) beta[kk][j] -= tmp[j];
            }
            free(tmp);
        }
    }
    for (int l = 0; l < L && status == 0; ++l) {
        status = solve_level(&A[l], beta[l], alpha[l], tol, max_iter, direct_max_n, NULL);
        if (beta_out) memcpy(beta_out[l], beta[l], sizeof(double) * (size_t)n[l]);
    }
    for (int l = 0; l < L; ++l) { csr_free(&A[l]); free(beta[l]); free(t[l]); }
    free(A); free(beta); free(t);
    return status;
}

/* ------------------------------------------------------------------------- */
/* O7  Thresholded factor and its forward substitution                        */
/* ------------------------------------------------------------------------- */

/* (id - M~(T)) beta = f with M~ = -X~ blocks (eq:perturbedmatrix P:846-861,
 * eq:perturbed_split P:865-869; reading C-7 for the sign), solved by forward
 * substitution in level order (the Jacobi iteration reaches the same vector
 * after L sweeps, Theorem jacobi):
 *   beta^(1) = f^(1);
 *   beta^(k) = f^(k) - sum_{l<k} sum_i X~_kl[j,i] beta_i^(l),
 * where X~_kl[j,i] = chi_i^(l)(x_j^(k)) if ||x_j^(k) - x_i^(l)||^2 < (T q_l)^2
 * (strict, coarse column level's q, reading C-5) and the Lagrange function
 * chi_i^(l) = sum_h c_i[h] Phi_l(. - x_h^(l)), c_i = A_l^{-1} e_i (eq:chi
 * P:373-377), by dense Cholesky (A_l SPD).  Then alpha^(l) =
 * A_l^{-1} beta^(l) (eq:blockdiagonal_levelwise P:616), also by Cholesky.
 * Columns are processed in level order, so every beta^(l) used is final.
 * nnz_out (nullable): number of stored factor entries.  Intended for small
 * coarse levels (dense O(N(l)^3)). */
int mo_thresholded(int d, int k, int L, const int64_t *n, const double *const *pts,
                   const double *delta, const double *q, double T, const double *const *f,
                   double *const *beta, double *const *alpha, int64_t *nnz_out)
{
    int64_t nnz = 0;
    for (int l = 0; l < L; ++l) memcpy(beta[l], f[l], sizeof(double) * (size_t)n[l]);
    double *e = NULL, *c = NULL;
    for (int l = 0; l + 1 < L; ++l) {
        mo_csr A;
        if (build_A(d, k, n[l], pts[l], delta[l], &A)) return -1;
        e = (double *)realloc(e, sizeof(double) * (size_t)n[l]);
        c = (double *)realloc(c, sizeof(double) * (size_t)n[l]);
        const double R = T * q[l], R2 = R * R;
        int st = 0;
        double *F = chol_factor(A.n, A.row_ptr, A.col, A.val, &st);
        if (!F) { csr_free(&A); return st; }
        for (int64_t i = 0; i < n[l]; ++i) {
            for (int64_t h = 0; h < n[l]; ++h) e[h] = 0.0;
            e[i] = 1.0;
            chol_solve(A.n, F, e, c);
            for (int kk = l + 1; kk < L; ++kk)
                for (int64_t j = 0; j < n[kk]; ++j) {
                    const double *xj = pts[kk] + j * d;
                    if (!(dist2(d, xj, pts[l] + i * d) < R2)) continue;
                    double chi = 0.0;
                    for (int64_t h = 0; h < n[l]; ++h)
                        chi += c[h] * mo_kernel(d, k, delta[l], xj, pts[l] + h * d);
                    beta[kk][j] -= chi * beta[l][i];
                    ++nnz;
                }
        }
        free(F);
        csr_free(&A);
    }
    free(e);
    free(c);
    for (int l = 0; l < L; ++l) {
        mo_csr A;
        if (build_A(d, k, n[l], pts[l], delta[l], &A)) return -1;
        int st = mo_cholesky_solve(A.n, A.row_ptr, A.col, A.val, beta[l], alpha[l]);
        csr_free(&A);
        if (st) return 2;
    }
    if (nnz_out) *nnz_out = nnz;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Geometry                                                                   */
/* ------------------------------------------------------------------------- */

/* q_X = 1/2 min_{j != k} ||x_j - x_k||_2, brute force. */
double mo_separation(int d, int64_t n, const double *P)
{
    double best = INFINITY;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            double r2 = dist2(d, P + i * d, P + j * d);
            if (r2 < best) best = r2;
        }
    return 0.5 * sqrt(best);
}

/* One row of the level residual of eq:mas at row j of level l:
 * (A_l alpha^{(l)})_j + sum_{k<l} (B_{lk} alpha^{(k)})_j - f^{(l)}_j,
 * evaluated by brute force over all columns (for sampled full-size checks).
 * Also returns in *absrow the sum of |terms| (a scale for tolerances). */
double mo_mas_row_residual(int d, int k, int l, const int64_t *n,
                           const double *const *pts, const double *delta,
                           const double *const *alpha, double f_j, int64_t j,
                           double *absrow)
{
    const double *x = pts[l] + j * d;
    double s = 0.0, a = fabs(f_j);
    for (int kk = 0; kk <= l; ++kk)
        for (int64_t c = 0; c < n[kk]; ++c) {
            double v = mo_kernel(d, k, delta[kk], x, pts[kk] + c * d);
            if (v != 0.0) { s += v * alpha[kk][c]; a += fabs(v * alpha[kk][c]); }
        }
    if (absrow) *absrow = a;
    return s - f_j;
}

/* Threads of the -fopenmp build (the CPU baseline's multi-core leg); returns
 * the count in effect (1 when built without OpenMP). */
int mo_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* msk_example.c -- the C-ABI used from plain C99 (no Python, no torch).
 *
 * Paper grids l = 1..3 on [0,1]^2 (Table 1: (2^l + 1)^2 points, delta_l =
 * 4 sqrt(2) 2^-(l+1), q_l = 2^-(l+1), phi_{3,1}), samples of the Franke function
 * (eq:Franke P:1278), host buffers everywhere.  Solves, evaluates s_L on the
 * finest grid and checks the interpolation property s_L = f on X_L.
 *
 *   gcc -std=c99 -O2 examples/msk_example.c -I include -L paper_2503_04914_b200 -lmsk \
 *       -Wl,-rpath,$PWD/paper_2503_04914_b200 -lm -o /tmp/msk_example && /tmp/msk_example
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "msk.h"

static double franke(double x, double y) {
    return 0.75 * exp(-((9 * x - 2) * (9 * x - 2) + (9 * y - 2) * (9 * y - 2)) / 4) +
           0.75 * exp(-(9 * x + 1) * (9 * x + 1) / 49 - (9 * y + 1) / 10) +
           0.5 * exp(-((9 * x - 7) * (9 * x - 7) + (9 * y - 3) * (9 * y - 3)) / 4) -
           0.2 * exp(-(9 * x - 4) * (9 * x - 4) - (9 * y - 7) * (9 * y - 7));
}

#define CHECK(call)                                                                  \
    do {                                                                             \
        msk_status s_ = (call);                                                      \
        if (s_ != MSK_OK) {                                                          \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)s_, msk_last_error()); \
            return 2;                                                                \
        }                                                                            \
    } while (0)

int main(void) {
    enum { L = 3, D = 2 };
    int64_t n[L];
    double *pts[L], *f[L], *alpha[L], delta[L], q[L];
    for (int l = 0; l < L; ++l) {
        const int m = (1 << (l + 1)) + 1;  /* grid level l+1 */
        n[l] = (int64_t)m * m;
        pts[l] = malloc(sizeof(double) * D * n[l]);
        f[l] = malloc(sizeof(double) * n[l]);
        alpha[l] = malloc(sizeof(double) * n[l]);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                const int64_t r = (int64_t)i * m + j;
                pts[l][2 * r] = (double)i / (m - 1);
                pts[l][2 * r + 1] = (double)j / (m - 1);
                f[l][r] = franke(pts[l][2 * r], pts[l][2 * r + 1]);
            }
        delta[l] = 4.0 * sqrt(2.0) * pow(2.0, -(l + 2));
        q[l] = pow(2.0, -(l + 2));
    }
    msk_ctx *ctx = NULL;
    msk_hierarchy *h = NULL;
    msk_solve_info info;
    CHECK(msk_ctx_create(0, NULL, 0, 1, NULL, &ctx));
    CHECK(msk_hierarchy_create(ctx, D, L, n, (const double *const *)pts, delta, q, 1, MSK_FLAG_NONE, &h));
    CHECK(msk_assemble(h, 0.0, 0.0));
    CHECK(msk_solve(h, (const double *const *)f, 1e-12, 1000, MSK_SCHED_PRUNED, alpha, &info));
    double *s = malloc(sizeof(double) * n[L - 1]);
    CHECK(msk_evaluate(h, n[L - 1], pts[L - 1], s));
    double err = 0.0;
    for (int64_t i = 0; i < n[L - 1]; ++i) err = fmax(err, fabs(s[i] - f[L - 1][i]));
    printf("{\"library\": \"%s\", \"points\": [%lld, %lld, %lld], \"cg_iters\": [%d, %d, %d], "
           "\"max_interpolation_error\": %.3e}\n",
           msk_version(), (long long)n[0], (long long)n[1], (long long)n[2], info.cg_iters[0], info.cg_iters[1],
           info.cg_iters[2], err);
    msk_hierarchy_destroy(h);
    msk_ctx_destroy(ctx);
    for (int l = 0; l < L; ++l) { free(pts[l]); free(f[l]); free(alpha[l]); }
    free(s);
    return err < 1e-10 ? 0 : 1;
}

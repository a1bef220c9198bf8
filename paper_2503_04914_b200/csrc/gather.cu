// gather.cu -- matrix-free multi-level kernel sums (a3 rectangular blocks,
// a5 Jacobi B products, a9 evaluation).
//
//   out_i = base_i + sign * sum_{l} delta_l^-d sum_{n: r < delta_l} phi(r/delta_l) c^{(l)}_n
//
// One thread per target point; targets are in spatial order (sorted by a
// cell grid) so a warp's candidate cells overlap and the coordinate /
// coefficient loads hit L1/L2.  Summation order per target is fixed (levels
// ascending, candidates ascending) => deterministic.
//   B products (eq:mas P:287): base = f^{(k)}, sign = -1, the
//   levels l < k with c = t^{(l)} (reading C-7 for the sign).
//   Evaluation (eq:fapproximation P:295): base = 0, sign = +1, all levels.
#include "kernels.cuh"
#include "neighbors.cuh"

namespace msk {

namespace {
constexpr int NT = 256;

template <int D, int K>
__global__ void __launch_bounds__(NT) k_gather(GatherArgs a) {
    __shared__ long long sm[NT / 32 + 1];
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    long long hits = 0;
    if (i < a.nt) {
        double x[3];
#pragma unroll
        for (int t = 0; t < D; ++t) x[t] = a.tx[t][i];
        double acc = 0.0;
        for (int l = 0; l < a.nlev; ++l) {
            const LevelView &L = a.lev[l];
            const double d2 = L.delta2, inv = L.inv_delta;
            const double *__restrict__ c = L.coef;
            double s = 0.0;
            for_each_range<D>(L, x, [&](int b, int e) {
                for (int j = b; j < e; ++j) {
                    double y[3];
#pragma unroll
                    for (int t = 0; t < D; ++t) y[t] = L.x[t][j];
                    double r2 = dist2_nofma<D>(x, y);
                    if (r2 < d2) {
                        s = fma(wendland<K>(sqrt(r2) * inv), c[j], s);
                        ++hits;
                    }
                }
            });
            acc = fma(L.scale, s, acc);
        }
        double v = a.sign * acc;
        if (a.base) v = a.base[a.base_perm ? a.base_perm[i] : i] + v;
        a.out[a.out_perm ? a.out_perm[i] : i] = v;
    }
    if (a.hits) {
        long long tot = block_sum_ll<NT>(hits, sm);
        if (threadIdx.x == 0) atomicAdd(a.hits, (unsigned long long)tot);
    }
}
}  // namespace

void gather(const GatherArgs &a, cudaStream_t st, int *launches) {
    if (a.nt == 0) return;
    unsigned nb = ceil_div_u(a.nt, NT);
#define MSK_G(DD, KK) k_gather<DD, KK><<<nb, NT, 0, st>>>(a)
    if (a.d == 2) {
        if (a.k == 0) MSK_G(2, 0); else if (a.k == 1) MSK_G(2, 1); else MSK_G(2, 2);
    } else {
        if (a.k == 0) MSK_G(3, 0); else if (a.k == 1) MSK_G(3, 1); else MSK_G(3, 2);
    }
#undef MSK_G
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

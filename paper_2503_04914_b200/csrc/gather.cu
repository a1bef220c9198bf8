// gather.cu -- matrix-free multi-level kernel sums (a3 rectangular blocks,
// a5 Jacobi B products, a9 evaluation).
//
//   out_i = base_i + sign * sum_{l} delta_l^-d sum_{n: r < delta_l} phi(r/delta_l) c^{(l)}_n
//
// One thread per target point; targets are in spatial order (sorted by a
// cell grid) so a warp's candidate cells overlap and the source records hit
// L1/L2.  Sources are packed 32-byte records (x, y, z, c) (2-D: (x, y, c, 0)),
// one 2 x 128-bit load per candidate.
//
// Two passes per level keep the warp convergent: (1) the cheap test
// r^2 < delta^2 (no-FMA, reading C-4) over all candidates, recording the
// indices of the hits in a per-thread list; (2) a dense loop over the hits
// evaluating sqrt and phi.  (A single pass would execute the divergent hit
// path on almost every candidate iteration: with ~15 % hits per lane, some
// lane of the warp hits nearly always.)  Summation order per target is fixed
// (levels ascending, candidates ascending) => deterministic.
//   B products (eq:mas P:287): base = f^{(k)}, sign = -1, the
//   levels l < k with c = t^{(l)} (reading C-7 for the sign).
//   Evaluation (eq:fapproximation P:295): base = 0, sign = +1, all levels.
#include "kernels.cuh"
#include "neighbors.cuh"

namespace msk {

namespace {
constexpr int NT = 256;
constexpr int HMAX = 40;  // hit-list capacity per thread (flushed when full)

template <int D>
__device__ __forceinline__ double rec_dist2(const double *x, const double4 &R) {
    double y[3] = {R.x, R.y, R.z};
    return dist2_nofma<D>(x, y);
}

template <int D>
__device__ __forceinline__ double rec_coef(const double4 &R) {
    return D == 3 ? R.w : R.z;
}

template <int D, int K>
__global__ void __launch_bounds__(NT, 3) k_gather(GatherArgs a) {
    __shared__ long long sm[NT / 32 + 1];
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    long long hits = 0;
    if (i < a.nt) {
        double x[3];
#pragma unroll
        for (int t = 0; t < D; ++t) x[t] = a.tx[t][i];
        double acc = 0.0;
        int hl[HMAX];
        for (int l = 0; l < a.nlev; ++l) {
            const LevelView &L = a.lev[l];
            const double d2 = L.delta2, inv = L.inv_delta;
            const double4 *__restrict__ rec = L.rec;
            double s = 0.0;
            int nh = 0;
            auto flush = [&]() {
                for (int h = 0; h < nh; ++h) {
                    const double4 R = rec[hl[h]];
                    const double r2 = rec_dist2<D>(x, R);
                    s = fma(wendland<K>(sqrt(r2) * inv), rec_coef<D>(R), s);
                }
                hits += nh;
                nh = 0;
            };
            for_each_range<D>(L, x, [&](int b, int e) {
                int j = b;
                for (; j + 1 < e; j += 2) {
                    const double4 R0 = rec[j], R1 = rec[j + 1];
                    const bool h0 = rec_dist2<D>(x, R0) < d2, h1 = rec_dist2<D>(x, R1) < d2;
                    if (nh + 2 > HMAX) flush();
                    if (h0) hl[nh++] = j;
                    if (h1) hl[nh++] = j + 1;
                }
                if (j < e) {
                    const double4 R0 = rec[j];
                    if (nh + 1 > HMAX) flush();
                    if (rec_dist2<D>(x, R0) < d2) hl[nh++] = j;
                }
            });
            flush();
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

__global__ void k_pack(int64_t n, int d, const double *__restrict__ x0, const double *__restrict__ x1,
                       const double *__restrict__ x2, const double *__restrict__ c,
                       double4 *__restrict__ rec) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    rec[i] = d == 3 ? make_double4(x0[i], x1[i], x2[i], c[i]) : make_double4(x0[i], x1[i], c[i], 0.0);
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

void pack_records(int64_t n, int d, const double *xs, const double *coef, double4 *rec,
                  cudaStream_t st, int *launches) {
    if (n == 0) return;
    k_pack<<<ceil_div_u(n, NT), NT, 0, st>>>(n, d, xs, xs + n, d == 3 ? xs + 2 * n : nullptr, coef, rec);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

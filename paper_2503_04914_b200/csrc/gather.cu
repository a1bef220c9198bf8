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
#include <cmath>

#include <stdlib.h>

#include "kernels.cuh"
#include "neighbors.cuh"
#include "wscan.cuh"

namespace msk {

namespace {
#ifndef MSK_GNT
#define MSK_GNT 256
#endif
#ifndef MSK_HMAX
#define MSK_HMAX 40
#endif
// survivors per trip of the exact pass (records loaded up front, same order):
// 2-D 4 (C2 B products 0.97 -> 0.86 ms, evaluation 0.17 -> 0.13 ms), 3-D 1
// (2: 5.16 -> 5.29 / 5.88 -> 6.00 ms, spills at 64 registers)
#ifndef MSK_G_U2
#define MSK_G_U2 4
#endif
#ifndef MSK_G_U3
#define MSK_G_U3 1
#endif
#ifndef MSK_GMINB
#define MSK_GMINB 4
#endif
constexpr int NT = MSK_GNT;
constexpr int HMAX = MSK_HMAX;  // hit-list capacity per thread (flushed when full)

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
__global__ void __launch_bounds__(NT, MSK_GMINB) k_gather(GatherArgs a) {
    __shared__ long long sm[NT / 32 + 1];
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    long long hits = 0;
    if (i < a.nt) {
        double x[3];
        float xf[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int t = 0; t < D; ++t) {
            x[t] = a.tx[t][i];
            xf[t] = (float)(x[t] - a.lev[0].g.lo[t]);  // same origin for every level
        }
        double acc = 0.0;
        int hl[HMAX];
        for (int l = 0; l < a.nlev; ++l) {
            const LevelView &L = a.lev[l];
            const double d2 = L.delta2, inv = L.inv_delta;
            const double4 *__restrict__ rec = L.rec;
            const float4 *__restrict__ frec = L.frec;
            const float fthr = L.fthr;
            double s = 0.0;
            int nh = 0;
            // exact FP64 test (reading C-4) + phi on the candidates that passed the prefilter
            auto flush = [&]() {
                int h = 0;
                constexpr int GU = D == 2 ? MSK_G_U2 : MSK_G_U3;
                for (; GU > 1 && h + GU <= nh; h += GU) {  // records loaded up front, same order
                    double4 R[GU];
#pragma unroll
                    for (int u = 0; u < GU; ++u) R[u] = rec[hl[h + u]];
#pragma unroll
                    for (int u = 0; u < GU; ++u) {
                        const double r2 = rec_dist2<D>(x, R[u]);
                        if (r2 < d2) {
                            s = fma(wendland<K>(sqrt(r2) * inv), rec_coef<D>(R[u]), s);
                            ++hits;
                        }
                    }
                }
                for (; h < nh; ++h) {
                    const double4 R = rec[hl[h]];
                    const double r2 = rec_dist2<D>(x, R);
                    if (r2 < d2) {
                        s = fma(wendland<K>(sqrt(r2) * inv), rec_coef<D>(R), s);
                        ++hits;
                    }
                }
                nh = 0;
            };
            for_each_range<D>(L, x, [&](int b, int e) {
                // conservative FP32 prefilter on 16-byte records; 4 candidates per
                // trip (independent loads in flight: eval 6.21 -> 5.94 ms), then 2, then 1
                int j = b;
                for (; j + 3 < e; j += 4) {
                    const float4 F0 = frec[j], F1 = frec[j + 1], F2 = frec[j + 2], F3 = frec[j + 3];
                    float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
                    float a1 = xf[0] - F1.x, b1 = xf[1] - F1.y, c1 = xf[2] - F1.z;
                    float a2 = xf[0] - F2.x, b2 = xf[1] - F2.y, c2 = xf[2] - F2.z;
                    float a3 = xf[0] - F3.x, b3 = xf[1] - F3.y, c3 = xf[2] - F3.z;
                    const bool h0 = fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr;
                    const bool h1 = fmaf(c1, c1, fmaf(b1, b1, a1 * a1)) < fthr;
                    const bool h2 = fmaf(c2, c2, fmaf(b2, b2, a2 * a2)) < fthr;
                    const bool h3 = fmaf(c3, c3, fmaf(b3, b3, a3 * a3)) < fthr;
                    if (nh + 4 > HMAX) flush();
                    if (h0) hl[nh++] = j;
                    if (h1) hl[nh++] = j + 1;
                    if (h2) hl[nh++] = j + 2;
                    if (h3) hl[nh++] = j + 3;
                }
                for (; j + 1 < e; j += 2) {
                    const float4 F0 = frec[j], F1 = frec[j + 1];
                    float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
                    float a1 = xf[0] - F1.x, b1 = xf[1] - F1.y, c1 = xf[2] - F1.z;
                    const bool h0 = fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr;
                    const bool h1 = fmaf(c1, c1, fmaf(b1, b1, a1 * a1)) < fthr;
                    if (nh + 2 > HMAX) flush();
                    if (h0) hl[nh++] = j;
                    if (h1) hl[nh++] = j + 1;
                }
                if (j < e) {
                    const float4 F0 = frec[j];
                    float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
                    if (nh + 1 > HMAX) flush();
                    if (fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr) hl[nh++] = j;
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

// k_gather with the warp-cooperative candidate scan (wscan.cuh): same hits,
// same order, same arithmetic => bit-identical to k_gather.  128-thread CTAs
// (4 warps x 4.8 KB of static shared memory).
constexpr int NTW = 128;
#ifndef MSK_GW_MINB
#define MSK_GW_MINB 6
#endif
template <int D, int K>
__global__ void __launch_bounds__(NTW, MSK_GW_MINB) k_gather_w(GatherArgs a) {
    __shared__ wscan::WarpSmem Ws[NTW / 32];
    __shared__ long long sm[NTW / 32 + 1];
    wscan::WarpSmem &W = Ws[threadIdx.x >> 5];
    const int64_t i = (int64_t)blockIdx.x * NTW + threadIdx.x;
    const bool on = i < a.nt;
    long long hits = 0;
    double x[3] = {0.0, 0.0, 0.0};
    float xf[3] = {0.f, 0.f, 0.f};
    if (on) {
#pragma unroll
        for (int t = 0; t < D; ++t) {
            x[t] = a.tx[t][i];
            xf[t] = (float)(x[t] - a.lev[0].g.lo[t]);  // same origin for every level
        }
    }
    double acc = 0.0;
    int hl[wscan::HM];
    for (int l = 0; l < a.nlev; ++l) {
        const LevelView &L = a.lev[l];
        const double d2 = L.delta2, inv = L.inv_delta;
        const double4 *__restrict__ rec = L.rec;
        double s = 0.0;
        auto flush = [&](int nh) {
            int h = 0;
            for (; h + 1 < nh; h += 2) {  // two records in flight
                const double4 R0 = rec[hl[h]], R1 = rec[hl[h + 1]];
                const double r20 = rec_dist2<D>(x, R0), r21 = rec_dist2<D>(x, R1);
                if (r20 < d2) {
                    s = fma(wendland<K>(sqrt(r20) * inv), rec_coef<D>(R0), s);
                    ++hits;
                }
                if (r21 < d2) {
                    s = fma(wendland<K>(sqrt(r21) * inv), rec_coef<D>(R1), s);
                    ++hits;
                }
            }
            if (h < nh) {
                const double4 R0 = rec[hl[h]];
                const double r20 = rec_dist2<D>(x, R0);
                if (r20 < d2) {
                    s = fma(wendland<K>(sqrt(r20) * inv), rec_coef<D>(R0), s);
                    ++hits;
                }
            }
        };
        wscan::scan_level<D>(L, x, xf, on, W, hl, flush);
        acc = fma(L.scale, s, acc);
    }
    if (on) {
        double v = a.sign * acc;
        if (a.base) v = a.base[a.base_perm ? a.base_perm[i] : i] + v;
        a.out[a.out_perm ? a.out_perm[i] : i] = v;
    }
    if (a.hits) {
        long long tot = block_sum_ll<NTW>(hits, sm);
        if (threadIdx.x == 0) atomicAdd(a.hits, (unsigned long long)tot);
    }
}

// k_gather_m with the warp-cooperative scan (bit-identical per column)
template <int D, int K, int R>
__global__ void __launch_bounds__(NTW, 3) k_gather_mw(GatherMArgs a) {
    __shared__ wscan::WarpSmem Ws[NTW / 32];
    __shared__ long long sm[NTW / 32 + 1];
    wscan::WarpSmem &W = Ws[threadIdx.x >> 5];
    const int64_t i = (int64_t)blockIdx.x * NTW + threadIdx.x;
    const bool on = i < a.nt;
    long long hits = 0;
    double x[3] = {0.0, 0.0, 0.0};
    float xf[3] = {0.f, 0.f, 0.f};
    if (on) {
#pragma unroll
        for (int t = 0; t < D; ++t) {
            x[t] = a.tx[t][i];
            xf[t] = (float)(x[t] - a.lev[0].g.lo[t]);
        }
    }
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int hl[wscan::HM];
    for (int l = 0; l < a.nlev; ++l) {
        const LevelView &L = a.lev[l];
        const double d2 = L.delta2, inv = L.inv_delta;
        const double4 *__restrict__ rec = L.rec;
        const double *__restrict__ cf = a.coef[l];
        const int64_t ldc = a.ldc;
        double s[R];
#pragma unroll
        for (int r = 0; r < R; ++r) s[r] = 0.0;
        auto flush = [&](int nh) {
            for (int h = 0; h < nh; ++h) {
                const int j = hl[h];
                const double4 Q = rec[j];
                const double r2 = rec_dist2<D>(x, Q);
                if (r2 < d2) {
                    const double w = wendland<K>(sqrt(r2) * inv);
#pragma unroll
                    for (int r = 0; r < R; ++r) s[r] = fma(w, cf[(int64_t)j * ldc + r], s[r]);
                    ++hits;
                }
            }
        };
        wscan::scan_level<D>(L, x, xf, on, W, hl, flush);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(L.scale, s[r], acc[r]);
    }
    if (on) {
        const int64_t bi = a.base_perm ? a.base_perm[i] : i;
        const int64_t oi = a.out_perm ? a.out_perm[i] : i;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double v = a.sign * acc[r];
            if (a.base) v = (r < a.bcols ? a.base[bi * a.ldb + a.bcol0 + r] : 0.0) + v;
            if (r < a.wcols) a.out[oi * a.ldo + a.ocol0 + r] = v;
        }
    }
    if (a.hits) {
        long long tot = block_sum_ll<NTW>(hits, sm);
        if (threadIdx.x == 0) atomicAdd(a.hits, (unsigned long long)tot);
    }
}

template <int D, int K, int R>
__global__ void __launch_bounds__(NT, 3) k_gather_m(GatherMArgs a) {
    __shared__ long long sm[NT / 32 + 1];
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    long long hits = 0;
    if (i < a.nt) {
        double x[3];
        float xf[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int t = 0; t < D; ++t) {
            x[t] = a.tx[t][i];
            xf[t] = (float)(x[t] - a.lev[0].g.lo[t]);
        }
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;
        int hl[HMAX];
        for (int l = 0; l < a.nlev; ++l) {
            const LevelView &L = a.lev[l];
            const double d2 = L.delta2, inv = L.inv_delta;
            const double4 *__restrict__ rec = L.rec;
            const float4 *__restrict__ frec = L.frec;
            const double *__restrict__ cf = a.coef[l];
            const int64_t ldc = a.ldc;
            const float fthr = L.fthr;
            double s[R];
#pragma unroll
            for (int r = 0; r < R; ++r) s[r] = 0.0;
            int nh = 0;
            auto flush = [&]() {
                for (int h = 0; h < nh; ++h) {
                    const int j = hl[h];
                    const double4 Q = rec[j];
                    const double r2 = rec_dist2<D>(x, Q);
                    if (r2 < d2) {
                        const double w = wendland<K>(sqrt(r2) * inv);
#pragma unroll
                        for (int r = 0; r < R; ++r) s[r] = fma(w, cf[(int64_t)j * ldc + r], s[r]);
                        ++hits;
                    }
                }
                nh = 0;
            };
            for_each_range<D>(L, x, [&](int b, int e) {
                int j = b;
                for (; j + 1 < e; j += 2) {
                    const float4 F0 = frec[j], F1 = frec[j + 1];
                    float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
                    float a1 = xf[0] - F1.x, b1 = xf[1] - F1.y, c1 = xf[2] - F1.z;
                    const bool h0 = fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr;
                    const bool h1 = fmaf(c1, c1, fmaf(b1, b1, a1 * a1)) < fthr;
                    if (nh + 2 > HMAX) flush();
                    if (h0) hl[nh++] = j;
                    if (h1) hl[nh++] = j + 1;
                }
                if (j < e) {
                    const float4 F0 = frec[j];
                    float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
                    if (nh + 1 > HMAX) flush();
                    if (fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr) hl[nh++] = j;
                }
            });
            flush();
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fma(L.scale, s[r], acc[r]);
        }
        const int64_t bi = a.base_perm ? a.base_perm[i] : i;
        const int64_t oi = a.out_perm ? a.out_perm[i] : i;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double v = a.sign * acc[r];
            if (a.base) v = (r < a.bcols ? a.base[bi * a.ldb + a.bcol0 + r] : 0.0) + v;
            if (r < a.wcols) a.out[oi * a.ldo + a.ocol0 + r] = v;
        }
    }
    if (a.hits) {
        long long tot = block_sum_ll<NT>(hits, sm);
        if (threadIdx.x == 0) atomicAdd(a.hits, (unsigned long long)tot);
    }
}

template <int D, int K>
__global__ void __launch_bounds__(NT) k_gather_t(GatherTArgs a) {
    const int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= a.nt) return;
    double x[3];
#pragma unroll
    for (int t = 0; t < D; ++t) x[t] = a.tx[t][i];
    double acc = 0.0;
    for (int s = 0; s < a.nsrc; ++s) {
        const LevelView &L = a.src[s];
        const double *__restrict__ y = a.y[s];
        double sum = 0.0;
        for_each_range_m<D>(L, x, a.reach[s], [&](int b, int e) {
            for (int j = b; j < e; ++j) {
                double z[3];
#pragma unroll
                for (int t = 0; t < D; ++t) z[t] = L.x[t][j];
                const double r2 = dist2_nofma<D>(x, z);
                if (r2 < a.delta2) sum = fma(wendland<K>(sqrt(r2) * a.inv_delta), y[j], sum);
            }
        });
        acc = fma(a.scale, sum, acc);
    }
    a.out[i] = acc;
}

__global__ void k_dot_partial(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                              double *__restrict__ part) {
    __shared__ double red[NT / 32 + 2];
    double t = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
        t = fma(a[i], b[i], t);
    t = block_sum<NT>(t, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_sum_partials(const double *__restrict__ part, int np, double *__restrict__ out) {
    __shared__ double red[NT / 32 + 2];
    double t = 0.0;
    for (int i = threadIdx.x; i < np; i += NT) t += part[i];
    t = block_sum<NT>(t, red);
    if (threadIdx.x == 0) *out = t;
}

__global__ void k_scale(double *v, double s, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i < n) v[i] *= s;
}

__global__ void k_pack(int64_t n, int d, const double *__restrict__ x0, const double *__restrict__ x1,
                       const double *__restrict__ x2, const double *__restrict__ c,
                       double4 *__restrict__ rec) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    rec[i] = d == 3 ? make_double4(x0[i], x1[i], x2[i], c[i]) : make_double4(x0[i], x1[i], c[i], 0.0);
}

__global__ void k_fpack(int64_t n, int d, const double *__restrict__ x0, const double *__restrict__ x1,
                        const double *__restrict__ x2, double lo0, double lo1, double lo2,
                        float4 *__restrict__ frec) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    frec[i] = make_float4((float)(x0[i] - lo0), (float)(x1[i] - lo1), d == 3 ? (float)(x2[i] - lo2) : 0.f, 0.f);
}
}  // namespace

void pack_frecords(int64_t n, int d, const double *xs, const double *lo, float4 *frec, cudaStream_t st,
                   int *launches) {
    if (n == 0) return;
    k_fpack<<<ceil_div_u(n, NT), NT, 0, st>>>(n, d, xs, xs + n, d == 3 ? xs + 2 * n : nullptr, lo[0], lo[1],
                                             d == 3 ? lo[2] : 0.0, frec);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

// Conservative FP32 prefilter threshold: with coordinates
// stored as float(x - lo), |x - lo| <= M for every pair that can be within
// delta, each float difference is off by at most e = 2^-24 (2M + delta) + tiny,
// so a pair with r < delta has r_f <= delta + sqrt(d) e and, after the float
// sum of squares, r2_f < (delta + sqrt(d) e)^2 (1 + 8 2^-24).  Any candidate
// with r2_f >= that bound is outside the support for sure; the survivors get
// the exact FP64 test.
float prefilter_threshold(double delta, double M, int d) {
    const double u = std::ldexp(1.0, -24);
    const double e = u * (2.0 * M + delta) * (1.0 + 1e-6) + std::ldexp(1.0, -60);
    const double t = (delta + std::sqrt((double)d) * e) * (delta + std::sqrt((double)d) * e) * (1.0 + 8.0 * u);
    float f = (float)t;
    if ((double)f < t) f = std::nextafter(f, INFINITY);
    return std::nextafter(f, INFINITY);
}

// The per-thread kernels (k_gather, k_gather_m, k_mf_spmv) are the default;
// MSK_GATHER_WARP=1 selects the warp-cooperative ones (wscan.cuh; same bits).
// Same-box A/B on C3: B products 5.23 ms per-thread vs 6.2-7.6
// warp (broadcast threshold 0 .. 4 x 3^d cells), evaluation 5.95 vs 7.0-8.2 --
// the broadcast scan costs more instructions than the loads it saves.
bool gather_v1() {
    static const bool v1 = getenv("MSK_GATHER_WARP") == nullptr || getenv("MSK_GATHER_V1") != nullptr;
    return v1;
}

void gather(const GatherArgs &a, cudaStream_t st, int *launches) {
    if (a.nt == 0) return;
    if (!gather_v1()) {
        const unsigned nbw = ceil_div_u(a.nt, NTW);
#define MSK_GW(DD, KK) k_gather_w<DD, KK><<<nbw, NTW, 0, st>>>(a)
        if (a.d == 2) {
            if (a.k == 0) MSK_GW(2, 0); else if (a.k == 1) MSK_GW(2, 1); else MSK_GW(2, 2);
        } else {
            if (a.k == 0) MSK_GW(3, 0); else if (a.k == 1) MSK_GW(3, 1); else MSK_GW(3, 2);
        }
#undef MSK_GW
        MSK_CHECK_LAUNCH();
        if (launches) *launches += 1;
        return;
    }
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

void gather_multi(const GatherMArgs &a, cudaStream_t st, int *launches) {
    if (a.nt == 0) return;
    unsigned nb = ceil_div_u(a.nt, NT);
    if (a.R != 2 && a.R != 4) throw Error(1, "gather_multi: R must be 2 or 4");
    const bool v1 = gather_v1();
    const unsigned nbw = ceil_div_u(a.nt, NTW);
#define MSK_GM(DD, KK, RR)                                               \
    do {                                                                 \
        if (v1) k_gather_m<DD, KK, RR><<<nb, NT, 0, st>>>(a);            \
        else k_gather_mw<DD, KK, RR><<<nbw, NTW, 0, st>>>(a);            \
    } while (0)
#define MSK_GMK(DD, RR)                                                                  \
    do {                                                                               \
        if (a.k == 0) MSK_GM(DD, 0, RR); else if (a.k == 1) MSK_GM(DD, 1, RR); else MSK_GM(DD, 2, RR); \
    } while (0)
    if (a.d == 2) { if (a.R == 2) MSK_GMK(2, 2); else MSK_GMK(2, 4); }
    else { if (a.R == 2) MSK_GMK(3, 2); else MSK_GMK(3, 4); }
#undef MSK_GMK
#undef MSK_GM
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void gather_t(const GatherTArgs &a, cudaStream_t st, int *launches) {
    if (a.nt == 0 || a.nsrc == 0) return;
    unsigned nb = ceil_div_u(a.nt, NT);
#define MSK_GT(DD, KK) k_gather_t<DD, KK><<<nb, NT, 0, st>>>(a)
    if (a.d == 2) {
        if (a.k == 0) MSK_GT(2, 0); else if (a.k == 1) MSK_GT(2, 1); else MSK_GT(2, 2);
    } else {
        if (a.k == 0) MSK_GT(3, 0); else if (a.k == 1) MSK_GT(3, 1); else MSK_GT(3, 2);
    }
#undef MSK_GT
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

// scratch: >= 297 doubles
double dev_dot(const double *a, const double *b, int64_t n, double *scratch, cudaStream_t st) {
    constexpr int NB = 296;  // fixed grid: a fixed summation tree
    k_dot_partial<<<NB, NT, 0, st>>>(a, b, n, scratch);
    MSK_CHECK_LAUNCH();
    k_sum_partials<<<1, NT, 0, st>>>(scratch, NB, scratch + NB);
    MSK_CHECK_LAUNCH();
    double s = 0.0;
    MSK_CUDA(cudaMemcpyAsync(&s, scratch + NB, sizeof s, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    return s;
}

void dev_scale(double *v, double s, int64_t n, cudaStream_t st) {
    if (n == 0) return;
    k_scale<<<ceil_div_u(n, NT), NT, 0, st>>>(v, s, n);
    MSK_CHECK_LAUNCH();
}

void pack_records(int64_t n, int d, const double *xs, const double *coef, double4 *rec,
                  cudaStream_t st, int *launches) {
    if (n == 0) return;
    k_pack<<<ceil_div_u(n, NT), NT, 0, st>>>(n, d, xs, xs + n, d == 3 ? xs + 2 * n : nullptr, coef, rec);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

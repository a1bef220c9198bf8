// misc.cu -- permutations between caller order and spatial order.
#include <string.h>

#include "kernels.cuh"

namespace msk {

namespace {
constexpr int NT = 256;
__global__ void k_pgather(int64_t n, const double *__restrict__ src, const int32_t *__restrict__ perm,
                          double *__restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}
__global__ void k_pscatter(int64_t n, const double *__restrict__ src, const int32_t *__restrict__ perm,
                           double *__restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i < n) dst[perm[i]] = src[i];
}
// order-preserving map of doubles to unsigned integers (exact min / max)
__device__ __forceinline__ unsigned long long ord_key(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_minmax(int64_t n, int d, const double *__restrict__ pts, unsigned long long *mm) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        for (int a = 0; a < d; ++a) {
            unsigned long long k = ord_key(pts[i * d + a]);
            lo[a] = k < lo[a] ? k : lo[a];
            hi[a] = k > hi[a] ? k : hi[a];
        }
    }
    for (int a = 0; a < d; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, lo[a], o);
            lo[a] = t < lo[a] ? t : lo[a];
            t = __shfl_xor_sync(0xffffffffu, hi[a], o);
            hi[a] = t > hi[a] ? t : hi[a];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&mm[a], lo[a]);
            atomicMax(&mm[3 + a], hi[a]);
        }
    }
}
}  // namespace

void minmax_points(int64_t n, int d, const double *pts, unsigned long long *mm, cudaStream_t st,
                   int *launches) {
    if (n == 0) return;
    int64_t nb = (n + NT - 1) / NT;
    k_minmax<<<(unsigned)(nb < 1184 ? nb : 1184), NT, 0, st>>>(n, d, pts, mm);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

double ord_key_to_double(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    memcpy(&v, &b, sizeof v);
    return v;
}

void permute_gather(int64_t n, const double *src, const int32_t *perm, double *dst, cudaStream_t st,
                    int *launches) {
    if (n == 0) return;
    k_pgather<<<ceil_div_u(n, NT), NT, 0, st>>>(n, src, perm, dst);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void permute_scatter(int64_t n, const double *src, const int32_t *perm, double *dst, cudaStream_t st,
                     int *launches) {
    if (n == 0) return;
    k_pscatter<<<ceil_div_u(n, NT), NT, 0, st>>>(n, src, perm, dst);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

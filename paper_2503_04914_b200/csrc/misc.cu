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

// Bounding box of n row-major d-dimensional points as ordered keys (exact).
// The array is read as flat doubles (coalesced); a thread's stride is a
// multiple of d, so each thread sees one axis only.
__global__ void k_minmax(int64_t n, int d, const double *__restrict__ pts, unsigned long long *mm) {
    __shared__ unsigned long long slo[3], shi[3];
    if (threadIdx.x < 3) {
        slo[threadIdx.x] = ~0ull;
        shi[threadIdx.x] = 0ull;
    }
    __syncthreads();
    const int64_t total = n * d;
    const int64_t nthreads = (int64_t)gridDim.x * NT;
    const int64_t stride = nthreads - nthreads % d;  // multiple of d
    const int64_t g = (int64_t)blockIdx.x * NT + threadIdx.x;
    unsigned long long lo = ~0ull, hi = 0ull;
    if (g < stride) {
        for (int64_t k = g; k < total; k += stride) {
            const unsigned long long key = ord_key(pts[k]);
            lo = key < lo ? key : lo;
            hi = key > hi ? key : hi;
        }
        const int a = (int)(g % d);
        atomicMin(&slo[a], lo);
        atomicMax(&shi[a], hi);
    }
    __syncthreads();
    if (threadIdx.x < d) {
        atomicMin(&mm[threadIdx.x], slo[threadIdx.x]);
        atomicMax(&mm[3 + threadIdx.x], shi[threadIdx.x]);
    }
}
__global__ void k_sum_i32(int64_t n, const int32_t *__restrict__ v, unsigned long long *out) {
    unsigned long long t = 0;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
        t += (unsigned long long)(unsigned)v[i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, t);
}
}  // namespace

// sum of n non-negative int32 values (host result)
int64_t sum_i32(const int32_t *v, int64_t n, cudaStream_t st) {
    unsigned long long *d = nullptr, h = 0;
    MSK_CUDA(cudaMallocAsync((void **)&d, sizeof h, st));
    MSK_CUDA(cudaMemsetAsync(d, 0, sizeof h, st));
    if (n > 0) {
        const int64_t nb = (n + NT - 1) / NT;
        k_sum_i32<<<(unsigned)(nb < 1184 ? nb : 1184), NT, 0, st>>>(n, v, d);
        MSK_CHECK_LAUNCH();
    }
    MSK_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    MSK_CUDA(cudaFreeAsync(d, st));
    return (int64_t)h;
}

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

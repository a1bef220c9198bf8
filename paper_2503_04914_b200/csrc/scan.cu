// scan.cu -- device-wide exclusive prefix sum (reduce-then-scan, 3 launches
// per recursion level).  Used for cell ranges (int32) and CSR row pointers
// (int64).  Deterministic (integer arithmetic).
#include "kernels.cuh"

namespace msk {

namespace {
constexpr int SNT = 512;            // threads per block
constexpr int SIPT = 8;             // items per thread
constexpr int SITEMS = SNT * SIPT;  // items per block

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// exclusive scan of one value per thread across the block; returns the
// exclusive prefix and writes the block total to *total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *smem, T *total) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T incl = warp_incl_scan(v);
    if (lane == 31) smem[w] = incl;
    __syncthreads();
    if (w == 0) {
        T s = lane < SNT / 32 ? smem[lane] : T(0);
        T si = warp_incl_scan(s);
        if (lane < SNT / 32) smem[lane] = si - s;
        if (lane == SNT / 32 - 1) smem[SNT / 32] = si;
    }
    __syncthreads();
    T r = smem[w] + incl - v;
    *total = smem[SNT / 32];
    __syncthreads();
    return r;
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(SNT) k_scan_reduce(const TI *__restrict__ in, int64_t n,
                                                     TO *__restrict__ sums) {
    __shared__ TO sm[SNT / 32 + 1];
    int64_t base = (int64_t)blockIdx.x * SITEMS + (int64_t)threadIdx.x * SIPT;
    TO s = 0;
#pragma unroll
    for (int i = 0; i < SIPT; ++i)
        if (base + i < n) s += (TO)in[base + i];
    TO tot;
    block_excl_scan<TO>(s, sm, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// out[i] = offs[block] + exclusive prefix within block; out[n] = total when
// the block holds element n-1 (offs == nullptr means a single block).
template <typename TI, typename TO>
__global__ void __launch_bounds__(SNT) k_scan_apply(const TI *__restrict__ in, int64_t n,
                                                    TO *__restrict__ out,
                                                    const TO *__restrict__ offs) {
    __shared__ TO sm[SNT / 32 + 1];
    int64_t base = (int64_t)blockIdx.x * SITEMS + (int64_t)threadIdx.x * SIPT;
    TO v[SIPT];
    TO s = 0;
#pragma unroll
    for (int i = 0; i < SIPT; ++i) {
        v[i] = base + i < n ? (TO)in[base + i] : TO(0);
        s += v[i];
    }
    TO tot;
    TO pre = block_excl_scan<TO>(s, sm, &tot);
    TO off = offs ? offs[blockIdx.x] : TO(0);
    TO run = off + pre;
#pragma unroll
    for (int i = 0; i < SIPT; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (base <= n - 1 && n - 1 < base + SIPT) out[n] = run;  // run = total after last element
}

template <typename TI, typename TO>
void scan_impl(const TI *in, int64_t n, TO *out, cudaStream_t st, int *launches) {
    if (n <= 0) {
        MSK_CUDA(cudaMemsetAsync(out, 0, sizeof(TO), st));
        return;
    }
    int64_t nb = (n + SITEMS - 1) / SITEMS;
    if (nb == 1) {
        k_scan_apply<TI, TO><<<1, SNT, 0, st>>>(in, n, out, nullptr);
        MSK_CHECK_LAUNCH();
        if (launches) *launches += 1;
        return;
    }
    TO *sums = nullptr;
    MSK_CUDA(cudaMallocAsync((void **)&sums, sizeof(TO) * (size_t)(nb + 1), st));
    k_scan_reduce<TI, TO><<<(unsigned)nb, SNT, 0, st>>>(in, n, sums);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
    scan_impl<TO, TO>(sums, nb, sums, st, launches);  // in-place exclusive scan of block sums
    k_scan_apply<TI, TO><<<(unsigned)nb, SNT, 0, st>>>(in, n, out, sums);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
    MSK_CUDA(cudaFreeAsync(sums, st));
}
}  // namespace

void exclusive_scan_i32(const int32_t *in, int64_t n, int32_t *out, cudaStream_t st, int *launches) {
    scan_impl<int32_t, int32_t>(in, n, out, st, launches);
}
void exclusive_scan_i64(const int32_t *in, int64_t n, int64_t *out, cudaStream_t st, int *launches) {
    scan_impl<int32_t, int64_t>(in, n, out, st, launches);
}

}  // namespace msk

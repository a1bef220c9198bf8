// common.cuh -- shared device helpers of libmsk (sm_100a, FP64).
//
// Nothing here is shared with oracle/ (which is independent test code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <nvtx3/nvToolsExt.h>

#include <stdexcept>
#include <string>

namespace msk {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string &m) : std::runtime_error(m), status(s) {}
};

#define MSK_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::msk::Error(e_ == cudaErrorMemoryAllocation ? 2 : 3,                   \
                               std::string(#call) + ": " + cudaGetErrorString(e_));       \
    } while (0)

#define MSK_CHECK_LAUNCH() MSK_CUDA(cudaGetLastError())

// Device-side bounds checks of the bounds build (python -m
// paper_2503_04914_b200.build --bounds -> libmsk_bounds.so; the stand-in for
// compute-sanitizer memcheck, which this GPU pool does not offer): a failed
// check prints its location and traps (the launch fails with an error).
#ifdef MSK_BOUNDS
#include <cstdio>
#define MSK_DASSERT(c)                                                                      \
    do {                                                                                     \
        if (!(c)) {                                                                          \
            printf("MSK_DASSERT failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,   \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                                   \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define MSK_DASSERT(c) \
    do {               \
    } while (0)
#endif

// MSK_DEBUG_SYNC=1: synchronise after each orchestrated launch and name the
// failing step (diagnostics for device faults; off by default).
inline void debug_sync(cudaStream_t st, const char *what) {
    static int on = -1;
    if (on < 0) on = getenv("MSK_DEBUG_SYNC") != nullptr;
    if (!on) return;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw Error(3, std::string(what) + ": " + cudaGetErrorString(e));
}

// NVTX range on the calling host thread (every C-ABI call, every level of a
// solve, the B products / CG / evaluation chunks): profilers attribute the
// kernels launched inside it (ncu --nvtx --nvtx-include "msk_solve/level 2/CG/").
// NVTX v3 is header-only; without a tool attached a push/pop is a no-op call.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    explicit NvtxRange(const std::string &name) { nvtxRangePushA(name.c_str()); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

constexpr int kMaxLevels = 16;

// ---------------------------------------------------------------- geometry
// Grid of one level: cell side c >= delta (1 + 2^-20) along the leading axes
// and c / zf along the LAST axis (z in 3-D, y in 2-D; zf a power of two, so
// inv[last] = zf * inv_cell exactly); row-major x-major keys key = (ix * ny +
// iy) * nz + iz (nz = 1 in 2-D).  A pair with r < delta lies in cells whose
// indices differ by at most 1 along the leading axes and by at most zf along
// the last one (the thin last-axis cells trim each of
// the 3^(d-1) contiguous candidate ranges from 3 delta to (2 zf + 1) delta / zf).
struct Grid {
    double lo[3];
    double inv_cell;  // 1 / c (leading axes)
    double inv[3];    // per axis: inv_cell, or zf * inv_cell on the last axis
    int zf;           // last-axis refinement (1 = cubic cells)
    int64_t dim[3];   // nx, ny, nz (nz = 1 for d = 2)
    int64_t ncells;
};

// One level as seen by the device kernels (points in spatial order, SoA).
struct LevelView {
    int64_t n;
    const double *x[3];         // SoA coordinates, spatial order
    const int32_t *cell_start;  // ncells + 1
    Grid g;
    double delta2;              // delta * delta, computed once on the host (reading C-4)
    double inv_delta;           // 1 / delta
    double scale;               // delta^-d
    const double *coef;         // coefficient vector (spatial order) for gathers
    const double4 *rec;         // packed (x, y, z, coef) records (2-D: (x, y, coef, 0)) for gathers
    const float4 *frec;         // FP32 coordinates relative to g.lo (conservative prefilter)
    float fthr;                 // prefilter threshold: r2_f >= fthr  =>  r^2 >= delta^2 for sure
    float bcells;               // warp scans (wscan.cuh): broadcast when the warp's box has <= bcells cells
};

// squared distance, left to right, round-to-nearest, no FMA (reading C-4)
template <int D>
__device__ __forceinline__ double dist2_nofma(const double *a, const double *b) {
    double t = __dsub_rn(a[0], b[0]);
    double s = __dmul_rn(t, t);
    t = __dsub_rn(a[1], b[1]);
    s = __dadd_rn(s, __dmul_rn(t, t));
    if (D == 3) {
        t = __dsub_rn(a[2], b[2]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

// Wendland phi_{d,k}(r) for d in {2,3}: l = floor(d/2) + k + 1 = k + 2
// (reading C-3; P:1275 for k = 1).  Valid for 0 <= r < 1.
template <int K>
__device__ __forceinline__ double wendland(double r) {
    double s = fmax(1.0 - r, 0.0);  // r*inv_delta may round to 1 + ulp at the boundary
    double s2 = s * s;
    if (K == 0) return s2;
    if (K == 1) return (s2 * s2) * fma(4.0, r, 1.0);
    // K == 2
    double s6 = s2 * s2 * s2;
    return s6 * fma(fma(35.0, r, 18.0), r, 3.0) * (1.0 / 3.0);
}

// cell coordinate of x along axis a, not clamped
__device__ __forceinline__ int64_t cell_coord(const Grid &g, int a, double x) {
    return (int64_t)floor(__dmul_rn(__dsub_rn(x, g.lo[a]), g.inv[a]));
}

// --------------------------------------------------------- reductions
// Deterministic block sum: fixed xor-shuffle tree per warp, warp partials
// summed in warp order by warp 0.  Result valid in all threads.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *smem /* >= NT/32 + 1 */) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) smem[w] = v;
    __syncthreads();
    if (w == 0) {
        double t = lane < NT / 32 ? smem[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) smem[NT / 32] = t;
    }
    __syncthreads();
    return smem[NT / 32];
}

// R independent block sums with block_sum's tree per value (bit-identical to R
// block_sum calls); smem >= R * (NT/32 + 1).  Results returned in v.
template <int NT, int R>
__device__ __forceinline__ void block_sum_r(double (&v)[R], double *smem) {
    constexpr int W = NT / 32 + 1;
#pragma unroll
    for (int r = 0; r < R; ++r)
        for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) smem[r * W + w] = v[r];
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double t = lane < NT / 32 ? smem[r * W + lane] : 0.0;
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) smem[r * W + NT / 32] = t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = smem[r * W + NT / 32];
}

template <int NT>
__device__ __forceinline__ long long block_sum_ll(long long v, long long *smem) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) smem[w] = v;
    __syncthreads();
    if (w == 0) {
        long long t = lane < NT / 32 ? smem[lane] : 0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) smem[NT / 32] = t;
    }
    __syncthreads();
    return smem[NT / 32];
}

inline unsigned ceil_div_u(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace msk

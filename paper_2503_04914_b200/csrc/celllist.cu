// celllist.cu -- a1: uniform-grid cell list per level (replaces the paper's
// kd-tree).  Counting sort by cell key: histogram -> exclusive
// scan (cell ranges) -> scatter -> per-cell insertion sort by caller index
// (stable order, so the whole build is deterministic) -> SoA gather.
#include "kernels.cuh"

namespace msk {

namespace {
constexpr int NT = 256;

template <int D>
__device__ __forceinline__ int64_t point_key(const Grid &g, const double *p) {
    int64_t c[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
        int64_t v = cell_coord(g, a, p[a]);
        v = v < 0 ? 0 : (v >= g.dim[a] ? g.dim[a] - 1 : v);
        c[a] = v;
    }
    return (c[0] * g.dim[1] + c[1]) * g.dim[2] + c[2];
}

template <int D>
__global__ void __launch_bounds__(NT) k_keys(int64_t n, const double *__restrict__ pts, Grid g,
                                             int64_t *__restrict__ key, int32_t *__restrict__ count) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    double p[3];
#pragma unroll
    for (int a = 0; a < D; ++a) p[a] = pts[i * D + a];
    int64_t k = point_key<D>(g, p);
    key[i] = k;
    atomicAdd(&count[k], 1);
}

__global__ void __launch_bounds__(NT) k_scatter(int64_t n, const int64_t *__restrict__ key,
                                                const int32_t *__restrict__ cell_start,
                                                int32_t *__restrict__ fill,
                                                int32_t *__restrict__ perm) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    int64_t k = key[i];
    int pos = cell_start[k] + atomicAdd(&fill[k], 1);
    perm[pos] = (int32_t)i;
}

// insertion sort of each cell's slice of perm (cells hold O(1) points)
__global__ void __launch_bounds__(NT) k_cell_sort(int64_t ncells, const int32_t *__restrict__ cs,
                                                  int32_t *__restrict__ perm) {
    int64_t c = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (c >= ncells) return;
    int b = cs[c], e = cs[c + 1];
    for (int i = b + 1; i < e; ++i) {
        int32_t v = perm[i];
        int j = i - 1;
        while (j >= b && perm[j] > v) {
            perm[j + 1] = perm[j];
            --j;
        }
        perm[j + 1] = v;
    }
}

template <int D>
__global__ void __launch_bounds__(NT) k_gather_sorted(int64_t n, const double *__restrict__ pts,
                                                      const int32_t *__restrict__ perm,
                                                      const int64_t *__restrict__ key_orig,
                                                      double *x0, double *x1, double *x2,
                                                      int64_t *__restrict__ key_sorted) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    int64_t src = perm[i];
    x0[i] = pts[src * D + 0];
    x1[i] = pts[src * D + 1];
    if (D == 3) x2[i] = pts[src * D + 2];
    if (key_sorted) key_sorted[i] = key_orig[src];
}
}  // namespace

void build_cell_list(int d, int64_t n, const double *pts_rm, const Grid &g, bool stable,
                     const CellListOut &out, cudaStream_t st, int *launches) {
    int64_t *key = nullptr;
    int32_t *count = nullptr;
    MSK_CUDA(cudaMallocAsync((void **)&key, sizeof(int64_t) * (size_t)n, st));
    MSK_CUDA(cudaMallocAsync((void **)&count, sizeof(int32_t) * (size_t)g.ncells, st));
    MSK_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t) * (size_t)g.ncells, st));
    unsigned nb = ceil_div_u(n, NT);
    if (d == 2) k_keys<2><<<nb, NT, 0, st>>>(n, pts_rm, g, key, count);
    else k_keys<3><<<nb, NT, 0, st>>>(n, pts_rm, g, key, count);
    MSK_CHECK_LAUNCH();
    exclusive_scan_i32(count, g.ncells, out.cell_start, st, launches);
    MSK_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t) * (size_t)g.ncells, st));
    k_scatter<<<nb, NT, 0, st>>>(n, key, out.cell_start, count, out.perm);
    MSK_CHECK_LAUNCH();
    if (stable) {
        k_cell_sort<<<ceil_div_u(g.ncells, NT), NT, 0, st>>>(g.ncells, out.cell_start, out.perm);
        MSK_CHECK_LAUNCH();
        if (launches) *launches += 1;
    }
    if (d == 2)
        k_gather_sorted<2><<<nb, NT, 0, st>>>(n, pts_rm, out.perm, key, out.xs[0], out.xs[1],
                                              nullptr, out.keys);
    else
        k_gather_sorted<3><<<nb, NT, 0, st>>>(n, pts_rm, out.perm, key, out.xs[0], out.xs[1],
                                              out.xs[2], out.keys);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 3;
    MSK_CUDA(cudaFreeAsync(count, st));
    MSK_CUDA(cudaFreeAsync(key, st));
}

}  // namespace msk

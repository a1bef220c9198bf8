// neighbors.cuh -- candidate enumeration over a level's cell list.
//
// For a target x, the candidates are the points of the cells whose indices
// differ from x's (unclamped) cell by at most one per axis, intersected with
// the grid.  With row-major keys the cells along the last axis are
// contiguous, so a 3-D query is 9 contiguous ranges and a 2-D query 3.
// Visiting ranges in increasing key order yields candidates in increasing
// spatial index.
#pragma once
#include "common.cuh"

namespace msk {

template <int D, typename F>
__device__ __forceinline__ void for_each_range(const LevelView &L, const double *x, F &&f) {
    int64_t c[3];
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = cell_coord(L.g, a, x[a]);
    const int64_t la = D - 1;
    int64_t lo_last = c[la] - 1 < 0 ? 0 : c[la] - 1;
    int64_t hi_last = c[la] + 1 >= L.g.dim[la] ? L.g.dim[la] - 1 : c[la] + 1;
    if (lo_last > hi_last) return;
    int64_t x0 = c[0] - 1 < 0 ? 0 : c[0] - 1;
    int64_t x1 = c[0] + 1 >= L.g.dim[0] ? L.g.dim[0] - 1 : c[0] + 1;
    if (D == 2) {
        for (int64_t ix = x0; ix <= x1; ++ix) {
            int64_t kb = ix * L.g.dim[1];
            f(L.cell_start[kb + lo_last], L.cell_start[kb + hi_last + 1]);
        }
    } else {
        int64_t y0 = c[1] - 1 < 0 ? 0 : c[1] - 1;
        int64_t y1 = c[1] + 1 >= L.g.dim[1] ? L.g.dim[1] - 1 : c[1] + 1;
        for (int64_t ix = x0; ix <= x1; ++ix)
            for (int64_t iy = y0; iy <= y1; ++iy) {
                int64_t kb = (ix * L.g.dim[1] + iy) * L.g.dim[2];
                f(L.cell_start[kb + lo_last], L.cell_start[kb + hi_last + 1]);
            }
    }
}

// Same enumeration with a reach of m cells per axis (radius up to m cell
// sides): used for the truncation radius T q_l of the thresholded factor,
// which spans several cells of the level grid.
template <int D, typename F>
__device__ __forceinline__ void for_each_range_m(const LevelView &L, const double *x, int m, F &&f) {
    int64_t c[3];
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = cell_coord(L.g, a, x[a]);
    const int64_t la = D - 1;
    int64_t lo_last = c[la] - m < 0 ? 0 : c[la] - m;
    int64_t hi_last = c[la] + m >= L.g.dim[la] ? L.g.dim[la] - 1 : c[la] + m;
    if (lo_last > hi_last) return;
    int64_t x0 = c[0] - m < 0 ? 0 : c[0] - m;
    int64_t x1 = c[0] + m >= L.g.dim[0] ? L.g.dim[0] - 1 : c[0] + m;
    if (D == 2) {
        for (int64_t ix = x0; ix <= x1; ++ix) {
            int64_t kb = ix * L.g.dim[1];
            f(L.cell_start[kb + lo_last], L.cell_start[kb + hi_last + 1]);
        }
    } else {
        int64_t y0 = c[1] - m < 0 ? 0 : c[1] - m;
        int64_t y1 = c[1] + m >= L.g.dim[1] ? L.g.dim[1] - 1 : c[1] + m;
        for (int64_t ix = x0; ix <= x1; ++ix)
            for (int64_t iy = y0; iy <= y1; ++iy) {
                int64_t kb = (ix * L.g.dim[1] + iy) * L.g.dim[2];
                f(L.cell_start[kb + lo_last], L.cell_start[kb + hi_last + 1]);
            }
    }
}

}  // namespace msk

// neighbors.cuh -- candidate enumeration over a level's cell list.
//
// For a target x, the candidates are the points of the cells whose indices
// differ from x's (unclamped) cell by at most one along the leading axes and
// at most zf along the last (thin) axis, intersected with the grid.  With row-major keys the cells along the last axis are
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
    const int64_t la = D - 1, z = L.g.zf;  // last axis: zf thin cells span delta
    int64_t lo_last = c[la] - z < 0 ? 0 : c[la] - z;
    int64_t hi_last = c[la] + z >= L.g.dim[la] ? L.g.dim[la] - 1 : c[la] + z;
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

// The exact neighbours {j : r^2(x, x_j) < delta^2} (no-FMA r^2, reading C-4)
// of x among cols' points, in ascending j: f(j, r2) per hit.  Candidates pass
// a conservative FP32 prefilter on the 16-byte records cols.frec first (see
// prefilter_threshold in gather.cu: it never rejects a true neighbour), the
// survivors are buffered (HM per thread, keeps the warp convergent) and get
// the exact FP64 test.  Requires cols.frec (relative to cols.g.lo).
// ABOVE: only candidates j >= jmin (the ranges clipped; a symmetric count
// visits each pair once, from its lower index).
template <int D, int HM = 32, bool ABOVE = false, typename F>
__device__ __forceinline__ void for_each_hit(const LevelView &cols, const double *x, F &&f, int jmin = 0) {
    float xf[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < D; ++a) xf[a] = (float)(x[a] - cols.g.lo[a]);
    const float fthr = cols.fthr;
    const double d2 = cols.delta2;
    const float4 *__restrict__ frec = cols.frec;
    int hl[HM];
    int nh = 0;
    auto flush = [&]() {
        for (int h = 0; h < nh; ++h) {
            const int j = hl[h];
            double y[3];
#pragma unroll
            for (int a = 0; a < D; ++a) y[a] = cols.x[a][j];
            const double r2 = dist2_nofma<D>(x, y);
            if (r2 < d2) f(j, r2);
        }
        nh = 0;
    };
    for_each_range<D>(cols, x, [&](int b, int e) {
        if (ABOVE && b < jmin) b = jmin;
        int j = b;
        for (; j + 3 < e; j += 4) {  // four candidates per trip (independent loads)
            const float4 F0 = frec[j], F1 = frec[j + 1], F2 = frec[j + 2], F3 = frec[j + 3];
            const float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
            const float a1 = xf[0] - F1.x, b1 = xf[1] - F1.y, c1 = xf[2] - F1.z;
            const float a2 = xf[0] - F2.x, b2 = xf[1] - F2.y, c2 = xf[2] - F2.z;
            const float a3 = xf[0] - F3.x, b3 = xf[1] - F3.y, c3 = xf[2] - F3.z;
            const bool h0 = fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr;
            const bool h1 = fmaf(c1, c1, fmaf(b1, b1, a1 * a1)) < fthr;
            const bool h2 = fmaf(c2, c2, fmaf(b2, b2, a2 * a2)) < fthr;
            const bool h3 = fmaf(c3, c3, fmaf(b3, b3, a3 * a3)) < fthr;
            if (nh + 4 > HM) flush();
            if (h0) hl[nh++] = j;
            if (h1) hl[nh++] = j + 1;
            if (h2) hl[nh++] = j + 2;
            if (h3) hl[nh++] = j + 3;
        }
        for (; j + 1 < e; j += 2) {  // two candidates per trip (independent loads)
            const float4 F0 = frec[j], F1 = frec[j + 1];
            const float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
            const float a1 = xf[0] - F1.x, b1 = xf[1] - F1.y, c1 = xf[2] - F1.z;
            const bool h0 = fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr;
            const bool h1 = fmaf(c1, c1, fmaf(b1, b1, a1 * a1)) < fthr;
            if (nh + 2 > HM) flush();
            if (h0) hl[nh++] = j;
            if (h1) hl[nh++] = j + 1;
        }
        if (j < e) {
            const float4 F0 = frec[j];
            const float a0 = xf[0] - F0.x, b0 = xf[1] - F0.y, c0 = xf[2] - F0.z;
            if (nh + 1 > HM) flush();
            if (fmaf(c0, c0, fmaf(b0, b0, a0 * a0)) < fthr) hl[nh++] = j;
        }
    });
    flush();
}

// Same enumeration with a reach of m cells along the leading axes (radius
// below m cell sides) and m * zf thin cells along the last one: used for the
// truncation radius T q_l of the thresholded factor, which spans several cells
// of the level grid.
template <int D, typename F>
__device__ __forceinline__ void for_each_range_m(const LevelView &L, const double *x, int m, F &&f) {
    int64_t c[3];
#pragma unroll
    for (int a = 0; a < D; ++a) c[a] = cell_coord(L.g, a, x[a]);
    const int64_t la = D - 1, mz = (int64_t)m * L.g.zf;
    int64_t lo_last = c[la] - mz < 0 ? 0 : c[la] - mz;
    int64_t hi_last = c[la] + mz >= L.g.dim[la] ? L.g.dim[la] - 1 : c[la] + mz;
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

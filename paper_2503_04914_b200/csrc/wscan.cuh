// wscan.cuh -- warp-cooperative candidate scan over one level's cell list,
// with the warp's neighbourhood staged in shared memory (a3 matrix-free
// SpMV, a5 B products, a9 evaluation; DESIGN.md §7 "Matrix-free kernel sums").
//
// A warp owns 32 consecutive targets (spatially sorted, so their cells are
// close).  Per level:
//   1. every lane computes its 3^d candidate cells (clamped, as
//      for_each_range); the warp reduces them to a box of cells;
//   2. if the box has at most LevelView::bcells cells (default 2.5 x 3^d) (the targets share cells:
//      every coarser source level), it is a few "columns" (3-D: (ix, iy);
//      2-D: ix) whose cells along the last axis are contiguous in key order,
//      i.e. ONE contiguous range of points each: the columns' cell_start rows
//      are staged in shared memory, then their FP32 prefilter records are
//      copied (cp.async, 16 B per lane) into a per-warp buffer, and EVERY lane
//      tests EVERY staged record (one broadcast LDS.128 serves the warp; the
//      loop is warp-uniform, so hit-list flushes are warp-uniform too);
//   3. otherwise (fine source levels: the targets span many cells) every lane
//      enumerates its own 3^d cells from global memory (through L1);
//   4. survivors of the conservative FP32 prefilter go to a per-lane hit list;
//      flush() runs the exact FP64 test (reading C-4) and the kernel
//      evaluation on them (caller-supplied).
// Candidates are visited in ascending spatial index in both modes (columns in
// key order, ranges ascending), and the broadcast mode's extra candidates all
// fail the exact test, so the hits and their order -- and the sums -- are
// those of the per-thread enumeration (for_each_range): bit-identical.
#pragma once
#include <climits>

#include "common.cuh"
#include "neighbors.cuh"
#include "tma.cuh"

namespace msk {
namespace wscan {

#ifndef MSK_WS_CAP
#define MSK_WS_CAP 256    // staged FP32 records per warp
#endif
#ifndef MSK_WS_HM
#define MSK_WS_HM 40      // hit-list capacity per lane (flushed when full)
#endif
#ifndef MSK_WS_CSCAP
#define MSK_WS_CSCAP 128  // staged cell_start entries per warp
#endif
constexpr int CAP = MSK_WS_CAP, HM = MSK_WS_HM, CSCAP = MSK_WS_CSCAP, MAXCOL = 32;

struct __align__(16) WarpSmem {
    float4 rec[CAP];        // staged prefilter records, columns concatenated
    int cs[CSCAP];          // cell_start rows of the box columns, (nz + 1) per column
    int colgb[MAXCOL];      // first global point index of each column
    int colfo[MAXCOL + 1];  // offset of each column in rec[] (+ total)
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// conservative FP32 prefilter (prefilter_threshold in gather.cu): false =>
// r^2 >= delta^2 for sure
__device__ __forceinline__ bool pre(const float *xf, const float4 &F, float thr) {
    const float a = xf[0] - F.x, b = xf[1] - F.y, c = xf[2] - F.z;
    return fmaf(c, c, fmaf(b, b, a * a)) < thr;
}

// One level for the warp.  x / xf: the lane's target (FP64, FP32 relative to
// the common origin); on: the lane has a target.  hl: the lane's hit list;
// flush(nh): process hl[0..nh) (ascending global index) in order.  Must be
// called by all 32 lanes (warp-collective).
//
// Mode by box size: at most L.bcells cells (the warp's targets share
// cells: coarse source levels) => broadcast from shared memory, flushes
// warp-uniform (all lanes flush together when any list is nearly full);
// otherwise every lane enumerates its own 3^d cells from global memory (L1).
template <int D, class Flush>
__device__ __forceinline__ void scan_level(const LevelView &L, const double *x, const float *xf, bool on,
                                           WarpSmem &W, int (&hl)[HM], Flush &&flush) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float thr = L.fthr;
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    bool valid = on;
    if (on) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int64_t c = cell_coord(L.g, a, x[a]);
            const int64_t rr = a == D - 1 ? L.g.zf : 1;  // thin last-axis cells
            const int64_t l = c - rr < 0 ? 0 : c - rr;
            const int64_t h = c + rr >= L.g.dim[a] ? L.g.dim[a] - 1 : c + rr;
            if (l > h) valid = false;
            else { lo[a] = (int)l; hi[a] = (int)h; }
        }
    }
    if (!valid) {
#pragma unroll
        for (int a = 0; a < 3; ++a) { lo[a] = INT_MAX; hi[a] = INT_MIN; }
    }
    int b0[3], b1[3];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        b0[a] = __reduce_min_sync(FULL, lo[a]);
        b1[a] = __reduce_max_sync(FULL, hi[a]);
    }
    if (b0[0] == INT_MAX) return;  // warp-uniform: no lane has candidates
    const int64_t nx = (int64_t)b1[0] - b0[0] + 1;
    const int64_t ny = D == 3 ? (int64_t)b1[1] - b0[1] + 1 : 1;
    const int zl = b0[D - 1];
    const int64_t nz = (int64_t)b1[D - 1] - zl + 1;
    int nh = 0;
    bool bc = nx * ny <= MAXCOL && nx * ny * (nz + 1) <= CSCAP && (float)(nx * ny * nz) <= L.bcells;
    if (bc) {  // warp-uniform
        const int ncol = (int)(nx * ny), w = (int)nz + 1, nyi = (int)ny;
        __syncwarp();  // the previous level's readers of W are done
        for (int t = lane; t < ncol * w; t += 32) {
            const int ci = t / w, z = t - ci * w;
            const int64_t ix = b0[0] + ci / nyi;
            const int64_t key = D == 3 ? (ix * L.g.dim[1] + (b0[1] + ci % nyi)) * L.g.dim[2] + zl + z
                                       : ix * L.g.dim[1] + zl + z;
            MSK_DASSERT(t < CSCAP && key >= 0 && key <= L.g.ncells);
            W.cs[t] = L.cell_start[key];
        }
        __syncwarp();
        int len = 0, gb = 0;
        if (lane < ncol) {
            gb = W.cs[lane * w];
            len = W.cs[lane * w + w - 1] - gb;
        }
        int inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        const int T = __shfl_sync(FULL, inc, 31);
        if (lane < ncol) {
            W.colgb[lane] = gb;
            W.colfo[lane] = inc - len;
        }
        if (lane == 0) W.colfo[ncol] = T;
        bc = T <= CAP;
        if (bc) {
            __syncwarp();
            for (int ci = 0; ci < ncol; ++ci) {
                const int g0 = W.colgb[ci], f0 = W.colfo[ci], n0 = W.colfo[ci + 1] - f0;
                for (int t = lane; t < n0; t += 32) {
                    MSK_DASSERT(f0 + t < CAP && g0 + t >= 0 && g0 + t < L.n);
                    cp_async16(&W.rec[f0 + t], &L.frec[g0 + t]);
                }
            }
            cp_async_wait_all();
            __syncwarp();
            // every lane tests every staged record (one broadcast LDS.128 per
            // record for the warp), in key order = ascending global index
            for (int ci = 0; ci < ncol; ++ci) {
                const int f1 = W.colfo[ci + 1], gadd = W.colgb[ci] - W.colfo[ci];
                int s = W.colfo[ci];
                for (; s + 3 < f1; s += 4) {
                    if (__any_sync(FULL, nh + 4 > HM)) {  // warp-uniform flush
                        if (nh) flush(nh);
                        nh = 0;
                    }
                    const float4 F0 = W.rec[s], F1 = W.rec[s + 1], F2 = W.rec[s + 2], F3 = W.rec[s + 3];
                    const bool h0 = valid && pre(xf, F0, thr), h1 = valid && pre(xf, F1, thr);
                    const bool h2 = valid && pre(xf, F2, thr), h3 = valid && pre(xf, F3, thr);
                    if (h0) hl[nh++] = s + gadd;
                    if (h1) hl[nh++] = s + 1 + gadd;
                    if (h2) hl[nh++] = s + 2 + gadd;
                    if (h3) hl[nh++] = s + 3 + gadd;
                }
                for (; s < f1; ++s) {
                    if (__any_sync(FULL, nh + 1 > HM)) {
                        if (nh) flush(nh);
                        nh = 0;
                    }
                    if (valid && pre(xf, W.rec[s], thr)) hl[nh++] = s + gadd;
                }
            }
        }
    }
    if (!bc && valid) {
        // the lane's own 3^d cells straight from global memory (through L1)
        const float4 *__restrict__ frec = L.frec;
        for_each_range<D>(L, x, [&](int b, int e) {
            int j = b;
            for (; j + 3 < e; j += 4) {
                const float4 F0 = frec[j], F1 = frec[j + 1], F2 = frec[j + 2], F3 = frec[j + 3];
                const bool h0 = pre(xf, F0, thr), h1 = pre(xf, F1, thr);
                const bool h2 = pre(xf, F2, thr), h3 = pre(xf, F3, thr);
                if (nh + 4 > HM) {
                    flush(nh);
                    nh = 0;
                }
                if (h0) hl[nh++] = j;
                if (h1) hl[nh++] = j + 1;
                if (h2) hl[nh++] = j + 2;
                if (h3) hl[nh++] = j + 3;
            }
            for (; j < e; ++j) {
                const bool h0 = pre(xf, frec[j], thr);
                if (nh + 1 > HM) {
                    flush(nh);
                    nh = 0;
                }
                if (h0) hl[nh++] = j;
            }
        });
    }
    if (nh) flush(nh);
    __syncwarp();
}

}  // namespace wscan
}  // namespace msk

// wscan.cuh -- warp-cooperative candidate scan over one level's cell list,
// with the warp's neighbourhood staged in shared memory (a3 matrix-free
// SpMV, a5 B products, a9 evaluation; DESIGN.md §7 "Matrix-free kernel sums").
//
// A warp owns 32 consecutive targets (spatially sorted, so their cells are
// close).  Per level:
//   1. every lane computes its 3^d candidate cells (clamped, as
//      for_each_range); the warp reduces them to a box of cells;
//   2. the box is a set of "columns" (3-D: (ix, iy); 2-D: ix) whose cells
//      along the last axis are contiguous in key order, so each column is ONE
//      contiguous range of points: the columns' cell_start rows are staged in
//      shared memory, then the FP32 prefilter records of every column are
//      bulk-copied (cp.async, 16 B per lane) into a per-warp buffer;
//   3. candidates are tested from shared memory, either
//        broadcast -- every lane tests every staged record (one LDS.128
//                     serves the warp; no divergence), when the box holds at
//                     most MSK_WS_BRATIO x the largest per-lane candidate
//                     count (coarse source levels: targets share cells), or
//        per lane  -- each lane tests its own 3^(d-1) column ranges (fine
//                     levels: the warp's targets span many cells);
//   4. survivors of the conservative FP32 prefilter go to a per-lane hit list
//      in shared memory; flush() runs the exact FP64 test (reading C-4) and
//      the kernel evaluation on them (caller-supplied).
// Candidates are visited in ascending spatial index in both modes (columns in
// key order, ranges ascending), and the broadcast mode's extra candidates all
// fail the exact test, so the hits and their order -- and the sums -- are
// those of the per-thread enumeration (for_each_range): bit-identical.
// A box that does not fit (too many columns, cells or records) falls back to
// the per-lane enumeration straight from global memory.
#pragma once
#include <climits>

#include "common.cuh"
#include "neighbors.cuh"
#include "tma.cuh"

namespace msk {
namespace wscan {

#ifndef MSK_WS_CAP
#define MSK_WS_CAP 384    // staged FP32 records per warp
#endif
#ifndef MSK_WS_HM
#define MSK_WS_HM 24      // hit-list capacity per lane (flushed when full)
#endif
#ifndef MSK_WS_CSCAP
#define MSK_WS_CSCAP 256  // staged cell_start entries per warp
#endif
#ifndef MSK_WS_BRATIO
#define MSK_WS_BRATIO 1.8f
#endif
constexpr int CAP = MSK_WS_CAP, HM = MSK_WS_HM, CSCAP = MSK_WS_CSCAP, MAXCOL = 32;

struct __align__(16) WarpSmem {
    float4 rec[CAP];      // staged prefilter records, columns concatenated
    int hl[HM * 32];      // hit lists, [slot][lane] (conflict-free)
    int cs[CSCAP];        // cell_start rows of the box columns, (nz + 1) per column
    int colgb[MAXCOL];    // first global point index of each column
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
// the common origin); on: the lane has a target.  flush(nh): process the
// lane's hits W.hl[h * 32 + lane], h < nh (ascending global index), in order.
// Must be called by all 32 lanes (warp-collective).
template <int D, class Flush>
__device__ __forceinline__ void scan_level(const LevelView &L, const double *x, const float *xf, bool on,
                                           WarpSmem &W, Flush &&flush) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float thr = L.fthr;
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    bool valid = on;
    if (on) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int64_t c = cell_coord(L.g, a, x[a]);
            const int64_t l = c - 1 < 0 ? 0 : c - 1;
            const int64_t h = c + 1 >= L.g.dim[a] ? L.g.dim[a] - 1 : c + 1;
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
    auto append = [&](int j) {
        if (nh == HM) {
            flush(nh);
            nh = 0;
        }
        W.hl[nh * 32 + lane] = j;
        ++nh;
    };
    // candidates [s0, s1) of the staged buffer; global index = s + gadd
    auto scan_range = [&](int s0, int s1, int gadd, bool ok) {
        int s = s0;
        for (; s + 3 < s1; s += 4) {
            const float4 F0 = W.rec[s], F1 = W.rec[s + 1], F2 = W.rec[s + 2], F3 = W.rec[s + 3];
            const bool h0 = ok && pre(xf, F0, thr), h1 = ok && pre(xf, F1, thr);
            const bool h2 = ok && pre(xf, F2, thr), h3 = ok && pre(xf, F3, thr);
            if (h0) append(s + gadd);
            if (h1) append(s + 1 + gadd);
            if (h2) append(s + 2 + gadd);
            if (h3) append(s + 3 + gadd);
        }
        for (; s < s1; ++s)
            if (ok && pre(xf, W.rec[s], thr)) append(s + gadd);
    };
    bool staged = nx * ny <= MAXCOL && nx * ny * (nz + 1) <= CSCAP;  // warp-uniform
    if (staged) {
        const int ncol = (int)(nx * ny), w = (int)nz + 1, nyi = (int)ny;
        __syncwarp();  // the previous level's readers of W are done
        for (int t = lane; t < ncol * w; t += 32) {
            const int ci = t / w, z = t - ci * w;
            const int64_t ix = b0[0] + ci / nyi;
            const int64_t key = D == 3 ? (ix * L.g.dim[1] + (b0[1] + ci % nyi)) * L.g.dim[2] + zl + z
                                       : ix * L.g.dim[1] + zl + z;
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
        staged = T <= CAP;
        if (staged) {
            // largest per-lane candidate count decides the mode
            int own = 0;
            if (valid) {
                const int zlo = lo[D - 1] - zl, zhi = hi[D - 1] - zl + 1;
                for (int ix = lo[0]; ix <= hi[0]; ++ix)
                    for (int iy = (D == 3 ? lo[1] : 0); iy <= (D == 3 ? hi[1] : 0); ++iy) {
                        const int ci = (ix - b0[0]) * nyi + (D == 3 ? iy - b0[1] : 0);
                        own += W.cs[ci * w + zhi] - W.cs[ci * w + zlo];
                    }
            }
            const int ownmax = __reduce_max_sync(FULL, own);
            const bool bcast = (float)T <= MSK_WS_BRATIO * (float)ownmax;
            __syncwarp();
            for (int ci = 0; ci < ncol; ++ci) {
                const int g0 = W.colgb[ci], f0 = W.colfo[ci], n0 = W.colfo[ci + 1] - f0;
                for (int t = lane; t < n0; t += 32) cp_async16(&W.rec[f0 + t], &L.frec[g0 + t]);
            }
            cp_async_wait_all();
            __syncwarp();
            if (bcast) {
                for (int ci = 0; ci < ncol; ++ci) {
                    const int f0 = W.colfo[ci], f1 = W.colfo[ci + 1];
                    scan_range(f0, f1, W.colgb[ci] - f0, valid);
                }
            } else if (valid) {
                const int zlo = lo[D - 1] - zl, zhi = hi[D - 1] - zl + 1;
                for (int ix = lo[0]; ix <= hi[0]; ++ix)
                    for (int iy = (D == 3 ? lo[1] : 0); iy <= (D == 3 ? hi[1] : 0); ++iy) {
                        const int ci = (ix - b0[0]) * nyi + (D == 3 ? iy - b0[1] : 0);
                        const int base = W.colfo[ci] - W.colgb[ci];
                        scan_range(W.cs[ci * w + zlo] + base, W.cs[ci * w + zhi] + base, -base, true);
                    }
            }
        }
    }
    if (!staged && valid) {
        // fallback: the lane's own ranges straight from global memory
        const float4 *__restrict__ frec = L.frec;
        for_each_range<D>(L, x, [&](int b, int e) {
            int j = b;
            for (; j + 1 < e; j += 2) {
                const float4 F0 = frec[j], F1 = frec[j + 1];
                const bool h0 = pre(xf, F0, thr), h1 = pre(xf, F1, thr);
                if (h0) append(j);
                if (h1) append(j + 1);
            }
            if (j < e && pre(xf, frec[j], thr)) append(j);
        });
    }
    if (nh) flush(nh);
    __syncwarp();
}

}  // namespace wscan
}  // namespace msk

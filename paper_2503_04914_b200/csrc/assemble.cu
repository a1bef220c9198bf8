// assemble.cu -- a2: CSR pattern and values of A_l (and of B_{kl} blocks for
// export).  Pattern: r^2 < delta^2 with r^2 evaluated left to right without
// FMA and delta^2 computed once on the host (reading C-4) -- bit-exact with
// the definition; candidates are screened by the conservative FP32 prefilter
// first (for_each_hit, neighbors.cuh), which never drops a true neighbour.  Values Phi_delta(r) = delta^-d phi(r / delta)
// (eq:kernelscaling P:67) with the column level's delta (reading C-1).
#include <stdlib.h>
#include <string.h>

#include "kernels.cuh"
#include "neighbors.cuh"

namespace msk {

namespace {
constexpr int NT = 256;

template <int D>
__global__ void __launch_bounds__(NT) k_count(LevelView rows, LevelView cols, int same,
                                              int32_t *__restrict__ cnt,
                                              unsigned long long *__restrict__ min_r2_bits, int64_t row0) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    if (i < rows.n) {
        double x[3];
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = rows.x[a][i];
        int c = 0;
        for_each_hit<D>(cols, x, [&](int j, double r2) {
            ++c;
            if (same && j != i + row0 && r2 < best) best = r2;  // row0: rows is a slice of cols
        });
        cnt[i] = c;
    }
    if (min_r2_bits) {
        // block min of non-negative doubles via their ordered bit patterns
        unsigned long long bits = (unsigned long long)__double_as_longlong(best);
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = t < bits ? t : bits;
        }
        if ((threadIdx.x & 31) == 0) atomicMin(min_r2_bits, bits);
    }
}

// The same counts for a whole level against itself (same, no row slice), each
// pair visited once: row i tests only the candidates j > i, and a hit adds to
// both rows (integer atomics: exact, order-free); the diagonal counts for i.
// Half the candidate tests of k_count.  cnt must be zero on entry.
template <int D>
__global__ void __launch_bounds__(NT) k_count_sym(LevelView v, int32_t *__restrict__ cnt,
                                                  unsigned long long *__restrict__ min_r2_bits) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    if (i < v.n) {
        double x[3];
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = v.x[a][i];
        int c = 1;  // (i, i)
        for_each_hit<D, 32, true>(v, x, [&](int j, double r2) {
            ++c;
            MSK_DASSERT(j > i && j < v.n);
            atomicAdd(&cnt[j], 1);
            if (r2 < best) best = r2;
        }, (int)i + 1);
        atomicAdd(&cnt[i], c);
    }
    if (min_r2_bits) {
        unsigned long long bits = (unsigned long long)__double_as_longlong(best);
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = t < bits ? t : bits;
        }
        if ((threadIdx.x & 31) == 0) atomicMin(min_r2_bits, bits);
    }
}

// Nearest pair of a level beyond its support (q = 1/2 min distance when no
// pair lies within delta): every candidate within m cells per axis,
// r^2 without FMA (reading C-4).  A pair closer than m cell sides is always
// found, so the caller grows m until the minimum is below m cell sides.
template <int D>
__global__ void __launch_bounds__(NT) k_min_r2_reach(LevelView v, int m, unsigned long long *__restrict__ min_r2_bits) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    if (i < v.n) {
        double x[3];
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = v.x[a][i];
        for_each_range_m<D>(v, x, m, [&](int b, int e) {
            for (int j = b; j < e; ++j) {
                if (j == i) continue;
                double y[3];
#pragma unroll
                for (int a = 0; a < D; ++a) y[a] = v.x[a][j];
                const double r2 = dist2_nofma<D>(x, y);
                best = r2 < best ? r2 : best;
            }
        });
    }
    unsigned long long bits = (unsigned long long)__double_as_longlong(best);
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, bits, o);
        bits = t < bits ? t : bits;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(min_r2_bits, bits);
}

template <int D, int K>
__global__ void __launch_bounds__(NT) k_fill(LevelView rows, LevelView cols,
                                             const int64_t *__restrict__ row_ptr,
                                             int32_t *__restrict__ col, double *__restrict__ val) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= rows.n) return;
    double x[3];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = rows.x[a][i];
    int64_t p = row_ptr[i];
    const double inv = cols.inv_delta, sc = cols.scale;
    for_each_hit<D>(cols, x, [&](int j, double r2) {
        col[p] = j;
        if (val) val[p] = sc * wendland<K>(sqrt(r2) * inv);
        ++p;
    });
}
template <int D>
__global__ void __launch_bounds__(NT) k_hit_range(LevelView rows, LevelView cols,
                                                  unsigned long long *__restrict__ mm) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    unsigned long long lo = ~0ull, hi = 0;
    if (i < rows.n) {
        double x[3];
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = rows.x[a][i];
        for_each_hit<D>(cols, x, [&](int j, double) {
            lo = (unsigned long long)j < lo ? (unsigned long long)j : lo;
            hi = (unsigned long long)j > hi ? (unsigned long long)j : hi;
        });
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, lo, o);
        lo = t < lo ? t : lo;
        t = __shfl_xor_sync(0xffffffffu, hi, o);
        hi = t > hi ? t : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}
}  // namespace

void hit_range(int d, const LevelView &rows, const LevelView &cols, unsigned long long *mm, cudaStream_t st) {
    unsigned long long init[2] = {~0ull, 0ull};
    MSK_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
    if (rows.n == 0) return;
    unsigned nb = ceil_div_u(rows.n, NT);
    if (d == 2) k_hit_range<2><<<nb, NT, 0, st>>>(rows, cols, mm);
    else k_hit_range<3><<<nb, NT, 0, st>>>(rows, cols, mm);
    MSK_CHECK_LAUNCH();
}

void count_pattern(int d, const LevelView &rows, const LevelView &cols, bool same, int32_t *cnt,
                   unsigned long long *min_r2_bits, cudaStream_t st, int *launches, int64_t row0) {
    if (rows.n == 0) return;
    unsigned nb = ceil_div_u(rows.n, NT);
    static const bool sym = getenv("MSK_COUNT_SYM") == nullptr || atoi(getenv("MSK_COUNT_SYM")) != 0;
    if (sym && same && row0 == 0 && rows.n == cols.n) {  // a whole level against itself
        MSK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)rows.n, st));
        if (d == 2) k_count_sym<2><<<nb, NT, 0, st>>>(rows, cnt, min_r2_bits);
        else k_count_sym<3><<<nb, NT, 0, st>>>(rows, cnt, min_r2_bits);
        MSK_CHECK_LAUNCH();
        if (launches) *launches += 1;
        return;
    }
    if (d == 2) k_count<2><<<nb, NT, 0, st>>>(rows, cols, same ? 1 : 0, cnt, min_r2_bits, row0);
    else k_count<3><<<nb, NT, 0, st>>>(rows, cols, same ? 1 : 0, cnt, min_r2_bits, row0);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

void fill_pattern(int d, int k, const LevelView &rows, const LevelView &cols,
                  const int64_t *row_ptr, int32_t *col, double *val, cudaStream_t st,
                  int *launches) {
    if (rows.n == 0) return;
    unsigned nb = ceil_div_u(rows.n, NT);
#define MSK_FILL(DD, KK) k_fill<DD, KK><<<nb, NT, 0, st>>>(rows, cols, row_ptr, col, val)
    if (d == 2) {
        if (k == 0) MSK_FILL(2, 0); else if (k == 1) MSK_FILL(2, 1); else MSK_FILL(2, 2);
    } else {
        if (k == 0) MSK_FILL(3, 0); else if (k == 1) MSK_FILL(3, 1); else MSK_FILL(3, 2);
    }
#undef MSK_FILL
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

// min r^2 over the pairs of level v whose cells differ by at most m per axis
double min_r2_reach(int d, const LevelView &v, int m, cudaStream_t st) {
    unsigned long long *dm = nullptr, hm = 0x7ff0000000000000ull;
    MSK_CUDA(cudaMallocAsync((void **)&dm, sizeof hm, st));
    MSK_CUDA(cudaMemcpyAsync(dm, &hm, sizeof hm, cudaMemcpyHostToDevice, st));
    if (v.n > 0) {
        if (d == 2) k_min_r2_reach<2><<<ceil_div_u(v.n, NT), NT, 0, st>>>(v, m, dm);
        else k_min_r2_reach<3><<<ceil_div_u(v.n, NT), NT, 0, st>>>(v, m, dm);
        MSK_CHECK_LAUNCH();
    }
    MSK_CUDA(cudaMemcpyAsync(&hm, dm, sizeof hm, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    MSK_CUDA(cudaFreeAsync(dm, st));
    double r2;
    memcpy(&r2, &hm, sizeof r2);
    return r2;
}

}  // namespace msk

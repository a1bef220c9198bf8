// cg.cu -- a4/a8: block-diagonal conjugate gradients (Theorem cg P:603-661,
// Algorithm 1, eq:blockdiagonal_levelwise P:616) as ONE
// persistent cooperative launch per phase.
//
// The paper runs one stream per level and synchronises with the host twice
// per iteration.  Here every level of the batch owns
// a contiguous group of co-resident CTAs; each group runs its own CG loop
// with its own device-side barrier and deterministic reductions, so the whole
// solve of all levels is one launch with no host round trips:
//
//   x = 0, r = b, p = b, bb = rr = b.b
//   while rr > tol^2 bb and it < max_iter:          (reading C-9)
//       q = A p ; pq = p.q          -- CSR-stream SpMV fused with the dot
//       alpha = rr / pq
//       x += alpha p ; r -= alpha q ; rr' = r.r      -- fused update + dot
//       beta = rr' / rr ; p = r + beta p
//
// SpMV (CSR-stream): a CTA takes a tile of NT consecutive rows (spatial
// order), streams the tile's contiguous nnz range with fully coalesced loads
// of val/col, gathers p[col] (L2-resident thanks to the spatial sort) and
// stages the products in shared memory; each thread then sums its row in
// ascending column order (deterministic).
//
// Reductions: fixed xor-shuffle tree per warp -> fixed warp order -> one
// partial per CTA -> after the group barrier every CTA sums the partials in
// the same fixed order.  All CTAs of a group therefore hold bit-identical
// scalars and take identical control flow; results do not depend on timing.
#include <cooperative_groups.h>
#include <cuda/atomic>

#include <vector>

#include "kernels.cuh"

namespace msk {

namespace {
constexpr int NT = 256;     // threads per CTA == rows per tile
constexpr int CAP = 4096;   // staged products per chunk (32 KB of shared memory)
constexpr int U = 4;        // independent gathers in flight per thread
constexpr int CH = 4;       // tiles per reduction chunk (the unit of work distribution)

struct CGBatch {
    int nlev;
    CGLevelArgs lev[kMaxLevels];
};

__device__ __forceinline__ void group_barrier(unsigned long long *ctr, int nb,
                                              unsigned long long &round) {
    __syncthreads();
    if (nb > 1) {
        round += (unsigned long long)nb;
        if (threadIdx.x == 0) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> a(*ctr);
            __threadfence();
            a.fetch_add(1ull, cuda::memory_order_release);
            unsigned long long spins = 0;
            while (a.load(cuda::memory_order_acquire) < round) {
                __nanosleep(64);
                if (++spins > (1ull << 31)) __trap();  // never hang the device forever
            }
            __threadfence();
        }
        __syncthreads();
    }
}

// Deterministic all-reduce over the chunk partials of one group.  Each chunk
// (CH consecutive tiles) is owned by exactly one CTA, which has written its
// partial; after the group barrier every CTA sums all partials in the same
// fixed order.  The result depends only on n (not on the number of CTAs in
// the group or on the GPU), so a level gives bit-identical results whether
// it is solved alone or batched with other levels.
__device__ __forceinline__ double chunk_allreduce(const double *partials, int64_t nchunks, int nb,
                                                  unsigned long long *ctr,
                                                  unsigned long long &round, double *s_red) {
    group_barrier(ctr, nb, round);
    double t = 0.0;
    for (int64_t j = threadIdx.x; j < nchunks; j += NT) t += __ldcg(&partials[j]);
    return block_sum<NT>(t, s_red);
}

// q = A p on rows [r0, r0+nr); returns this thread's q (row r0+tid) or 0.
__device__ __forceinline__ double spmv_tile(int64_t r0, int nr, const int64_t *__restrict__ row_ptr,
                                            const int32_t *__restrict__ col,
                                            const double *__restrict__ val, const double *p,
                                            double *s_prod, int64_t *s_rp) {
    const int tid = threadIdx.x;
    for (int t = tid; t <= nr; t += NT) s_rp[t] = __ldg(&row_ptr[r0 + t]);
    __syncthreads();
    const int64_t k0 = s_rp[0], k1 = s_rp[nr];
    int64_t myb = 0, mye = 0;
    if (tid < nr) { myb = s_rp[tid]; mye = s_rp[tid + 1]; }
    double acc = 0.0;
    for (int64_t cb = k0; cb < k1; cb += CAP) {
        const int64_t ce = cb + CAP < k1 ? cb + CAP : k1;
        for (int64_t k = cb + tid; k < ce; k += NT * U) {
            double v[U];
            int c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int64_t kk = k + (int64_t)u * NT;
                if (kk < ce) { v[u] = __ldg(&val[kk]); c[u] = __ldg(&col[kk]); }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int64_t kk = k + (int64_t)u * NT;
                if (kk < ce) s_prod[kk - cb] = v[u] * p[c[u]];
            }
        }
        __syncthreads();
        if (tid < nr) {
            int64_t lo = myb > cb ? myb : cb, hi = mye < ce ? mye : ce;
            for (int64_t k = lo; k < hi; ++k) acc += s_prod[k - cb];
        }
        __syncthreads();
    }
    return acc;
}

__global__ void __launch_bounds__(NT, 4) k_cg(CGBatch B) {
    __shared__ double s_prod[CAP];
    __shared__ int64_t s_rp[NT + 1];
    __shared__ double s_red[NT / 32 + 2];

    int g = 0;
    while (g + 1 < B.nlev && (int)blockIdx.x >= B.lev[g + 1].block_begin) ++g;
    const CGLevelArgs &L = B.lev[g];
    const int nb = L.nblocks, me = (int)blockIdx.x - L.block_begin;
    const int tid = threadIdx.x;
    const int64_t n = L.n;
    const int64_t ntiles = (n + NT - 1) / NT;
    const int64_t nchunks = (ntiles + CH - 1) / CH;
    double *__restrict__ x = L.x;
    double *__restrict__ r = L.r;
    double *p = L.p;  // written by other CTAs between barriers: plain (coherent) loads
    double *__restrict__ q = L.q;
    double *part = L.partials;  // 3 * nchunks
    unsigned long long round = 0;
    // chunk c = tiles [c*CH, min((c+1)*CH, ntiles)), owned by CTA c mod nb
#define MSK_FOR_CHUNK_TILES(c, t) \
    for (int64_t t = (c) * CH, t##_e = ((c) + 1) * CH < ntiles ? ((c) + 1) * CH : ntiles; t < t##_e; ++t)

    // ---- init: x = 0, r = p = b, bb = b.b
    for (int64_t c = me; c < nchunks; c += nb) {
        double acc = 0.0;
        MSK_FOR_CHUNK_TILES(c, t) {
            int64_t i = t * NT + tid;
            if (i < n) {
                double bi = L.b_src ? __ldg(&L.b_src[__ldg(&L.b_perm[i])]) : __ldg(&L.b[i]);
                x[i] = 0.0;
                r[i] = bi;
                p[i] = bi;
                acc += bi * bi;
            }
        }
        double s = block_sum<NT>(acc, s_red);
        if (tid == 0) part[c] = s;
    }
    const double bb = chunk_allreduce(part, nchunks, nb, L.barrier, round, s_red);
    double rr = bb;
    int it = 0, status = 0;
    if (bb > 0.0) {
        const double stop = L.tol2 * bb;
        for (;;) {
            if (rr <= stop) break;
            if (it >= L.max_iter) { status = 1; break; }
            // ---- q = A p, pq = p.q
            for (int64_t c = me; c < nchunks; c += nb) {
                double acc = 0.0;
                MSK_FOR_CHUNK_TILES(c, t) {
                    int64_t r0 = t * NT;
                    int nr = (int)(n - r0 < NT ? n - r0 : NT);
                    double qi = spmv_tile(r0, nr, L.row_ptr, L.col, L.val, p, s_prod, s_rp);
                    if (tid < nr) {
                        q[r0 + tid] = qi;
                        acc += p[r0 + tid] * qi;
                    }
                }
                double s = block_sum<NT>(acc, s_red);
                if (tid == 0) part[nchunks + c] = s;
            }
            const double pq = chunk_allreduce(part + nchunks, nchunks, nb, L.barrier, round, s_red);
            const double alpha = rr / pq;
            // ---- x += alpha p, r -= alpha q, rr' = r.r
            for (int64_t c = me; c < nchunks; c += nb) {
                double acc = 0.0;
                MSK_FOR_CHUNK_TILES(c, t) {
                    int64_t i = t * NT + tid;
                    if (i < n) {
                        double pi = p[i];
                        x[i] += alpha * pi;
                        double ri = r[i] - alpha * q[i];
                        r[i] = ri;
                        acc += ri * ri;
                    }
                }
                double s = block_sum<NT>(acc, s_red);
                if (tid == 0) part[2 * nchunks + c] = s;
            }
            const double rrn = chunk_allreduce(part + 2 * nchunks, nchunks, nb, L.barrier, round, s_red);
            const double beta = rrn / rr;
            rr = rrn;
            // ---- p = r + beta p
            for (int64_t c = me; c < nchunks; c += nb) {
                MSK_FOR_CHUNK_TILES(c, t) {
                    int64_t i = t * NT + tid;
                    if (i < n) p[i] = r[i] + beta * p[i];
                }
            }
            group_barrier(L.barrier, nb, round);
            ++it;
        }
    }
    if (L.x_out) {
        for (int64_t c = me; c < nchunks; c += nb) {
            MSK_FOR_CHUNK_TILES(c, t) {
                int64_t i = t * NT + tid;
                if (i < n) L.x_out[__ldg(&L.x_perm[i])] = x[i];
            }
        }
    }
#undef MSK_FOR_CHUNK_TILES
    if (me == 0 && tid == 0) {
        *L.out_iters = it;
        L.out_rr[0] = rr;
        L.out_rr[1] = bb;
        *L.out_status = status;
    }
}

__global__ void __launch_bounds__(NT) k_spmv(int64_t n, const int64_t *__restrict__ row_ptr,
                                             const int32_t *__restrict__ col,
                                             const double *__restrict__ val,
                                             const double *__restrict__ v, double *__restrict__ y) {
    __shared__ double s_prod[CAP];
    __shared__ int64_t s_rp[NT + 1];
    int64_t r0 = (int64_t)blockIdx.x * NT;
    int nr = (int)(n - r0 < NT ? n - r0 : NT);
    double qi = spmv_tile(r0, nr, row_ptr, col, val, v, s_prod, s_rp);
    if ((int)threadIdx.x < nr) y[r0 + threadIdx.x] = qi;
}

int g_max_resident = 0;
}  // namespace

int cg_max_resident_blocks() {
    if (g_max_resident == 0) {
        int dev = 0, sms = 0, per = 0;
        MSK_CUDA(cudaGetDevice(&dev));
        MSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cg, NT, 0));
        g_max_resident = sms * (per > 0 ? per : 1);
    }
    return g_max_resident;
}

// levels[i].nblocks == 0 => the launcher assigns CTAs proportionally to work.
void cg_batched(CGLevelArgs *levels, int nlev, cudaStream_t st, int *launches) {
    if (nlev <= 0) return;
    if (nlev > kMaxLevels) throw Error(1, "cg_batched: too many levels");
    const int total = cg_max_resident_blocks();
    if (total < nlev) throw Error(3, "cg_batched: fewer resident CTAs than levels");
    std::vector<double> work(nlev);
    double wsum = 0.0;
    for (int l = 0; l < nlev; ++l) {
        work[l] = (double)levels[l].nnz + 12.0 * (double)levels[l].n;  // ~bytes/8 per iteration
        wsum += work[l];
    }
    // CTA allocation: proportional to work, at least one, at most one per chunk.
    int used = 0;
    std::vector<int> nbk(nlev);
    std::vector<int64_t> nch(nlev);
    int64_t ptot = 0;
    for (int l = 0; l < nlev; ++l) {
        int64_t tiles = (levels[l].n + NT - 1) / NT;
        nch[l] = (tiles + CH - 1) / CH;
        if (nch[l] < 1) nch[l] = 1;
        ptot += 3 * nch[l];
        int want = levels[l].nblocks > 0
                       ? levels[l].nblocks
                       : (int)((double)(total - nlev) * work[l] / (wsum > 0 ? wsum : 1.0)) + 1;
        if (want > nch[l]) want = (int)nch[l];
        if (want < 1) want = 1;
        nbk[l] = want;
        used += want;
    }
    while (used > total) {  // trim the largest groups
        int big = 0;
        for (int l = 1; l < nlev; ++l) if (nbk[l] > nbk[big]) big = l;
        --nbk[big];
        --used;
    }
    // workspace: chunk partials (3 per chunk per level) + barrier counters
    double *partials = nullptr;
    unsigned long long *bars = nullptr;
    MSK_CUDA(cudaMallocAsync((void **)&partials, sizeof(double) * (size_t)ptot, st));
    MSK_CUDA(cudaMallocAsync((void **)&bars, sizeof(unsigned long long) * (size_t)nlev, st));
    MSK_CUDA(cudaMemsetAsync(bars, 0, sizeof(unsigned long long) * (size_t)nlev, st));
    CGBatch B;
    B.nlev = nlev;
    int begin = 0;
    int64_t poff = 0;
    for (int l = 0; l < nlev; ++l) {
        B.lev[l] = levels[l];
        B.lev[l].nblocks = nbk[l];
        B.lev[l].block_begin = begin;
        B.lev[l].partials = partials + poff;
        B.lev[l].barrier = bars + l;
        begin += nbk[l];
        poff += 3 * nch[l];
    }
    void *args[] = {&B};
    MSK_CUDA(cudaLaunchCooperativeKernel((void *)k_cg, dim3(used), dim3(NT), args, 0, st));
    if (launches) *launches += 1;
    MSK_CUDA(cudaFreeAsync(partials, st));
    MSK_CUDA(cudaFreeAsync(bars, st));
}

void spmv_csr(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *val,
              const double *v, double *y, cudaStream_t st, int *launches) {
    if (n == 0) return;
    k_spmv<<<ceil_div_u(n, NT), NT, 0, st>>>(n, row_ptr, col, val, v, y);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

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
//   x = 0, r = b, bb = rr = b.b, beta = alpha' = 0
//   while rr > tol^2 bb and it < max_iter:          (reading C-9)
//       w = A r ; p = r + beta p ; q = w + beta q ; x += alpha' p_old ;
//       pq = p.q                     -- ONE pass: SpMV + updates + dot [barrier]
//       alpha = rr / pq
//       r -= alpha q ; rr' = r.r      -- fused update + dot           [barrier]
//       beta = rr' / rr ; alpha' = alpha
//   x += alpha' p                     -- the last deferred x update
//
// This is Algorithm 1's CG with q = A p formed by the
// recurrence q = A r + beta q (A p = A r + beta A p_old), which lets the
// x/p update ride on the SpMV pass: two device-wide barriers per iteration
// instead of three, the same 88 bytes of vector traffic per row.  In exact
// arithmetic the iterates are those of the textbook loop; in floating point
// they differ by rounding only (parity: tests/test_gpu_parity.py).
//
// SpMV: a CTA takes a tile of NT consecutive rows (spatial order).  One
// thread streams the tile's contiguous CSR slices (values, columns) into
// shared memory with a bulk-async copy (TMA, cp.async.bulk, L2 evict-first
// so the gathered vector r stays L2-resident) completing on an mbarrier; the
// threads then only issue the irregular gathers r[col] (U independent loads
// in flight per thread), and each thread sums its row in ascending column
// order (deterministic).
//
// Work unit and reductions: a level's tiles are grouped into chunks of CH
// tiles (CH fixed by n alone); chunk c belongs to CTA c mod nb.  Each chunk
// writes one partial per dot product (fixed xor-shuffle tree per warp ->
// fixed warp order); after the group barrier every CTA sums all chunk
// partials in the same fixed order.  The result therefore depends only on n,
// not on the number of CTAs, the GPU or the other levels of the batch, and
// all CTAs of a group take identical control flow.
#include <cuda/atomic>

#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "neighbors.cuh"
#include "tma.cuh"
#include "wscan.cuh"

namespace msk {

namespace {
constexpr int NT = 256;       // threads per CTA == rows per tile
constexpr int NW = NT / 32;   // warps per CTA
#ifndef MSK_U
#define MSK_U 4
#endif
#ifndef MSK_CAPT
#define MSK_CAPT 2048
#endif
#ifndef MSK_MINB
#define MSK_MINB 3
#endif
#ifndef MSK_MF_U2
#define MSK_MF_U2 4  // matrix-free SpMV: survivors per trip, 2-D (C2 finest 68.4 -> 54.5 ms)
#endif
#ifndef MSK_MF_U3
#define MSK_MF_U3 2  // 3-D (C3 finest 166 -> 144 ms; 4: 149 ms)
#endif
#ifndef MSK_MF_P
#define MSK_MF_P 4   // candidates per trip of the prefilter (4: C2 finest 54.6 -> 52.2 ms, C3 144 -> 138)
#endif
#ifndef MSK_MF_MINB
#define MSK_MF_MINB 4
#endif
#ifndef MSK_ASYNC_MIN_C
#define MSK_ASYNC_MIN_C 4096
#endif
constexpr int U = MSK_U;      // independent gathers in flight per lane (row-parallel)
constexpr int MAXCH = 4;      // max tiles per chunk
constexpr int RPCAP = MAXCH * NT + 4;  // staged row pointers per chunk

struct CGBatch {
    int nlev;
    CGLevelArgs lev[kMaxLevels];
};

// ---- CTA-level pipeline (used by k_cg): large bulk copies, double-buffered.
// The piece capacity C (CSR entries per stage) is a template parameter: the
// launcher picks C from the mean row length so that a piece spans ~200+ rows
// (each thread owns rows, so a piece of few long rows leaves threads idle):
// C = 2048 (values 16 KB + columns 8 KB, 3 CTAs/SM) for short rows (d = 3),
// C = 4096 (2 CTAs/SM) for long rows (d = 2, ~25 per row).  Same-box A/B:
// C3 finest level 33.5 ms (2048) vs 37.7 (4096); C5 finest 1546 vs 1246 ms.
constexpr int CAPT0 = MSK_CAPT;   // short-row variant
constexpr int MINB0 = MSK_MINB;
constexpr int CAPT1 = 4096;       // long-row / few-chunk variant
constexpr int MINB1 = 2;
constexpr int CAPT2 = 2432;       // mid-size levels (one-tile chunks: 256 rows x ~9 entries fit one piece)
constexpr int MINB2 = 3;
constexpr int NSTG = 2;           // pipeline stages (NSTG - 1 pieces in flight ahead)
template <int C>
struct __align__(16) CtaStageT {
    double val[C];
    int32_t col[C + 8];
};
template <int C>
struct __align__(16) CGSharedTT {
    CtaStageT<C> st[NSTG];    // ring of CSR slices (a stream of pieces)
    int64_t rp[2][RPCAP];     // row pointers of the current and the next chunk
    double red[NT / 32 + 2];
    uint64_t bar_st[NSTG];
    uint64_t bar_rp[2];
    unsigned arr[NSTG];  // asynchronous stage release: warps done with the stage (+8 per use)
};

// ctr == nullptr: the group is one thread-block cluster (small levels, see
// cg_batched) and the hardware cluster barrier (release / acquire at cluster
// scope) replaces the counter in global memory.
__device__ __forceinline__ void group_barrier(unsigned long long *ctr, int nb,
                                              unsigned long long &round) {
    if (ctr == nullptr) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    __syncthreads();
    if (nb > 1) {
        round += (unsigned long long)nb;
        if (threadIdx.x == 0) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> a(*ctr);
            // release: this CTA's writes (ordered before by __syncthreads) become
            // visible to every CTA that acquires the counter (no extra fence)
            a.fetch_add(1ull, cuda::memory_order_release);
            unsigned long long spins = 0;
            while (a.load(cuda::memory_order_acquire) < round) {
                __nanosleep(32);
                if (++spins > (1ull << 31)) __trap();  // never hang the device forever
            }
        }
        __syncthreads();
    }
}

// Per-thread share of a fixed-order chunk sum: partials j = tid, tid + NT, ...
// added left to right (the order every reduction of the solver uses).  The
// loads are issued 8 at a time ahead of the dependent adds (one L2 round trip
// per 8 partials instead of per partial); the summation order is unchanged.
__device__ __forceinline__ double strided_sum(const double *partials, int64_t nchunks) {
    double t = 0.0;
    int64_t j = threadIdx.x;
    for (; j + 7 * NT < nchunks; j += 8 * NT) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(&partials[j + u * NT]);
#pragma unroll
        for (int u = 0; u < 8; ++u) t += v[u];
    }
    for (; j < nchunks; j += NT) t += __ldcg(&partials[j]);
    return t;
}

// Deterministic all-reduce over the chunk partials of one group: after the
// group barrier every CTA sums all partials in the same fixed order.
__device__ __forceinline__ double chunk_allreduce(const double *partials, int64_t nchunks, int nb,
                                                  unsigned long long *ctr,
                                                  unsigned long long &round, double *s_red) {
    group_barrier(ctr, nb, round);
    return block_sum<NT>(strided_sum(partials, nchunks), s_red);
}

// ---------------------------------------------------------------------------
// CTA-level pipelined SpMV phase over all chunks of this CTA: w = A r, then
// per row p = r + beta p, q = w + beta q, x += alpha' p_old (first iteration:
// p = r, q = w, x = 0), with p.q partials per chunk.  The CTA's CSR entries are streamed as a sequence of
// pieces (<= CAPTE entries, two bulk copies each) through two stages: piece
// P+1 is in flight while piece P is consumed.  Row pointers of the next chunk
// are prefetched into the second rp buffer.  Each thread owns row
// t*NT + tid of every tile t of the chunk and gathers p for the entries of
// its rows that fall into the piece (row-parallel, U loads in flight),
// accumulating in ascending column order.
struct PipeState {
    uint32_t P;   // pieces consumed so far (stage P%NSTG, parity (P/NSTG)&1)
    uint32_t CS;  // chunks visited so far (rp buffer CS&1, parity (CS>>1)&1)
};

template <class SH>
__device__ __forceinline__ void issue_rp(SH &S, int b, const int64_t *row_ptr, int64_t r0, int nrows,
                                         uint64_t pol) {
    const int64_t lo = r0 & ~(int64_t)1;
    const int64_t hi = (r0 + nrows + 2) & ~(int64_t)1;
    const uint32_t bytes = (uint32_t)((hi - lo) * 8);
    mbar_arrive_expect_tx(&S.bar_rp[b], bytes);
    tma_load_1d(S.rp[b], row_ptr + lo, bytes, &S.bar_rp[b], pol);
}

template <class SH>
__device__ __forceinline__ void issue_piece_t(SH &S, int b, const int32_t *col, const double *val,
                                              int64_t kb, int64_t ke, uint64_t pol) {
    const int64_t vlo = kb & ~(int64_t)1, vhi = (ke + 1) & ~(int64_t)1;
    const int64_t clo = kb & ~(int64_t)3, chi = (ke + 3) & ~(int64_t)3;
    const uint32_t vb = (uint32_t)((vhi - vlo) * 8), cb = (uint32_t)((chi - clo) * 4);
    mbar_arrive_expect_tx(&S.bar_st[b], vb + cb);
    tma_load_1d(S.st[b].val, val + vlo, vb, &S.bar_st[b], pol);
    tma_load_1d(S.st[b].col, col + clo, cb, &S.bar_st[b], pol);
}

// the same piece with 16-bit columns (col16): the stage's column area holds 2 x
// (C + 8) of them
template <class SH>
__device__ __forceinline__ void issue_piece_16(SH &S, int b, const uint16_t *col16, const double *val,
                                               int64_t kb, int64_t ke, uint64_t pol) {
    const int64_t vlo = kb & ~(int64_t)1, vhi = (ke + 1) & ~(int64_t)1;
    const int64_t clo = kb & ~(int64_t)7, chi = (ke + 7) & ~(int64_t)7;
    const uint32_t vb = (uint32_t)((vhi - vlo) * 8), cb = (uint32_t)((chi - clo) * 2);
    mbar_arrive_expect_tx(&S.bar_st[b], vb + cb);
    tma_load_1d(S.st[b].val, val + vlo, vb, &S.bar_st[b], pol);
    tma_load_1d(S.st[b].col, col16 + clo, cb, &S.bar_st[b], pol);
}

// branch-free (lanes of a warp use different windows): two-way selects only
__device__ __forceinline__ int col16_decode(uint32_t c, const int4 &b) {
    const bool odd = (c >> 14) & 1u, upper = (c >> 15) & 1u;
    const int lo = odd ? b.y : b.x;
    const int hi = odd ? b.w : b.z;
    return (upper ? hi : lo) + (int)(c & 0x3FFFu);
}

// Chunks handled: cbase + me + k*nb for k = 0.. while < cbase + nloc (cbase =
// 0, nloc = all chunks on one GPU; the owned chunk range of a partition in
// the distributed CG).  L.row_ptr is indexed by global row.
// PLAIN: y = A v only (msk_apply_block): v = L.r, y = L.q, no updates, no dot.
struct NoPush {
    __device__ __forceinline__ void operator()(int64_t, double) const {}
};
template <int C, bool PLAIN = false, class Push = NoPush, bool C16 = false>
__device__ __forceinline__ void spmv_phase(CGSharedTT<C> &S, const CGLevelArgs &L, int me, int nb, int64_t cbase,
                                           int64_t nloc, int CH, double *part_out, PipeState &ps, uint64_t pol,
                                           bool first, double alpha_prev, double beta,
                                           const Push &push = Push()) {
    // C16: 16-bit columns (L.col16 + per-chunk window bases L.cbase), 10 B per entry
    auto issue = [&](int b, int64_t kb, int64_t ke) {
        if constexpr (C16) issue_piece_16(S, b, L.col16, L.val, kb, ke, pol);
        else issue_piece_t(S, b, L.col, L.val, kb, ke, pol);
    };
    constexpr int CAPTE = C - 2;  // usable entries per piece (alignment slack)
    // Asynchronous stage release (pieces of >= MSK_ASYNC_MIN_C entries): when
    // piece j + 2 lies in the same chunk, the last warp to finish piece j
    // refills its stage and no warp waits for the others; otherwise (and at
    // chunk ends) a CTA barrier.  Same-box A/B: C2 finest level (4096-entry
    // pieces, 2 CTAs/SM) 20.15 -> 18.69 ms; with 2048-entry pieces (C3) it
    // is 1-2 % slower, so those keep the barrier.
    constexpr bool ASYNC = C >= MSK_ASYNC_MIN_C;
    const int tid = threadIdx.x;
    const int64_t n = L.n;
    const int64_t K = me < nloc ? (nloc - 1 - me) / nb + 1 : 0;  // my chunks
    if (K == 0) return;
    const double *rv = L.r;  // written by other CTAs in the previous phase (after the barrier)
    auto chunk_rows = [&](int64_t k, int64_t &cr0, int &crows) {
        const int64_t c = cbase + me + k * nb;
        cr0 = c * CH * NT;
        crows = (int)(n - cr0 < (int64_t)CH * NT ? n - cr0 : (int64_t)CH * NT);
    };
    auto rp_off = [&](int64_t cr0) { return (int)(cr0 - (cr0 & ~(int64_t)1)); };
    int64_t cr0;
    int crows;
    if (tid == 0) {
        chunk_rows(0, cr0, crows);
        issue_rp(S, ps.CS & 1, L.row_ptr, cr0, crows, pol);
        if (K > 1) {
            chunk_rows(1, cr0, crows);
            issue_rp(S, (ps.CS + 1) & 1, L.row_ptr, cr0, crows, pol);
        }
    }
    mbar_wait(&S.bar_rp[ps.CS & 1], (ps.CS >> 1) & 1u);
    chunk_rows(0, cr0, crows);
    {
        const int64_t *rp = S.rp[ps.CS & 1] + rp_off(cr0);
        const int64_t K0 = rp[0], K1 = rp[crows];
        if (tid == 0) issue(ps.P & 1, K0, K0 + CAPTE < K1 ? K0 + CAPTE : K1);
    }
    for (int64_t k = 0; k < K; ++k) {
        chunk_rows(k, cr0, crows);
        const uint32_t cs = ps.CS + (uint32_t)k;
        // the epilogue's own-row vectors of the NEXT chunk -> L2 (hidden behind
        // this chunk's pieces; 33.38 -> 33.1 ms on the C3 finest level)
        if (!PLAIN && tid == 0 && L.clen && k + 1 < K) {
            // the next chunk's gathered r: its column windows -> L2 (r was written by
            // every CTA in the last pass and competes with the streamed CSR for L2)
            const int64_t cn = cbase + me + (k + 1) * nb;
            const int4 b = __ldg(&L.cbase[cn]), e = __ldg(&L.clen[cn]);
            const int bb[4] = {b.x, b.y, b.z, b.w}, ee[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                if (ee[w] <= 0) continue;
                const uintptr_t a0 = (uintptr_t)(rv + bb[w]) & ~(uintptr_t)15;
                const uintptr_t a1 = ((uintptr_t)(rv + bb[w] + ee[w]) + 15) & ~(uintptr_t)15;
                prefetch_l2((const void *)a0, (uint32_t)(a1 - a0));
            }
        }
        if (!PLAIN && tid == 0 && !first && k + 1 < K) {
            int64_t nr0;
            int nrows;
            chunk_rows(k + 1, nr0, nrows);
            // 16-byte aligned interior of each slice (vector bases are only 8-byte aligned)
            for (const double *v : {(const double *)L.p, (const double *)L.q, (const double *)L.x}) {
                const uintptr_t a0 = ((uintptr_t)(v + nr0) + 15) & ~(uintptr_t)15;
                const uintptr_t a1 = (uintptr_t)(v + nr0 + nrows) & ~(uintptr_t)15;
                if (a1 > a0) prefetch_l2((const void *)a0, (uint32_t)(a1 - a0));
            }
        }
        const int64_t *rp = S.rp[cs & 1] + rp_off(cr0);
        const int64_t K1 = rp[crows];
        int4 wb = make_int4(0, 0, 0, 0);
        if constexpr (C16) wb = __ldg(&L.cbase[cbase + me + k * nb]);
        int64_t rb[MAXCH], re[MAXCH];
        double acc[MAXCH];
#pragma unroll
        for (int t = 0; t < MAXCH; ++t) {
            const int r = t * NT + tid;
            const bool ok = t < CH && r < crows;
            rb[t] = ok ? rp[r] : 0;
            re[t] = ok ? rp[r + 1] : 0;
            acc[t] = 0.0;
        }
        for (int64_t kb = rp[0]; kb < K1;) {
            const int64_t ke = kb + CAPTE < K1 ? kb + CAPTE : K1;
            // the next piece (rest of this chunk, or the first piece of the next
            // one) goes into the other stage, which held piece P-1 (consumed)
            // ASYNC: piece j + 1 was already issued at the end of piece j - 1
            // unless this is the chunk's first piece
            const bool pre_issued = ASYNC && kb != rp[0];
            if (ke < K1) {
                if (tid == 0 && !pre_issued)
                    issue((ps.P + 1) & 1, ke, ke + CAPTE < K1 ? ke + CAPTE : K1);
            } else if (k + 1 < K) {
                mbar_wait(&S.bar_rp[(cs + 1) & 1], ((cs + 1) >> 1) & 1u);
                if (tid == 0) {
                    int64_t nr0;
                    int nrows;
                    chunk_rows(k + 1, nr0, nrows);
                    const int64_t *nrp = S.rp[(cs + 1) & 1] + rp_off(nr0);
                    const int64_t a = nrp[0], e = nrp[nrows];
                    issue((ps.P + 1) & 1, a, a + CAPTE < e ? a + CAPTE : e);
                }
            }
            mbar_wait(&S.bar_st[ps.P & 1], (ps.P >> 1) & 1u);
            const CtaStageT<C> &cur = S.st[ps.P & 1];
            const int voff = (int)(kb & 1), coff = C16 ? (int)(kb & 7) : (int)(kb & 3);
            const uint16_t *col16 = reinterpret_cast<const uint16_t *>(cur.col);
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                if (t >= CH) break;
                // clamp in 64-bit before narrowing (entry offsets exceed 2^31)
                const int64_t lo64 = rb[t] > kb ? rb[t] : kb, hi64 = re[t] < ke ? re[t] : ke;
                const int lo = (int)(lo64 - kb);
                const int hi = hi64 > lo64 ? (int)(hi64 - kb) : lo;
                for (int e = lo; e < hi; e += U) {
                    double pv[U], vv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int ee = e + u;
                        const int cj = ee < hi ? (C16 ? col16_decode(col16[coff + ee], wb) : cur.col[coff + ee]) : 0;
                        MSK_DASSERT(ee >= hi || (coff + ee < (C16 ? 2 * (C + 8) : C + 8) && voff + ee < C &&
                                                 cj >= 0 && cj < n));
                        pv[u] = ee < hi ? rv[cj] : 0.0;
                        vv[u] = ee < hi ? cur.val[voff + ee] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (e + u < hi) acc[t] = fma(vv[u], pv[u], acc[t]);
                }
            }
            // stage P%NSTG consumed by every thread: it may be refilled.  (Per-warp
            // release through "empty" mbarriers instead was slower: 35.1 vs 33.4 ms.)
            if (ASYNC && kb + 2 * CAPTE < K1) {
                // piece j + 2 lies in this chunk: the last warp to finish piece j
                // refills its stage; the other warps go on without waiting
                // Ordering: __syncwarp orders the warp's reads of the stage before
                // lane 0's arrival; the arrival is a release (and the last one an
                // acquire) at CTA scope, so every warp's generic-proxy reads of
                // the stage happen-before the refill; fence.proxy.async then
                // orders them before the async-proxy (TMA) write.
                constexpr unsigned NW = NT / 32;
                __syncwarp();
                if ((tid & 31) == 0) {
                    cuda::atomic_ref<unsigned, cuda::thread_scope_block> arr(S.arr[ps.P & 1]);
                    const unsigned old = arr.fetch_add(1u, cuda::memory_order_acq_rel);
                    if (old % NW == NW - 1) {
                        fence_proxy_async_smem();
                        const int64_t k2 = kb + 2 * CAPTE;
                        issue(ps.P & 1, k2, k2 + CAPTE < K1 ? k2 + CAPTE : K1);
                    }
                }
            } else {
                __syncthreads();
            }
            ++ps.P;
            kb = ke;
        }
        double dot = 0.0;
        if (PLAIN) {
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                const int r = t * NT + tid;
                if (t < CH && r < crows) L.q[cr0 + r] = acc[t];
            }
        } else {
            double *__restrict__ x = L.x;
            double *__restrict__ p = L.p;
            double *__restrict__ q = L.q;
            double ri[MAXCH], po[MAXCH], qo[MAXCH], xo[MAXCH];
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                const int r = t * NT + tid;
                const bool ok = t < CH && r < crows;
                const int64_t i = cr0 + r;
                ri[t] = ok ? rv[i] : 0.0;
                po[t] = ok && !first ? p[i] : 0.0;
                qo[t] = ok && !first ? q[i] : 0.0;
                xo[t] = ok && !first ? x[i] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                const int r = t * NT + tid;
                if (t < CH && r < crows) {
                    const int64_t i = cr0 + r;
                    const double pn = first ? ri[t] : ri[t] + beta * po[t];
                    const double qn = first ? acc[t] : acc[t] + beta * qo[t];
                    p[i] = pn;
                    q[i] = qn;
                    x[i] = first ? 0.0 : xo[t] + alpha_prev * po[t];
                    dot += pn * qn;
                }
            }
        }
        const double s = block_sum<NT>(dot, S.red);  // its barriers also retire rp buffer cs&1
        if (tid == 0) {
            if (!PLAIN) {
                part_out[cbase + me + k * nb] = s;
                push(cbase + me + k * nb, s);  // partitioned CG over peer memory: the peers' copies
            }
            if (k + 2 < K) {
                int64_t nr0;
                int nrows;
                chunk_rows(k + 2, nr0, nrows);
                issue_rp(S, cs & 1, L.row_ptr, nr0, nrows, pol);
            }
        }
    }
    ps.CS += (uint32_t)K;
}

template <int C, int MB>
__global__ void __launch_bounds__(NT, MB) k_cg(CGBatch B) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CGSharedTT<C> &S = *reinterpret_cast<CGSharedTT<C> *>(smem_raw);

    int g = 0;
    while (g + 1 < B.nlev && (int)blockIdx.x >= B.lev[g + 1].block_begin) ++g;
    const CGLevelArgs &L = B.lev[g];
    const int nb = L.nblocks, me = (int)blockIdx.x - L.block_begin;
    const int tid = threadIdx.x;
    const int64_t n = L.n;
    const int CH = L.chunk_tiles;
    const int64_t ntiles = (n + NT - 1) / NT;
    const int64_t nchunks = (ntiles + CH - 1) / CH;
    double *part = L.partials;  // 3 * nchunks
    unsigned long long round = 0;
    PipeState ps{0u, 0u};
    if (tid == 0) {
        for (int b = 0; b < NSTG; ++b) mbar_init(&S.bar_st[b], 1);
        mbar_init(&S.bar_rp[0], 1);
        mbar_init(&S.bar_rp[1], 1);
        S.arr[0] = S.arr[1] = 0u;
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();

    // ---- init: r = b, bb = b.b (x, p, q are first written by iteration 0)
    for (int64_t c = me; c < nchunks; c += nb) {
        double acc = 0.0;
        for (int t = 0; t < CH; ++t) {
            int64_t i = (c * CH + t) * NT + tid;
            if (i < n) {
                double bi = L.b_src ? __ldg(&L.b_src[__ldg(&L.b_perm[i])]) : __ldg(&L.b[i]);
                L.r[i] = bi;
                acc += bi * bi;
            }
        }
        double s = block_sum<NT>(acc, S.red);
        if (tid == 0) part[c] = s;
    }
    const double bb = chunk_allreduce(part, nchunks, nb, L.barrier, round, S.red);
    double rr = bb;
    int it = 0, status = 0;
    // optional phase timing (CTA 0 of the group, thread 0; MSK_CG_PHASES=1)
    const bool tdbg = L.dbg != nullptr && me == 0 && tid == 0;
    unsigned long long tph[6] = {0, 0, 0, 0, 0, 0}, tprev = 0;
    auto tick = [&](int k) {
        if (tdbg) {
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (k >= 0) tph[k] += now - tprev;
            tprev = now;
        }
    };
    double alpha = 0.0, beta = 0.0;
    if (bb > 0.0) {
        const double stop = L.tol2 * bb;
        for (;;) {
            if (rr <= stop) break;
            if (it >= L.max_iter) { status = 1; break; }
            tick(-1);
            // ---- w = A r ; p = r + beta p ; q = w + beta q ; x += alpha p_old ; pq = p.q
            if (L.col16)
                spmv_phase<C, false, NoPush, true>(S, L, me, nb, 0, nchunks, CH, part + nchunks, ps, pol, it == 0,
                                                   alpha, beta);
            else
                spmv_phase(S, L, me, nb, 0, nchunks, CH, part + nchunks, ps, pol, it == 0, alpha, beta);
            tick(0);
            const double pq = chunk_allreduce(part + nchunks, nchunks, nb, L.barrier, round, S.red);
            tick(1);
            alpha = rr / pq;
            if (L.coef && me == 0 && tid == 0 && it < L.coef_cap) L.coef[2 * it] = alpha;
            // ---- r -= alpha q, rr' = r.r
            {
                double *__restrict__ r = L.r;
                const double *__restrict__ q = L.q;
                for (int64_t c = me; c < nchunks; c += nb) {
                    double rv[MAXCH], qv[MAXCH];
#pragma unroll
                    for (int t = 0; t < MAXCH; ++t) {
                        int64_t i = (c * CH + t) * NT + tid;
                        bool ok = t < CH && i < n;
                        rv[t] = ok ? r[i] : 0.0;
                        qv[t] = ok ? q[i] : 0.0;
                    }
                    double acc = 0.0;
#pragma unroll
                    for (int t = 0; t < MAXCH; ++t) {
                        int64_t i = (c * CH + t) * NT + tid;
                        if (t < CH && i < n) {
                            double ri = rv[t] - alpha * qv[t];
                            r[i] = ri;
                            acc += ri * ri;
                        }
                    }
                    double s = block_sum<NT>(acc, S.red);
                    if (tid == 0) part[2 * nchunks + c] = s;
                }
            }
            tick(2);
            const double rrn = chunk_allreduce(part + 2 * nchunks, nchunks, nb, L.barrier, round, S.red);
            tick(3);
            beta = rrn / rr;
            rr = rrn;
            if (L.coef && me == 0 && tid == 0 && it < L.coef_cap) L.coef[2 * it + 1] = beta;
            ++it;
        }
    }
    if (tdbg)
        for (int k = 0; k < 6; ++k) L.dbg[k] = tph[k];
    // ---- the last deferred update x += alpha p (own rows: no barrier needed)
    for (int64_t c = me; c < nchunks; c += nb)
        for (int t = 0; t < CH; ++t) {
            int64_t i = (c * CH + t) * NT + tid;
            if (i < n) {
                const double xi = it > 0 ? L.x[i] + alpha * L.p[i] : 0.0;
                L.x[i] = xi;
                if (L.x_out) L.x_out[__ldg(&L.x_perm[i])] = xi;
            }
        }
    if (me == 0 && tid == 0) {
        *L.out_iters = it;
        L.out_rr[0] = rr;
        L.out_rr[1] = bb;
        *L.out_status = status;
    }
}

// ---------------------------------------------------------------------------
// Multi-RHS CG (msk_solve_multi): one level, R right-hand sides sharing every
// CSR piece (the matrix is streamed once per iteration for all R columns).
// Per column the arithmetic is k_cg's, in the same order (chunk partials,
// block_sum tree, fma order in the rows), with per-column scalars; a column
// that has met its stopping rule is frozen (alpha = beta = 0 from then on:
// x, r unchanged exactly), so every column equals its single-RHS solve bit for
// bit.  Vectors are [n][R] row-major (x with row stride ldx).
template <int C, int R>
struct __align__(16) CGSharedR {
    CGSharedTT<C> b;
    double redr[R * (NT / 32 + 1)];
};

template <int R>
__device__ __forceinline__ void chunk_allreduce_r(const double *partials, int64_t nchunks, int nb,
                                                  unsigned long long *ctr, unsigned long long &round,
                                                  double *s_red, double (&out)[R]) {
    group_barrier(ctr, nb, round);
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = 0.0;
    int64_t j = threadIdx.x;
    for (; j + 3 * NT < nchunks; j += 4 * NT) {  // loads ahead of the adds, same order (strided_sum)
        double v[4][R];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) v[u][r] = __ldcg(&partials[(j + u * NT) * R + r]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) out[r] += v[u][r];
    }
    for (; j < nchunks; j += NT) {
#pragma unroll
        for (int r = 0; r < R; ++r) out[r] += __ldcg(&partials[j * R + r]);
    }
    block_sum_r<NT, R>(out, s_red);
}

template <int C, int R>
__device__ __forceinline__ void spmv_phase_r(CGSharedR<C, R> &SR, const CGRArgs &A, int me, int nb, int CH,
                                             double *part_out, PipeState &ps, uint64_t pol, bool first,
                                             const double (&alpha_prev)[R], const double (&beta)[R]) {
    constexpr int CAPTE = C - 2;
    constexpr int UR = 2;  // gathers (R doubles each) in flight per thread
    CGSharedTT<C> &S = SR.b;
    const int tid = threadIdx.x;
    const int64_t n = A.n;
    const int64_t ntiles = (n + NT - 1) / NT, nloc = (ntiles + CH - 1) / CH;
    const int64_t K = me < nloc ? (nloc - 1 - me) / nb + 1 : 0;
    if (K == 0) return;
    const double *rv = A.r;
    auto chunk_rows = [&](int64_t k, int64_t &cr0, int &crows) {
        const int64_t c = me + k * nb;
        cr0 = c * CH * NT;
        crows = (int)(n - cr0 < (int64_t)CH * NT ? n - cr0 : (int64_t)CH * NT);
    };
    auto rp_off = [&](int64_t cr0) { return (int)(cr0 - (cr0 & ~(int64_t)1)); };
    int64_t cr0;
    int crows;
    if (tid == 0) {
        chunk_rows(0, cr0, crows);
        issue_rp(S, ps.CS & 1, A.row_ptr, cr0, crows, pol);
        if (K > 1) {
            chunk_rows(1, cr0, crows);
            issue_rp(S, (ps.CS + 1) & 1, A.row_ptr, cr0, crows, pol);
        }
    }
    mbar_wait(&S.bar_rp[ps.CS & 1], (ps.CS >> 1) & 1u);
    chunk_rows(0, cr0, crows);
    {
        const int64_t *rp = S.rp[ps.CS & 1] + rp_off(cr0);
        const int64_t K0 = rp[0], K1 = rp[crows];
        if (tid == 0) issue_piece_t(S, ps.P & 1, A.col, A.val, K0, K0 + CAPTE < K1 ? K0 + CAPTE : K1, pol);
    }
    for (int64_t k = 0; k < K; ++k) {
        chunk_rows(k, cr0, crows);
        const uint32_t cs = ps.CS + (uint32_t)k;
        const int64_t *rp = S.rp[cs & 1] + rp_off(cr0);
        const int64_t K1 = rp[crows];
        int64_t rb[MAXCH], re[MAXCH];
        double acc[MAXCH][R];
#pragma unroll
        for (int t = 0; t < MAXCH; ++t) {
            const int r = t * NT + tid;
            const bool ok = t < CH && r < crows;
            rb[t] = ok ? rp[r] : 0;
            re[t] = ok ? rp[r + 1] : 0;
#pragma unroll
            for (int c = 0; c < R; ++c) acc[t][c] = 0.0;
        }
        for (int64_t kb = rp[0]; kb < K1;) {
            const int64_t ke = kb + CAPTE < K1 ? kb + CAPTE : K1;
            if (ke < K1) {
                if (tid == 0)
                    issue_piece_t(S, (ps.P + 1) & 1, A.col, A.val, ke, ke + CAPTE < K1 ? ke + CAPTE : K1, pol);
            } else if (k + 1 < K) {
                mbar_wait(&S.bar_rp[(cs + 1) & 1], ((cs + 1) >> 1) & 1u);
                if (tid == 0) {
                    int64_t nr0;
                    int nrows;
                    chunk_rows(k + 1, nr0, nrows);
                    const int64_t *nrp = S.rp[(cs + 1) & 1] + rp_off(nr0);
                    const int64_t a = nrp[0], e = nrp[nrows];
                    issue_piece_t(S, (ps.P + 1) & 1, A.col, A.val, a, a + CAPTE < e ? a + CAPTE : e, pol);
                }
            }
            mbar_wait(&S.bar_st[ps.P & 1], (ps.P >> 1) & 1u);
            const CtaStageT<C> &cur = S.st[ps.P & 1];
            const int voff = (int)(kb & 1), coff = (int)(kb & 3);
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                if (t >= CH) break;
                const int64_t lo64 = rb[t] > kb ? rb[t] : kb, hi64 = re[t] < ke ? re[t] : ke;
                const int lo = (int)(lo64 - kb);
                const int hi = hi64 > lo64 ? (int)(hi64 - kb) : lo;
                for (int e = lo; e < hi; e += UR) {
                    double pv[UR][R], vv[UR];
#pragma unroll
                    for (int u = 0; u < UR; ++u) {
                        const int ee = e + u;
                        const bool ok = ee < hi;
                        const double2 *src = reinterpret_cast<const double2 *>(rv + (int64_t)(ok ? cur.col[coff + ee] : 0) * R);
#pragma unroll
                        for (int c = 0; c < R; c += 2) {
                            const double2 w2 = ok ? src[c / 2] : make_double2(0.0, 0.0);
                            pv[u][c] = w2.x;
                            pv[u][c + 1] = w2.y;
                        }
                        vv[u] = ok ? cur.val[voff + ee] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < UR; ++u)
                        if (e + u < hi) {
#pragma unroll
                            for (int c = 0; c < R; ++c) acc[t][c] = fma(vv[u], pv[u][c], acc[t][c]);
                        }
                }
            }
            __syncthreads();
            ++ps.P;
            kb = ke;
        }
        double dot[R];
#pragma unroll
        for (int c = 0; c < R; ++c) dot[c] = 0.0;
        {
            // all loads of the chunk's rows first (independent, in flight together), then the stores
            double *__restrict__ xw = A.x;
            double *__restrict__ pw = A.p;
            double *__restrict__ qw = A.q;
            constexpr int TB = R >= 4 ? 2 : MAXCH;  // rows per load batch (register budget)
#pragma unroll
            for (int t0 = 0; t0 < MAXCH; t0 += TB) {
                double ri[TB][R], po[TB][R], qo[TB][R], xo[TB][R];
#pragma unroll
                for (int tt = 0; tt < TB; ++tt) {
                    const int t = t0 + tt;
                    const int r = t * NT + tid;
                    const bool ok = t < CH && r < crows;
                    const int64_t i = cr0 + r;
#pragma unroll
                    for (int c = 0; c < R; ++c) {
                        ri[tt][c] = ok ? rv[i * R + c] : 0.0;
                        po[tt][c] = ok && !first ? pw[i * R + c] : 0.0;
                        qo[tt][c] = ok && !first ? qw[i * R + c] : 0.0;
                        xo[tt][c] = ok && !first ? xw[i * A.ldx + c] : 0.0;
                    }
                }
#pragma unroll
                for (int tt = 0; tt < TB; ++tt) {
                    const int t = t0 + tt;
                    const int r = t * NT + tid;
                    if (t < CH && r < crows) {
                        const int64_t i = cr0 + r;
#pragma unroll
                        for (int c = 0; c < R; ++c) {
                            const double pn = first ? ri[tt][c] : ri[tt][c] + beta[c] * po[tt][c];
                            const double qn = first ? acc[t][c] : acc[t][c] + beta[c] * qo[tt][c];
                            pw[i * R + c] = pn;
                            qw[i * R + c] = qn;
                            xw[i * A.ldx + c] = first ? 0.0 : xo[tt][c] + alpha_prev[c] * po[tt][c];
                            dot[c] += pn * qn;
                        }
                    }
                }
            }
        }
        block_sum_r<NT, R>(dot, SR.redr);
        if (tid == 0) {
            const int64_t c0 = me + k * nb;
#pragma unroll
            for (int c = 0; c < R; ++c) part_out[c0 * R + c] = dot[c];
            if (k + 2 < K) {
                int64_t nr0;
                int nrows;
                chunk_rows(k + 2, nr0, nrows);
                issue_rp(S, cs & 1, A.row_ptr, nr0, nrows, pol);
            }
        }
    }
    ps.CS += (uint32_t)K;
}

template <int C, int MB, int R>
__global__ void __launch_bounds__(NT, MB) k_cgr(CGRArgs A, int nb, int CH, double *part,
                                                unsigned long long *barrier) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CGSharedR<C, R> &SR = *reinterpret_cast<CGSharedR<C, R> *>(smem_raw);
    CGSharedTT<C> &S = SR.b;
    const int me = (int)blockIdx.x, tid = threadIdx.x;
    const int64_t n = A.n;
    const int64_t ntiles = (n + NT - 1) / NT;
    const int64_t nchunks = (ntiles + CH - 1) / CH;
    unsigned long long round = 0;
    PipeState ps{0u, 0u};
    if (tid == 0) {
        for (int b = 0; b < NSTG; ++b) mbar_init(&S.bar_st[b], 1);
        mbar_init(&S.bar_rp[0], 1);
        mbar_init(&S.bar_rp[1], 1);
        S.arr[0] = S.arr[1] = 0u;
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    // ---- init: r = b, bb = b.b per column
    for (int64_t c = me; c < nchunks; c += nb) {
        double acc[R];
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = 0.0;
        for (int t = 0; t < CH; ++t) {
            const int64_t i = (c * CH + t) * NT + tid;
            if (i < n) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    double bi;
                    if (A.b) bi = __ldg(&A.b[i * R + k]);
                    else bi = k < A.nvalid ? __ldg(&A.b_src[(int64_t)__ldg(&A.b_perm[i]) * A.ldb + A.col0 + k]) : 0.0;
                    A.r[i * R + k] = bi;
                    acc[k] += bi * bi;
                }
            }
        }
        block_sum_r<NT, R>(acc, SR.redr);
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < R; ++k) part[c * R + k] = acc[k];
        }
    }
    double bb[R], rr[R], alpha[R], beta[R];
    chunk_allreduce_r<R>(part, nchunks, nb, barrier, round, SR.redr, bb);
    int itc[R];
    bool act[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        rr[k] = bb[k];
        alpha[k] = 0.0;
        beta[k] = 0.0;
        itc[k] = 0;
    }
    int it = 0;
    for (;;) {
        bool any = false;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            act[k] = bb[k] > 0.0 && rr[k] > A.tol2 * bb[k] && it < A.max_iter;
            any = any || act[k];
        }
        if (!any) break;
        // ---- pass 1: w = A r ; p, q, x updates ; pq
        spmv_phase_r<C, R>(SR, A, me, nb, CH, part + nchunks * R, ps, pol, it == 0, alpha, beta);
        double pq[R];
        chunk_allreduce_r<R>(part + nchunks * R, nchunks, nb, barrier, round, SR.redr, pq);
#pragma unroll
        for (int k = 0; k < R; ++k) alpha[k] = act[k] ? rr[k] / pq[k] : 0.0;
        // ---- pass 2: r -= alpha q ; rr
        for (int64_t c = me; c < nchunks; c += nb) {
            double acc[R];
#pragma unroll
            for (int k = 0; k < R; ++k) acc[k] = 0.0;
            double *__restrict__ rw = A.r;
            const double *__restrict__ qr = A.q;
            double rv4[MAXCH][R], qv4[MAXCH][R];
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                const int64_t i = (c * CH + t) * NT + tid;
                const bool ok = t < CH && i < n;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    rv4[t][k] = ok ? rw[i * R + k] : 0.0;
                    qv4[t][k] = ok ? qr[i * R + k] : 0.0;
                }
            }
#pragma unroll
            for (int t = 0; t < MAXCH; ++t) {
                const int64_t i = (c * CH + t) * NT + tid;
                if (t < CH && i < n) {
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const double ri = rv4[t][k] - alpha[k] * qv4[t][k];
                        rw[i * R + k] = ri;
                        acc[k] += ri * ri;
                    }
                }
            }
            block_sum_r<NT, R>(acc, SR.redr);
            if (tid == 0) {
#pragma unroll
                for (int k = 0; k < R; ++k) part[(2 * nchunks + c) * R + k] = acc[k];
            }
        }
        double rrn[R];
        chunk_allreduce_r<R>(part + 2 * nchunks * R, nchunks, nb, barrier, round, SR.redr, rrn);
#pragma unroll
        for (int k = 0; k < R; ++k) {
            beta[k] = act[k] ? rrn[k] / rr[k] : 0.0;
            if (act[k]) {
                rr[k] = rrn[k];
                ++itc[k];
            }
        }
        ++it;
    }
    // ---- the last deferred x update, then caller order
    for (int64_t c = me; c < nchunks; c += nb)
        for (int t = 0; t < CH; ++t) {
            const int64_t i = (c * CH + t) * NT + tid;
            if (i < n) {
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const double xi = it > 0 ? A.x[i * A.ldx + k] + alpha[k] * A.p[i * R + k] : 0.0;
                    A.x[i * A.ldx + k] = xi;
                    if (A.x_out && k < A.nvalid) A.x_out[(int64_t)__ldg(&A.x_perm[i]) * A.ldo + A.col0 + k] = xi;
                }
            }
        }
    if (me == 0 && tid == 0) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            A.out_iters[k] = itc[k];
            A.out_rr[2 * k] = rr[k];
            A.out_rr[2 * k + 1] = bb[k];
            A.out_status[k] = bb[k] > 0.0 && rr[k] > A.tol2 * bb[k] ? 1 : 0;
        }
    }
}

// standalone y = A v (msk_apply_block): the CG's pipelined SpMV pass without
// the CG epilogue, persistent grid (one CTA per resident slot, chunks round robin)
template <int C, int MB>
__global__ void __launch_bounds__(NT, MB) k_spmv_t(CGLevelArgs L, int CH) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CGSharedTT<C> &S = *reinterpret_cast<CGSharedTT<C> *>(smem_raw);
    if (threadIdx.x == 0) {
        for (int b = 0; b < NSTG; ++b) mbar_init(&S.bar_st[b], 1);
        mbar_init(&S.bar_rp[0], 1);
        mbar_init(&S.bar_rp[1], 1);
        S.arr[0] = S.arr[1] = 0u;
        fence_mbar_init();
    }
    __syncthreads();
    PipeState ps{0u, 0u};
    const int64_t nch = ((L.n + NT - 1) / NT + CH - 1) / CH;
    spmv_phase<C, true>(S, L, blockIdx.x, gridDim.x, 0, nch, CH, nullptr, ps, policy_evict_first(), false, 0.0,
                        0.0);
}

// ---------------------------------------------------------------------------
// Distributed CG (one partition = a contiguous range of whole chunks of one
// level).  The same arithmetic as k_cg, split into phase kernels so that the
// chunk partials can be all-reduced (NCCL or the single-process emulation)
// and the halo of r exchanged between phases.  Scalars live on the device;
// kernels do nothing once the CG has stopped.  Because every partial is
// computed per chunk exactly as in k_cg and summed over all chunks in the
// same fixed order, the result is bit-identical to the single-GPU solve for
// any number of partitions.
__device__ __forceinline__ void dcg_check_top(DistCGScalars &s, double tol2, int max_iter) {
    if (!(s.bb > 0.0) || s.rr <= tol2 * s.bb) {
        s.active = 0;
    } else if (s.it >= max_iter) {
        s.active = 0;
        s.status = 1;
    } else {
        s.active = 1;
    }
}

// ---------------------------------------------------------------------------
// Partitioned CG over peer memory (PeerCGArgs, kernels.cuh).  One persistent
// cooperative launch per rank runs the whole CG of its row block; W ranks in
// ONE launch in the single-GPU emulation (rank = blockIdx.x / nb).
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_sys_add(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// the fixed-order chunk sum of chunk_allreduce (no barrier: the caller's
// cross-rank barrier has made every chunk partial visible)
__device__ __forceinline__ double chunk_sum(const double *partials, int64_t nchunks, double *s_red) {
    return block_sum<NT>(strided_sum(partials, nchunks), s_red);
}

struct PeerPush {  // thread 0 stores a chunk partial into every rank's copy
    const PeerCGArgs *A;
    int64_t off;
    __device__ __forceinline__ void operator()(int64_t c, double s) const {
        for (int w = 0; w < A->W; ++w)
            if (A->R[w].part) A->R[w].part[off + c] = s;
    }
};

template <int C, int MB>
__global__ void __launch_bounds__(NT, MB) k_pcg(const __grid_constant__ PeerCGArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CGSharedTT<C> &S = *reinterpret_cast<CGSharedTT<C> *>(smem_raw);
    const int W = A.W, nb = A.nb, tid = threadIdx.x;
    const int m = A.rank >= 0 ? A.rank : (int)blockIdx.x / nb;
    const int me = (int)blockIdx.x - (A.rank >= 0 ? 0 : m * nb);
    const PeerRank &Rm = A.R[m];
    CGLevelArgs L = A.L;
    L.x = Rm.x; L.r = Rm.r; L.p = Rm.p; L.q = Rm.q;
    L.row_ptr = Rm.row_ptr; L.col = Rm.col; L.val = Rm.val;
    const int64_t n = L.n, nch = A.nchunks, c0 = Rm.c0, c1 = Rm.c1;
    const int CH = L.chunk_tiles;
    double *part = Rm.part;
    if (tid == 0) {
        for (int b = 0; b < NSTG; ++b) mbar_init(&S.bar_st[b], 1);
        mbar_init(&S.bar_rp[0], 1);
        mbar_init(&S.bar_rp[1], 1);
        S.arr[0] = S.arr[1] = 0u;
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    unsigned long long round = 0;
    unsigned long long xround = *Rm.nbar;  // barriers of earlier launches (identical on every rank)
    // cross-rank barrier: every thread's peer stores are fenced at system scope,
    // the rank's CTAs meet (group barrier), its leader adds 1 to every rank's
    // counter (release, system scope), every CTA waits for W arrivals (acquire)
    auto xbarrier = [&]() {
        __syncthreads();
        if (tid == 0) fence_acq_rel_sys();  // cumulative: the CTA's peer stores, ordered by the bar.sync
        group_barrier(Rm.gbar, nb, round);
        ++xround;
        if (me == 0 && tid == 0) {
            // one system-scope release fence, then relaxed adds (fence + relaxed
            // write = release); the group barrier's acquire made every CTA's
            // stores (each fenced above) happen-before this fence
            fence_acq_rel_sys();
            for (int w = 0; w < W; ++w) red_relaxed_sys_add(A.R[w].xcnt, 1ull);
        }
        if (tid == 0) {
            const unsigned long long want = (unsigned long long)W * xround;
            unsigned long long spins = 0;
            while (ld_relaxed_sys(Rm.xcnt) < want) {  // poll relaxed, then one acquire
                __nanosleep(32);
                if (++spins > (1ull << 31)) __trap();  // never hang the device forever
            }
            (void)ld_acquire_sys(Rm.xcnt);
        }
        __syncthreads();
    };
    // r of a row this rank owns -> the peers whose SpMV reads it (their halo)
    const int64_t slo = Rm.slo, shi = Rm.shi;
    auto push_halo = [&](int64_t i, double v) {
        if (i < slo || i >= shi) return;  // interior row: no peer reads it
        for (int w = 0; w < W; ++w)
            if (w != m && i >= A.R[w].hlo && i < A.R[w].hhi) A.R[w].r[i] = v;
    };
    auto push_part = [&](int64_t off, int64_t c, double v) {
        for (int w = 0; w < W; ++w) A.R[w].part[off + c] = v;
    };

    // ---- init: r = b on the owned rows (+ halo copies), bb partials
    for (int64_t c = c0 + me; c < c1; c += nb) {
        double acc = 0.0;
        for (int t = 0; t < CH; ++t) {
            const int64_t i = (c * CH + t) * NT + tid;
            if (i < n) {
                const double bi = L.b_src ? __ldg(&L.b_src[__ldg(&L.b_perm[i])]) : __ldg(&L.b[i]);
                L.r[i] = bi;
                push_halo(i, bi);
                acc += bi * bi;
            }
        }
        const double s = block_sum<NT>(acc, S.red);
        if (tid == 0) push_part(0, c, s);
    }
    xbarrier();
    const double bb = chunk_sum(part, nch, S.red);
    double rr = bb;
    int it = 0, status = 0;
    double alpha = 0.0, beta = 0.0;
    PipeState ps{0u, 0u};
    const PeerPush pq_push{&A, nch};
    if (bb > 0.0) {
        const double stop = L.tol2 * bb;
        for (;;) {
            if (rr <= stop) break;
            if (it >= L.max_iter) { status = 1; break; }
            // ---- w = A r ; p = r + beta p ; q = w + beta q ; x += alpha p_old ; pq partials
            spmv_phase<C, false, PeerPush>(S, L, me, nb, c0, c1 - c0, CH, part + nch, ps, pol, it == 0, alpha,
                                           beta, pq_push);
            xbarrier();
            const double pq = chunk_sum(part + nch, nch, S.red);
            alpha = rr / pq;
            if (L.coef && m == 0 && me == 0 && tid == 0 && it < L.coef_cap) L.coef[2 * it] = alpha;
            // ---- r -= alpha q on the owned rows (+ halo copies), rr' partials
            for (int64_t c = c0 + me; c < c1; c += nb) {
                double rv[MAXCH], qv[MAXCH];
#pragma unroll
                for (int t = 0; t < MAXCH; ++t) {
                    const int64_t i = (c * CH + t) * NT + tid;
                    const bool ok = t < CH && i < n;
                    rv[t] = ok ? L.r[i] : 0.0;
                    qv[t] = ok ? L.q[i] : 0.0;
                }
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t < MAXCH; ++t) {
                    const int64_t i = (c * CH + t) * NT + tid;
                    if (t < CH && i < n) {
                        const double ri = rv[t] - alpha * qv[t];
                        L.r[i] = ri;
                        push_halo(i, ri);
                        acc += ri * ri;
                    }
                }
                const double s = block_sum<NT>(acc, S.red);
                if (tid == 0) push_part(2 * nch, c, s);
            }
            xbarrier();
            const double rrn = chunk_sum(part + 2 * nch, nch, S.red);
            beta = rrn / rr;
            rr = rrn;
            if (L.coef && m == 0 && me == 0 && tid == 0 && it < L.coef_cap) L.coef[2 * it + 1] = beta;
            ++it;
        }
    }
    // ---- the last deferred x += alpha p on the owned rows, pushed to every rank's alpha
    for (int64_t c = c0 + me; c < c1; c += nb)
        for (int t = 0; t < CH; ++t) {
            const int64_t i = (c * CH + t) * NT + tid;
            if (i < n) {
                const double xi = it > 0 ? L.x[i] + alpha * L.p[i] : 0.0;
                L.x[i] = xi;
                for (int w = 0; w < W; ++w) A.R[w].alpha[i] = xi;
            }
        }
    xbarrier();
    if (me == 0 && tid == 0) {
        *Rm.nbar = xround;
        if (m == 0 || A.rank >= 0) {
            *L.out_iters = it;
            L.out_rr[0] = rr;
            L.out_rr[1] = bb;
            *L.out_status = status;
        }
    }
}

__global__ void __launch_bounds__(NT) k_dcg_init(DistCGArgs A) {
    __shared__ double red[NT / 32 + 2];
    const CGLevelArgs &L = A.L;
    const int CH = L.chunk_tiles, tid = threadIdx.x;
    for (int64_t c = A.c0 + blockIdx.x; c < A.c1; c += gridDim.x) {
        double acc = 0.0;
        for (int t = 0; t < CH; ++t) {
            int64_t i = (c * CH + t) * NT + tid;
            if (i < L.n) {
                double bi = L.b_src ? __ldg(&L.b_src[__ldg(&L.b_perm[i])]) : __ldg(&L.b[i]);
                L.r[i] = bi;
                acc += bi * bi;
            }
        }
        double s = block_sum<NT>(acc, red);
        if (tid == 0) A.part_send[c] = s;
    }
}

template <int C, int MB>
__global__ void __launch_bounds__(NT, MB) k_dcg_spmv(DistCGArgs A) {
    if (!A.sc->active) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CGSharedTT<C> &S = *reinterpret_cast<CGSharedTT<C> *>(smem_raw);
    if (threadIdx.x == 0) {
        for (int b = 0; b < NSTG; ++b) mbar_init(&S.bar_st[b], 1);
        mbar_init(&S.bar_rp[0], 1);
        mbar_init(&S.bar_rp[1], 1);
        S.arr[0] = S.arr[1] = 0u;
        fence_mbar_init();
    }
    __syncthreads();
    PipeState ps{0u, 0u};
    const DistCGScalars &sc = *A.sc;
    spmv_phase(S, A.L, blockIdx.x, gridDim.x, A.c0, A.c1 - A.c0, A.L.chunk_tiles, A.part_send, ps,
               policy_evict_first(), sc.it == 0, sc.alpha, sc.beta);
}

__global__ void __launch_bounds__(NT) k_dcg_rupd(DistCGArgs A) {
    if (!A.sc->active) return;
    __shared__ double red[NT / 32 + 2];
    const CGLevelArgs &L = A.L;
    const int CH = L.chunk_tiles, tid = threadIdx.x;
    const double alpha = A.sc->alpha;
    for (int64_t c = A.c0 + blockIdx.x; c < A.c1; c += gridDim.x) {
        double acc = 0.0;
        for (int t = 0; t < CH; ++t) {
            int64_t i = (c * CH + t) * NT + tid;
            if (i < L.n) {
                double ri = L.r[i] - alpha * L.q[i];
                L.r[i] = ri;
                acc += ri * ri;
            }
        }
        double s = block_sum<NT>(acc, red);
        if (tid == 0) A.part_send[c] = s;
    }
}

// after the loop: the last deferred x += alpha p on the owned rows (x = 0
// when no iteration ran)
__global__ void __launch_bounds__(NT) k_dcg_xfin(DistCGArgs A) {
    const CGLevelArgs &L = A.L;
    const int CH = L.chunk_tiles, tid = threadIdx.x;
    const bool any = A.sc->it > 0;
    const double alpha = A.sc->alpha;
    for (int64_t c = A.c0 + blockIdx.x; c < A.c1; c += gridDim.x)
        for (int t = 0; t < CH; ++t) {
            int64_t i = (c * CH + t) * NT + tid;
            if (i < L.n) L.x[i] = any ? L.x[i] + alpha * L.p[i] : 0.0;
        }
}

// Matrix-free pass 1 (MSK_FLAG_MATRIX_FREE): per owned row i, w = sum_j
// Phi(x_i - x_j) r_j with Phi evaluated exactly as k_fill stores it
// (scale * phi(sqrt(r2) / delta)) and the hits visited in ascending j -- the
// CSR column order -- so w, and with the same epilogue and chunk partials as
// spmv_phase the whole CG, is bit-identical to the assembled path.
// Candidates: conservative FP32 prefilter (gather.cu), then the exact no-FMA
// test (reading C-4) on the survivors.
template <int D, int K>
__global__ void __launch_bounds__(NT, MSK_MF_MINB) k_mf_spmv(DistCGArgs A, LevelView V) {
    if (!A.sc->active) return;
    __shared__ double red[NT / 32 + 2];
    constexpr int HM = 40;
    const CGLevelArgs &L = A.L;
    const int CH = L.chunk_tiles, tid = threadIdx.x;
    const bool first = A.sc->it == 0;
    const double alpha_prev = A.sc->alpha, beta = A.sc->beta;
    const double *rv = L.r;
    const double d2 = V.delta2, inv = V.inv_delta, scl = V.scale;
    const float fthr = V.fthr;
    const float4 *__restrict__ frec = V.frec;
    const double4 *__restrict__ rec = V.rec;
    for (int64_t c = A.c0 + blockIdx.x; c < A.c1; c += gridDim.x) {
        double dot = 0.0;
        for (int t = 0; t < CH; ++t) {
            const int64_t i = (c * CH + t) * NT + tid;
            if (i >= L.n) continue;
            double x[3];
            float xf[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int a = 0; a < D; ++a) {
                x[a] = V.x[a][i];
                xf[a] = (float)(x[a] - V.g.lo[a]);
            }
            double acc = 0.0;
            int hl[HM];
            int nh = 0;
            auto flush = [&]() {
                int h = 0;
                // MFU survivors per trip: their records and gathered r values are
                // loaded up front (independent loads in flight), then accumulated in
                // ascending order as before (a miss adds nothing: bit-identical)
                constexpr int MFU = D == 2 ? MSK_MF_U2 : MSK_MF_U3;
                for (; MFU > 1 && h + MFU <= nh; h += MFU) {
                    double4 R[MFU];
                    double rj[MFU];
#pragma unroll
                    for (int u = 0; u < MFU; ++u) {
                        const int j = hl[h + u];
                        R[u] = rec[j];
                        rj[u] = rv[j];
                    }
#pragma unroll
                    for (int u = 0; u < MFU; ++u) {
                        const double y[3] = {R[u].x, R[u].y, R[u].z};
                        const double r2 = dist2_nofma<D>(x, y);
                        if (r2 < d2) {
                            const double v = scl * wendland<K>(sqrt(r2) * inv);
                            acc = fma(v, rj[u], acc);
                        }
                    }
                }
                for (; h < nh; ++h) {
                    const int j = hl[h];
                    const double4 R = rec[j];  // packed coordinates (the .w slot is unused here)
                    const double y[3] = {R.x, R.y, R.z};
                    const double r2 = dist2_nofma<D>(x, y);
                    if (r2 < d2) {
                        const double v = scl * wendland<K>(sqrt(r2) * inv);
                        acc = fma(v, rv[j], acc);
                    }
                }
                nh = 0;
            };
            for_each_range<D>(V, x, [&](int b, int e) {
                int j = b;
#if MSK_MF_P == 4
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
#endif
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
            // epilogue: the expressions of spmv_phase
            const double ri = rv[i];
            const double po = first ? 0.0 : L.p[i], qo = first ? 0.0 : L.q[i], xo = first ? 0.0 : L.x[i];
            const double pn = first ? ri : ri + beta * po;
            const double qn = first ? acc : acc + beta * qo;
            L.p[i] = pn;
            L.q[i] = qn;
            L.x[i] = first ? 0.0 : xo + alpha_prev * po;
            dot += pn * qn;
        }
        const double s = block_sum<NT>(dot, red);
        if (tid == 0) A.part_send[c] = s;
    }
}

// k_mf_spmv with the warp-cooperative, shared-memory-staged candidate scan
// (wscan.cuh): warp w of the CTA owns rows base + 32 w + lane of each tile --
// the rows this thread owns in k_mf_spmv -- and the hits are the same, in the
// same order, so w and the chunk partials are bit-identical.  Dynamic shared
// memory: 8 x WarpSmem (static).
template <int D, int K>
__global__ void __launch_bounds__(NT, 3) k_mf_spmv_w(DistCGArgs A, LevelView V) {
    if (!A.sc->active) return;
    __shared__ wscan::WarpSmem Ws[NT / 32];
    __shared__ double red[NT / 32 + 2];
    wscan::WarpSmem &W = Ws[threadIdx.x >> 5];
    const CGLevelArgs &L = A.L;
    const int CH = L.chunk_tiles, tid = threadIdx.x;
    const bool first = A.sc->it == 0;
    const double alpha_prev = A.sc->alpha, beta = A.sc->beta;
    const double *rv = L.r;
    const double d2 = V.delta2, inv = V.inv_delta, scl = V.scale;
    const double4 *__restrict__ rec = V.rec;
    for (int64_t c = A.c0 + blockIdx.x; c < A.c1; c += gridDim.x) {
        double dot = 0.0;
        for (int t = 0; t < CH; ++t) {
            const int64_t i = (c * CH + t) * NT + tid;
            const bool on = i < L.n;
            double x[3] = {0.0, 0.0, 0.0};
            float xf[3] = {0.f, 0.f, 0.f};
            if (on) {
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    x[a] = V.x[a][i];
                    xf[a] = (float)(x[a] - V.g.lo[a]);
                }
            }
            double acc = 0.0;
            int hl[wscan::HM];
            auto flush = [&](int nh) {
                int h = 0;
                for (; h + 1 < nh; h += 2) {  // two records in flight
                    const int j0 = hl[h], j1 = hl[h + 1];
                    const double4 R0 = rec[j0], R1 = rec[j1];
                    const double p0 = rv[j0], p1 = rv[j1];
                    const double y0[3] = {R0.x, R0.y, R0.z}, y1[3] = {R1.x, R1.y, R1.z};
                    const double r20 = dist2_nofma<D>(x, y0), r21 = dist2_nofma<D>(x, y1);
                    if (r20 < d2) acc = fma(scl * wendland<K>(sqrt(r20) * inv), p0, acc);
                    if (r21 < d2) acc = fma(scl * wendland<K>(sqrt(r21) * inv), p1, acc);
                }
                if (h < nh) {
                    const int j0 = hl[h];
                    const double4 R0 = rec[j0];
                    const double y0[3] = {R0.x, R0.y, R0.z};
                    const double r20 = dist2_nofma<D>(x, y0);
                    if (r20 < d2) acc = fma(scl * wendland<K>(sqrt(r20) * inv), rv[j0], acc);
                }
            };
            wscan::scan_level<D>(V, x, xf, on, W, hl, flush);
            if (on) {
                // epilogue: the expressions of spmv_phase
                const double ri = rv[i];
                const double po = first ? 0.0 : L.p[i], qo = first ? 0.0 : L.q[i], xo = first ? 0.0 : L.x[i];
                const double pn = first ? ri : ri + beta * po;
                const double qn = first ? acc : acc + beta * qo;
                L.p[i] = pn;
                L.q[i] = qn;
                L.x[i] = first ? 0.0 : xo + alpha_prev * po;
                dot += pn * qn;
            }
        }
        const double s = block_sum<NT>(dot, red);
        if (tid == 0) A.part_send[c] = s;
    }
}

// mode 0: after init (bb); 1: after SpMV (pq, alpha); 2: after the r update
// (rr', beta); 3: end of iteration (it++, stopping test).  One CTA; the sum
// over chunks uses the order of chunk_allreduce.
__global__ void __launch_bounds__(NT) k_dcg_scalar(DistCGArgs A, int mode) {
    __shared__ double red[NT / 32 + 2];
    DistCGScalars &s = *A.sc;
    if (mode != 0 && !s.active) return;
    double v = 0.0;
    if (mode != 3) {
        double t = 0.0;
        if (A.gw == 0) {
            t = strided_sum(A.part_recv, A.nchunks);
        } else {  // all-gathered blocks: the same chunks in the same order
            int r = 0;
            for (int64_t j = threadIdx.x; j < A.nchunks; j += NT) {
                while (j >= A.gc0[r + 1]) ++r;
                t += __ldcg(&A.part_recv[r * A.gcmax + j - A.gc0[r]]);
            }
        }
        v = block_sum<NT>(t, red);
    }
    if (threadIdx.x != 0) return;
    if (mode == 0) {
        s.bb = v;
        s.rr = v;
        s.alpha = 0.0;
        s.beta = 0.0;
        s.it = 0;
        s.status = 0;
        dcg_check_top(s, A.L.tol2, A.L.max_iter);
    } else if (mode == 1) {
        s.pq = v;
        s.alpha = s.rr / v;
        if (A.L.coef && s.it < A.L.coef_cap) A.L.coef[2 * s.it] = s.alpha;
    } else if (mode == 2) {
        s.beta = v / s.rr;
        s.rr = v;
        if (A.L.coef && s.it < A.L.coef_cap) A.L.coef[2 * s.it + 1] = s.beta;
    } else {
        s.it += 1;
        dcg_check_top(s, A.L.tol2, A.L.max_iter);
    }
}

__global__ void k_sum_arrays(int W, DistPtrs srcs, double *dst, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int w = 0; w < W; ++w) s += srcs.p[w][i];
    dst[i] = s;
}

__global__ void k_col_minmax(int64_t nnz, const int32_t *__restrict__ col, unsigned long long *mm) {
    unsigned long long lo = ~0ull, hi = 0;
    for (int64_t p = (int64_t)blockIdx.x * NT + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * NT) {
        unsigned long long c = (unsigned long long)col[p];
        lo = c < lo ? c : lo;
        hi = c > hi ? c : hi;
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

// the two piece-capacity variants of k_cg / k_dcg_spmv
struct CGVariant {
    const void *cg, *dcg;
    size_t smem;
    int resident;  // co-resident CTAs of k_cg on the device
};
// Per device: cudaFuncSetAttribute applies to the current device's context
// only, and co-residency depends on the device.  Set once per device under a
// mutex (several host threads -- e.g. the threaded-rank tests -- may race here).
constexpr int kMaxDevices = 64;
CGVariant g_var_dev[kMaxDevices][3];
bool g_var_done[kMaxDevices] = {false};
std::mutex g_var_mu;
thread_local CGVariant *g_var = g_var_dev[0];

void set_smem_attrs() {
    int dev = 0;
    MSK_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) throw Error(3, "set_smem_attrs: device index out of range");
    std::lock_guard<std::mutex> lk(g_var_mu);
    g_var = g_var_dev[dev];
    if (g_var_done[dev]) return;
    g_var[0] = {(const void *)k_cg<CAPT0, MINB0>, (const void *)k_dcg_spmv<CAPT0, MINB0>,
                sizeof(CGSharedTT<CAPT0>), 0};
    g_var[1] = {(const void *)k_cg<CAPT1, MINB1>, (const void *)k_dcg_spmv<CAPT1, MINB1>,
                sizeof(CGSharedTT<CAPT1>), 0};
    g_var[2] = {(const void *)k_cg<CAPT2, MINB2>, (const void *)k_dcg_spmv<CAPT2, MINB2>,
                sizeof(CGSharedTT<CAPT2>), 0};
    int sms = 0;
    MSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    for (int vi = 0; vi < 3; ++vi) {
        CGVariant &v = g_var[vi];
        MSK_CUDA(cudaFuncSetAttribute(v.cg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem));
        MSK_CUDA(cudaFuncSetAttribute(v.dcg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem));
        int per = 0;
        MSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, v.cg, NT, v.smem));
        v.resident = sms * (per > 0 ? per : 1);
    }
    MSK_CUDA(cudaFuncSetAttribute(k_pcg<CAPT0, MINB0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(CGSharedTT<CAPT0>)));
    MSK_CUDA(cudaFuncSetAttribute(k_pcg<CAPT1, MINB1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(CGSharedTT<CAPT1>)));
    // the other dynamic-shared-memory kernels of this file (multi-RHS CG, plain SpMV)
    MSK_CUDA(cudaFuncSetAttribute(k_cgr<2048, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(CGSharedR<2048, 2>)));
    MSK_CUDA(cudaFuncSetAttribute(k_cgr<2048, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(CGSharedR<2048, 4>)));
    MSK_CUDA(cudaFuncSetAttribute(k_spmv_t<CAPT0, MINB0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(CGSharedTT<CAPT0>)));
    MSK_CUDA(cudaFuncSetAttribute(k_spmv_t<CAPT1, MINB1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(CGSharedTT<CAPT1>)));
    g_var_done[dev] = true;
}

// variant by mean row length (entries per row of the work being launched)
#ifndef MSK_LONGROW
#define MSK_LONGROW 16.0
#endif
int cg_variant(double nnz, double rows) { return rows > 0 && nnz >= MSK_LONGROW * rows ? 1 : 0; }
}  // namespace

int cg_max_resident_blocks() {
    set_smem_attrs();
    int r = g_var[0].resident;
    for (int vi = 0; vi < 3; ++vi) r = g_var[vi].resident < r ? g_var[vi].resident : r;
    return r;
}

// tiles per chunk: a function of n only (keeps results launch-independent,
// and the same for the single-GPU, partitioned and multi-RHS paths).  Larger
// chunks amortise the per-chunk work (row-pointer copy, partial reduction):
// 4 tiles from 1024 tiles up, 2 from 512 (same-box A/B: C3 level 4 -18 %,
// level 3 -7 %, C2 levels 4-5 -13/-7 %; 2 tiles at 256 tiles would halve the
// CTAs of C2 level 3 and cost 28 %).
int cg_chunk_tiles(int64_t n) {
    int64_t tiles = (n + NT - 1) / NT;
    return tiles >= 1024 ? 4 : tiles >= 512 ? 2 : 1;
}

// levels[i].nblocks == 0 => the launcher assigns CTAs proportionally to work.
void cg_batched(CGLevelArgs *levels, int nlev, cudaStream_t st, int *launches) {
    if (nlev <= 0) return;
    if (nlev > kMaxLevels) throw Error(1, "cg_batched: too many levels");
    set_smem_attrs();
    double snnz = 0.0, srows = 0.0;
    int64_t schunks = 0;
    int dom = 0;  // the level with the most work decides the chunk shape
    for (int l = 0; l < nlev; ++l) {
        snnz += (double)levels[l].nnz;
        srows += (double)levels[l].n;
        const int64_t tiles = (levels[l].n + NT - 1) / NT, ch = cg_chunk_tiles(levels[l].n);
        schunks += (tiles + ch - 1) / ch;
        if (levels[l].nnz > levels[dom].nnz) dom = l;
    }
    // long rows, or so few chunks that occupancy is moot: the large-piece
    // variant (a small level's 256-row chunk then fits one piece); one-tile
    // chunks of mid-size levels: 2432-entry pieces (one piece per chunk; C3
    // levels 3/4 -12 %/-9 %); the finest levels (4-tile chunks) keep 2048, the
    // larger smem carve-out costs them L1 for the gathers (+11 %).
    int vi = 0;
    if (cg_variant(snnz, srows) == 1 || schunks <= g_var[1].resident) vi = 1;
    else if (cg_chunk_tiles(levels[dom].n) == 1) vi = 2;
    const CGVariant &var = g_var[vi];
    const int total = var.resident;
    if (total < nlev) throw Error(3, "cg_batched: fewer resident CTAs than levels");
    std::vector<double> work(nlev);
    double wsum = 0.0;
    for (int l = 0; l < nlev; ++l) {
        work[l] = (double)levels[l].nnz + 12.0 * (double)levels[l].n;  // ~bytes/8 per iteration
        wsum += work[l];
        for (const void *ptr : {(const void *)levels[l].row_ptr, (const void *)levels[l].col,
                                (const void *)levels[l].val})
            if (((uintptr_t)ptr & 15u) != 0) throw Error(3, "cg_batched: CSR arrays must be 16-byte aligned");
    }
    // CTA allocation: proportional to work, at least one, at most one per chunk.
    int used = 0;
    std::vector<int> nbk(nlev), chk(nlev);
    std::vector<int64_t> nch(nlev);
    int64_t ptot = 0;
    for (int l = 0; l < nlev; ++l) {
        int64_t tiles = (levels[l].n + NT - 1) / NT;
        chk[l] = cg_chunk_tiles(levels[l].n);
        nch[l] = (tiles + chk[l] - 1) / chk[l];
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
        B.lev[l].chunk_tiles = chk[l];
        B.lev[l].partials = partials + poff;
        B.lev[l].barrier = bars + l;
        begin += nbk[l];
        poff += 3 * nch[l];
    }
    void *args[] = {&B};
    // One small level (<= 16 chunks): a single thread-block cluster, one CTA per
    // chunk, synchronised by the hardware cluster barrier instead of a counter in
    // global memory (the iteration of a small level is latency bound): C3 levels
    // 1/2 -10/-13 %, C2 levels 1/2 -16/-13 %.  With several chunks per CTA (64
    // chunks on 16 CTAs) the cooperative launch is 2.3x faster, hence the bound.
    // Same chunks, same partials, same order: bit-identical to the cooperative
    // launch.  Falls back to it if the cluster cannot be scheduled.
    if (nlev == 1 && nch[0] <= 16 && !getenv("MSK_NO_CLUSTER")) {
        const int cl = (int)(nch[0] < 16 ? nch[0] : 16);
        CGBatch C = B;
        C.lev[0].nblocks = cl;
        C.lev[0].barrier = nullptr;
        void *cargs[] = {&C};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = var.smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(var.cg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (cudaLaunchKernelExC(&cfg, var.cg, cargs) == cudaSuccess) {
            if (launches) *launches += 1;
            MSK_CUDA(cudaFreeAsync(partials, st));
            MSK_CUDA(cudaFreeAsync(bars, st));
            return;
        }
        cudaGetLastError();  // clear, then the cooperative launch
    }
    MSK_CUDA(cudaLaunchCooperativeKernel(var.cg, dim3(used), dim3(NT), args, var.smem, st));
    if (launches) *launches += 1;
    MSK_CUDA(cudaFreeAsync(partials, st));
    MSK_CUDA(cudaFreeAsync(bars, st));
}

void cg_multi(const CGRArgs &a, int R, cudaStream_t st, int *launches) {
    if (a.n == 0) return;
    if (R != 2 && R != 4) throw Error(1, "cg_multi: R must be 2 or 4");
    constexpr int CM = 2048;
    const void *fn = R == 2 ? (const void *)k_cgr<CM, 2, 2> : (const void *)k_cgr<CM, 2, 4>;
    const size_t smem = R == 2 ? sizeof(CGSharedR<CM, 2>) : sizeof(CGSharedR<CM, 4>);
    set_smem_attrs();  // per device, includes k_cgr's attribute
    int dev = 0, sms = 0, per = 0;
    MSK_CUDA(cudaGetDevice(&dev));
    MSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, smem));
    const int CH = cg_chunk_tiles(a.n);
    const int64_t nch = ((a.n + NT - 1) / NT + CH - 1) / CH;
    int nb = sms * (per > 0 ? per : 1);
    if (nb > nch) nb = (int)nch;
    double *part = nullptr;
    unsigned long long *bar = nullptr;
    MSK_CUDA(cudaMallocAsync((void **)&part, sizeof(double) * (size_t)(3 * nch * R), st));
    MSK_CUDA(cudaMallocAsync((void **)&bar, sizeof(unsigned long long), st));
    MSK_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned long long), st));
    CGRArgs A = a;
    int CHv = CH;
    void *args[] = {&A, &nb, &CHv, &part, &bar};
    MSK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(nb), dim3(NT), args, smem, st));
    if (launches) *launches += 1;
    MSK_CUDA(cudaFreeAsync(part, st));
    MSK_CUDA(cudaFreeAsync(bar, st));
}

namespace {
unsigned dcg_grid(const DistCGArgs &a, int per_sm) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t nc = a.c1 - a.c0;
    int64_t g = (int64_t)sms * per_sm;
    return (unsigned)(nc < 1 ? 1 : (nc < g ? nc : g));
}
}  // namespace

// 16-bit columns per reduction chunk: greedy windows of 2^14 indices from the
// smallest column up (at most 4; a chunk's columns fall into ~3 clusters, one
// per x-offset of its rows' cells), entry = window << 14 | (column - base).
__global__ void __launch_bounds__(NT) k_col16(int64_t n, int CH, const int64_t *__restrict__ rp,
                                              const int32_t *__restrict__ col, uint16_t *__restrict__ col16,
                                              int4 *__restrict__ cbase, int4 *__restrict__ clen,
                                              int *__restrict__ fail) {
    __shared__ int red[NW];
    const int64_t c = blockIdx.x;
    const int64_t r0 = c * CH * NT, r1 = r0 + (int64_t)CH * NT < n ? r0 + (int64_t)CH * NT : n;
    const int64_t e0 = rp[r0], e1 = rp[r1];
    const int tid = threadIdx.x;
    auto block_min = [&](int v) {
        v = __reduce_min_sync(0xffffffffu, v);
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        int m = red[0];
        for (int w = 1; w < NW; ++w) m = red[w] < m ? red[w] : m;
        return m;
    };
    int base[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
    int64_t lower = INT64_MIN;
    for (int w = 0; w < 4; ++w) {
        int m = INT_MAX;
        for (int64_t e = e0 + tid; e < e1; e += NT) {
            const int v = col[e];
            if ((int64_t)v >= lower && v < m) m = v;
        }
        m = block_min(m);
        if (m == INT_MAX) break;
        base[w] = m;
        lower = (int64_t)m + 16384;
    }
    int ext[4] = {0, 0, 0, 0};  // per window: largest offset + 1 (the extent read by the gathers)
    for (int64_t e = e0 + tid; e < e1; e += NT) {
        const int v = col[e];
        const int w = (v >= base[1]) + (v >= base[2]) + (v >= base[3]);
        const int64_t off = (int64_t)v - base[w];
        if (off < 0 || off >= 16384) {
            atomicOr(fail, 1);
            continue;
        }
        ext[w] = (int)off + 1 > ext[w] ? (int)off + 1 : ext[w];
        if (col16) col16[e] = (uint16_t)((w << 14) | (int)off);
    }
    for (int w = 0; w < 4; ++w) ext[w] = -block_min(-ext[w]);
    if (tid == 0) {
        cbase[c] = make_int4(base[0], base[1], base[2], base[3]);
        if (clen) clen[c] = make_int4(ext[0], ext[1], ext[2], ext[3]);
    }
}

// co-resident CTAs of k_pcg's variant for a level (the per-rank grid is
// this / W in the emulation, all of it on a GPU of its own)
int pcg_resident_blocks(double nnz, double rows) {
    set_smem_attrs();
    return g_var[cg_variant(nnz, rows)].resident;
}

void pcg_launch(const PeerCGArgs &a, cudaStream_t st) {
    set_smem_attrs();
    const int vi = cg_variant((double)a.L.nnz, (double)a.L.n);
    const CGVariant &var = g_var[vi];
    const void *fn = vi == 0 ? (const void *)k_pcg<CAPT0, MINB0> : (const void *)k_pcg<CAPT1, MINB1>;
    const unsigned grid = (unsigned)(a.rank >= 0 ? a.nb : a.nb * a.W);
    if ((int)grid > var.resident) throw Error(3, "pcg_launch: grid exceeds the co-resident CTAs");
    PeerCGArgs A = a;
    void *args[] = {&A};
    MSK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(NT), args, var.smem, st));
}

bool col16_build(int64_t n, const int64_t *row_ptr, const int32_t *col, uint16_t *col16, int4 *cbase,
                 int4 *clen, cudaStream_t st) {
    if (n <= 0) return false;
    const int CH = cg_chunk_tiles(n);
    const int64_t nch = ((n + NT - 1) / NT + CH - 1) / CH;
    int *fail = nullptr, hf = 0;
    MSK_CUDA(cudaMallocAsync((void **)&fail, sizeof(int), st));
    MSK_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), st));
    k_col16<<<(unsigned)nch, NT, 0, st>>>(n, CH, row_ptr, col, col16, cbase, clen, fail);
    MSK_CHECK_LAUNCH();
    MSK_CUDA(cudaMemcpyAsync(&hf, fail, sizeof(int), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    MSK_CUDA(cudaFreeAsync(fail, st));
    return hf == 0;
}

void dcg_init(const DistCGArgs &a, cudaStream_t st) {
    k_dcg_init<<<dcg_grid(a, 8), NT, 0, st>>>(a);
    MSK_CHECK_LAUNCH();
}
void dcg_spmv(const DistCGArgs &a, cudaStream_t st) {
    set_smem_attrs();
    const double rows = (double)(a.c1 - a.c0) * a.L.chunk_tiles * NT;
    const CGVariant &var = g_var[cg_variant((double)a.L.nnz, rows)];
    void *args[] = {(void *)&a};
    MSK_CUDA(cudaLaunchKernel(var.dcg, dim3(dcg_grid(a, 3)), dim3(NT), args, var.smem, st));
}
void dcg_rupd(const DistCGArgs &a, cudaStream_t st) {
    k_dcg_rupd<<<dcg_grid(a, 8), NT, 0, st>>>(a);
    MSK_CHECK_LAUNCH();
}
void dcg_xfin(const DistCGArgs &a, cudaStream_t st) {
    k_dcg_xfin<<<dcg_grid(a, 8), NT, 0, st>>>(a);
    MSK_CHECK_LAUNCH();
}
void dcg_mf_spmv(const DistCGArgs &a, const LevelView &v, int d, int k, cudaStream_t st) {
    const bool v1 = gather_v1();
#define MSK_MF(DD, KK)                                                                   \
    do {                                                                                 \
        if (v1) k_mf_spmv<DD, KK><<<dcg_grid(a, MSK_MF_MINB), NT, 0, st>>>(a, v);                  \
        else k_mf_spmv_w<DD, KK><<<dcg_grid(a, 3), NT, 0, st>>>(a, v);                   \
    } while (0)
    if (d == 2) {
        if (k == 0) MSK_MF(2, 0); else if (k == 1) MSK_MF(2, 1); else MSK_MF(2, 2);
    } else {
        if (k == 0) MSK_MF(3, 0); else if (k == 1) MSK_MF(3, 1); else MSK_MF(3, 2);
    }
#undef MSK_MF
    MSK_CHECK_LAUNCH();
}
void dcg_scalar(const DistCGArgs &a, int mode, cudaStream_t st) {
    k_dcg_scalar<<<1, NT, 0, st>>>(a, mode);
    MSK_CHECK_LAUNCH();
}
void sum_arrays(int W, const DistPtrs &srcs, double *dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_sum_arrays<<<ceil_div_u(n, NT), NT, 0, st>>>(W, srcs, dst, n);
    MSK_CHECK_LAUNCH();
}
void col_minmax(int64_t nnz, const int32_t *col, unsigned long long *mm, cudaStream_t st) {
    unsigned long long init[2] = {~0ull, 0ull};
    MSK_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
    if (nnz <= 0) return;
    int64_t nb = (nnz + NT - 1) / NT;
    k_col_minmax<<<(unsigned)(nb < 1184 ? nb : 1184), NT, 0, st>>>(nnz, col, mm);
    MSK_CHECK_LAUNCH();
}

void spmv_csr(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *val,
              const double *v, double *y, cudaStream_t st, int *launches) {
    if (n == 0) return;
    set_smem_attrs();  // per device, includes k_spmv_t's attribute
    CGLevelArgs L{};
    L.n = n;
    L.row_ptr = row_ptr;
    L.col = col;
    L.val = val;
    L.r = const_cast<double *>(v);
    L.q = y;
    int64_t nnz = 0;
    MSK_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof nnz, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    const int CH = cg_chunk_tiles(n);
    const int64_t nch = ((n + NT - 1) / NT + CH - 1) / CH;
    const int vi = cg_variant((double)nnz, (double)n);  // long rows: 4096-entry pieces
    const int grid = (int)(nch < g_var[vi].resident ? nch : g_var[vi].resident);
    if (vi == 1)
        k_spmv_t<CAPT1, MINB1><<<grid, NT, sizeof(CGSharedTT<CAPT1>), st>>>(L, CH);
    else
        k_spmv_t<CAPT0, MINB0><<<grid, NT, sizeof(CGSharedTT<CAPT0>), st>>>(L, CH);
    MSK_CHECK_LAUNCH();
    if (launches) *launches += 1;
}

}  // namespace msk

// capi_solve.cu -- msk_solve (a5 Jacobi schedules, a7 thresholded sweep, a4/a8
// block CG, partitioned levels) and msk_evaluate (a9, host-buffer pipelining).
#include "capi_internal.cuh"

// =================================================================== solve
namespace capi {

struct LevelStat {
    int iters, status;
    double rr, bb;
};

// one CG launch over the given levels; returns per-level stats (host) after sync
CGLevelArgs cg_args(msk_hierarchy *h, int l, double tol, int max_iter, const double *b,
                    const double *b_src, double *x, double *x_out, int *d_iters, double *d_rr,
                    int *d_status) {
    LevelData &D = h->lev[l];
    CGLevelArgs a{};
    a.n = D.n;
    a.nnz = D.nnz;
    a.row_ptr = D.row_ptr;
    a.col = D.col;
    a.val = D.val;
    a.col16 = D.col16;
    a.cbase = D.cbase;
    a.clen = D.clen;
    a.b = b;
    a.b_src = b_src;
    a.b_perm = b_src ? D.perm : nullptr;
    a.x = x;
    a.r = h->ws_r(l);
    a.p = h->ws_p(l);
    a.q = h->ws_q(l);
    a.x_out = x_out;
    a.x_perm = x_out ? D.perm : nullptr;
    a.tol2 = tol * tol;
    a.max_iter = max_iter;
    a.nblocks = 0;
    a.out_iters = d_iters;
    a.out_rr = d_rr;
    a.out_status = d_status;
    return a;
}

// Condition number estimate from m CG steps (the Lanczos connection):
// T = tridiag with T00 = 1/a0, Tjj = 1/aj + b(j-1)/a(j-1), T(j,j+1) = sqrt(bj)/aj;
// its extreme eigenvalues (Sturm-sequence bisection) approximate those of A.
double lanczos_kappa(const double *coef, int m) {
    if (m <= 0) return 0.0;
    std::vector<double> dg(m), off(m > 1 ? m - 1 : 1, 0.0);
    for (int j = 0; j < m; ++j) {
        const double a = coef[2 * j];
        dg[j] = 1.0 / a + (j > 0 ? coef[2 * j - 1] / coef[2 * j - 2] : 0.0);
        if (j + 1 < m) off[j] = std::sqrt(std::max(coef[2 * j + 1], 0.0)) / a;
    }
    double lo = dg[0], hi = dg[0];
    for (int j = 0; j < m; ++j) {
        const double r = (j > 0 ? std::fabs(off[j - 1]) : 0.0) + (j + 1 < m ? std::fabs(off[j]) : 0.0);
        lo = std::min(lo, dg[j] - r);
        hi = std::max(hi, dg[j] + r);
    }
    auto below = [&](double x) {  // number of eigenvalues < x
        int c = 0;
        double q = dg[0] - x;
        if (q < 0) ++c;
        for (int j = 1; j < m; ++j) {
            if (q == 0.0) q = 1e-300;
            q = dg[j] - x - off[j - 1] * off[j - 1] / q;
            if (q < 0) ++c;
        }
        return c;
    };
    auto bisect = [&](int k) {  // the k-th smallest eigenvalue (k = 1..m)
        double a = lo, b = hi;
        for (int it = 0; it < 200 && b - a > 1e-15 * std::max(std::fabs(a), std::fabs(b)); ++it) {
            const double mid = 0.5 * (a + b);
            if (below(mid) >= k) b = mid; else a = mid;
        }
        return 0.5 * (a + b);
    };
    const double lmin = bisect(1), lmax = bisect(m);
    return lmin > 0.0 ? lmax / lmin : 0.0;
}

double cg_bytes(const LevelData &D, int iters) {
    // algorithmic bytes: per iteration 12 B/nnz (val + col)
    // + 88 B/row (SpMV pass: row_ptr 8, gathered r 8, p/q/x read + write 48;
    // r pass: r, q read + r write 24); iteration 0 reads no p/q/x (-24 B/row);
    // init 16 B/row (b read, r write); final x update 24 B/row (x, p read, x write)
    if (iters <= 0) return 24.0 * (double)D.n;
    return (double)iters * (12.0 * (double)D.nnz + 88.0 * (double)D.n) + 16.0 * (double)D.n;
}

}  // namespace capi

namespace {
// MSK_DIST_P2P=0: the partitioned CG as host-driven phase kernels with NCCL
// collectives (or device copies in the emulation) instead of k_pcg
bool dist_p2p_enabled() {
    const char *e = getenv("MSK_DIST_P2P");
    return !(e && e[0] == '0');
}

// Peer memory of partitioned level l for k_pcg across processes (one GPU per
// rank): allocate this rank's r / partials / result / counters with cudaMalloc,
// all-gather the IPC handles over NCCL, open the peers'.  Every rank makes the
// same calls; a failure anywhere (e.g. ranks sharing one device in one process,
// no peer access) is agreed on by an all-reduce and every rank falls back to
// the phase path.  Cached in the context per level index and reused by every
// later hierarchy of the context (grown collectively when a level is larger).
bool peer_setup(msk_hierarchy *h, int l, int64_t nch) {
    auto &M = h->ctx->peer[l];
    const int64_t n = h->lev[l].n;
    if (M.tried && !M.ok) return false;              // this context cannot map peers
    if (M.ok && M.ncap >= n && M.chcap >= nch) return true;  // reuse (every rank decides alike)
    cudaStream_t st = h->st();
    if (M.ok) {  // grow: all ranks are here (same n, nch); no kernel may use the old buffers
        MSK_CUDA(cudaStreamSynchronize(st));
        M.release();
    }
    M.tried = true;
    M.ncap = n;
    M.chcap = nch;
    const int W = h->ctx->world, me = h->ctx->rank;
    int fail = 0;
    auto ck = [&](cudaError_t e) {
        if (e != cudaSuccess) { cudaGetLastError(); fail = 1; }
    };
    ck(cudaMalloc((void **)&M.r, sizeof(double) * (size_t)n));
    ck(cudaMalloc((void **)&M.part, sizeof(double) * (size_t)(3 * nch)));
    ck(cudaMalloc((void **)&M.alpha, sizeof(double) * (size_t)n));
    ck(cudaMalloc((void **)&M.cnt, sizeof(unsigned long long) * 3));
    constexpr int NB = 4;  // handles per rank, then the device UUID
    struct Blob {
        cudaIpcMemHandle_t hd[NB];
        unsigned char uuid[16];
    };
    Blob mine;
    memset(&mine, 0, sizeof mine);
    if (!fail) {
        ck(cudaMemset(M.cnt, 0, sizeof(unsigned long long) * 3));
        ck(cudaIpcGetMemHandle(&mine.hd[0], M.r));
        ck(cudaIpcGetMemHandle(&mine.hd[1], M.part));
        ck(cudaIpcGetMemHandle(&mine.hd[2], M.alpha));
        ck(cudaIpcGetMemHandle(&mine.hd[3], M.cnt));
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, h->ctx->device));
        if (!fail) memcpy(mine.uuid, &prop.uuid, 16);
    }
    const size_t hb = sizeof(Blob);
    unsigned char *dh = dalloc<unsigned char>(hb * (size_t)(W + 1), st);
    MSK_CUDA(cudaMemcpyAsync(dh + hb * W, &mine, hb, cudaMemcpyHostToDevice, st));
    MSK_NCCL(nccl_api()->AllGather(dh + hb * W, dh, hb, ncclUint8, h->ctx->comm, st));
    std::vector<Blob> blobs((size_t)W);
    MSK_CUDA(cudaMemcpyAsync(blobs.data(), dh, hb * W, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    // ranks that share a device (threads as ranks, several processes on one
    // GPU) must not run kernels that wait on each other: phase path instead
    for (int a = 0; a < W && !fail; ++a)
        for (int b = a + 1; b < W; ++b)
            if (memcmp(blobs[a].uuid, blobs[b].uuid, 16) == 0) fail = 1;
    std::vector<cudaIpcMemHandle_t> all((size_t)(NB * W));
    for (int w = 0; w < W; ++w)
        for (int k = 0; k < NB; ++k) all[(size_t)(NB * w + k)] = blobs[w].hd[k];
    M.pr.assign(W, nullptr); M.ppart.assign(W, nullptr); M.palpha.assign(W, nullptr); M.pcnt.assign(W, nullptr);
    for (int w = 0; w < W && !fail; ++w) {
        if (w == me) {
            M.pr[w] = M.r; M.ppart[w] = M.part; M.palpha[w] = M.alpha; M.pcnt[w] = M.cnt;
            continue;
        }
        void *p[NB] = {nullptr, nullptr, nullptr, nullptr};
        for (int k = 0; k < NB && !fail; ++k) {
            ck(cudaIpcOpenMemHandle(&p[k], all[(size_t)(NB * w + k)], cudaIpcMemLazyEnablePeerAccess));
            if (!fail) M.opened.push_back(p[k]);
        }
        M.pr[w] = (double *)p[0]; M.ppart[w] = (double *)p[1]; M.palpha[w] = (double *)p[2];
        M.pcnt[w] = (unsigned long long *)p[3];
    }
    // agreement: every rank takes the peer path, or none does
    int *df = (int *)dh;
    MSK_CUDA(cudaMemcpyAsync(df + 1, &fail, sizeof(int), cudaMemcpyHostToDevice, st));
    MSK_NCCL(nccl_api()->AllReduce(df + 1, df, 1, ncclInt32, ncclSum, h->ctx->comm, st));
    int tot = 0;
    MSK_CUDA(cudaMemcpyAsync(&tot, df, sizeof(int), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(dh, st);
    M.ok = tot == 0;
    return M.ok;
}
// v (spatial order) complete on every rank from each rank's rows [rows[r],
// rows[r+1]): one in-place all-gather of equal blocks (the largest share),
// then the blocks moved to their rows -- instead of a zero-filled all-reduce
void allgather_rows(msk_hierarchy *h, double *v, const std::vector<int64_t> &rows, cudaStream_t st) {
    const int W = h->ctx->world, me = h->ctx->rank;
    int64_t smax = 1;
    for (int r = 0; r < W; ++r) smax = std::max(smax, rows[r + 1] - rows[r]);
    double *buf = dalloc<double>((size_t)(smax * W), st);
    if (rows[me + 1] > rows[me])
        MSK_CUDA(cudaMemcpyAsync(buf + me * smax, v + rows[me], sizeof(double) * (size_t)(rows[me + 1] - rows[me]),
                                 cudaMemcpyDeviceToDevice, st));
    MSK_NCCL(nccl_api()->AllGather(buf + me * smax, buf, (size_t)smax, ncclFloat64, h->ctx->comm, st));
    for (int r = 0; r < W; ++r)
        if (r != me && rows[r + 1] > rows[r])
            MSK_CUDA(cudaMemcpyAsync(v + rows[r], buf + r * smax, sizeof(double) * (size_t)(rows[r + 1] - rows[r]),
                                     cudaMemcpyDeviceToDevice, st));
    dfree(buf, st);
}
}  // namespace

extern "C" msk_status msk_solve(msk_hierarchy *h, const double *const *f, double tol,
                                int32_t max_iter, uint32_t schedule, double *const *alpha,
                                msk_solve_info *info) {
    API_BEGIN
    require(h && f && alpha, "msk_solve: NULL argument");
    require(tol > 0.0 && tol < 1.0, "msk_solve: tol must be in (0,1)");
    require(max_iter >= 1, "msk_solve: max_iter must be >= 1");
    require(schedule == MSK_SCHED_PRUNED || schedule == MSK_SCHED_LITERAL, "msk_solve: unknown schedule");
    if (!h->assembled) throw Error(MSK_ERR_STATE, "msk_solve: call msk_assemble first");
    for (int l = 0; l < h->L; ++l) require(f[l] && alpha[l], "msk_solve: NULL level pointer");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const int L = h->L;
    const double inner_tol = tol / 10.0;  // reading C-10
    const bool mf = (h->flags & MSK_FLAG_MATRIX_FREE) != 0;
    h->ensure_ws();
    for (int l = 0; l < L; ++l)
        if (!h->lev[l].alpha) h->lev[l].alpha = dalloc<double>((size_t)h->lev[l].n, st);

    std::vector<DevBuf> fd;
    std::vector<DevOut> ad;
    fd.reserve(L);
    ad.reserve(L);
    // host buffers: f^(l) copied in on a copy stream (level order, one event per
    // level) and alpha^(l) copied out as soon as level l is final (PRUNED), so
    // the transfers overlap the solve of the other levels
    cudaStream_t cin = h->ctx->copy_in(), cout = h->ctx->copy_out();
    for (int l = 0; l < L; ++l) {
        fd.emplace_back(f[l], (size_t)h->lev[l].n, st, true);
        ad.emplace_back(alpha[l], (size_t)h->lev[l].n, st);
    }
    std::vector<Ev> ev_f((size_t)L), ev_a((size_t)L);
    CopyStreamsGuard copy_guard{cin, cout};  // destroyed before fd / ad
    {
        Ev ready;
        ready.record(st);
        ready.wait_on(cin);
        for (int l = 0; l < L; ++l) {
            fd[l].copy_async(cin);
            ev_f[l].record(cin);
        }
    }
    auto wait_f = [&](int l) { ev_f[l].wait_on(st); };
    auto out_alpha = [&](int l) {  // alpha^(l) final in ad[l].ptr (caller order)
        ev_a[l].record(st);
        ad[l].flush_async(cout, ev_a[l].e);
    };
    // device-side per-launch stats: [slot][level]
    const int nslots = schedule == MSK_SCHED_LITERAL ? L + 1 : 1;
    int *d_it = dalloc<int>((size_t)(nslots * L), st);
    int *d_stat = dalloc<int>((size_t)(nslots * L), st);
    double *d_rr = dalloc<double>((size_t)(2 * nslots * L), st);
    MSK_CUDA(cudaMemsetAsync(d_it, 0, sizeof(int) * nslots * L, st));
    MSK_CUDA(cudaMemsetAsync(d_stat, 0, sizeof(int) * nslots * L, st));
    MSK_CUDA(cudaMemsetAsync(d_rr, 0, sizeof(double) * 2 * nslots * L, st));
    const int coef_cap = std::min(max_iter, 4096);
    double *d_coef = dalloc<double>((size_t)(2 * coef_cap) * nslots * L, st);
    auto set_coef = [&](CGLevelArgs &a, int idx) {
        a.coef = d_coef + (size_t)(2 * coef_cap) * idx;
        a.coef_cap = coef_cap;
    };
    unsigned long long *d_hits = dalloc<unsigned long long>(1, st);
    MSK_CUDA(cudaMemsetAsync(d_hits, 0, sizeof(unsigned long long), st));

    int launches = 0;
    Timer ttot(st);
    std::vector<Timer *> cg_t, ga_t;
    std::vector<int> cg_t_level;  // level index, or -1 for a multi-level launch
    auto time_cg = [&](int lvl) {
        cg_t.push_back(new Timer(st));
        cg_t_level.push_back(lvl);
        cg_t.back()->start();
    };
    auto time_ga = [&]() {
        ga_t.push_back(new Timer(st));
        ga_t.back()->start();
    };
    // B products for target level k from coefficient vectors coef[0..k-1]
    auto b_products = [&](int k, double *const *coef_spatial, double *out_spatial) {
        GatherArgs ga{};
        ga.d = h->d;
        ga.k = h->k;
        ga.nt = h->lev[k].n;
        for (int a = 0; a < h->d; ++a) ga.tx[a] = h->lev[k].xs + (size_t)a * h->lev[k].n;
        ga.nlev = k;
        for (int l = 0; l < k; ++l) ga.lev[l] = h->view(l, coef_spatial[l]);
        ga.base = fd[k].ptr;
        ga.base_perm = h->lev[k].perm;
        ga.sign = -1.0;
        ga.out = out_spatial;
        ga.out_perm = nullptr;
        ga.hits = d_hits;
        NvtxRange nv("B products");
        time_ga();
        gather(ga, st, &launches);
        ga_t.back()->stop();
    };

    // B products for rows [r0, r1) of target level k only (a partitioned level's owned rows)
    auto b_products_rows = [&](int k, double *const *coef_spatial, double *out_spatial, int64_t r0, int64_t r1) {
        GatherArgs ga{};
        ga.d = h->d;
        ga.k = h->k;
        ga.nt = r1 - r0;
        for (int a = 0; a < h->d; ++a) ga.tx[a] = h->lev[k].xs + (size_t)a * h->lev[k].n + r0;
        ga.nlev = k;
        for (int l = 0; l < k; ++l) ga.lev[l] = h->view(l, coef_spatial[l]);
        ga.base = fd[k].ptr;
        ga.base_perm = h->lev[k].perm + r0;
        ga.sign = -1.0;
        ga.out = out_spatial + r0;
        ga.out_perm = nullptr;
        ga.hits = d_hits;
        time_ga();
        gather(ga, st, &launches);
        ga_t.back()->stop();
    };

    ttot.start();
    std::vector<double *> alpha_sp(L), t_sp(L);
    for (int l = 0; l < L; ++l) {
        alpha_sp[l] = h->lev[l].alpha;
        t_sp[l] = h->ws_t(l);
    }

    // ---- distributed solve of one partitioned level:
    // beta on the owned rows, then the CG as phase kernels with all-reduced
    // chunk partials and halo exchange of r; alpha assembled on every rank.
    // beta_ready: beta^(l) is already in ws_beta(l) (thresholded factor, a7)
    // slot: stats slot (LITERAL: one per sweep + the final solves); out: the
    // complete solution vector (spatial order, every rank); to_caller: also
    // write it to the caller's alpha^(l)
    auto dist_level = [&](int l, double tl, bool beta_ready, int slot = 0, double *out = nullptr,
                          bool to_caller = true) {
        if (!out) out = alpha_sp[l];
        const int si = slot * L + l;
        auto &Dd = h->dist[l];
        LevelData &D = h->lev[l];
        const int64_t n = D.n;
        const int CH = cg_chunk_tiles(n);
        const int64_t nch = (n + (int64_t)CH * 256 - 1) / ((int64_t)CH * 256);
        // a partitioned level, or (matrix-free, not partitioned) one partition of all rows
        const bool part = Dd.on;
        std::vector<msk_hierarchy::PartLocal> whole;
        if (!part) {
            msk_hierarchy::PartLocal P;
            P.lo = 0; P.hi = n; P.c0 = 0; P.c1 = nch; P.nnz = D.nnz; P.hlo = 0; P.hhi = n;
            whole.push_back(P);
        }
        auto &parts = part ? Dd.local : whole;
        const int np = (int)parts.size();
        const bool emu = part && h->ctx->emulated;
        const int W = part ? h->ctx->world : 1;
        std::vector<double *> X(np), R(np), Pv(np), Q(np), send(np);
        std::vector<double *> owned_alloc;
        double *recv = dalloc<double>((size_t)nch, st);
        DistCGScalars *sc = dalloc<DistCGScalars>((size_t)np, st);
        // real ranks: chunk partials are all-gathered, each rank's owned chunks as
        // one block of gcmax (the largest owned count) -- no zero-filled arrays
        int64_t gcmax = 0;
        std::vector<int64_t> gc0;
        if (part && !emu) {
            const int64_t cpr = (int64_t)CH * 256;
            for (int w = 0; w <= W; ++w) gc0.push_back(w < W ? Dd.rows[w] / cpr : nch);
            for (int w = 0; w < W; ++w) gcmax = std::max(gcmax, gc0[w + 1] - gc0[w]);
            gcmax = std::max<int64_t>(gcmax, 1);
        }
        double *gbuf = part && !emu ? dalloc<double>((size_t)(gcmax * W), st) : nullptr;
        for (int i = 0; i < np; ++i) {
            if (emu) {
                double *blk = dalloc<double>((size_t)(4 * n), st);
                owned_alloc.push_back(blk);
                X[i] = blk; R[i] = blk + n; Pv[i] = blk + 2 * n; Q[i] = blk + 3 * n;
            } else {
                X[i] = h->ws_t(l); R[i] = h->ws_r(l); Pv[i] = h->ws_p(l); Q[i] = h->ws_q(l);
            }
            send[i] = dalloc<double>((size_t)nch, st);
            if (!gbuf) MSK_CUDA(cudaMemsetAsync(send[i], 0, sizeof(double) * (size_t)nch, st));
        }
        // beta^(l) on the owned rows (B products of the coarser, complete levels)
        if (l > 0 && !beta_ready) {
            for (auto &P : parts) {
                GatherArgs ga{};
                ga.d = h->d;
                ga.k = h->k;
                ga.nt = P.hi - P.lo;
                for (int a = 0; a < h->d; ++a) ga.tx[a] = D.xs + (size_t)a * n + P.lo;
                ga.nlev = l;
                for (int k = 0; k < l; ++k) ga.lev[k] = h->view(k, alpha_sp[k]);
                ga.base = fd[l].ptr;
                ga.base_perm = D.perm + P.lo;
                ga.sign = -1.0;
                ga.out = h->ws_beta(l) + P.lo;
                ga.hits = d_hits;
                time_ga();
                gather(ga, st, &launches);
                ga_t.back()->stop();
            }
        }
        std::vector<DistCGArgs> args(np);
        for (int i = 0; i < np; ++i) {
            const auto &P = parts[i];
            DistCGArgs &A = args[i];
            A.L = cg_args(h, l, tl, max_iter, l == 0 ? nullptr : h->ws_beta(l), l == 0 ? fd[0].ptr : nullptr,
                          X[i], nullptr, nullptr, nullptr, nullptr);
            A.L.r = R[i];
            A.L.p = Pv[i];
            A.L.q = Q[i];
            A.L.row_ptr = P.rp ? P.rp - P.lo : nullptr;  // indexed by global row
            A.L.col = P.col;
            A.L.val = P.val;
            A.L.col16 = nullptr;
            A.L.cbase = nullptr;
            A.L.clen = nullptr;
            A.L.nnz = P.nnz;
            A.L.chunk_tiles = CH;
            A.c0 = P.c0;
            A.c1 = P.c1;
            A.nchunks = nch;
            A.part_send = send[i];
            A.part_recv = part ? recv : send[i];  // one partition: nothing to reduce
            if (gbuf) {  // chunk c of this rank -> gbuf[rank * gcmax + c - c0]
                const int me = h->ctx->rank;
                A.part_send = gbuf + me * gcmax - gc0[me];
                A.part_recv = gbuf;
                A.gw = W;
                A.gcmax = gcmax;
                for (int w = 0; w <= W; ++w) A.gc0[w] = gc0[w];
            }
            A.sc = sc + i;
            if (i == 0) set_coef(A.L, si);
        }
        auto allreduce = [&]() {
            if (!part) return;
            if (emu) {
                DistPtrs ptrs{};
                for (int i = 0; i < np; ++i) ptrs.p[i] = send[i];
                sum_arrays(np, ptrs, recv, nch, st);
            } else {  // in place: this rank's block is already at rank * gcmax
                MSK_NCCL(nccl_api()->AllGather(gbuf + h->ctx->rank * gcmax, gbuf, (size_t)gcmax, ncclFloat64,
                                               h->ctx->comm, st));
            }
        };
        // halo plans (msk_halo_plan): per local partition, send/recv row ranges per peer
        std::vector<std::vector<int64_t>> sl(np, std::vector<int64_t>(W)), sh = sl, rl = sl, rh = sl;
        for (int i = 0; i < np && part; ++i)
            msk_halo_plan(W, parts[i].rank, Dd.rows.data(), Dd.hlo.data(), Dd.hhi.data(), sl[i].data(),
                          sh[i].data(), rl[i].data(), rh[i].data());
        auto halo = [&]() {
            if (!part) return;
            if (emu) {  // partition i receives from partition s by a device copy
                for (int i = 0; i < np; ++i)
                    for (int s = 0; s < W; ++s)
                        if (rl[i][s] < rh[i][s])
                            MSK_CUDA(cudaMemcpyAsync(R[i] + rl[i][s], R[s] + rl[i][s],
                                                     sizeof(double) * (size_t)(rh[i][s] - rl[i][s]),
                                                     cudaMemcpyDeviceToDevice, st));
            } else {
                MSK_NCCL(nccl_api()->GroupStart());
                for (int s = 0; s < W; ++s) {
                    if (sl[0][s] < sh[0][s])
                        MSK_NCCL(nccl_api()->Send(R[0] + sl[0][s], (size_t)(sh[0][s] - sl[0][s]), ncclFloat64, s,
                                                  h->ctx->comm, st));
                    if (rl[0][s] < rh[0][s])
                        MSK_NCCL(nccl_api()->Recv(R[0] + rl[0][s], (size_t)(rh[0][s] - rl[0][s]), ncclFloat64, s,
                                                  h->ctx->comm, st));
                }
                MSK_NCCL(nccl_api()->GroupEnd());
            }
        };
        if (mf) h->pack(l, h->ws_r(l), &launches);  // packed coordinates for k_mf_spmv
        const bool p2p = part && !mf && dist_p2p_enabled() && (emu || peer_setup(h, l, nch));
        if (p2p && !emu) {
            // ---- one GPU per rank: this rank's k_pcg over the peers' mapped buffers
            auto &M = h->ctx->peer[l];
            const auto &P = Dd.local[0];
            PeerCGArgs pa{};
            pa.L = args[0].L;
            pa.L.out_iters = d_it + si;
            pa.L.out_rr = d_rr + 2 * si;
            pa.L.out_status = d_stat + si;
            pa.L.nnz = D.nnz;
            pa.nchunks = nch;
            pa.W = W;
            pa.rank = h->ctx->rank;
            pa.nb = pcg_resident_blocks((double)D.nnz, (double)n);
            MSK_CUDA(cudaMemsetAsync(M.cnt + 2, 0, sizeof(unsigned long long), st));  // own group barrier
            for (int w = 0; w < W; ++w) {
                PeerRank &pr = pa.R[w];
                pr.r = M.pr[w];
                pr.part = M.ppart[w];
                pr.alpha = M.palpha[w];
                pr.xcnt = M.pcnt[w];
                pr.nbar = M.pcnt[w] + 1;
                pr.gbar = M.pcnt[w] + 2;
                pr.hlo = Dd.hlo[w];
                pr.hhi = Dd.hhi[w];
                const int64_t cpr = (int64_t)CH * 256;
                pr.c0 = Dd.rows[w] / cpr;
                pr.c1 = (Dd.rows[w + 1] + cpr - 1) / cpr;
                if (w == h->ctx->rank) {
                    pr.x = X[0]; pr.p = Pv[0]; pr.q = Q[0];
                    pr.row_ptr = P.rp - P.lo; pr.col = P.col; pr.val = P.val;
                }
            }
            for (int w = 0; w < W; ++w) {  // rows of rank w that another rank reads
                int64_t a = Dd.rows[w + 1], b = Dd.rows[w];
                for (int v = 0; v < W; ++v) {
                    if (v == w) continue;
                    const int64_t s0 = std::max(Dd.rows[w], Dd.hlo[v]), s1 = std::min(Dd.rows[w + 1], Dd.hhi[v]);
                    if (s0 < s1) { a = std::min(a, s0); b = std::max(b, s1); }
                }
                pa.R[w].slo = a;
                pa.R[w].shi = b;
            }
            time_cg(l);
            pcg_launch(pa, st);
            launches += 1;
            cg_t.back()->stop();
            MSK_CUDA(cudaMemcpyAsync(out, M.alpha, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
            if (to_caller) permute_scatter(n, out, D.perm, ad[l].ptr, st, &launches);
            for (double *p : send) dfree(p, st);
            dfree(recv, st);
            dfree(sc, st);
            dfree(gbuf, st);
            return;
        }
        if (p2p && emu) {
            // ---- the whole CG of the level in ONE launch over peer memory (k_pcg):
            // every partition is a group of CTAs; partials and halo rows of r are
            // stored into the other partitions' buffers, the groups meet in a
            // device-side barrier
            double *pbuf = dalloc<double>((size_t)(3 * nch * np), st);
            unsigned long long *cnt = dalloc<unsigned long long>((size_t)(3 * np), st);
            MSK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 3 * np, st));
            PeerCGArgs pa{};
            pa.L = args[0].L;
            pa.L.x = pa.L.r = pa.L.p = pa.L.q = nullptr;
            pa.L.out_iters = d_it + si;
            pa.L.out_rr = d_rr + 2 * si;
            pa.L.out_status = d_stat + si;
            pa.L.nnz = D.nnz;
            pa.nchunks = nch;
            pa.W = np;
            pa.rank = -1;
            pa.nb = std::max(1, pcg_resident_blocks((double)D.nnz, (double)n) / np);
            for (int i = 0; i < np; ++i) {
                const auto &P = parts[i];
                PeerRank &pr = pa.R[i];
                pr.x = X[i];
                pr.r = R[i];
                pr.p = Pv[i];
                pr.q = Q[i];
                pr.part = pbuf + (size_t)(3 * nch) * i;
                pr.alpha = out;  // every partition pushes its owned rows into the one result
                pr.xcnt = cnt + 3 * i;
                pr.nbar = cnt + 3 * i + 1;
                pr.gbar = cnt + 3 * i + 2;
                pr.row_ptr = P.rp - P.lo;
                pr.col = P.col;
                pr.val = P.val;
                pr.c0 = P.c0;
                pr.c1 = P.c1;
                pr.hlo = P.hlo;
                pr.hhi = P.hhi;
            }
            for (int i = 0; i < np; ++i) {  // rows of partition i that another partition reads
                int64_t a = parts[i].hi, b = parts[i].lo;
                for (int j = 0; j < np; ++j) {
                    if (j == i) continue;
                    const int64_t s0 = std::max(parts[i].lo, parts[j].hlo), s1 = std::min(parts[i].hi, parts[j].hhi);
                    if (s0 < s1) { a = std::min(a, s0); b = std::max(b, s1); }
                }
                pa.R[i].slo = a;
                pa.R[i].shi = b;
            }
            time_cg(l);
            pcg_launch(pa, st);
            launches += 1;
            cg_t.back()->stop();
            dfree(pbuf, st);
            dfree(cnt, st);
            if (to_caller) permute_scatter(n, out, D.perm, ad[l].ptr, st, &launches);
            for (double *p : owned_alloc) dfree(p, st);
            for (double *p : send) dfree(p, st);
            dfree(recv, st);
            dfree(sc, st);
            return;
        }
        time_cg(l);
        for (int i = 0; i < np; ++i) dcg_init(args[i], st);
        allreduce();
        for (int i = 0; i < np; ++i) dcg_scalar(args[i], 0, st);
        halo();
        launches += 3 * np;
        for (int done = 0;;) {
            for (int k = 0; k < 8; ++k) {
                for (int i = 0; i < np; ++i) {
                    if (mf) dcg_mf_spmv(args[i], h->view(l), h->d, h->k, st);
                    else dcg_spmv(args[i], st);
                }
                allreduce();
                for (int i = 0; i < np; ++i) dcg_scalar(args[i], 1, st);
                for (int i = 0; i < np; ++i) dcg_rupd(args[i], st);
                allreduce();
                for (int i = 0; i < np; ++i) dcg_scalar(args[i], 2, st);
                for (int i = 0; i < np; ++i) dcg_scalar(args[i], 3, st);
                halo();
                launches += 6 * np + (emu ? 2 : 0);
            }
            done += 8;
            DistCGScalars hs;
            MSK_CUDA(cudaMemcpyAsync(&hs, sc, sizeof hs, cudaMemcpyDeviceToHost, st));
            MSK_CUDA(cudaStreamSynchronize(st));
            if (!hs.active || done > max_iter + 16) break;
        }
        for (int i = 0; i < np; ++i) dcg_xfin(args[i], st);
        launches += np;
        cg_t.back()->stop();
        // alpha^(l) complete on every rank (spatial order), then caller order
        if (!part) {
            if (out != X[0])
                MSK_CUDA(cudaMemcpyAsync(out, X[0], sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
        } else if (emu) {
            for (int i = 0; i < np; ++i) {
                const auto &P = parts[i];
                MSK_CUDA(cudaMemcpyAsync(out + P.lo, X[i] + P.lo, sizeof(double) * (size_t)(P.hi - P.lo),
                                         cudaMemcpyDeviceToDevice, st));
            }
        } else {
            const auto &P = Dd.local[0];
            if (out != X[0])
                MSK_CUDA(cudaMemcpyAsync(out + P.lo, X[0] + P.lo, sizeof(double) * (size_t)(P.hi - P.lo),
                                         cudaMemcpyDeviceToDevice, st));
            allgather_rows(h, out, Dd.rows, st);
        }
        if (to_caller) permute_scatter(n, out, D.perm, ad[l].ptr, st, &launches);
        MSK_CUDA(cudaMemcpyAsync(d_it + si, &sc->it, sizeof(int), cudaMemcpyDeviceToDevice, st));
        MSK_CUDA(cudaMemcpyAsync(d_stat + si, &sc->status, sizeof(int), cudaMemcpyDeviceToDevice, st));
        MSK_CUDA(cudaMemcpyAsync(d_rr + 2 * si, &sc->rr, sizeof(double), cudaMemcpyDeviceToDevice, st));
        MSK_CUDA(cudaMemcpyAsync(d_rr + 2 * si + 1, &sc->bb, sizeof(double), cudaMemcpyDeviceToDevice, st));
        for (double *p : owned_alloc) dfree(p, st);
        for (double *p : send) dfree(p, st);
        dfree(recv, st);
        dfree(sc, st);
        dfree(gbuf, st);
    };
    bool any_dist = false;
    for (int l = 0; l < L; ++l) any_dist = any_dist || h->dist[l].on;

    const bool thresholded = h->T > 0.0;
    if (thresholded || schedule != MSK_SCHED_PRUNED)
        for (int l = 0; l < L; ++l) wait_f(l);
    if (thresholded) {
        // a7: Jacobi on (id - M~(T)) beta = f (eq:perturbed_split P:865-869),
        // beta^(k) = f^(k) - sum_{l<k} X~_kl beta^(l) with the stored factor;
        // PRUNED = forward substitution (each block row once, in level order),
        // LITERAL = L full sweeps from beta_0 = f.  Then D_L alpha = beta by the
        // block-diagonal CG on ALL levels in one batched launch (Algorithm 1).
        double *fsp = h->ws_r(0);
        for (int l = 0; l < L; ++l)
            permute_gather(h->lev[l].n, fd[l].ptr, h->lev[l].perm, fsp + h->off[l], st, &launches);
        double *beta = h->ws_beta(0);
        if (schedule == MSK_SCHED_PRUNED) {
            MSK_CUDA(cudaMemcpyAsync(beta, fsp, sizeof(double) * h->ntot, cudaMemcpyDeviceToDevice, st));
            time_ga();
            for (int k = 1; k < L; ++k) {
                const auto &Dk = h->dist[k];
                if (!Dk.on) {
                    thresh_residual(h->off[k], h->off[k + 1], h->trow_ptr, h->tcol, h->tval, beta, beta, beta, st,
                                    &launches, h->tbucket, h->tmax_active);
                    continue;
                }
                // partitioned level: the owned rows, then beta^(k) complete on every
                // rank for the finer levels' rows (zero-padded sum: exact)
                for (const auto &P : Dk.local)
                    thresh_residual(h->off[k] + P.lo, h->off[k] + P.hi, h->trow_ptr, h->tcol, h->tval, beta, beta,
                                    beta, st, &launches, h->tbucket, h->tmax_active);
                if (!h->ctx->emulated) allgather_rows(h, beta + h->off[k], Dk.rows, st);
            }
            ga_t.back()->stop();
        } else {
            double *cur = h->ws_beta(0), *nxt = h->ws_t(0);
            MSK_CUDA(cudaMemcpyAsync(cur, fsp, sizeof(double) * h->ntot, cudaMemcpyDeviceToDevice, st));
            MSK_CUDA(cudaMemcpyAsync(nxt, fsp, sizeof(double) * h->ntot, cudaMemcpyDeviceToDevice, st));
            time_ga();
            for (int sweep = 0; sweep < L; ++sweep) {
                thresh_residual(h->off[1], h->ntot, h->trow_ptr, h->tcol, h->tval, fsp, cur, nxt, st, &launches,
                                h->tbucket, h->tmax_active);
                std::swap(cur, nxt);
            }
            ga_t.back()->stop();
            beta = cur;
        }
        std::vector<CGLevelArgs> a;
        for (int l = 0; l < L; ++l) {
            if (h->dist[l].on) continue;  // partitioned levels: below
            a.push_back(cg_args(h, l, tol, max_iter, beta + h->off[l], nullptr, alpha_sp[l], ad[l].ptr,
                                d_it + l, d_rr + 2 * l, d_stat + l));
            set_coef(a.back(), l);
        }
        if (!a.empty()) {
            time_cg(-1);
            cg_batched(a.data(), (int)a.size(), st, &launches);
            cg_t.back()->stop();
        }
        // (distributed context) the partitioned levels: beta^(l) = ws_beta(l) from the Jacobi
        for (int l = 0; l < L; ++l)
            if (h->dist[l].on) dist_level(l, tol, true);
    } else if (schedule == MSK_SCHED_PRUNED) {
        // Algorithm 2 with every inner solve done once, when its input is final:
        // beta^(l) = f^(l) - sum_{k<l} B_lk t^(k); t^(l) = A_l^{-1} beta^(l);
        // alpha^(l) = t^(l) (the final block CG of a converged block is the
        // same solve); the finest level is solved at tol.
        for (int l = 0; l < L; ++l) {
            NvtxRange nvl("level " + std::to_string(l));
            const double tl = l + 1 < L ? inner_tol : tol;
            wait_f(l);
            if (h->dist[l].on || mf) {
                dist_level(l, tl, false);
                out_alpha(l);
                debug_sync(st, "dist_level");
                if (l + 1 < L) h->pack(l, alpha_sp[l], &launches);
                continue;
            }
            CGLevelArgs a;
            if (l == 0) {
                a = cg_args(h, l, tl, max_iter, nullptr, fd[0].ptr, alpha_sp[l], ad[l].ptr,
                            d_it + l, d_rr + 2 * l, d_stat + l);
                set_coef(a, l);
            } else {
                b_products(l, alpha_sp.data(), h->ws_beta(l));
                a = cg_args(h, l, tl, max_iter, h->ws_beta(l), nullptr, alpha_sp[l], ad[l].ptr,
                            d_it + l, d_rr + 2 * l, d_stat + l);
                set_coef(a, l);
            }
            debug_sync(st, "b_products");
            NvtxRange nvc("CG");
            time_cg(l);
            cg_batched(&a, 1, st, &launches);
            cg_t.back()->stop();
            out_alpha(l);
            debug_sync(st, "cg");
            if (l + 1 < L) h->pack(l, alpha_sp[l], &launches);  // source records for later B products
            debug_sync(st, "pack");
        }
    } else {
        // Literal Algorithm 2: beta_0 = f; L sweeps of
        //   t^(l) = A_l^{-1} beta^(l) (l < L, inner tol, one batched launch),
        //   beta^(k) = f^(k) - sum_{l<k} B_kl t^(l)  (k >= 2)
        // then the block-diagonal CG (Algorithm 1) on all levels at tol.
        for (int l = 0; l < L; ++l) permute_gather(h->lev[l].n, fd[l].ptr, h->lev[l].perm, h->ws_beta(l), st, &launches);
        for (int sweep = 0; sweep < L; ++sweep) {
            if (L > 1) {
                std::vector<CGLevelArgs> a;
                for (int l = 0; l + 1 < L; ++l) {
                    if (h->dist[l].on || mf) continue;  // below
                    a.push_back(cg_args(h, l, inner_tol, max_iter, h->ws_beta(l), nullptr, t_sp[l], nullptr,
                                        d_it + sweep * L + l, d_rr + 2 * (sweep * L + l), d_stat + sweep * L + l));
                    set_coef(a.back(), sweep * L + l);
                }
                if (!a.empty()) {
                    time_cg(-1);
                    cg_batched(a.data(), (int)a.size(), st, &launches);
                    cg_t.back()->stop();
                }
                // partitioned inner levels (distributed context): the partitioned CG,
                // t^(l) complete on every rank afterwards; matrix-free levels: the
                // phase kernels with k_mf_spmv
                for (int l = 0; l + 1 < L; ++l)
                    if (h->dist[l].on || mf) dist_level(l, inner_tol, true, sweep, t_sp[l], false);
                for (int l = 0; l + 1 < L; ++l) h->pack(l, t_sp[l], &launches);
                for (int k = 1; k < L; ++k) {
                    const auto &Dk = h->dist[k];
                    if (Dk.on && !h->ctx->emulated)  // this rank's rows of a partitioned level
                        b_products_rows(k, t_sp.data(), h->ws_beta(k), Dk.local[0].lo, Dk.local[0].hi);
                    else
                        b_products(k, t_sp.data(), h->ws_beta(k));
                }
            }
        }
        std::vector<CGLevelArgs> a;
        for (int l = 0; l < L; ++l) {
            if (h->dist[l].on || mf) continue;
            a.push_back(cg_args(h, l, tol, max_iter, h->ws_beta(l), nullptr, alpha_sp[l], ad[l].ptr,
                                d_it + L * L + l, d_rr + 2 * (L * L + l), d_stat + L * L + l));
            set_coef(a.back(), L * L + l);
        }
        if (!a.empty()) {
            time_cg(-1);
            cg_batched(a.data(), (int)a.size(), st, &launches);
            cg_t.back()->stop();
        }
        for (int l = 0; l < L; ++l)
            if (h->dist[l].on || mf) dist_level(l, tol, true, L, alpha_sp[l], true);
    }
    ttot.stop();
    for (int l = 0; l < L; ++l) ad[l].flush();
    {  // the copy streams' work completes before the results are read / buffers freed on st
        for (int l = 0; l < L; ++l) wait_f(l);
        Ev done;
        done.record(cout);
        done.wait_on(st);
    }
    std::vector<int> it((size_t)(nslots * L)), stat((size_t)(nslots * L));
    std::vector<double> rr((size_t)(2 * nslots * L));
    unsigned long long hits = 0;
    MSK_CUDA(cudaMemcpyAsync(it.data(), d_it, sizeof(int) * it.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(stat.data(), d_stat, sizeof(int) * stat.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(rr.data(), d_rr, sizeof(double) * rr.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(&hits, d_hits, sizeof hits, cudaMemcpyDeviceToHost, st));
    const int fin_slot = schedule == MSK_SCHED_LITERAL && !thresholded ? L : 0;
    std::vector<double> coefs((size_t)(2 * coef_cap) * L);
    MSK_CUDA(cudaMemcpyAsync(coefs.data(), d_coef + (size_t)(2 * coef_cap) * fin_slot * L,
                             sizeof(double) * coefs.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(d_it, st); dfree(d_stat, st); dfree(d_rr, st); dfree(d_hits, st); dfree(d_coef, st);

    msk_solve_info loc;
    memset(&loc, 0, sizeof loc);
    loc.L = L;
    loc.jacobi_sweeps = schedule == MSK_SCHED_LITERAL ? L : 0;
    const int fin = schedule == MSK_SCHED_LITERAL && !thresholded ? L : 0;  // slot of the final solves
    if (thresholded) hits = (unsigned long long)(h->tnnz_active * (schedule == MSK_SCHED_LITERAL ? L : 1));
    std::string noconv;
    for (int s = 0; s < (thresholded ? 1 : nslots); ++s)
        for (int l = 0; l < L; ++l) {
            int idx = s * L + l;
            bool used = thresholded || schedule == MSK_SCHED_PRUNED || s == fin || l + 1 < L;
            if (!used) continue;
            if (stat[idx] && noconv.empty()) {
                char buf[160];
                snprintf(buf, sizeof buf, "level %d: rel. residual %.3e after %d iterations", l,
                         rr[2 * idx + 1] > 0 ? sqrt(rr[2 * idx] / rr[2 * idx + 1]) : 0.0, it[idx]);
                noconv = buf;
            }
            loc.nnz_cg += (double)it[idx] * (double)h->lev[l].nnz;
            loc.bytes_cg += cg_bytes(h->lev[l], it[idx]);
            if (s == fin) {
                loc.cg_iters[l] = it[idx];
                loc.kappa_est[l] = lanczos_kappa(coefs.data() + (size_t)(2 * coef_cap) * l,
                                                 std::min(it[idx], coef_cap));
                loc.rel_res[l] = rr[2 * idx + 1] > 0 ? sqrt(rr[2 * idx] / rr[2 * idx + 1]) : 0.0;
                loc.bytes_cg_level[l] += cg_bytes(h->lev[l], it[idx]);
            } else {
                loc.inner_iters[l] += it[idx];
            }
        }
    loc.nnz_gather = (double)hits;
    for (size_t i = 0; i < cg_t.size(); ++i) {
        double t = cg_t[i]->ms();
        loc.t_cg_ms += t;
        if (cg_t_level[i] >= 0) loc.t_cg_level_ms[cg_t_level[i]] += t;
        delete cg_t[i];
    }
    for (auto *t : ga_t) {
        loc.t_gather_ms += t->ms();
        delete t;
    }
    loc.t_total_ms = ttot.ms();
    loc.launches = launches;
    if (info) *info = loc;
    if (!noconv.empty()) throw Error(MSK_ERR_NOCONV, noconv);
    h->solved = true;
    API_END
}

// ================================================================ evaluate
namespace {
// Host-buffer evaluation on one GPU, pipelined in chunks of evaluation points:
// chunk c+1 is copied in (copy stream) while chunk c is sorted and evaluated
// (compute stream) and chunk c-1's values are copied out (second copy
// stream).  Every output depends only on its own point (fixed summation
// order), so the result is identical to the one-shot path.
void evaluate_pipelined(msk_hierarchy *h, int64_t m, const double *x, double *s, msk_eval_info *info) {
    cudaStream_t st = h->st(), cin = h->ctx->copy_in(), cout = h->ctx->copy_out();
    const int d = h->d, L = h->L;
    int launches = 0;
    // chunk boundaries: every chunk covers the whole domain, so each one re-reads
    // the levels' records (~0.26 ms per chunk on C3); a short first chunk starts
    // the computation early, growing chunks keep it fed from the copy stream, a
    // short last chunk leaves little copy-out after the last kernel (C3, 1e7
    // points: 1 Mi-point uniform chunks 11.2 ms, this schedule 9.4 ms; one-shot on device 6.6)
    std::vector<int64_t> bnd{0};
    if (const char *e = getenv("MSK_EVAL_CHUNK")) {  // test hook: uniform chunks
        const int64_t chunk = std::max<int64_t>(256, atoll(e));
        for (int64_t c = chunk; c < m; c += chunk) bnd.push_back(c);
    } else if (m >= (1 << 21)) {
        for (double fr : {0.10, 0.30, 0.60, 0.95}) bnd.push_back((int64_t)(fr * (double)m));
    }
    bnd.push_back(m);
    const int64_t nc = (int64_t)bnd.size() - 1;
    int64_t chunk = 0;
    for (int64_t c = 0; c < nc; ++c) chunk = std::max(chunk, bnd[c + 1] - bnd[c]);
    Timer ttot(st);
    ttot.start();
    const LevelData &F = h->lev[L - 1];
    const Grid g = F.g;
    double *xd = dalloc<double>((size_t)(m * d), st);
    double *sd = dalloc<double>((size_t)m, st);
    const int64_t cmax = std::min(chunk, m);
    double *xs = dalloc<double>((size_t)(cmax * d), st);
    int32_t *perm = dalloc<int32_t>((size_t)cmax, st);
    int32_t *cs = dalloc<int32_t>((size_t)(g.ncells + 1), st);
    unsigned long long *d_hits = dalloc<unsigned long long>(1, st);
    MSK_CUDA(cudaMemsetAsync(d_hits, 0, sizeof(unsigned long long), st));
    for (int l = 0; l < L; ++l) h->pack(l, h->lev[l].alpha, &launches);
    CopyStreamsGuard copy_guard{cin, cout};
    Ev ready;
    ready.record(st);  // allocations (stream-ordered on st) before the copy streams touch them
    ready.wait_on(cin);
    ready.wait_on(cout);
    std::vector<Ev> ein((size_t)nc), eout((size_t)nc);
    std::vector<Timer *> tso, tev;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t c0 = bnd[c], c1 = bnd[c + 1], nck = c1 - c0;
        MSK_CUDA(cudaMemcpyAsync(xd + c0 * d, x + c0 * d, sizeof(double) * (size_t)(nck * d),
                                 cudaMemcpyHostToDevice, cin));
        ein[c].record(cin);
    }
    for (int64_t c = 0; c < nc; ++c) {
        NvtxRange nvc("evaluate chunk " + std::to_string(c));
        const int64_t c0 = bnd[c], c1 = bnd[c + 1], nck = c1 - c0;
        ein[c].wait_on(st);
        CellListOut co{};
        co.perm = perm;
        for (int a = 0; a < d; ++a) co.xs[a] = xs + (size_t)a * nck;
        co.cell_start = cs;
        tso.push_back(new Timer(st));
        tso.back()->start();
        build_cell_list(d, nck, xd + c0 * d, g, false, co, st, &launches);
        tso.back()->stop();
        GatherArgs ga{};
        ga.d = d;
        ga.k = h->k;
        ga.nt = nck;
        for (int a = 0; a < d; ++a) ga.tx[a] = xs + (size_t)a * nck;
        ga.nlev = L;
        for (int l = 0; l < L; ++l) ga.lev[l] = h->view(l, h->lev[l].alpha);
        ga.base = nullptr;
        ga.sign = 1.0;
        ga.out = sd + c0;
        ga.out_perm = perm;
        ga.hits = d_hits;
        tev.push_back(new Timer(st));
        tev.back()->start();
        gather(ga, st, &launches);
        tev.back()->stop();
        eout[c].record(st);
        eout[c].wait_on(cout);
        MSK_CUDA(cudaMemcpyAsync(s + c0, sd + c0, sizeof(double) * (size_t)nck, cudaMemcpyDeviceToHost, cout));
    }
    Ev done;
    done.record(cout);
    done.wait_on(st);
    ttot.stop();
    unsigned long long hits = 0;
    MSK_CUDA(cudaMemcpyAsync(&hits, d_hits, sizeof hits, cudaMemcpyDeviceToHost, st));
    dfree(xd, st); dfree(sd, st); dfree(xs, st); dfree(perm, st); dfree(cs, st); dfree(d_hits, st);
    MSK_CUDA(cudaStreamSynchronize(st));
    double tsort = 0, teval = 0;
    for (auto *t : tso) { tsort += t->ms(); delete t; }
    for (auto *t : tev) { teval += t->ms(); delete t; }
    if (info) {
        info->nnz = (double)hits;
        info->t_sort_ms = tsort;
        info->t_eval_ms = teval;
        info->t_total_ms = ttot.ms();
        info->launches = launches;
    }
}
}  // namespace

extern "C" msk_status msk_evaluate_ex(msk_hierarchy *h, int64_t m, const double *x, double *s,
                                      msk_eval_info *info) {
    API_BEGIN
    require(h != nullptr, "msk_evaluate: NULL hierarchy");
    require(m >= 0, "msk_evaluate: m < 0");
    require(m == 0 || (x && s), "msk_evaluate: NULL argument");
    require(m < (1ll << 31) - 1, "msk_evaluate: m too large for one call");
    if (!h->solved) throw Error(MSK_ERR_STATE, "msk_evaluate: call msk_solve first");
    if (info) memset(info, 0, sizeof *info);
    if (m == 0) return MSK_OK;
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    if (h->ctx->world == 1 && !is_device_ptr(x) && !is_device_ptr(s)) {
        evaluate_pipelined(h, m, x, s, info);
        return MSK_OK;
    }
    cudaStream_t st = h->st();
    const int d = h->d, L = h->L;
    int launches = 0;
    Timer ttot(st), tsort(st), teval(st);
    ttot.start();
    DevBuf xd(x, (size_t)(m * d), st);
    DevOut sd(s, (size_t)m, st);
    // spatially sort the evaluation points on the finest level's grid (order
    // only affects locality: each output is independent of it)
    const LevelData &F = h->lev[L - 1];
    Grid g = F.g;
    double *xs = dalloc<double>((size_t)(m * d), st);
    int32_t *perm = dalloc<int32_t>((size_t)m, st);
    int32_t *cs = dalloc<int32_t>((size_t)(g.ncells + 1), st);
    CellListOut co{};
    co.perm = perm;
    for (int a = 0; a < d; ++a) co.xs[a] = xs + (size_t)a * m;
    co.cell_start = cs;
    // distributed context: a stable sort makes the order identical on every
    // rank, and each partition evaluates one contiguous share of it
    const int W = h->ctx->world;
    tsort.start();
    build_cell_list(d, m, xd.ptr, g, W > 1, co, st, &launches);
    tsort.stop();
    unsigned long long *d_hits = dalloc<unsigned long long>(1, st);
    MSK_CUDA(cudaMemsetAsync(d_hits, 0, sizeof(unsigned long long), st));
    for (int l = 0; l < L; ++l) h->pack(l, h->lev[l].alpha, &launches);
    teval.start();
    // distributed: rank r evaluates the share [r smax, (r+1) smax) of the sorted
    // points into a spatial-order buffer; one in-place all-gather of the shares
    // (not a zero-filled all-reduce) and a permutation give every rank all of
    // s_L -- or, with MSK_FLAG_OUTPUT_LOCAL, only its own share is written
    const int64_t smax = (m + W - 1) / W;
    const bool local_only = (h->flags & MSK_FLAG_OUTPUT_LOCAL) != 0;
    if (local_only && W > 1 && !h->ctx->emulated && sd.host)  // the other entries keep the caller's values
        MSK_CUDA(cudaMemcpyAsync(sd.ptr, s, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, st));
    double *ssp = W > 1 ? dalloc<double>((size_t)(smax * W), st) : nullptr;
    for (int r = 0; r < W; ++r) {
        if (W > 1 && !h->ctx->emulated && r != h->ctx->rank) continue;
        const int64_t lo = std::min(m, smax * r), hi = std::min(m, smax * (r + 1));
        if (hi <= lo) continue;
        GatherArgs ga{};
        ga.d = d;
        ga.k = h->k;
        ga.nt = hi - lo;
        for (int a = 0; a < d; ++a) ga.tx[a] = xs + (size_t)a * m + lo;
        ga.nlev = L;
        for (int l = 0; l < L; ++l) ga.lev[l] = h->view(l, h->lev[l].alpha);
        ga.base = nullptr;
        ga.sign = 1.0;
        ga.out = W > 1 ? ssp + lo : sd.ptr;
        ga.out_perm = W > 1 ? nullptr : perm + lo;
        ga.hits = d_hits;
        gather(ga, st, &launches);
    }
    if (W > 1) {
        const int me = h->ctx->rank;
        if (!h->ctx->emulated && !local_only)
            MSK_NCCL(nccl_api()->AllGather(ssp + smax * me, ssp, (size_t)smax, ncclFloat64, h->ctx->comm, st));
        const bool all = h->ctx->emulated || !local_only;
        const int64_t lo = all ? 0 : std::min(m, smax * me), hi = all ? m : std::min(m, smax * (me + 1));
        if (hi > lo) permute_scatter(hi - lo, ssp + lo, perm + lo, sd.ptr, st, &launches);
        dfree(ssp, st);
    }
    teval.stop();
    sd.flush();
    ttot.stop();
    unsigned long long hits = 0;
    MSK_CUDA(cudaMemcpyAsync(&hits, d_hits, sizeof hits, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(xs, st); dfree(perm, st); dfree(cs, st); dfree(d_hits, st);
    if (info) {
        info->nnz = (double)hits;
        info->t_sort_ms = tsort.ms();
        info->t_eval_ms = teval.ms();
        info->t_total_ms = ttot.ms();
        info->launches = launches;
    }
    API_END
}

extern "C" msk_status msk_evaluate(msk_hierarchy *h, int64_t m, const double *x, double *s) {
    return msk_evaluate_ex(h, m, x, s, nullptr);
}


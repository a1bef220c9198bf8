// capi_extra.cu -- multi-RHS solve/evaluation (NEXT-3), truncation diagnostics
// (NEXT-2) and the row-level entry points msk_apply_block / msk_cg_level.
#include "capi_internal.cuh"

// ============================================================ multi-RHS
// NEXT-3: several right-hand sides f_1..f_nrhs on the same
// hierarchy (exact mode, PRUNED schedule, one GPU, assembled A_l).  Columns are
// solved in groups of 4 (or 2): each CSR piece and each kernel evaluation of
// the B products serves the whole group.  Per column the arithmetic is that of
// msk_solve -- every column is bit-identical to its single-RHS solve.
extern "C" msk_status msk_solve_multi(msk_hierarchy *h, int32_t nrhs, const double *const *f, double tol,
                                      int32_t max_iter, double *const *alpha, int32_t *iters, double *t_ms) {
    API_BEGIN
    require(h && f && alpha, "msk_solve_multi: NULL argument");
    require(nrhs >= 1 && nrhs <= 1024, "msk_solve_multi: nrhs must be in [1, 1024]");
    require(tol > 0.0 && tol < 1.0 && max_iter >= 1, "msk_solve_multi: bad tol / max_iter");
    if (!h->assembled) throw Error(MSK_ERR_STATE, "msk_solve_multi: call msk_assemble first");
    require(!(h->T > 0.0), "msk_solve_multi: exact mode only (msk_assemble with T <= 0)");
    require(!(h->flags & MSK_FLAG_MATRIX_FREE), "msk_solve_multi: needs assembled A_l");
    require(h->ctx->world == 1, "msk_solve_multi: single GPU in this version");
    for (int l = 0; l < h->L; ++l) require(f[l] && alpha[l], "msk_solve_multi: NULL level pointer");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const int L = h->L;
    const double inner_tol = tol / 10.0;  // reading C-10
    h->release_multi();
    // column groups of 2 (an odd tail is padded with a zero column).  Groups of 4
    // are supported by the kernels but measured slower per column on C3 (37.8
    // vs 36.9 ms per right-hand side; single solves: 46.2): at 4 columns the
    // per-thread vector state exceeds the register budget of 3 CTAs per SM.
    for (int c = 0, pc = 0; c < nrhs;) {
        const int rem = nrhs - c, R = getenv("MSK_MULTI_R4") && rem >= 3 ? 4 : 2;
        h->grp0.push_back(c);
        h->grpR.push_back(R);
        h->grpP.push_back(pc);
        c += std::min(R, rem);
        pc += R;
        h->nrhs_pad = pc;
    }
    h->nrhs_m = nrhs;
    const int NP = h->nrhs_pad;
    std::vector<DevBuf> fd;
    std::vector<DevOut> ad;
    fd.reserve(L);
    ad.reserve(L);
    for (int l = 0; l < L; ++l) {
        fd.emplace_back(f[l], (size_t)(h->lev[l].n * nrhs), st);
        ad.emplace_back(alpha[l], (size_t)(h->lev[l].n * nrhs), st);
        h->alpham[l] = dalloc<double>((size_t)(h->lev[l].n * NP), st);
    }
    // workspace: r, p, q, beta per level for one group (R <= 4 columns)
    double *wsm = dalloc<double>((size_t)(4 * 4 * h->ntot), st);
    auto wsv = [&](int which, int l, int R) { return wsm + (size_t)which * 4 * h->ntot + (size_t)h->off[l] * R; };
    for (int l = 0; l < L; ++l) h->pack(l, wsm, nullptr);  // packed coordinates for the B products
    const int ng = (int)h->grp0.size();
    int *d_it = dalloc<int>((size_t)(4 * L * ng), st);
    int *d_stat = dalloc<int>((size_t)(4 * L * ng), st);
    double *d_rr = dalloc<double>((size_t)(8 * L * ng), st);
    MSK_CUDA(cudaMemsetAsync(d_it, 0, sizeof(int) * 4 * L * ng, st));
    MSK_CUDA(cudaMemsetAsync(d_stat, 0, sizeof(int) * 4 * L * ng, st));
    Timer tm(st);
    tm.start();
    int launches = 0;
    for (int g = 0; g < ng; ++g) {
        const int R = h->grpR[g], c0 = h->grp0[g], pc = h->grpP[g];
        const int nvalid = std::min(R, nrhs - c0);
        for (int l = 0; l < L; ++l) {
            const LevelData &D = h->lev[l];
            const double tl = l + 1 < L ? inner_tol : tol;
            CGRArgs a{};
            a.n = D.n;
            a.nnz = D.nnz;
            a.row_ptr = D.row_ptr;
            a.col = D.col;
            a.val = D.val;
            a.ldb = nrhs;
            a.col0 = c0;
            a.nvalid = nvalid;
            if (l == 0) {
                a.b_src = fd[0].ptr;
                a.b_perm = D.perm;
            } else {
                GatherMArgs ga{};
                ga.d = h->d;
                ga.k = h->k;
                ga.R = R;
                ga.nt = D.n;
                for (int t = 0; t < h->d; ++t) ga.tx[t] = D.xs + (size_t)t * D.n;
                ga.nlev = l;
                for (int k = 0; k < l; ++k) {
                    ga.lev[k] = h->view(k);
                    ga.coef[k] = h->alpham[k] + (size_t)h->lev[k].n * pc;  // group block [n][R]
                }
                ga.ldc = R;
                ga.base = fd[l].ptr;
                ga.base_perm = D.perm;
                ga.ldb = nrhs;
                ga.bcol0 = c0;
                ga.bcols = nvalid;
                ga.sign = -1.0;
                ga.out = wsv(3, l, R);
                ga.out_perm = nullptr;
                ga.ldo = R;
                ga.ocol0 = 0;
                ga.wcols = R;
                gather_multi(ga, st, &launches);
                a.b = wsv(3, l, R);
            }
            a.x = h->alpham[l] + (size_t)D.n * pc;  // group block [n][R] (contiguous rows)
            a.ldx = R;
            a.r = wsv(0, l, R);
            a.p = wsv(1, l, R);
            a.q = wsv(2, l, R);
            a.x_out = ad[l].ptr;
            a.x_perm = D.perm;
            a.ldo = nrhs;
            a.tol2 = tl * tl;
            a.max_iter = max_iter;
            const int slot = (g * L + l) * 4;
            a.out_iters = d_it + slot;
            a.out_rr = d_rr + 2 * slot;
            a.out_status = d_stat + slot;
            cg_multi(a, R, st, &launches);
        }
    }
    tm.stop();
    for (int l = 0; l < L; ++l) ad[l].flush();
    std::vector<int> hit((size_t)(4 * L * ng)), hst((size_t)(4 * L * ng));
    std::vector<double> hrr((size_t)(8 * L * ng));
    MSK_CUDA(cudaMemcpyAsync(hit.data(), d_it, sizeof(int) * hit.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(hst.data(), d_stat, sizeof(int) * hst.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(hrr.data(), d_rr, sizeof(double) * hrr.size(), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(wsm, st); dfree(d_it, st); dfree(d_stat, st); dfree(d_rr, st);
    if (t_ms) *t_ms = tm.ms();
    std::string noconv;
    for (int g = 0; g < ng; ++g)
        for (int l = 0; l < L; ++l)
            for (int k = 0; k < std::min(h->grpR[g], nrhs - h->grp0[g]); ++k) {
                const int slot = (g * L + l) * 4 + k, col = h->grp0[g] + k;
                if (iters) iters[(size_t)l * nrhs + col] = hit[slot];
                if (hst[slot] && noconv.empty()) {
                    char buf[200];
                    snprintf(buf, sizeof buf, "level %d, rhs %d: rel. residual %.3e after %d iterations", l, col,
                             hrr[2 * slot + 1] > 0 ? sqrt(hrr[2 * slot] / hrr[2 * slot + 1]) : 0.0, hit[slot]);
                    noconv = buf;
                }
            }
    if (!noconv.empty()) throw Error(MSK_ERR_NOCONV, noconv);
    API_END
}

// s[i][r] = f_L of right-hand side r at x_i (after msk_solve_multi); s is m x nrhs
extern "C" msk_status msk_evaluate_multi(msk_hierarchy *h, int64_t m, const double *x, double *s) {
    API_BEGIN
    require(h != nullptr, "msk_evaluate_multi: NULL hierarchy");
    require(m >= 0 && m < (1ll << 31) - 1, "msk_evaluate_multi: bad m");
    require(m == 0 || (x && s), "msk_evaluate_multi: NULL argument");
    if (h->nrhs_m == 0) throw Error(MSK_ERR_STATE, "msk_evaluate_multi: call msk_solve_multi first");
    if (m == 0) return MSK_OK;
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const int d = h->d, L = h->L, nrhs = h->nrhs_m;
    DevBuf xd(x, (size_t)(m * d), st);
    DevOut sd(s, (size_t)(m * nrhs), st);
    const LevelData &F = h->lev[L - 1];
    const Grid g = F.g;
    double *xs = dalloc<double>((size_t)(m * d), st);
    int32_t *perm = dalloc<int32_t>((size_t)m, st);
    int32_t *cs = dalloc<int32_t>((size_t)(g.ncells + 1), st);
    CellListOut co{};
    co.perm = perm;
    for (int a = 0; a < d; ++a) co.xs[a] = xs + (size_t)a * m;
    co.cell_start = cs;
    build_cell_list(d, m, xd.ptr, g, false, co, st, nullptr);
    for (int l = 0; l < L; ++l) h->pack(l, h->alpham[l], nullptr);  // coordinates (the .w slot is unused)
    for (size_t gi = 0; gi < h->grp0.size(); ++gi) {
        GatherMArgs ga{};
        ga.d = d;
        ga.k = h->k;
        ga.R = h->grpR[gi];
        ga.nt = m;
        for (int a = 0; a < d; ++a) ga.tx[a] = xs + (size_t)a * m;
        ga.nlev = L;
        for (int l = 0; l < L; ++l) {
            ga.lev[l] = h->view(l);
            ga.coef[l] = h->alpham[l] + (size_t)h->lev[l].n * h->grpP[gi];
        }
        ga.ldc = h->grpR[gi];
        ga.base = nullptr;
        ga.sign = 1.0;
        ga.out = sd.ptr;
        ga.out_perm = perm;
        ga.ldo = nrhs;
        ga.ocol0 = h->grp0[gi];
        ga.wcols = std::min(h->grpR[gi], nrhs - h->grp0[gi]);
        gather_multi(ga, st, nullptr);
    }
    sd.flush();
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(xs, st); dfree(perm, st); dfree(cs, st);
    API_END
}

// ================================================= truncation diagnostics
// NEXT-2: ||M_L||_2 (Figure 1) by power iteration
// on M^T M with M applied matrix-free: M v = -(B A^{-1}) v blockwise (the
// lower blocks -X_kl = -B_kl A_l^{-1}, reading C-7), M^T u = -A^{-1} (B^T u)
// blockwise; the A_l^{-1} are CG solves (one batched launch per application),
// B and B^T kernel sums (gather / gather_t).  sigma = ||M v|| with ||v|| = 1.
namespace {
__global__ void k_start_vector(double *v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (i < n) v[i] = (double)(((uint64_t)(i + 1) * 2654435761ull) & 0xffffffffull) * 0x1p-32 - 0.5;
}
}  // namespace

extern "C" msk_status msk_m_norm_ex(msk_hierarchy *h, int32_t which, int32_t max_iter, double rel_tol,
                                    double cg_tol, double *norm, int32_t *iters) {
    API_BEGIN
    require(h && norm, "msk_m_norm: NULL argument");
    require(which >= 0 && which <= 2, "msk_m_norm: which must be 0 (M), 1 (M - M~(T)) or 2 (M~(T))");
    if (which >= 1 && !(h->T > 0.0))
        throw Error(MSK_ERR_STATE, "msk_m_norm: M - M~(T) needs the thresholded factor (msk_assemble with T > 0)");
    require(max_iter >= 1 && rel_tol > 0.0 && cg_tol > 0.0 && cg_tol < 1.0, "msk_m_norm: bad arguments");
    if (!h->assembled) throw Error(MSK_ERR_STATE, "msk_m_norm: call msk_assemble first");
    require(!(h->flags & MSK_FLAG_MATRIX_FREE) && h->ctx->world == 1,
            "msk_m_norm: needs assembled A_l on one GPU");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const int L = h->L;
    const int64_t N = h->ntot;
    *norm = 0.0;
    if (iters) *iters = 0;
    if (L < 2) return MSK_OK;
    h->ensure_ws();
    double *v = dalloc<double>((size_t)N, st), *u = dalloc<double>((size_t)N, st);
    double *w = dalloc<double>((size_t)N, st), *t = dalloc<double>((size_t)N, st);
    double *scratch = dalloc<double>(300, st);
    int *d_it = dalloc<int>((size_t)L, st), *d_stat = dalloc<int>((size_t)L, st);
    // M - M~(T) = -(X - X~): add X~ v (stored CSR) to M v and X~^T u (its transpose) to M^T u
    int64_t *cptr = nullptr, *cpos = nullptr;
    int32_t *crow = nullptr, *ccol = nullptr;
    double *nv = nullptr;
    const int64_t ncols = h->off[L - 1];
    if (which >= 1) {
        cptr = dalloc<int64_t>((size_t)(ncols + 1), st);
        cpos = dalloc<int64_t>((size_t)h->tnnz + 1, st);
        crow = dalloc<int32_t>((size_t)h->tnnz + 1, st);
        thresh_csc(N - h->off[1], h->off[1], h->tnnz, ncols, h->trow_ptr, h->tcol, cptr, cpos, crow, ccol, st,
                   nullptr);
        nv = dalloc<double>((size_t)N, st);
    }
    double *d_rr = dalloc<double>((size_t)(2 * L), st);
    k_start_vector<<<ceil_div_u(N, 256), 256, 0, st>>>(v, N);
    MSK_CHECK_LAUNCH();
    dev_scale(v, 1.0 / sqrt(dev_dot(v, v, N, scratch, st)), N, st);
    // A_l^{-1} for l < L-1 on all those levels in one launch: x_l = A_l^{-1} b_l
    auto solve_coarse = [&](const double *b, double *x) {
        std::vector<CGLevelArgs> a;
        for (int l = 0; l + 1 < L; ++l)
            a.push_back(cg_args(h, l, cg_tol, 20000, b + h->off[l], nullptr, x + h->off[l], nullptr, d_it + l,
                                d_rr + 2 * l, d_stat + l));
        cg_batched(a.data(), (int)a.size(), st, nullptr);
    };
    double sigma = 0.0;
    int it = 0;
    for (; it < max_iter; ++it) {
        // u = M v  (which = 2: u = M~ v = -X~ v only)
        if (which == 2) MSK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * (size_t)N, st));
        else solve_coarse(v, t);
        if (which != 2) MSK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * (size_t)h->lev[0].n, st));
        for (int l = 0; l + 1 < L && which != 2; ++l) h->pack(l, t + h->off[l], nullptr);
        for (int k = 1; k < L && which != 2; ++k) {
            GatherArgs ga{};
            ga.d = h->d;
            ga.k = h->k;
            ga.nt = h->lev[k].n;
            for (int a = 0; a < h->d; ++a) ga.tx[a] = h->lev[k].xs + (size_t)a * h->lev[k].n;
            ga.nlev = k;
            for (int l = 0; l < k; ++l) ga.lev[l] = h->view(l, t + h->off[l]);
            ga.sign = -1.0;
            ga.out = u + h->off[k];
            gather(ga, st, nullptr);
        }
        if (which == 2) {  // u = 0 - X~ v
            thresh_residual(h->off[1], N, h->trow_ptr, h->tcol, h->tval, u, v, u, st, nullptr, h->tbucket,
                            h->tmax_active);
        }
        if (which == 1) {  // u += X~ v  (thresh_residual: out = base - sum val * (-v))
            MSK_CUDA(cudaMemcpyAsync(nv, v, sizeof(double) * (size_t)N, cudaMemcpyDeviceToDevice, st));
            dev_scale(nv, -1.0, N, st);
            thresh_residual(h->off[1], N, h->trow_ptr, h->tcol, h->tval, u, nv, u, st, nullptr, h->tbucket,
                            h->tmax_active);
        }
        const double s_new = sqrt(dev_dot(u, u, N, scratch, st));
        // w = M^T u = -A^{-1} (B^T u) on the coarse levels, 0 on the finest
        for (int l = 0; l + 1 < L && which != 2; ++l) {
            GatherTArgs gt{};
            gt.d = h->d;
            gt.k = h->k;
            gt.nt = h->lev[l].n;
            for (int a = 0; a < h->d; ++a) gt.tx[a] = h->lev[l].xs + (size_t)a * h->lev[l].n;
            const double dl = h->lev[l].delta;
            gt.delta2 = dl * dl;
            gt.inv_delta = 1.0 / dl;
            gt.scale = -pow(dl, -(double)h->d);  // the minus sign of M^T
            gt.nsrc = 0;
            for (int k = l + 1; k < L; ++k) {
                gt.src[gt.nsrc] = h->view(k);
                gt.y[gt.nsrc] = u + h->off[k];
                gt.reach[gt.nsrc] = (int)std::min(floor(dl * h->lev[k].g.inv_cell) + 1.0, 1e6);
                ++gt.nsrc;
            }
            gt.out = t + h->off[l];
            gather_t(gt, st, nullptr);
        }
        if (which == 2) MSK_CUDA(cudaMemsetAsync(w, 0, sizeof(double) * (size_t)N, st));
        else solve_coarse(t, w);
        MSK_CUDA(cudaMemsetAsync(w + h->off[L - 1], 0, sizeof(double) * (size_t)h->lev[L - 1].n, st));
        if (which >= 1)  // w += X~^T u  (which = 2: the sign of M~^T is immaterial to the norm)
            csc_spmv_add(ncols, cptr, cpos, crow, h->tval, u, w, st, h->tbucket, h->tmax_active);
        const double wn = sqrt(dev_dot(w, w, N, scratch, st));
        const bool done = it > 0 && fabs(s_new - sigma) <= rel_tol * s_new;
        sigma = s_new;
        if (done || !(wn > 0.0)) { ++it; break; }
        MSK_CUDA(cudaMemcpyAsync(v, w, sizeof(double) * (size_t)N, cudaMemcpyDeviceToDevice, st));
        dev_scale(v, 1.0 / wn, N, st);
    }
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(v, st); dfree(u, st); dfree(w, st); dfree(t, st); dfree(scratch, st);
    dfree(d_it, st); dfree(d_stat, st); dfree(d_rr, st);
    dfree(cptr, st); dfree(cpos, st); dfree(crow, st); dfree(ccol, st); dfree(nv, st);
    *norm = sigma;
    if (iters) *iters = it;
    API_END
}

extern "C" msk_status msk_m_norm(msk_hierarchy *h, int32_t max_iter, double rel_tol, double cg_tol,
                                 double *norm, int32_t *iters) {
    return msk_m_norm_ex(h, 0, max_iter, rel_tol, cg_tol, norm, iters);
}


extern "C" msk_status msk_apply_block(msk_hierarchy *h, int row_level, int col_level, const double *v,
                                      double *y, double *t_ms) {
    API_BEGIN
    require(h && v && y, "msk_apply_block: NULL argument");
    require(row_level >= 0 && row_level < h->L && col_level >= 0 && col_level <= row_level,
            "msk_apply_block: need 0 <= col_level <= row_level < L");
    if (row_level == col_level && !h->assembled) throw Error(MSK_ERR_STATE, "msk_apply_block: assemble first");
    if (row_level == col_level && h->dist[row_level].on)
        throw Error(MSK_ERR_STATE, "msk_apply_block: level is partitioned across ranks");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const LevelData &R = h->lev[row_level], &C = h->lev[col_level];
    DevBuf vd(v, (size_t)C.n, st);
    DevOut yd(y, (size_t)R.n, st);
    double *vs = dalloc<double>((size_t)C.n, st);
    permute_gather(C.n, vd.ptr, C.perm, vs, st, nullptr);
    Timer tm(st);
    if (row_level == col_level && R.row_ptr) {
        double *ys = dalloc<double>((size_t)R.n, st);
        tm.start();
        spmv_csr(R.n, R.row_ptr, R.col, R.val, vs, ys, st, nullptr);
        tm.stop();
        permute_scatter(R.n, ys, R.perm, yd.ptr, st, nullptr);
        dfree(ys, st);
    } else {
        GatherArgs ga{};
        ga.d = h->d;
        ga.k = h->k;
        ga.nt = R.n;
        for (int a = 0; a < h->d; ++a) ga.tx[a] = R.xs + (size_t)a * R.n;
        ga.nlev = 1;
        h->pack(col_level, vs, nullptr);
        ga.lev[0] = h->view(col_level, vs);
        ga.sign = 1.0;
        ga.out = yd.ptr;
        ga.out_perm = R.perm;
        tm.start();
        gather(ga, st, nullptr);
        tm.stop();
    }
    yd.flush();
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(vs, st);
    if (t_ms) *t_ms = tm.ms();
    API_END
}

extern "C" msk_status msk_cg_level(msk_hierarchy *h, int level, const double *b, double *x, double tol,
                                   int32_t max_iter, int32_t *iters, double *rel_res, double *t_ms) {
    API_BEGIN
    require(h && b && x, "msk_cg_level: NULL argument");
    require(level >= 0 && level < h->L, "msk_cg_level: bad level");
    require(tol > 0.0 && tol < 1.0 && max_iter >= 1, "msk_cg_level: bad tol / max_iter");
    if (!h->assembled) throw Error(MSK_ERR_STATE, "msk_cg_level: assemble first");
    if (h->dist[level].on) throw Error(MSK_ERR_STATE, "msk_cg_level: level is partitioned across ranks");
    if (h->flags & MSK_FLAG_MATRIX_FREE)
        throw Error(MSK_ERR_STATE, "msk_cg_level: matrix-free hierarchy (no stored A_l); use msk_solve");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    h->ensure_ws();
    const LevelData &D = h->lev[level];
    DevBuf bd(b, (size_t)D.n, st);
    DevOut xd(x, (size_t)D.n, st);
    double *xs = dalloc<double>((size_t)D.n, st);
    int *d_it = dalloc<int>(2, st);
    double *d_rr = dalloc<double>(2, st);
    CGLevelArgs a = cg_args(h, level, tol, max_iter, nullptr, bd.ptr, xs, xd.ptr, d_it, d_rr, d_it + 1);
    const bool phases = getenv("MSK_CG_PHASES") != nullptr;  // diagnostic phase timing
    unsigned long long *dbg = nullptr;
    if (phases) {
        dbg = dalloc<unsigned long long>(6, st);
        MSK_CUDA(cudaMemsetAsync(dbg, 0, 6 * sizeof(unsigned long long), st));
        a.dbg = dbg;
    }
    Timer tm(st);
    tm.start();
    cg_batched(&a, 1, st, nullptr);
    tm.stop();
    xd.flush();
    if (phases) {
        unsigned long long hd[6];
        MSK_CUDA(cudaMemcpyAsync(hd, dbg, sizeof hd, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[msk] cg phases (ms, CTA 0): spmv+update %.3f bar1 %.3f r-update %.3f bar2 %.3f\n",
                hd[0] * 1e-6, hd[1] * 1e-6, hd[2] * 1e-6, hd[3] * 1e-6);
        dfree(dbg, st);
    }
    int hit[2];
    double hrr[2];
    MSK_CUDA(cudaMemcpyAsync(hit, d_it, sizeof hit, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(hrr, d_rr, sizeof hrr, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(xs, st); dfree(d_it, st); dfree(d_rr, st);
    if (iters) *iters = hit[0];
    if (rel_res) *rel_res = hrr[1] > 0 ? sqrt(hrr[0] / hrr[1]) : 0.0;
    if (t_ms) *t_ms = tm.ms();
    if (hit[1]) {
        char buf[160];
        snprintf(buf, sizeof buf, "level %d: rel. residual %.3e after %d iterations", level,
                 hrr[1] > 0 ? sqrt(hrr[0] / hrr[1]) : 0.0, hit[0]);
        throw Error(MSK_ERR_NOCONV, buf);
    }
    API_END
}


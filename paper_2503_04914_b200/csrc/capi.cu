// capi.cu -- the C-ABI of libmsk (include/msk.h): argument checking, device
// memory (stream-ordered pool), host/device pointer handling, and the
// orchestration of the hot-path kernels:
//   create   : a0 ingest + a1 cell lists + pattern row counts (q, duplicates)
//   assemble : a2 CSR of A_l
//   solve    : a5 Jacobi (pruned or literal schedule) + a4/a8 block CG
//   evaluate : a9
// Every step of the path runs in the kernels of this library; there is no
// host compute path and no CPU fallback.
#include "capi_internal.cuh"

thread_local std::string capi::g_err;

// ================================================================= context
extern "C" msk_status msk_ctx_create(int device, void *cuda_stream, int rank, int world_size,
                                     const void *nccl_unique_id, msk_ctx **out) {
    API_BEGIN
    require(out != nullptr, "msk_ctx_create: out is NULL");
    *out = nullptr;
    require(world_size >= 1 && world_size <= kMaxParts, "msk_ctx_create: world_size must be in 1..16");
    const bool emulated = world_size > 1 && rank == -1 && nccl_unique_id == nullptr;
    if (world_size == 1) require(rank == 0 && nccl_unique_id == nullptr, "msk_ctx_create: world_size 1 needs rank 0, no id");
    else if (!emulated)
        require(rank >= 0 && rank < world_size && nccl_unique_id != nullptr,
                "msk_ctx_create: distributed context needs 0 <= rank < world_size and an NCCL unique id "
                "(or rank = -1 and no id for the single-process emulation)");
    int ndev = 0;
    MSK_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "msk_ctx_create: bad device index");
    MSK_CUDA(cudaSetDevice(device));
    msk_ctx *c = new msk_ctx();
    c->device = device;
    c->world = world_size;
    c->rank = emulated ? 0 : rank;
    c->emulated = emulated;
    if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else {
        MSK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    if (world_size > 1 && !emulated) {
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof id);
        MSK_NCCL(nccl_api()->CommInitRank(&c->comm, world_size, id, rank));
    }
    // keep freed blocks in the stream-ordered pool: repeated create/solve
    // cycles then allocate without device-wide synchronisation
    cudaMemPool_t pool;
    MSK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~0ull;
    MSK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    cg_max_resident_blocks();
    *out = c;
    API_END
}

extern "C" void msk_ctx_destroy(msk_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto &M : ctx->peer) M.release();
    if (ctx->comm) nccl_api()->CommDestroy(ctx->comm);
    if (ctx->cin) { cudaStreamSynchronize(ctx->cin); cudaStreamDestroy(ctx->cin); }
    if (ctx->cout) { cudaStreamSynchronize(ctx->cout); cudaStreamDestroy(ctx->cout); }
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

extern "C" msk_status msk_nccl_unique_id(void *out) {
    API_BEGIN
    require(out != nullptr, "msk_nccl_unique_id: NULL argument");
    ncclUniqueId id;
    MSK_NCCL(nccl_api()->GetUniqueId(&id));
    memcpy(out, &id, sizeof id);
    API_END
}

// Halo plan of partition `rank` (host logic, no device): for every peer s,
// the rows it must send to s (the part of s's referenced column range
// [hlo[s], hhi[s]) that `rank` owns) and the rows it receives from s (the
// part of its own referenced range that s owns).  Empty ranges have lo == hi.
extern "C" msk_status msk_halo_plan(int world, int rank, const int64_t *rows, const int64_t *hlo,
                                    const int64_t *hhi, int64_t *send_lo, int64_t *send_hi, int64_t *recv_lo,
                                    int64_t *recv_hi) {
    API_BEGIN
    require(world >= 1 && rank >= 0 && rank < world && rows && hlo && hhi && send_lo && send_hi && recv_lo &&
                recv_hi,
            "msk_halo_plan: bad argument");
    for (int s = 0; s < world; ++s) {
        int64_t a = 0, b = 0, c = 0, e = 0;
        if (s != rank) {
            a = std::max(hlo[s], rows[rank]);
            b = std::min(hhi[s], rows[rank + 1]);
            c = std::max(hlo[rank], rows[s]);
            e = std::min(hhi[rank], rows[s + 1]);
        }
        send_lo[s] = a;
        send_hi[s] = std::max(a, b);
        recv_lo[s] = c;
        recv_hi[s] = std::max(c, e);
    }
    API_END
}

// Row partition of a level (host logic, no device): whole chunks of
// cg_chunk_tiles(n) * 256 rows, chunks split as evenly as possible.
extern "C" msk_status msk_partition_rows(int64_t n, int world, int64_t *bounds) {
    API_BEGIN
    require(n >= 0 && world >= 1 && bounds != nullptr, "msk_partition_rows: bad argument");
    const int64_t rows_per_chunk = (int64_t)cg_chunk_tiles(n) * 256;
    const int64_t nch = (n + rows_per_chunk - 1) / rows_per_chunk;
    for (int r = 0; r <= world; ++r) {
        const int64_t c = nch * r / world;
        bounds[r] = std::min(c * rows_per_chunk, n);
    }
    API_END
}

// Refinement of the last grid axis (Grid::zf): MSK_ZF (1, 2, 4, 8; default 2).
// Same-box A/B on C3: step 55.73 / 55.57 / 56.18 / 57.40 ms for
// zf = 1 / 2 / 4 / 8 -- thinner cells trim the candidate ranges (B products
// 5.56 -> 5.25 -> 5.14 ms) but multiply the cells the cell-list passes visit
// (create 2.58 -> 2.78 -> 3.26 ms).
int grid_zf() {
    static const int zf = [] {
        const char *e = getenv("MSK_ZF");
        const int v = e ? atoi(e) : 2;
        return v == 1 || v == 2 || v == 4 || v == 8 ? v : 2;
    }();
    return zf;
}

// Which levels to partition: a latency model of one CG
// iteration.  One GPU moves ~12 nnz + 88 n bytes at ~5 TB/s (measured k_cg:
// 4.9-5.4 TB/s), with a ~15 us floor (two device barriers and the grid's
// ramp; C3 levels 1-4 measure 5-15 us); W partitions move 1/W of the bytes
// each and add the partitioned path's barriers (k_pcg over NVLink: ~10 us
// per iteration; host-driven phase path with NCCL: ~60 us).  Partition when
// that is below 0.8 x the one-GPU time.  Identical on every rank (same inputs).
bool partition_pays(double nnz, double n, int W) {
    const char *e = getenv("MSK_DIST_P2P");
    const bool p2p = !(e && e[0] == '0');
    const double bw = 5e12, floor_s = 15e-6, ovh = p2p ? 10e-6 : 60e-6;
    const double bytes = 12.0 * nnz + 88.0 * n;
    const double t1 = std::max(floor_s, bytes / bw);
    const double tw = std::max(floor_s, bytes / ((double)W * bw)) + ovh;
    return tw < 0.8 * t1;
}

// =============================================================== hierarchy
extern "C" msk_status msk_hierarchy_create(msk_ctx *ctx, int d, int L, const int64_t *n,
                                           const double *const *points, const double *delta,
                                           const double *q, int wendland_k, uint32_t flags,
                                           msk_hierarchy **out) {
    msk_hierarchy *h = nullptr;
    try {
        require(ctx && out && n && points && delta, "msk_hierarchy_create: NULL argument");
        *out = nullptr;
        require(d == 2 || d == 3, "msk_hierarchy_create: d must be 2 or 3");
        require(L >= 1 && L <= kMaxLevels, "msk_hierarchy_create: L must be in 1..16");
        require(wendland_k >= 0 && wendland_k <= 2, "msk_hierarchy_create: k must be 0, 1 or 2");
        require((flags & ~(MSK_FLAG_DIST_ALL | MSK_FLAG_MATRIX_FREE | MSK_FLAG_OUTPUT_LOCAL)) == 0,
                "msk_hierarchy_create: unknown flags");
        for (int l = 0; l < L; ++l) {
            require(n[l] >= 1 && n[l] < (1ll << 31) - 1, "msk_hierarchy_create: n[l] out of range");
            require(points[l] != nullptr, "msk_hierarchy_create: NULL points");
            require(std::isfinite(delta[l]) && delta[l] > 0, "msk_hierarchy_create: delta must be finite and > 0");
            if (q) require(std::isfinite(q[l]) && q[l] > 0, "msk_hierarchy_create: q must be finite and > 0");
        }
        MSK_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        h = new msk_hierarchy();
        h->ctx = ctx;
        h->d = d;
        h->L = L;
        h->k = wendland_k;
        h->flags = flags;
        Timer tm(st);
        tm.start();
        int launches = 0;
        // ---- a0: ingest (device copies of host inputs) + bounding box
        std::vector<DevBuf> pts;
        pts.reserve(L);
        unsigned long long *mm = dalloc<unsigned long long>(6, st);
        unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
        MSK_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st));
        for (int l = 0; l < L; ++l) {
            pts.emplace_back(points[l], (size_t)(n[l] * d), st);
            minmax_points(n[l], d, pts.back().ptr, mm, st, &launches);
        }
        unsigned long long mmh[6];
        MSK_CUDA(cudaMemcpyAsync(mmh, mm, sizeof mmh, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaStreamSynchronize(st));
        dfree(mm, st);
        for (int a = 0; a < d; ++a) {
            h->lo[a] = ord_key_to_double(mmh[a]);
            h->hi[a] = ord_key_to_double(mmh[3 + a]);
            require(std::isfinite(h->lo[a]) && std::isfinite(h->hi[a]),
                    "msk_hierarchy_create: non-finite point coordinates");
        }
        // ---- a1: per-level uniform grid + cell list; pattern row counts
        std::vector<unsigned long long *> minr2(L);
        for (int l = 0; l < L; ++l) {
            LevelData &D = h->lev[l];
            D.n = n[l];
            D.delta = delta[l];
            h->off[l + 1] = h->off[l] + n[l];
            double cell = delta[l] * (1.0 + 0x1p-20);
            const int zf = grid_zf();
            for (;;) {
                // the cell count is formed in double first: extent / delta can be
                // large enough (3-D, > ~2.6e6 per axis) to overflow int64 products
                const double inv = 1.0 / cell;
                double invs[3], dims_d[3], ncells_d = 1.0;
                for (int a = 0; a < 3; ++a) {
                    invs[a] = a == d - 1 ? (double)zf * inv : inv;  // exact: zf is a power of two
                    dims_d[a] = a < d ? floor((h->hi[a] - h->lo[a]) * invs[a]) + 1.0 : 1.0;
                    ncells_d *= dims_d[a];
                }
                require(std::isfinite(ncells_d), "msk_hierarchy_create: non-finite cell grid");
                // bound the cell count (points much sparser than delta): larger
                // cells only add candidates, never lose neighbours
                if (ncells_d <= (double)zf * (8.0 * (double)n[l] + 4096.0)) {
                    Grid g{};
                    g.inv_cell = inv;
                    g.zf = zf;
                    g.ncells = 1;
                    for (int a = 0; a < 3; ++a) {
                        g.lo[a] = a < d ? h->lo[a] : 0.0;
                        g.inv[a] = invs[a];
                        g.dim[a] = (int64_t)dims_d[a];
                        g.ncells *= g.dim[a];
                    }
                    D.g = g;
                    break;
                }
                cell *= 1.5;
            }
            D.xs = dalloc<double>((size_t)(d * n[l]), st);
            D.perm = dalloc<int32_t>((size_t)n[l], st);
            D.cell_start = dalloc<int32_t>((size_t)(D.g.ncells + 1), st);
            CellListOut co{};
            co.perm = D.perm;
            for (int a = 0; a < d; ++a) co.xs[a] = D.xs + (size_t)a * n[l];
            co.cell_start = D.cell_start;
            co.keys = nullptr;
            build_cell_list(d, n[l], pts[l].ptr, D.g, true, co, st, &launches);
            {  // FP32 prefilter coordinates (relative to lo) and threshold
                double ext = 0.0;
                for (int a = 0; a < d; ++a) ext = std::max(ext, h->hi[a] - h->lo[a]);
                D.frec = dalloc<float4>((size_t)n[l], st);
                pack_frecords(n[l], d, D.xs, h->lo, D.frec, st, &launches);
                D.fthr = prefilter_threshold(delta[l], ext + delta[l], d);
            }
            D.cnt = dalloc<int32_t>((size_t)n[l], st);
            minr2[l] = dalloc<unsigned long long>(1, st);
            unsigned long long inf = 0x7ff0000000000000ull;
            MSK_CUDA(cudaMemcpyAsync(minr2[l], &inf, sizeof inf, cudaMemcpyHostToDevice, st));
            LevelView v = h->view(l);
            // distributed context: which levels are partitioned is decided here (the
            // latency model on an analytic nnz estimate, identical on every rank);
            // with one GPU per rank a partitioned level counts only its owned rows
            h->part_on[l] = false;
            const int W = ctx->world;
            if (W > 1) {
                const int64_t rpc = (int64_t)cg_chunk_tiles(n[l]) * 256;
                const int64_t nch = (n[l] + rpc - 1) / rpc;
                double vol = 1.0;
                for (int a = 0; a < d; ++a) vol *= std::max(h->hi[a] - h->lo[a], delta[l]);
                const double ball = d == 3 ? 4.18879020478639 * delta[l] * delta[l] * delta[l]
                                           : 3.14159265358979 * delta[l] * delta[l];
                const double nnz_est = (double)n[l] * std::max(1.0, (double)n[l] * ball / vol);
                h->part_on[l] = nch >= W && ((flags & MSK_FLAG_DIST_ALL) || partition_pays(nnz_est, (double)n[l], W));
            }
            int64_t r0 = 0, r1 = n[l];
            if (h->part_on[l] && !ctx->emulated) {
                std::vector<int64_t> b((size_t)W + 1);
                msk_partition_rows(n[l], W, b.data());
                r0 = b[ctx->rank];
                r1 = b[ctx->rank + 1];
                MSK_CUDA(cudaMemsetAsync(D.cnt, 0, sizeof(int32_t) * (size_t)n[l], st));
            }
            LevelView rv = v;
            rv.n = r1 - r0;
            for (int a = 0; a < d; ++a) rv.x[a] += r0;
            count_pattern(d, rv, v, true, D.cnt + r0, minr2[l], st, &launches, r0);
            D.cnt_lo = r0;
            D.cnt_hi = r1;
        }
        h->ntot = h->off[L];
        std::vector<unsigned long long> mr(L);
        // a level whose rows were counted in slices: the minimum over every rank's
        // slice (each pair is seen by its rows' owners: duplicates are still found)
        for (int l = 0; l < L; ++l) {
            if (!(h->part_on[l] && !ctx->emulated)) continue;
            const int W = ctx->world;
            unsigned long long *all = dalloc<unsigned long long>((size_t)W, st);
            MSK_NCCL(nccl_api()->AllGather(minr2[l], all, 1, ncclUint64, ctx->comm, st));
            std::vector<unsigned long long> hv((size_t)W);
            MSK_CUDA(cudaMemcpyAsync(hv.data(), all, sizeof(unsigned long long) * W, cudaMemcpyDeviceToHost, st));
            MSK_CUDA(cudaStreamSynchronize(st));
            const unsigned long long m = *std::min_element(hv.begin(), hv.end());
            MSK_CUDA(cudaMemcpyAsync(minr2[l], &m, sizeof m, cudaMemcpyHostToDevice, st));
            dfree(all, st);
        }
        for (int l = 0; l < L; ++l)
            MSK_CUDA(cudaMemcpyAsync(&mr[l], minr2[l], sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        tm.stop();
        MSK_CUDA(cudaStreamSynchronize(st));
        for (int l = 0; l < L; ++l) {
            dfree(minr2[l], st);
            double r2;
            memcpy(&r2, &mr[l], sizeof r2);
            require(r2 > 0.0, "msk_hierarchy_create: duplicate points in level " + std::to_string(l));
            if (!q && !std::isfinite(r2) && n[l] > 1) {
                // no pair within delta_l: widen the search (m cells per axis) until the
                // closest pair found is closer than m cell sides -- then it is the closest
                const LevelView v = h->view(l);
                const double cell = 1.0 / v.g.inv_cell;
                int64_t maxdim = 1;
                for (int a = 0; a < d; ++a) maxdim = std::max<int64_t>(maxdim, v.g.dim[a]);
                for (int64_t m = 2;; m *= 2) {
                    const int mm = (int)std::min<int64_t>(m, maxdim);
                    r2 = min_r2_reach(d, v, mm, st);
                    const double lim = (double)mm * cell * (1.0 - 1e-12);
                    if (mm >= maxdim || (std::isfinite(r2) && r2 < lim * lim)) break;
                }
            }
            h->lev[l].q = q ? q[l] : (std::isfinite(r2) ? 0.5 * sqrt(r2) : 0.5 * delta[l]);
        }
        h->t_create_ms = tm.ms();
        h->launches_create = launches;
        *out = h;
        return MSK_OK;
    } catch (const msk::Error &e) {
        set_err(e.what());
        if (h) { h->release(); delete h; }
        return (msk_status)e.status;
    } catch (const std::exception &e) {
        set_err(e.what());
        if (h) { h->release(); delete h; }
        return MSK_ERR_CUDA;
    }
}

extern "C" void msk_hierarchy_destroy(msk_hierarchy *h) {
    if (!h) return;
    cudaSetDevice(h->ctx->device);
    h->release();
    cudaStreamSynchronize(h->st());
    delete h;
}

extern "C" msk_status msk_hierarchy_info_get(const msk_hierarchy *h, msk_hierarchy_info *info) {
    API_BEGIN
    require(h && info, "msk_hierarchy_info_get: NULL argument");
    memset(info, 0, sizeof *info);
    info->d = h->d;
    info->L = h->L;
    info->k = h->k;
    for (int l = 0; l < h->L; ++l) {
        info->n[l] = h->lev[l].n;
        info->nnz_A[l] = h->lev[l].nnz;
        info->ncells[l] = h->lev[l].g.ncells;
        info->delta[l] = h->lev[l].delta;
        info->q[l] = h->lev[l].q;
    }
    info->t_create_ms = h->t_create_ms;
    info->t_assemble_ms = h->t_assemble_ms;
    info->launches_create = h->launches_create;
    info->launches_assemble = h->launches_assemble;
    API_END
}

// ================================================================ assemble
namespace {

// a6: the thresholded factor X~_{kl}(T) of all blocks k > l (eq:perturbedmatrix
// P:846-861): geometric pattern ||x_j^(k) - x_i^(l)||^2 < (T q_l)^2 (reading
// C-5), values chi_i^(l)(x_j^(k)) from Lagrange columns c_i = A_l^{-1} e_i
// solved by the multi-RHS CG at lagrange_tol (eq:chi P:373-377).
void build_factor(msk_hierarchy *h, double T, double lagrange_tol, double patch_R, int64_t patch_min_n,
                  int *launches) {
    cudaStream_t st = h->st();
    // MSK_DEBUG_PATCH: device time of each phase of the build (stderr)
    const bool dbg = getenv("MSK_DEBUG_PATCH") != nullptr;
    std::vector<std::pair<std::string, Timer *>> ph;
    auto mark = [&](const std::string &name) {
        if (!dbg) return;
        ph.emplace_back(name, new Timer(st));
        ph.back().second->start();
    };
    auto done = [&]() {
        if (!dbg || ph.empty()) return;
        ph.back().second->stop();
    };
    const int L = h->L, d = h->d;
    const int64_t ntot = h->ntot;
    // ---- pattern: rows = all points (level 0 rows empty), columns global
    int32_t *cnt = dalloc<int32_t>((size_t)ntot, st);
    MSK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)ntot, st));
    auto pattern_args = [&](int k) {
        ThreshPatternArgs a{};
        a.d = d;
        a.nt = h->lev[k].n;
        for (int q = 0; q < d; ++q) a.tx[q] = h->lev[k].xs + (size_t)q * h->lev[k].n;
        a.nlev = k;
        a.nb = (int)std::min<double>(floor(T), (double)kMaxTBucket);
        for (int l = 0; l < k; ++l) {
            a.lev[l] = h->view(l);
            const double R = T * h->lev[l].q;
            a.R2[l] = R * R;
            for (int t = 1; t <= a.nb; ++t) {  // the R2 recipe at integer T = t (reading C-5)
                const double Rt = (double)t * h->lev[l].q;
                a.tq2[l][t - 1] = Rt * Rt;
            }
            a.reach[l] = (int)std::min(floor(R * h->lev[l].g.inv_cell) + 1.0, 1e6);
            a.col_off[l] = h->off[l];
        }
        return a;
    };
    mark("pattern count");
    for (int k = 1; k < L; ++k) {
        ThreshPatternArgs a = pattern_args(k);
        a.cnt = cnt + h->off[k];
        thresh_count(a, st, launches);
    }
    done();
    h->trow_ptr = dalloc<int64_t>((size_t)(ntot + 1), st);
    exclusive_scan_i64(cnt, ntot, h->trow_ptr, st, launches);
    int64_t nnz = 0;
    MSK_CUDA(cudaMemcpyAsync(&nnz, h->trow_ptr + ntot, sizeof nnz, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(cnt, st);
    h->tnnz = nnz;
    h->tcol = dalloc<int32_t>((size_t)nnz, st);
    h->tval = dalloc<double>((size_t)nnz, st);
    h->tbucket = dalloc<uint8_t>((size_t)nnz, st);
    mark("pattern fill");
    for (int k = 1; k < L; ++k) {
        ThreshPatternArgs a = pattern_args(k);
        a.row_ptr = h->trow_ptr + h->off[k];
        a.col = h->tcol;
        a.bucket = h->tbucket;
        thresh_fill(a, st, launches);
    }
    done();
    mark("transpose index");
    // ---- transpose index over the coarse columns (levels 0..L-2)
    const int64_t ncols = h->off[L - 1];
    int64_t *cptr = dalloc<int64_t>((size_t)(ncols + 1), st);
    int64_t *cpos = dalloc<int64_t>((size_t)nnz, st);
    int32_t *crow = dalloc<int32_t>((size_t)nnz, st);
    int32_t *ccol = nullptr;  // columns are found by binary search in cptr (saves 4 B per entry)
    thresh_csc(ntot - h->off[1], h->off[1], nnz, ncols, h->trow_ptr, h->tcol, cptr, cpos, crow, ccol, st,
               launches);
    done();
    std::vector<int64_t> hcptr((size_t)(ncols + 1));
    MSK_CUDA(cudaMemcpyAsync(hcptr.data(), cptr, sizeof(int64_t) * (ncols + 1), cudaMemcpyDeviceToHost, st));
    int *dstat = dalloc<int>(2, st);
    MSK_CUDA(cudaMemsetAsync(dstat, 0, 2 * sizeof(int), st));
    int *pstat = dalloc<int>(6, st);  // patch path: CG failures, overflows, max iterations, max patch, count x 2
    MSK_CUDA(cudaMemsetAsync(pstat, 0, 6 * sizeof(int), st));
    MSK_CUDA(cudaStreamSynchronize(st));
    // ---- Lagrange columns, level by level, rounds of concurrent 32-column batches
    const int resident = 4 * 148;
    const double budget = 8e9;  // bytes of CG workspace per round
    for (int l = 0; l + 1 < L; ++l) {
        const LevelData &D = h->lev[l];
        if (patch_R > 0.0 && D.n > patch_min_n) {
            // ---- local-patch Lagrange functions, one CTA per column
            PatchArgs pa{};
            pa.d = d;
            pa.k = h->k;
            pa.L = L;
            pa.ncols = D.n;
            const double rho = patch_R * D.q;
            pa.rho2 = rho * rho;
            pa.reach = (int)std::min(floor(rho * D.g.inv_cell) + 1.0, 1e6);
            pa.Lv = h->view(l);
            pa.row_ptr = D.row_ptr;
            pa.col = D.col;
            pa.val = D.val;
            pa.tol2 = lagrange_tol * lagrange_tol;
            pa.max_iter = 5000;
            pa.cptr = cptr;
            pa.cpos = cpos;
            pa.crow = crow;
            pa.col_off = h->off[l];
            for (int q = 0; q <= L; ++q) pa.lev_off[q] = h->off[q];
            for (int q = 0; q < L; ++q) {
                pa.lev_xs[q] = h->lev[q].xs;
                pa.lev_n[q] = h->lev[q].n;
            }
            pa.val_out = h->tval;
            pa.fail = pstat;
            MSK_CUDA(cudaMemsetAsync(pstat + 4, 0, 2 * sizeof(int), st));
            patch_count(pa, D.cnt, pstat + 4, st);  // [4] max patch points, [5] max sum of their row lengths
            int hpz[2] = {0, 0};
            MSK_CUDA(cudaMemcpyAsync(hpz, pstat + 4, sizeof hpz, cudaMemcpyDeviceToHost, st));
            MSK_CUDA(cudaStreamSynchronize(st));
            const int hp = hpz[0];
            if (getenv("MSK_DEBUG_PATCH"))
                fprintf(stderr, "[msk] patch level %d: n %lld q %.6g rho %.6g reach %d cell %.6g pmax %d nnz bound %d\n",
                        l, (long long)D.n, D.q, rho, pa.reach, 1.0 / D.g.inv_cell, hp, hpz[1]);
            if (hp > 65535)
                throw Error(MSK_ERR_INVALID, "msk_assemble: local patch of " + std::to_string(hp) +
                                                 " points (> 65535); reduce patch_R");
            pa.pmax = hp;
            // the members' row lengths bound the patch-local entries (the workspace, and
            // with it the CTAs per SM, is sized by it instead of pmax x max row length)
            pa.nnzmax = (int)std::min<int64_t>((int64_t)hpz[1], (int64_t)hp * hp);
            {
                const int64_t side = 2 * (int64_t)pa.reach + 1, nq = d == 3 ? side * side : side;
                if (nq > 65535)
                    throw Error(MSK_ERR_INVALID, "msk_assemble: local patch spans too many cells; reduce patch_R");
                pa.nq = (int)nq;
            }
            const size_t smem = patch_smem_bytes(pa.pmax, pa.nnzmax, pa.nq);
            // larger patches run from a global workspace (patch_lagrange); bound it
            if (smem > (size_t)1 << 30)
                throw Error(MSK_ERR_INVALID, "msk_assemble: local patch too large (" + std::to_string(hp) +
                                                 " points); reduce patch_R");
            mark("level " + std::to_string(l) + " patches (k_patch)");
            patch_lagrange(pa, smem, st, launches);
            done();
            MSK_CUDA(cudaMemsetAsync(pstat + 4, 0, sizeof(int), st));
            continue;
        }
        const int64_t nb_total = (D.n + 31) / 32;
        const double slot_bytes = 4.0 * (double)D.n * 32.0 * 8.0;
        int64_t slots = std::min<int64_t>(nb_total, std::max<int64_t>(1, std::min<int64_t>(resident, (int64_t)(budget / slot_bytes))));
        double *ws = dalloc<double>((size_t)(slots * 4 * D.n * 32), st);
        for (int64_t b0 = 0; b0 < nb_total; b0 += slots) {
            const int64_t nb = std::min<int64_t>(slots, nb_total - b0);
            CGMultiArgs m{};
            m.n = D.n;
            m.ncols = D.n;
            m.row_ptr = D.row_ptr;
            m.col = D.col;
            m.val = D.val;
            m.tol2 = lagrange_tol * lagrange_tol;
            m.max_iter = 20000;
            m.batch0 = b0;
            m.nbatches = nb_total;
            m.ws = ws;
            m.fail = dstat;
            m.max_iters = dstat + 1;
            mark("level " + std::to_string(l) + " exact Lagrange CG");
            thresh_cg_multi(m, (int)nb, st, launches);
            done();
            const int64_t c0 = b0 * 32, c1 = std::min<int64_t>((b0 + nb) * 32, D.n);
            ThreshValueArgs v{};
            v.d = d;
            v.k = h->k;
            v.L = L;
            v.pos0 = hcptr[h->off[l] + c0];
            v.pos1 = hcptr[h->off[l] + c1];
            v.cpos = cpos;
            v.crow = crow;
            v.cptr = cptr;
            v.c_lo = h->off[l] + c0;
            v.c_hi = h->off[l] + c1;
            v.col_off = (int32_t)h->off[l];
            v.first_col = c0;
            for (int q = 0; q <= L; ++q) v.lev_off[q] = h->off[q];
            for (int q = 0; q < L; ++q) {
                v.lev_xs[q] = h->lev[q].xs;
                v.lev_n[q] = h->lev[q].n;
            }
            v.Lv = h->view(l);
            v.ws = ws;
            v.val = h->tval;
            mark("level " + std::to_string(l) + " values");
            thresh_values(v, st, launches);
            done();
        }
        dfree(ws, st);
    }
    int hstat[2], hps[5];
    MSK_CUDA(cudaMemcpyAsync(hstat, dstat, sizeof hstat, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(hps, pstat, sizeof hps, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(dstat, st); dfree(pstat, st); dfree(cptr, st); dfree(cpos, st); dfree(crow, st); dfree(ccol, st);
    if (dbg) {
        for (auto &p : ph) {
            fprintf(stderr, "[msk] factor build %-34s %9.3f ms\n", p.first.c_str(), p.second->ms());
            delete p.second;
        }
    }
    h->lagrange_max_iters = std::max(hstat[1], hps[2]);
    h->patch_max_points = hps[3];
    if (hstat[0]) throw Error(MSK_ERR_NOCONV, "msk_assemble: Lagrange CG did not converge in 20000 iterations");
    if (hps[1]) throw Error(MSK_ERR_INVALID, "msk_assemble: local patch overflow in " + std::to_string(hps[1]) +
                                                 " columns; reduce patch_R");
    if (hps[0]) throw Error(MSK_ERR_NOCONV, "msk_assemble: patch Lagrange CG did not converge in " +
                                                std::to_string(hps[0]) + " columns");
    // the factor is valid: only now does the hierarchy carry it
    h->T = T;
    h->T_active = T;
    h->tmax_active = 255;
    h->tnnz_active = h->tnnz;
}

}  // namespace

namespace {
void assemble_body(msk_hierarchy *h, double T, double lagrange_tol, double patch_R, int64_t patch_min_n, bool mf);


}

extern "C" msk_status msk_assemble_ex(msk_hierarchy *h, double T, double lagrange_tol, double patch_R,
                                      int64_t patch_min_n) {
    API_BEGIN
    require(std::isfinite(patch_R) && patch_min_n >= 0, "msk_assemble_ex: bad patch arguments");
    require(h != nullptr, "msk_assemble: NULL hierarchy");
    require(std::isfinite(T), "msk_assemble: T must be finite");
    require(!(T > 0.0) || (lagrange_tol > 0.0 && lagrange_tol < 1.0),
            "msk_assemble: lagrange_tol must be in (0,1) when T > 0");
    require(!(T > 0.0) || !(h->flags & MSK_FLAG_MATRIX_FREE),
            "msk_assemble: the thresholded factor needs assembled A_l (hierarchy is MSK_FLAG_MATRIX_FREE)");
    const bool mf = (h->flags & MSK_FLAG_MATRIX_FREE) != 0;
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    // a failed (re-)assembly leaves the hierarchy unassembled (MSK_ERR_STATE for
    // msk_solve), never with a half-built factor or freed CSR arrays
    h->assembled = false;
    h->solved = false;
    h->release_factor();
    h->release_dist();
    try {
        assemble_body(h, T, lagrange_tol, patch_R, patch_min_n, mf);
    } catch (...) {
        h->release_factor();
        h->release_dist();
        h->assembled = false;
        throw;
    }
    API_END
}

namespace {
void assemble_body(msk_hierarchy *h, double T, double lagrange_tol, double patch_R, int64_t patch_min_n, bool mf) {
    cudaStream_t st = h->st();
    Timer tm(st);
    tm.start();
    int launches = 0;
    std::vector<int64_t> nnz(h->L);
    // a partitioned level counted only its owned rows at create; the thresholded
    // factor build needs the full A_l of the column levels: count the others now
    for (int l = 0; l + 1 < h->L && T > 0.0; ++l) {
        LevelData &D = h->lev[l];
        if (D.cnt_lo == 0 && D.cnt_hi == D.n) continue;
        const LevelView v = h->view(l);
        for (int part = 0; part < 2; ++part) {
            const int64_t r0 = part == 0 ? 0 : D.cnt_hi, r1 = part == 0 ? D.cnt_lo : D.n;
            if (r1 <= r0) continue;
            LevelView rv = v;
            rv.n = r1 - r0;
            for (int a = 0; a < h->d; ++a) rv.x[a] += r0;
            count_pattern(h->d, rv, v, true, D.cnt + r0, nullptr, st, &launches, r0);
        }
        D.cnt_lo = 0;
        D.cnt_hi = D.n;
    }
    // distributed context: partition the large levels
    const int W = h->ctx->world;
    for (int l = 0; l < h->L && W > 1; ++l) {
        const int64_t n = h->lev[l].n;
        const int64_t rpc = (int64_t)cg_chunk_tiles(n) * 256;
        const int64_t nch = (n + rpc - 1) / rpc;
        if (h->part_on[l]) {  // decided in msk_hierarchy_create (latency model or DIST_ALL)
            auto &Dd = h->dist[l];
            Dd.on = true;
            Dd.rows.resize(W + 1);
            msk_partition_rows(n, W, Dd.rows.data());
            for (int r = 0; r < W; ++r) {
                if (!h->ctx->emulated && r != h->ctx->rank) continue;
                msk_hierarchy::PartLocal P;
                P.rank = r;
                P.lo = Dd.rows[r];
                P.hi = Dd.rows[r + 1];
                P.c0 = P.lo / rpc;
                P.c1 = (P.hi + rpc - 1) / rpc;
                Dd.local.push_back(P);
            }
        }
    }
    for (int l = 0; l < h->L; ++l) {
        LevelData &D = h->lev[l];
        dfree(D.row_ptr, st); dfree(D.col, st); dfree(D.val, st); dfree(D.col16, st); dfree(D.cbase, st);
        dfree(D.clen, st);
        D.row_ptr = nullptr; D.col = nullptr; D.val = nullptr; D.col16 = nullptr; D.cbase = nullptr;
        D.clen = nullptr;
        nnz[l] = 0;
        D.nnz = 0;  // (partitioned levels accumulate their partitions' entries below)
        if (h->dist[l].on) {  // owned rows only, per local partition
            for (auto &P : h->dist[l].local) {
                const int64_t m = P.hi - P.lo;
                P.rp = dalloc<int64_t>((size_t)(m + 3), st);
                MSK_CUDA(cudaMemsetAsync(P.rp + m + 1, 0, 2 * sizeof(int64_t), st));
                exclusive_scan_i64(D.cnt + P.lo, m, P.rp, st, &launches);
                MSK_CUDA(cudaMemcpyAsync(&P.nnz, P.rp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            }
            if (!(T > 0.0 && l + 1 < h->L)) continue;
            // thresholded factor in a distributed context: the column levels keep
            // their full A_l as well (the Lagrange build is replicated on every rank)
        }
        D.row_ptr = dalloc<int64_t>((size_t)(D.n + 3), st);  // + padding for 16-byte bulk copies
        MSK_CUDA(cudaMemsetAsync(D.row_ptr + D.n + 1, 0, 2 * sizeof(int64_t), st));
        exclusive_scan_i64(D.cnt, D.n, D.row_ptr, st, &launches);
        MSK_CUDA(cudaMemcpyAsync(&nnz[l], D.row_ptr + D.n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
    MSK_CUDA(cudaStreamSynchronize(st));
    for (int l = 0; l < h->L; ++l) {
        LevelData &D = h->lev[l];
        if (h->dist[l].on) {
            auto &Dd = h->dist[l];
            unsigned long long *mm = dalloc<unsigned long long>(2, st);
            for (auto &P : Dd.local) {
                if (mf) {  // no stored entries: nnz from the row counts, halo from the hit range
                    dfree(P.rp, st);
                    P.rp = nullptr;
                    LevelView rows = h->view(l), cols = h->view(l);
                    rows.n = P.hi - P.lo;
                    for (int a = 0; a < h->d; ++a) rows.x[a] += P.lo;
                    hit_range(h->d, rows, cols, mm, st);
                    unsigned long long hm[2];
                    MSK_CUDA(cudaMemcpyAsync(hm, mm, sizeof hm, cudaMemcpyDeviceToHost, st));
                    MSK_CUDA(cudaStreamSynchronize(st));
                    P.hlo = P.nnz ? std::min<int64_t>((int64_t)hm[0], P.lo) : P.lo;
                    P.hhi = P.nnz ? std::max<int64_t>((int64_t)hm[1] + 1, P.hi) : P.hi;
                    D.nnz += P.nnz;
                    continue;
                }
                P.col = dalloc<int32_t>((size_t)P.nnz + 4, st);
                P.val = dalloc<double>((size_t)P.nnz + 2, st);
                MSK_CUDA(cudaMemsetAsync(P.col + P.nnz, 0, 4 * sizeof(int32_t), st));
                MSK_CUDA(cudaMemsetAsync(P.val + P.nnz, 0, 2 * sizeof(double), st));
                LevelView rows = h->view(l), cols = h->view(l);
                rows.n = P.hi - P.lo;
                for (int a = 0; a < h->d; ++a) rows.x[a] += P.lo;
                fill_pattern(h->d, h->k, rows, cols, P.rp, P.col, P.val, st, &launches);
                col_minmax(P.nnz, P.col, mm, st);
                unsigned long long hm[2];
                MSK_CUDA(cudaMemcpyAsync(hm, mm, sizeof hm, cudaMemcpyDeviceToHost, st));
                MSK_CUDA(cudaStreamSynchronize(st));
                P.hlo = P.nnz ? std::min<int64_t>((int64_t)hm[0], P.lo) : P.lo;
                P.hhi = P.nnz ? std::max<int64_t>((int64_t)hm[1] + 1, P.hi) : P.hi;
                D.nnz += P.nnz;
            }
            dfree(mm, st);
            if (D.row_ptr) {  // full A_l of a column level (thresholded factor build)
                D.col = dalloc<int32_t>((size_t)nnz[l] + 4, st);
                D.val = dalloc<double>((size_t)nnz[l] + 2, st);
                MSK_CUDA(cudaMemsetAsync(D.col + nnz[l], 0, 4 * sizeof(int32_t), st));
                MSK_CUDA(cudaMemsetAsync(D.val + nnz[l], 0, 2 * sizeof(double), st));
                LevelView v = h->view(l);
                fill_pattern(h->d, h->k, v, v, D.row_ptr, D.col, D.val, st, &launches);
            }
            // every partition's halo range, known to all
            Dd.hlo.assign(W, 0);
            Dd.hhi.assign(W, 0);
            if (h->ctx->emulated) {
                for (auto &P : Dd.local) { Dd.hlo[P.rank] = P.hlo; Dd.hhi[P.rank] = P.hhi; }
            } else {
                int64_t *buf = dalloc<int64_t>((size_t)(2 * W + 2), st);
                int64_t mine[2] = {Dd.local[0].hlo, Dd.local[0].hhi};
                MSK_CUDA(cudaMemcpyAsync(buf + 2 * W, mine, sizeof mine, cudaMemcpyHostToDevice, st));
                MSK_NCCL(nccl_api()->AllGather(buf + 2 * W, buf, 2, ncclInt64, h->ctx->comm, st));
                std::vector<int64_t> all((size_t)(2 * W));
                MSK_CUDA(cudaMemcpyAsync(all.data(), buf, sizeof(int64_t) * 2 * W, cudaMemcpyDeviceToHost, st));
                MSK_CUDA(cudaStreamSynchronize(st));
                for (int r = 0; r < W; ++r) { Dd.hlo[r] = all[2 * r]; Dd.hhi[r] = all[2 * r + 1]; }
                dfree(buf, st);
            }
            continue;
        }
        D.nnz = nnz[l];
        if (mf) {  // matrix-free: the row counts (nnz) are all that is kept
            dfree(D.row_ptr, st);
            D.row_ptr = nullptr;
            continue;
        }
        D.col = dalloc<int32_t>((size_t)D.nnz + 4, st);  // + padding for 16-byte bulk copies
        D.val = dalloc<double>((size_t)D.nnz + 2, st);
        MSK_CUDA(cudaMemsetAsync(D.col + D.nnz, 0, 4 * sizeof(int32_t), st));
        MSK_CUDA(cudaMemsetAsync(D.val + D.nnz, 0, 2 * sizeof(double), st));
        LevelView v = h->view(l);
        fill_pattern(h->d, h->k, v, v, D.row_ptr, D.col, D.val, st, &launches);
        // MSK_COL16=1: k_cg streams 16-bit columns in per-chunk windows (10 B/nnz instead
        // of 12).  Off by default: same-box A/B C3 finest level 40.1 vs
        // 32.7 ms, C2 21.3 vs 19.4 ms -- the decode lengthens the gather's address chain,
        // and the SpMV pass is bound by that per-thread chain, not by bandwidth
        // The same per-chunk column windows can steer an L2 prefetch of the next chunk's
        // gathered r (MSK_RPREF=1).  Off by default: same-box A/B, C3 finest 32.91 ms
        // either way, level 5 3.46 vs 3.33 ms (the gathered r already hits L2).
        static const bool c16 = getenv("MSK_COL16") && getenv("MSK_COL16")[0] == '1';
        static const bool rpref = getenv("MSK_RPREF") && getenv("MSK_RPREF")[0] == '1';
        if ((c16 || rpref) && D.n >= 256) {
            const int CH = cg_chunk_tiles(D.n);
            const int64_t nch = ((D.n + 255) / 256 + CH - 1) / CH;
            if (c16) {
                D.col16 = dalloc<uint16_t>((size_t)D.nnz + 16, st);
                MSK_CUDA(cudaMemsetAsync(D.col16 + D.nnz, 0, 16 * sizeof(uint16_t), st));
            }
            D.cbase = dalloc<int4>((size_t)nch, st);
            if (rpref) D.clen = dalloc<int4>((size_t)nch, st);
            launches += 1;
            if (!col16_build(D.n, D.row_ptr, D.col, D.col16, D.cbase, D.clen, st)) {
                // some chunk spans more than 4 windows: no 16-bit stream (the windows
                // still steer the prefetch)
                dfree(D.col16, st);
                D.col16 = nullptr;
            }
        }
    }
    if (T > 0.0 && h->L > 1) build_factor(h, T, lagrange_tol, patch_R, patch_min_n, &launches);
    tm.stop();
    MSK_CUDA(cudaStreamSynchronize(st));
    h->t_assemble_ms = tm.ms();
    h->launches_assemble = launches;
    h->assembled = true;
}
}  // namespace

extern "C" msk_status msk_assemble(msk_hierarchy *h, double T, double lagrange_tol) {
    return msk_assemble_ex(h, T, lagrange_tol, 0.0, 0);
}

extern "C" msk_status msk_set_threshold(msk_hierarchy *h, double T) {
    API_BEGIN
    require(h != nullptr, "msk_set_threshold: NULL hierarchy");
    if (!(h->T > 0.0)) throw Error(MSK_ERR_STATE, "msk_set_threshold: no thresholded factor (msk_assemble with T > 0)");
    const int nb = (int)std::min<double>(floor(h->T), (double)kMaxTBucket);
    const bool all = T == h->T;
    require(all || (T == floor(T) && T >= 1.0 && T <= (double)nb),
            "msk_set_threshold: T must equal the build's T or be an integer in [1, floor(build T)] (<= 24)");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    h->tmax_active = all ? 255 : (int)T;
    h->T_active = T;
    h->tnnz_active = all ? h->tnnz : bucket_count(h->tbucket, h->tnnz, h->tmax_active, h->st());
    API_END
}

// ===================================================== row-level entry points
extern "C" msk_status msk_export_block(msk_hierarchy *h, int row_level, int col_level,
                                       int64_t *row_ptr, int32_t *col, double *val) {
    API_BEGIN
    require(h && row_ptr, "msk_export_block: NULL argument");
    require(row_level >= 0 && row_level < h->L && col_level >= 0 && col_level <= row_level,
            "msk_export_block: need 0 <= col_level <= row_level < L");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const LevelData &R = h->lev[row_level], &C = h->lev[col_level];
    const int64_t nr = R.n;
    int32_t *cnt = nullptr;
    int64_t *rp = nullptr;
    int32_t *cl = nullptr;
    double *vl = nullptr;
    bool own = true;
    int64_t nnz = 0;
    if (row_level == col_level && h->assembled && !h->dist[row_level].on && R.row_ptr) {
        rp = R.row_ptr; cl = R.col; vl = R.val; nnz = R.nnz;
        own = false;
    } else {
        LevelView rv = h->view(row_level), cv = h->view(col_level);
        cnt = dalloc<int32_t>((size_t)nr, st);
        count_pattern(h->d, rv, cv, row_level == col_level, cnt, nullptr, st, nullptr);
        rp = dalloc<int64_t>((size_t)(nr + 1), st);
        exclusive_scan_i64(cnt, nr, rp, st, nullptr);
        MSK_CUDA(cudaMemcpyAsync(&nnz, rp + nr, sizeof nnz, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaStreamSynchronize(st));
        cl = dalloc<int32_t>((size_t)nnz, st);
        vl = dalloc<double>((size_t)nnz, st);
        fill_pattern(h->d, h->k, rv, cv, rp, cl, vl, st, nullptr);
    }
    std::vector<int64_t> hrp((size_t)(nr + 1));
    std::vector<int32_t> hcl((size_t)nnz), rperm((size_t)nr), cperm((size_t)C.n);
    std::vector<double> hvl((size_t)nnz);
    MSK_CUDA(cudaMemcpyAsync(hrp.data(), rp, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost, st));
    if (nnz) {
        MSK_CUDA(cudaMemcpyAsync(hcl.data(), cl, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaMemcpyAsync(hvl.data(), vl, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st));
    }
    MSK_CUDA(cudaMemcpyAsync(rperm.data(), R.perm, sizeof(int32_t) * nr, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(cperm.data(), C.perm, sizeof(int32_t) * C.n, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    if (own) { dfree(cnt, st); dfree(rp, st); dfree(cl, st); dfree(vl, st); }
    // host re-indexing of the exported copy into caller order (diagnostic only)
    std::vector<int64_t> inv((size_t)nr);
    for (int64_t i = 0; i < nr; ++i) inv[rperm[i]] = i;
    int64_t pos = 0;
    std::vector<std::pair<int32_t, double>> tmp;
    for (int64_t j = 0; j < nr; ++j) {
        row_ptr[j] = pos;
        int64_t i = inv[j];
        tmp.clear();
        for (int64_t p = hrp[i]; p < hrp[i + 1]; ++p) tmp.emplace_back(cperm[hcl[p]], hvl[p]);
        std::sort(tmp.begin(), tmp.end());
        for (auto &e : tmp) {
            if (col) col[pos] = e.first;
            if (val) val[pos] = e.second;
            ++pos;
        }
    }
    row_ptr[nr] = pos;
    API_END
}

extern "C" msk_status msk_export_factor(msk_hierarchy *h, int row_level, int col_level, int64_t *row_ptr,
                                        int32_t *col, double *val, double *T_out) {
    API_BEGIN
    require(h && row_ptr, "msk_export_factor: NULL argument");
    require(row_level >= 0 && row_level < h->L && col_level >= 0 && col_level < row_level,
            "msk_export_factor: need 0 <= col_level < row_level < L");
    if (!(h->T > 0.0)) throw Error(MSK_ERR_STATE, "msk_export_factor: no thresholded factor (msk_assemble with T > 0)");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const LevelData &R = h->lev[row_level], &C = h->lev[col_level];
    const int64_t r0 = h->off[row_level], nr = R.n;
    std::vector<int64_t> hrp((size_t)(nr + 1));
    MSK_CUDA(cudaMemcpyAsync(hrp.data(), h->trow_ptr + r0, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    const int64_t p0 = hrp[0], np = hrp[nr] - hrp[0];
    std::vector<int32_t> hcl((size_t)np), rperm((size_t)nr), cperm((size_t)C.n);
    std::vector<double> hvl((size_t)np);
    std::vector<uint8_t> hbk((size_t)np);
    if (np) {
        MSK_CUDA(cudaMemcpyAsync(hcl.data(), h->tcol + p0, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaMemcpyAsync(hvl.data(), h->tval + p0, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaMemcpyAsync(hbk.data(), h->tbucket + p0, np, cudaMemcpyDeviceToHost, st));
    }
    MSK_CUDA(cudaMemcpyAsync(rperm.data(), R.perm, sizeof(int32_t) * nr, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(cperm.data(), C.perm, sizeof(int32_t) * C.n, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> inv((size_t)nr);
    for (int64_t i = 0; i < nr; ++i) inv[rperm[i]] = i;
    const int64_t c_lo = h->off[col_level], c_hi = h->off[col_level + 1];
    int64_t pos = 0;
    std::vector<std::pair<int32_t, double>> tmp;
    for (int64_t j = 0; j < nr; ++j) {
        row_ptr[j] = pos;
        const int64_t i = inv[j];
        tmp.clear();
        for (int64_t p = hrp[i] - p0; p < hrp[i + 1] - p0; ++p)
            if (hcl[p] >= c_lo && hcl[p] < c_hi && hbk[p] <= h->tmax_active)
                tmp.emplace_back(cperm[hcl[p] - c_lo], hvl[p]);
        std::sort(tmp.begin(), tmp.end());
        for (auto &e : tmp) {
            if (col) col[pos] = e.first;
            if (val) val[pos] = e.second;
            ++pos;
        }
    }
    row_ptr[nr] = pos;
    if (T_out) *T_out = h->T_active;
    API_END
}

extern "C" msk_status msk_export_cells(msk_hierarchy *h, int level, int32_t *perm, int32_t *cell_start,
                                       int64_t *cell_key, double *lo, double *cell, int64_t *dims) {
    API_BEGIN
    require(h != nullptr && level >= 0 && level < h->L, "msk_export_cells: bad argument");
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    const LevelData &D = h->lev[level];
    std::vector<int32_t> cs((size_t)(D.g.ncells + 1));
    MSK_CUDA(cudaMemcpyAsync(cs.data(), D.cell_start, sizeof(int32_t) * cs.size(), cudaMemcpyDeviceToHost, st));
    if (perm) MSK_CUDA(cudaMemcpyAsync(perm, D.perm, sizeof(int32_t) * D.n, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    if (cell_start) memcpy(cell_start, cs.data(), sizeof(int32_t) * cs.size());
    if (cell_key)
        for (int64_t c = 0; c < D.g.ncells; ++c)
            for (int32_t i = cs[c]; i < cs[c + 1]; ++i) cell_key[i] = c;
    for (int a = 0; a < h->d; ++a) {
        if (lo) lo[a] = D.g.lo[a];
        if (dims) dims[a] = D.g.dim[a];
    }
    if (cell) *cell = 1.0 / D.g.inv_cell;
    API_END
}

extern "C" msk_status msk_export_grid(msk_hierarchy *h, int level, double *lo, double *inv_cell, int64_t *dims) {
    API_BEGIN
    require(h != nullptr && level >= 0 && level < h->L, "msk_export_grid: bad argument");
    const LevelData &D = h->lev[level];
    for (int a = 0; a < h->d; ++a) {
        if (lo) lo[a] = D.g.lo[a];
        if (dims) dims[a] = D.g.dim[a];
        if (inv_cell) inv_cell[a] = D.g.inv[a];
    }
    API_END
}

extern "C" const char *msk_last_error(void) { return g_err.c_str(); }

extern "C" const char *msk_version(void) { return "libmsk 0.1 (sm_100a, FP64)"; }

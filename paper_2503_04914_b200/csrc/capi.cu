// capi.cu -- the C-ABI of libmsk (include/msk.h): argument checking, device
// memory (stream-ordered pool), host/device pointer handling, and the
// orchestration of the hot-path kernels:
//   create   : a0 ingest + a1 cell lists + pattern row counts (q, duplicates)
//   assemble : a2 CSR of A_l
//   solve    : a5 Jacobi (pruned or literal schedule) + a4/a8 block CG
//   evaluate : a9
// Every step of the path runs in the kernels of this library; there is no
// host compute path and no CPU fallback.
#include <math.h>
#include <stdio.h>

#include <cmath>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/msk.h"
#include "kernels.cuh"
#include "nccl_dl.cuh"

using namespace msk;

// ------------------------------------------------------------------ state
struct msk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // distributed solve: world partitions of every
    // large level; `emulated` runs all partitions in this process on one
    // device (testing), else one partition per rank over NCCL.
    int rank = 0, world = 1;
    bool emulated = false;
    ncclComm_t comm = nullptr;
    // copy streams for host-buffer calls (H2D / D2H overlapped with the compute
    // stream in chunks); created on first use
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaStream_t copy_in() {
        if (!cin) MSK_CUDA(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking));
        return cin;
    }
    cudaStream_t copy_out() {
        if (!cout) MSK_CUDA(cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking));
        return cout;
    }
};

namespace {

struct LevelData {
    int64_t n = 0;
    double delta = 0, q = 0;
    Grid g{};
    double *xs = nullptr;          // d * n SoA, spatial order
    int32_t *perm = nullptr;       // spatial -> caller
    int32_t *cell_start = nullptr; // ncells + 1
    int32_t *cnt = nullptr;        // A_l row counts (spatial order)
    int64_t nnz = 0;
    int64_t *row_ptr = nullptr;
    int32_t *col = nullptr;
    double *val = nullptr;
    double *alpha = nullptr;       // coefficients of the last solve, spatial order
    double4 *rec = nullptr;        // packed (coords, coefficient) records for gathers
    float4 *frec = nullptr;        // FP32 coordinates relative to lo (gather prefilter)
    float fthr = 0.f;              // prefilter threshold
};

thread_local std::string g_err;

void set_err(const std::string &s) { g_err = s; }

template <typename T>
T *dalloc(size_t count, cudaStream_t st) {
    T *p = nullptr;
    if (count == 0) count = 1;
    MSK_CUDA(cudaMallocAsync((void **)&p, sizeof(T) * count, st));
    return p;
}

void dfree(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// A device view of a caller buffer: the buffer itself if it is device memory,
// else a stream-ordered device copy.
struct DevBuf {
    const double *ptr = nullptr;
    double *owned = nullptr;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    const double *src = nullptr;  // deferred copy: host source (copy_async)
    size_t count = 0;
    DevBuf(const double *p, size_t c, cudaStream_t s, bool defer = false) : st(s), count(c) {
        if (is_device_ptr(p)) {
            ptr = p;
        } else {
            owned = dalloc<double>(c, s);
            if (defer) src = p;
            else if (c) MSK_CUDA(cudaMemcpyAsync(owned, p, sizeof(double) * c, cudaMemcpyHostToDevice, s));
            ptr = owned;
        }
    }
    // the deferred host->device copy on copy stream cs (after the allocation on st is ordered)
    void copy_async(cudaStream_t cs) {
        if (src && count)
            MSK_CUDA(cudaMemcpyAsync(owned, src, sizeof(double) * count, cudaMemcpyHostToDevice, cs));
        src = nullptr;
    }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : ptr(o.ptr), owned(o.owned), st(o.st), src(o.src), count(o.count) {
        o.owned = nullptr;
    }
    ~DevBuf() { dfree(owned, st); }
};

// A device output for a caller buffer; flush() copies back when it is host memory.
struct DevOut {
    double *ptr = nullptr;
    double *host = nullptr;
    size_t count = 0;
    cudaStream_t st = nullptr;
    DevOut() = default;
    DevOut(double *p, size_t c, cudaStream_t s) : count(c), st(s) {
        if (is_device_ptr(p)) {
            ptr = p;
        } else {
            host = p;
            ptr = dalloc<double>(c, s);
        }
    }
    DevOut(const DevOut &) = delete;
    DevOut &operator=(const DevOut &) = delete;
    bool flushed = false;
    DevOut(DevOut &&o) noexcept : ptr(o.ptr), host(o.host), count(o.count), st(o.st), flushed(o.flushed) {
        o.host = nullptr;
    }
    void flush() {
        if (host && count && !flushed)
            MSK_CUDA(cudaMemcpyAsync(host, ptr, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
        flushed = true;
    }
    // device->host copy on copy stream cs once `ready` (recorded on st) has fired
    void flush_async(cudaStream_t cs, cudaEvent_t ready) {
        if (host && count && !flushed) {
            MSK_CUDA(cudaStreamWaitEvent(cs, ready, 0));
            MSK_CUDA(cudaMemcpyAsync(host, ptr, sizeof(double) * count, cudaMemcpyDeviceToHost, cs));
        }
        flushed = true;
    }
    ~DevOut() {
        if (host) dfree(ptr, st);
    }
};

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    explicit Timer(cudaStream_t s) : st(s) {
        MSK_CUDA(cudaEventCreate(&a));
        MSK_CUDA(cudaEventCreate(&b));
    }
    void start() { MSK_CUDA(cudaEventRecord(a, st)); }
    void stop() { MSK_CUDA(cudaEventRecord(b, st)); }
    double ms() {  // after a stream synchronisation
        float t = 0;
        MSK_CUDA(cudaEventElapsedTime(&t, a, b));
        return t;
    }
    ~Timer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

// On scope exit (also when an error unwinds the call), wait for the copy
// streams: their transfers touch buffers that are freed on the compute stream.
struct CopyStreamsGuard {
    cudaStream_t a = nullptr, b = nullptr;
    ~CopyStreamsGuard() {
        if (a) cudaStreamSynchronize(a);
        if (b) cudaStreamSynchronize(b);
    }
};

// a synchronisation-only event
struct Ev {
    cudaEvent_t e = nullptr;
    Ev() { MSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
    Ev(const Ev &) = delete;
    Ev &operator=(const Ev &) = delete;
    ~Ev() { if (e) cudaEventDestroy(e); }
    void record(cudaStream_t s) { MSK_CUDA(cudaEventRecord(e, s)); }
    void wait_on(cudaStream_t s) { MSK_CUDA(cudaStreamWaitEvent(s, e, 0)); }
};

#define API_BEGIN try {
#define API_END                                                  \
    return MSK_OK;                                               \
    }                                                            \
    catch (const msk::Error &e) {                                \
        set_err(e.what());                                       \
        return (msk_status)e.status;                             \
    }                                                            \
    catch (const std::bad_alloc &) {                             \
        set_err("host allocation failed");                       \
        return MSK_ERR_NOMEM;                                    \
    }                                                            \
    catch (const std::exception &e) {                            \
        set_err(e.what());                                       \
        return MSK_ERR_CUDA;                                     \
    }

void require(bool ok, const std::string &msg) {
    if (!ok) throw Error(MSK_ERR_INVALID, msg);
}

}  // namespace

struct msk_hierarchy {
    msk_ctx *ctx = nullptr;
    int d = 0, L = 0, k = 0;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    LevelData lev[kMaxLevels];
    bool assembled = false, solved = false;
    int64_t ntot = 0;
    int64_t off[kMaxLevels + 1] = {0};
    double *ws = nullptr;  // CG workspace: r, p, q, beta, t (5 * ntot)
    // multi-RHS solve (msk_solve_multi): coefficients of all right-hand sides,
    // spatial order; per level one contiguous [n(l)][R] block per column group
    double *alpham[kMaxLevels] = {nullptr};
    int nrhs_m = 0, nrhs_pad = 0;
    std::vector<int> grp0, grpR, grpP;  // caller column, width R, padded column of each group
    double t_create_ms = 0, t_assemble_ms = 0;
    int launches_create = 0, launches_assemble = 0;
    // thresholded factor M~(T) (a6): one CSR over all points (rows of level 1
    // are empty), global level-major spatial column indices
    double T = 0.0;
    int64_t tnnz = 0;
    int64_t *trow_ptr = nullptr;
    int32_t *tcol = nullptr;
    double *tval = nullptr;
    int lagrange_max_iters = 0;
    int patch_max_points = 0;
    double t_lagrange_ms = 0;
    // distributed solve: per level, the row partition and this process's
    // partitions (one per rank over NCCL, all of them in the emulation)
    uint32_t flags = 0;
    struct PartLocal {
        int rank = 0;
        int64_t lo = 0, hi = 0, c0 = 0, c1 = 0, nnz = 0;
        int64_t *rp = nullptr;   // owned rows' CSR (local entries, global columns)
        int32_t *col = nullptr;
        double *val = nullptr;
        int64_t hlo = 0, hhi = 0;  // columns referenced by the owned rows: [hlo, hhi)
    };
    struct LevelDist {
        bool on = false;
        std::vector<int64_t> rows;       // world + 1 row bounds
        std::vector<int64_t> hlo, hhi;   // per rank
        std::vector<PartLocal> local;
    };
    LevelDist dist[kMaxLevels];

    void release_dist() {
        cudaStream_t s = st();
        for (int l = 0; l < kMaxLevels; ++l) {
            for (auto &P : dist[l].local) { dfree(P.rp, s); dfree(P.col, s); dfree(P.val, s); }
            dist[l] = LevelDist();
        }
    }

    void release_factor() {
        cudaStream_t s = st();
        dfree(trow_ptr, s); dfree(tcol, s); dfree(tval, s);
        trow_ptr = nullptr; tcol = nullptr; tval = nullptr;
        tnnz = 0;
        T = 0.0;
    }

    cudaStream_t st() const { return ctx->stream; }

    LevelView view(int l, const double *coef = nullptr) const {
        const LevelData &D = lev[l];
        LevelView v{};
        v.n = D.n;
        for (int a = 0; a < 3; ++a) v.x[a] = a < d ? D.xs + (size_t)a * D.n : nullptr;
        v.cell_start = D.cell_start;
        v.g = D.g;
        v.delta2 = D.delta * D.delta;
        v.inv_delta = 1.0 / D.delta;
        v.scale = pow(D.delta, -(double)d);
        v.coef = coef;
        v.rec = D.rec;
        v.frec = D.frec;
        v.fthr = D.fthr;
        return v;
    }

    // pack level l's coordinates with coefficient vector coef (spatial order)
    void pack(int l, const double *coef, int *launches) {
        LevelData &D = lev[l];
        if (!D.rec) D.rec = dalloc<double4>((size_t)D.n, st());
        pack_records(D.n, d, D.xs, coef, D.rec, st(), launches);
    }

    void ensure_ws() {
        if (!ws) ws = dalloc<double>((size_t)(5 * ntot), st());
    }
    double *ws_r(int l) { return ws + off[l]; }
    double *ws_p(int l) { return ws + ntot + off[l]; }
    double *ws_q(int l) { return ws + 2 * ntot + off[l]; }
    double *ws_beta(int l) { return ws + 3 * ntot + off[l]; }
    double *ws_t(int l) { return ws + 4 * ntot + off[l]; }

    void release() {
        cudaStream_t s = st();
        for (int l = 0; l < L; ++l) {
            LevelData &D = lev[l];
            dfree(D.xs, s); dfree(D.perm, s); dfree(D.cell_start, s); dfree(D.cnt, s);
            dfree(D.row_ptr, s); dfree(D.col, s); dfree(D.val, s); dfree(D.alpha, s); dfree(D.rec, s); dfree(D.frec, s);
            D = LevelData();
        }
        dfree(ws, s);
        ws = nullptr;
        release_multi();
        release_factor();
        release_dist();
    }
    void release_multi() {
        for (int l = 0; l < kMaxLevels; ++l) {
            dfree(alpham[l], st());
            alpham[l] = nullptr;
        }
        nrhs_m = nrhs_pad = 0;
        grp0.clear(); grpR.clear(); grpP.clear();
    }
};

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
        require((flags & ~(MSK_FLAG_DIST_ALL | MSK_FLAG_MATRIX_FREE)) == 0, "msk_hierarchy_create: unknown flags");
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
            for (;;) {
                Grid g{};
                g.inv_cell = 1.0 / cell;
                g.ncells = 1;
                for (int a = 0; a < 3; ++a) {
                    g.lo[a] = a < d ? h->lo[a] : 0.0;
                    g.dim[a] = a < d ? (int64_t)floor((h->hi[a] - h->lo[a]) * g.inv_cell) + 1 : 1;
                    g.ncells *= g.dim[a];
                }
                // bound the cell count (points much sparser than delta): larger
                // cells only add candidates, never lose neighbours
                if (g.ncells <= 8 * n[l] + 4096) {
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
            count_pattern(d, v, v, true, D.cnt, minr2[l], st, &launches);
        }
        h->ntot = h->off[L];
        std::vector<unsigned long long> mr(L);
        for (int l = 0; l < L; ++l)
            MSK_CUDA(cudaMemcpyAsync(&mr[l], minr2[l], sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        tm.stop();
        MSK_CUDA(cudaStreamSynchronize(st));
        for (int l = 0; l < L; ++l) {
            dfree(minr2[l], st);
            double r2;
            memcpy(&r2, &mr[l], sizeof r2);
            require(r2 > 0.0, "msk_hierarchy_create: duplicate points in level " + std::to_string(l));
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
        for (int l = 0; l < k; ++l) {
            a.lev[l] = h->view(l);
            const double R = T * h->lev[l].q;
            a.R2[l] = R * R;
            a.reach[l] = (int)std::min(floor(R * h->lev[l].g.inv_cell) + 1.0, 1e6);
            a.col_off[l] = h->off[l];
        }
        return a;
    };
    for (int k = 1; k < L; ++k) {
        ThreshPatternArgs a = pattern_args(k);
        a.cnt = cnt + h->off[k];
        thresh_count(a, st, launches);
    }
    h->trow_ptr = dalloc<int64_t>((size_t)(ntot + 1), st);
    exclusive_scan_i64(cnt, ntot, h->trow_ptr, st, launches);
    int64_t nnz = 0;
    MSK_CUDA(cudaMemcpyAsync(&nnz, h->trow_ptr + ntot, sizeof nnz, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(cnt, st);
    h->tnnz = nnz;
    h->tcol = dalloc<int32_t>((size_t)nnz, st);
    h->tval = dalloc<double>((size_t)nnz, st);
    for (int k = 1; k < L; ++k) {
        ThreshPatternArgs a = pattern_args(k);
        a.row_ptr = h->trow_ptr + h->off[k];
        a.col = h->tcol;
        thresh_fill(a, st, launches);
    }
    // ---- transpose index over the coarse columns (levels 0..L-2)
    const int64_t ncols = h->off[L - 1];
    int64_t *cptr = dalloc<int64_t>((size_t)(ncols + 1), st);
    int64_t *cpos = dalloc<int64_t>((size_t)nnz, st);
    int32_t *crow = dalloc<int32_t>((size_t)nnz, st);
    int32_t *ccol = nullptr;  // columns are found by binary search in cptr (saves 4 B per entry)
    thresh_csc(ntot - h->off[1], h->off[1], nnz, ncols, h->trow_ptr, h->tcol, cptr, cpos, crow, ccol, st,
               launches);
    std::vector<int64_t> hcptr((size_t)(ncols + 1));
    MSK_CUDA(cudaMemcpyAsync(hcptr.data(), cptr, sizeof(int64_t) * (ncols + 1), cudaMemcpyDeviceToHost, st));
    int *dstat = dalloc<int>(2, st);
    MSK_CUDA(cudaMemsetAsync(dstat, 0, 2 * sizeof(int), st));
    int *pstat = dalloc<int>(5, st);  // patch path: CG failures, overflows, max iterations, max patch, count
    MSK_CUDA(cudaMemsetAsync(pstat, 0, 5 * sizeof(int), st));
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
            patch_count(pa, pstat + 4, st);
            std::vector<int32_t> hc((size_t)D.n);
            int hp = 0;
            MSK_CUDA(cudaMemcpyAsync(&hp, pstat + 4, sizeof hp, cudaMemcpyDeviceToHost, st));
            MSK_CUDA(cudaMemcpyAsync(hc.data(), D.cnt, sizeof(int32_t) * (size_t)D.n, cudaMemcpyDeviceToHost, st));
            MSK_CUDA(cudaStreamSynchronize(st));
            const int maxrow = D.n ? *std::max_element(hc.begin(), hc.end()) : 0;
            if (getenv("MSK_DEBUG_PATCH"))
                fprintf(stderr, "[msk] patch level %d: n %lld q %.6g rho %.6g reach %d cell %.6g pmax %d maxrow %d\n", l,
                        (long long)D.n, D.q, rho, pa.reach, 1.0 / D.g.inv_cell, hp, maxrow);
            pa.pmax = hp;
            pa.nnzmax = (int)std::min<int64_t>((int64_t)hp * maxrow, (int64_t)hp * hp);
            const size_t smem = patch_smem_bytes(pa.pmax, pa.nnzmax);
            // larger patches run from a global workspace (patch_lagrange); bound it
            if (smem > (size_t)1 << 30)
                throw Error(MSK_ERR_INVALID, "msk_assemble: local patch too large (" + std::to_string(hp) +
                                                 " points); reduce patch_R");
            patch_lagrange(pa, smem, st, launches);
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
            thresh_cg_multi(m, (int)nb, st, launches);
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
            thresh_values(v, st, launches);
        }
        dfree(ws, st);
    }
    int hstat[2], hps[5];
    MSK_CUDA(cudaMemcpyAsync(hstat, dstat, sizeof hstat, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaMemcpyAsync(hps, pstat, sizeof hps, cudaMemcpyDeviceToHost, st));
    MSK_CUDA(cudaStreamSynchronize(st));
    dfree(dstat, st); dfree(pstat, st); dfree(cptr, st); dfree(cpos, st); dfree(crow, st); dfree(ccol, st);
    h->lagrange_max_iters = std::max(hstat[1], hps[2]);
    h->patch_max_points = hps[3];
    h->T = T;
    if (hstat[0]) throw Error(MSK_ERR_NOCONV, "msk_assemble: Lagrange CG did not converge in 20000 iterations");
    if (hps[1]) throw Error(MSK_ERR_INVALID, "msk_assemble: local patch overflow in " + std::to_string(hps[1]) +
                                                 " columns; reduce patch_R");
    if (hps[0]) throw Error(MSK_ERR_NOCONV, "msk_assemble: patch Lagrange CG did not converge in " +
                                                std::to_string(hps[0]) + " columns");
}

}  // namespace

extern "C" msk_status msk_assemble_ex(msk_hierarchy *h, double T, double lagrange_tol, double patch_R,
                                      int64_t patch_min_n) {
    API_BEGIN
    require(std::isfinite(patch_R) && patch_min_n >= 0, "msk_assemble_ex: bad patch arguments");
    require(h != nullptr, "msk_assemble: NULL hierarchy");
    require(std::isfinite(T), "msk_assemble: T must be finite");
    require(!(T > 0.0) || (lagrange_tol > 0.0 && lagrange_tol < 1.0),
            "msk_assemble: lagrange_tol must be in (0,1) when T > 0");
    require(!(T > 0.0) || h->ctx->world == 1, "msk_assemble: the thresholded factor is single-GPU in this version");
    require(!(T > 0.0) || !(h->flags & MSK_FLAG_MATRIX_FREE),
            "msk_assemble: the thresholded factor needs assembled A_l (hierarchy is MSK_FLAG_MATRIX_FREE)");
    const bool mf = (h->flags & MSK_FLAG_MATRIX_FREE) != 0;
    MSK_CUDA(cudaSetDevice(h->ctx->device));
    cudaStream_t st = h->st();
    h->release_factor();
    h->release_dist();
    Timer tm(st);
    tm.start();
    int launches = 0;
    std::vector<int64_t> nnz(h->L);
    // distributed context: partition the large levels
    const int W = h->ctx->world;
    for (int l = 0; l < h->L && W > 1; ++l) {
        const int64_t n = h->lev[l].n;
        const int64_t rpc = (int64_t)cg_chunk_tiles(n) * 256;
        const int64_t nch = (n + rpc - 1) / rpc;
        if (nch >= W && ((h->flags & MSK_FLAG_DIST_ALL) || n >= (1ll << 20))) {
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
        dfree(D.row_ptr, st); dfree(D.col, st); dfree(D.val, st);
        D.row_ptr = nullptr; D.col = nullptr; D.val = nullptr;
        nnz[l] = 0;
        if (h->dist[l].on) {  // owned rows only, per local partition
            for (auto &P : h->dist[l].local) {
                const int64_t m = P.hi - P.lo;
                P.rp = dalloc<int64_t>((size_t)(m + 3), st);
                MSK_CUDA(cudaMemsetAsync(P.rp + m + 1, 0, 2 * sizeof(int64_t), st));
                exclusive_scan_i64(D.cnt + P.lo, m, P.rp, st, &launches);
                MSK_CUDA(cudaMemcpyAsync(&P.nnz, P.rp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            }
            continue;
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
    }
    if (T > 0.0 && h->L > 1) build_factor(h, T, lagrange_tol, patch_R, patch_min_n, &launches);
    tm.stop();
    MSK_CUDA(cudaStreamSynchronize(st));
    h->t_assemble_ms = tm.ms();
    h->launches_assemble = launches;
    h->assembled = true;
    API_END
}

extern "C" msk_status msk_assemble(msk_hierarchy *h, double T, double lagrange_tol) {
    return msk_assemble_ex(h, T, lagrange_tol, 0.0, 0);
}

// =================================================================== solve
namespace {

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
    auto dist_level = [&](int l, double tl) {
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
        for (int i = 0; i < np; ++i) {
            if (emu) {
                double *blk = dalloc<double>((size_t)(4 * n), st);
                owned_alloc.push_back(blk);
                X[i] = blk; R[i] = blk + n; Pv[i] = blk + 2 * n; Q[i] = blk + 3 * n;
            } else {
                X[i] = h->ws_t(l); R[i] = h->ws_r(l); Pv[i] = h->ws_p(l); Q[i] = h->ws_q(l);
            }
            send[i] = dalloc<double>((size_t)nch, st);
            MSK_CUDA(cudaMemsetAsync(send[i], 0, sizeof(double) * (size_t)nch, st));
        }
        // beta^(l) on the owned rows (B products of the coarser, complete levels)
        if (l > 0) {
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
            A.L.nnz = P.nnz;
            A.L.chunk_tiles = CH;
            A.c0 = P.c0;
            A.c1 = P.c1;
            A.nchunks = nch;
            A.part_send = send[i];
            A.part_recv = part ? recv : send[i];  // one partition: nothing to reduce
            A.sc = sc + i;
            if (i == 0) set_coef(A.L, l);
        }
        auto allreduce = [&]() {
            if (!part) return;
            if (emu) {
                DistPtrs ptrs{};
                for (int i = 0; i < np; ++i) ptrs.p[i] = send[i];
                sum_arrays(np, ptrs, recv, nch, st);
            } else {
                MSK_NCCL(nccl_api()->AllReduce(send[0], recv, (size_t)nch, ncclFloat64, ncclSum, h->ctx->comm, st));
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
            MSK_CUDA(cudaMemcpyAsync(alpha_sp[l], X[0], sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
        } else if (emu) {
            for (int i = 0; i < np; ++i) {
                const auto &P = parts[i];
                MSK_CUDA(cudaMemcpyAsync(alpha_sp[l] + P.lo, X[i] + P.lo, sizeof(double) * (size_t)(P.hi - P.lo),
                                         cudaMemcpyDeviceToDevice, st));
            }
        } else {
            const auto &P = Dd.local[0];
            double *tmp = Q[0];
            MSK_CUDA(cudaMemsetAsync(tmp, 0, sizeof(double) * (size_t)n, st));
            MSK_CUDA(cudaMemcpyAsync(tmp + P.lo, X[0] + P.lo, sizeof(double) * (size_t)(P.hi - P.lo),
                                     cudaMemcpyDeviceToDevice, st));
            MSK_NCCL(nccl_api()->AllReduce(tmp, alpha_sp[l], (size_t)n, ncclFloat64, ncclSum, h->ctx->comm, st));
        }
        permute_scatter(n, alpha_sp[l], D.perm, ad[l].ptr, st, &launches);
        MSK_CUDA(cudaMemcpyAsync(d_it + l, &sc->it, sizeof(int), cudaMemcpyDeviceToDevice, st));
        MSK_CUDA(cudaMemcpyAsync(d_stat + l, &sc->status, sizeof(int), cudaMemcpyDeviceToDevice, st));
        MSK_CUDA(cudaMemcpyAsync(d_rr + 2 * l, &sc->rr, sizeof(double), cudaMemcpyDeviceToDevice, st));
        MSK_CUDA(cudaMemcpyAsync(d_rr + 2 * l + 1, &sc->bb, sizeof(double), cudaMemcpyDeviceToDevice, st));
        for (double *p : owned_alloc) dfree(p, st);
        for (double *p : send) dfree(p, st);
        dfree(recv, st);
        dfree(sc, st);
    };
    bool any_dist = false;
    for (int l = 0; l < L; ++l) any_dist = any_dist || h->dist[l].on;
    require(!any_dist || schedule == MSK_SCHED_PRUNED, "msk_solve: a distributed solve uses the PRUNED schedule");
    require(!mf || schedule == MSK_SCHED_PRUNED, "msk_solve: a matrix-free hierarchy uses the PRUNED schedule");

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
            for (int k = 1; k < L; ++k)
                thresh_residual(h->off[k], h->off[k + 1], h->trow_ptr, h->tcol, h->tval, beta, beta, beta, st,
                                &launches);
            ga_t.back()->stop();
        } else {
            double *cur = h->ws_beta(0), *nxt = h->ws_t(0);
            MSK_CUDA(cudaMemcpyAsync(cur, fsp, sizeof(double) * h->ntot, cudaMemcpyDeviceToDevice, st));
            MSK_CUDA(cudaMemcpyAsync(nxt, fsp, sizeof(double) * h->ntot, cudaMemcpyDeviceToDevice, st));
            time_ga();
            for (int sweep = 0; sweep < L; ++sweep) {
                thresh_residual(h->off[1], h->ntot, h->trow_ptr, h->tcol, h->tval, fsp, cur, nxt, st, &launches);
                std::swap(cur, nxt);
            }
            ga_t.back()->stop();
            beta = cur;
        }
        std::vector<CGLevelArgs> a;
        for (int l = 0; l < L; ++l) {
            a.push_back(cg_args(h, l, tol, max_iter, beta + h->off[l], nullptr, alpha_sp[l], ad[l].ptr,
                                d_it + l, d_rr + 2 * l, d_stat + l));
            set_coef(a.back(), l);
        }
        time_cg(-1);
        cg_batched(a.data(), L, st, &launches);
        cg_t.back()->stop();
    } else if (schedule == MSK_SCHED_PRUNED) {
        // Algorithm 2 with every inner solve done once, when its input is final:
        // beta^(l) = f^(l) - sum_{k<l} B_lk t^(k); t^(l) = A_l^{-1} beta^(l);
        // alpha^(l) = t^(l) (the final block CG of a converged block is the
        // same solve); the finest level is solved at tol.
        for (int l = 0; l < L; ++l) {
            const double tl = l + 1 < L ? inner_tol : tol;
            wait_f(l);
            if (h->dist[l].on || mf) {
                dist_level(l, tl);
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
                    a.push_back(cg_args(h, l, inner_tol, max_iter, h->ws_beta(l), nullptr, t_sp[l], nullptr,
                                        d_it + sweep * L + l, d_rr + 2 * (sweep * L + l), d_stat + sweep * L + l));
                    set_coef(a.back(), sweep * L + l);
                }
                time_cg(-1);
                cg_batched(a.data(), (int)a.size(), st, &launches);
                cg_t.back()->stop();
                for (int l = 0; l + 1 < L; ++l) h->pack(l, t_sp[l], &launches);
                for (int k = 1; k < L; ++k) b_products(k, t_sp.data(), h->ws_beta(k));
            }
        }
        std::vector<CGLevelArgs> a;
        for (int l = 0; l < L; ++l) {
            a.push_back(cg_args(h, l, tol, max_iter, h->ws_beta(l), nullptr, alpha_sp[l], ad[l].ptr,
                                d_it + L * L + l, d_rr + 2 * (L * L + l), d_stat + L * L + l));
            set_coef(a.back(), L * L + l);
        }
        time_cg(-1);
        cg_batched(a.data(), L, st, &launches);
        cg_t.back()->stop();
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
    if (thresholded) hits = (unsigned long long)(h->tnnz * (schedule == MSK_SCHED_LITERAL ? L : 1));
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
    int64_t chunk = 1 << 20;
    if (const char *e = getenv("MSK_EVAL_CHUNK")) chunk = std::max<int64_t>(256, atoll(e));  // test hook
    const int64_t nc = (m + chunk - 1) / chunk;
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
        const int64_t c0 = c * chunk, c1 = std::min(m, c0 + chunk), nck = c1 - c0;
        MSK_CUDA(cudaMemcpyAsync(xd + c0 * d, x + c0 * d, sizeof(double) * (size_t)(nck * d),
                                 cudaMemcpyHostToDevice, cin));
        ein[c].record(cin);
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t c0 = c * chunk, c1 = std::min(m, c0 + chunk), nck = c1 - c0;
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
    if (W > 1) MSK_CUDA(cudaMemsetAsync(sd.ptr, 0, sizeof(double) * (size_t)m, st));
    teval.start();
    for (int r = 0; r < W; ++r) {
        if (W > 1 && !h->ctx->emulated && r != h->ctx->rank) continue;
        const int64_t lo = m * r / W, hi = m * (r + 1) / W;
        GatherArgs ga{};
        ga.d = d;
        ga.k = h->k;
        ga.nt = hi - lo;
        for (int a = 0; a < d; ++a) ga.tx[a] = xs + (size_t)a * m + lo;
        ga.nlev = L;
        for (int l = 0; l < L; ++l) ga.lev[l] = h->view(l, h->lev[l].alpha);
        ga.base = nullptr;
        ga.sign = 1.0;
        ga.out = sd.ptr;
        ga.out_perm = perm + lo;
        ga.hits = d_hits;
        gather(ga, st, &launches);
    }
    if (W > 1 && !h->ctx->emulated)
        MSK_NCCL(nccl_api()->AllReduce(sd.ptr, sd.ptr, (size_t)m, ncclFloat64, ncclSum, h->ctx->comm, st));
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
    require(which == 0 || which == 1, "msk_m_norm: which must be 0 (M) or 1 (M - M~(T))");
    if (which == 1 && !(h->T > 0.0))
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
    if (which == 1) {
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
        // u = M v
        solve_coarse(v, t);
        MSK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * (size_t)h->lev[0].n, st));
        for (int l = 0; l + 1 < L; ++l) h->pack(l, t + h->off[l], nullptr);
        for (int k = 1; k < L; ++k) {
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
        if (which == 1) {  // u += X~ v  (thresh_residual: out = base - sum val * (-v))
            MSK_CUDA(cudaMemcpyAsync(nv, v, sizeof(double) * (size_t)N, cudaMemcpyDeviceToDevice, st));
            dev_scale(nv, -1.0, N, st);
            thresh_residual(h->off[1], N, h->trow_ptr, h->tcol, h->tval, u, nv, u, st, nullptr);
        }
        const double s_new = sqrt(dev_dot(u, u, N, scratch, st));
        // w = M^T u = -A^{-1} (B^T u) on the coarse levels, 0 on the finest
        for (int l = 0; l + 1 < L; ++l) {
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
        solve_coarse(t, w);
        MSK_CUDA(cudaMemsetAsync(w + h->off[L - 1], 0, sizeof(double) * (size_t)h->lev[L - 1].n, st));
        if (which == 1) csc_spmv_add(ncols, cptr, cpos, crow, h->tval, u, w, st);  // w += X~^T u
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

extern "C" msk_status msk_evaluate(msk_hierarchy *h, int64_t m, const double *x, double *s) {
    return msk_evaluate_ex(h, m, x, s, nullptr);
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
    if (np) {
        MSK_CUDA(cudaMemcpyAsync(hcl.data(), h->tcol + p0, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, st));
        MSK_CUDA(cudaMemcpyAsync(hvl.data(), h->tval + p0, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
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
            if (hcl[p] >= c_lo && hcl[p] < c_hi) tmp.emplace_back(cperm[hcl[p] - c_lo], hvl[p]);
        std::sort(tmp.begin(), tmp.end());
        for (auto &e : tmp) {
            if (col) col[pos] = e.first;
            if (val) val[pos] = e.second;
            ++pos;
        }
    }
    row_ptr[nr] = pos;
    if (T_out) *T_out = h->T;
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

extern "C" const char *msk_last_error(void) { return g_err.c_str(); }

extern "C" const char *msk_version(void) { return "libmsk 0.1 (sm_100a, FP64)"; }

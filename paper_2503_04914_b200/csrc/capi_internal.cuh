// capi_internal.cuh -- state and helpers shared by the C-ABI translation units
// (capi.cu: context, hierarchy, assembly, exports; capi_solve.cu: solve and
// evaluation; capi_extra.cu: multi-RHS, diagnostics, row-level entry points).
#pragma once
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
// Peer-memory buffers for k_pcg on separate GPUs, one set per level index:
// this rank's r, chunk partials, result and barrier counters (cudaMalloc,
// exported by IPC handle) and every rank's as mapped in this process.  They
// live in the CONTEXT and are reused by every hierarchy of the context (grown
// collectively when a level needs more), so a create/solve/destroy cycle
// pays no allocation or IPC mapping; the counters keep counting across solves.
struct PeerMem {
    bool tried = false, ok = false;
    int64_t ncap = 0, chcap = 0;  // capacities: rows, chunk partials (3 x chcap)
    double *r = nullptr, *part = nullptr, *alpha = nullptr;
    unsigned long long *cnt = nullptr;  // xcnt, nbar, gbar
    std::vector<double *> pr, ppart, palpha;
    std::vector<unsigned long long *> pcnt;
    std::vector<void *> opened;  // IPC-opened peer bases (closed on release)
    void release() {
        for (void *p : opened) cudaIpcCloseMemHandle(p);
        if (r) cudaFree(r);
        if (part) cudaFree(part);
        if (alpha) cudaFree(alpha);
        if (cnt) cudaFree(cnt);
        *this = PeerMem();
    }
};

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
    PeerMem peer[16];  // by level index (kMaxLevels)
};

namespace capi {

struct LevelData {
    int64_t n = 0;
    double delta = 0, q = 0;
    Grid g{};
    double *xs = nullptr;          // d * n SoA, spatial order
    int32_t *perm = nullptr;       // spatial -> caller
    int32_t *cell_start = nullptr; // ncells + 1
    int32_t *cnt = nullptr;        // A_l row counts (spatial order), valid on rows [cnt_lo, cnt_hi)
    int64_t cnt_lo = 0, cnt_hi = 0;
    int64_t nnz = 0;
    int64_t *row_ptr = nullptr;
    int32_t *col = nullptr;
    double *val = nullptr;
    uint16_t *col16 = nullptr;     // 16-bit columns for k_cg (cg.cu col16_build), or null
    int4 *cbase = nullptr;         //   their window bases per reduction chunk
    int4 *clen = nullptr;          //   and the extents (k_cg's L2 prefetch of the gathered r)
    double *alpha = nullptr;       // coefficients of the last solve, spatial order
    double4 *rec = nullptr;        // packed (coords, coefficient) records for gathers
    float4 *frec = nullptr;        // FP32 coordinates relative to lo (gather prefilter)
    float fthr = 0.f;              // prefilter threshold
};

extern thread_local std::string g_err;

inline void set_err(const std::string &s) { g_err = s; }

template <typename T>
T *dalloc(size_t count, cudaStream_t st) {
    T *p = nullptr;
    if (count == 0) count = 1;
    MSK_CUDA(cudaMallocAsync((void **)&p, sizeof(T) * count, st));
    return p;
}

inline void dfree(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

inline bool is_device_ptr(const void *p) {
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

#define API_BEGIN                          \
    ::msk::NvtxRange msk_nvtx_api_(__func__); \
    try {
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

inline void require(bool ok, const std::string &msg) {
    if (!ok) throw Error(MSK_ERR_INVALID, msg);
}

}  // namespace capi

using namespace capi;

// warp-scan broadcast limit (wscan.cuh): MSK_WS_BR x 3^d cells (default 2.5)
inline float ws_bcells(int d) {
    static const double br = getenv("MSK_WS_BR") ? atof(getenv("MSK_WS_BR")) : 2.5;
    return (float)(br * (d == 3 ? 27.0 : 9.0));
}

struct msk_hierarchy {
    msk_ctx *ctx = nullptr;
    int d = 0, L = 0, k = 0;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    LevelData lev[kMaxLevels];
    bool assembled = false, solved = false;
    bool part_on[kMaxLevels] = {false};  // distributed context: level partitioned in row blocks
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
    // T sweep (msk_set_threshold): per-entry distance bucket (smallest integer t with
    // r^2 < (t q_l)^2); entries with bucket > tmax_active are left out
    uint8_t *tbucket = nullptr;
    int tmax_active = 255;
    double T_active = 0.0;
    int64_t tnnz_active = 0;
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
        dfree(trow_ptr, s); dfree(tcol, s); dfree(tval, s); dfree(tbucket, s);
        trow_ptr = nullptr; tcol = nullptr; tval = nullptr; tbucket = nullptr;
        tnnz = 0;
        T = 0.0;
        T_active = 0.0;
        tmax_active = 255;
        tnnz_active = 0;
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
        v.bcells = ws_bcells(d);
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
            dfree(D.col16, s); dfree(D.cbase, s); dfree(D.clen, s);
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


// solve helpers (capi_solve.cu) used by other translation units
namespace capi {
CGLevelArgs cg_args(msk_hierarchy *h, int l, double tol, int max_iter, const double *b, const double *b_src,
                    double *x, double *x_out, int *d_iters, double *d_rr, int *d_status);
double cg_bytes(const LevelData &D, int iters);
double lanczos_kappa(const double *coef, int m);
}  // namespace capi

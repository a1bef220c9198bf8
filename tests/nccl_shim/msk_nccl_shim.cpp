// msk_nccl_shim.cpp -- TEST INFRASTRUCTURE.  An in-process stand-in for the
// subset of the NCCL API libmsk calls (nccl_dl.cuh), for ranks that are
// THREADS of one process.  libmsk picks it up through MSK_NCCL_LIBRARY.
//
// Purpose: run libmsk's rank >= 0 code path (one msk_ctx per rank, halo plans
// from the all-gathered column ranges, grouped send/recv of r halos,
// zero-filled all-reduces of chunk partials, alpha, beta and s_L) on a single
// GPU, with the transport replaced by host-staged copies.  It checks what a
// real NCCL job would deadlock or corrupt on: every rank must issue the same
// sequence of collectives with the same counts and types, and every receive
// must match a send of the same length from the named peer.
//
// Semantics: each call synchronises the caller's stream, stages its send data
// in host memory, waits for its peers' contributions and writes its receive
// buffer before returning (stronger than NCCL's stream ordering, so any
// program correct under NCCL is correct here).  All-reduce sums in rank order
// in the datatype (libmsk's all-reduces are zero-filled, so the order does
// not matter for its results).  Deadlocks are turned into errors after
// MSK_SHIM_TIMEOUT_S seconds (default 120).
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <tuple>
#include <vector>

namespace {

struct Contribution {
    int kind = 0;  // 1 all-reduce, 2 all-gather
    size_t count = 0;
    ncclDataType_t dt = ncclFloat64;
    ncclRedOp_t op = ncclSum;
    std::vector<char> data;
};

struct Collective {
    std::vector<Contribution> from;  // per rank
    int posted = 0, consumed = 0;
};

struct Group {
    int n = 0;
    std::mutex m;
    std::condition_variable cv;
    int joined = 0;
    std::map<long, Collective> coll;                                  // by collective sequence number
    std::map<std::pair<int, int>, std::deque<std::vector<char>>> box;  // (src, dst) -> messages
};

struct Comm {
    Group *g;
    int rank;
    long seq = 0;  // collectives issued by this rank
};

// calls served, by kind: all-reduce, all-gather, send, recv, comm init
std::atomic<long> g_stats[5];

std::mutex g_reg_m;
std::map<std::string, Group *> g_reg;

struct PendingP2P {
    bool send;
    const void *sbuf;
    void *rbuf;
    size_t bytes;
    int peer;
    Comm *comm;
    cudaStream_t st;
};
thread_local int t_group_depth = 0;
thread_local std::vector<PendingP2P> t_pending;

size_t dt_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
        default: return 0;
    }
}

std::chrono::seconds timeout() {
    const char *s = std::getenv("MSK_SHIM_TIMEOUT_S");
    return std::chrono::seconds(s ? std::atoi(s) : 120);
}

ncclResult_t fail(const char *what) {
    std::fprintf(stderr, "msk_nccl_shim: %s\n", what);
    return ncclInvalidUsage;
}

bool cuda_ok(cudaError_t e) {
    if (e == cudaSuccess) return true;
    std::fprintf(stderr, "msk_nccl_shim: CUDA error %s\n", cudaGetErrorString(e));
    return false;
}

// Stream-ordered copy on the rank's stream, complete on return (a plain
// cudaMemcpy from pageable memory may return before its DMA lands, and does
// not order against non-blocking streams).
bool copy_sync(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (!bytes) return true;
    return cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st)) && cuda_ok(cudaStreamSynchronize(st));
}

template <class T>
void sum_into(std::vector<char> &acc, const std::vector<char> &x) {
    T *a = reinterpret_cast<T *>(acc.data());
    const T *b = reinterpret_cast<const T *>(x.data());
    for (size_t i = 0; i < acc.size() / sizeof(T); ++i) a[i] += b[i];
}

ncclResult_t collective(Comm *c, int kind, const void *send, void *recv, size_t count, ncclDataType_t dt,
                        ncclRedOp_t op, cudaStream_t st) {
    const size_t es = dt_size(dt);
    if (!es) return fail("unsupported datatype");
    if (kind == 1 && op != ncclSum) return fail("only ncclSum is implemented");
    g_stats[kind - 1]++;
    Contribution me;
    me.kind = kind;
    me.count = count;
    me.dt = dt;
    me.op = op;
    me.data.resize(count * es);
    if (!copy_sync(me.data.data(), send, count * es, st)) return ncclUnhandledCudaError;
    Group *g = c->g;
    const long seq = c->seq++;
    std::vector<char> out;
    {
        std::unique_lock<std::mutex> l(g->m);
        Collective &C = g->coll[seq];
        if (C.from.empty()) C.from.resize(g->n);
        C.from[c->rank] = std::move(me);
        ++C.posted;
        g->cv.notify_all();
        if (!g->cv.wait_for(l, timeout(), [&] { return C.posted == g->n; }))
            return fail("collective timed out (a peer issued fewer collectives)");
        for (int r = 0; r < g->n; ++r) {
            const Contribution &x = C.from[r];
            if (x.kind != kind || x.count != count || x.dt != dt || x.op != op)
                return fail("mismatched collective across ranks (kind, count, datatype or op)");
        }
        if (kind == 1) {
            out = C.from[0].data;
            for (int r = 1; r < g->n; ++r) {
                if (dt == ncclFloat64) sum_into<double>(out, C.from[r].data);
                else if (dt == ncclFloat32) sum_into<float>(out, C.from[r].data);
                else if (dt == ncclInt64) sum_into<long long>(out, C.from[r].data);
                else if (dt == ncclUint64) sum_into<unsigned long long>(out, C.from[r].data);
                else if (dt == ncclInt32) sum_into<int>(out, C.from[r].data);
                else return fail("all-reduce datatype not implemented");
            }
        } else {
            out.resize(count * es * (size_t)g->n);
            for (int r = 0; r < g->n; ++r)
                if (count) std::memcpy(out.data() + (size_t)r * count * es, C.from[r].data.data(), count * es);
        }
        if (++C.consumed == g->n) g->coll.erase(seq);
    }
    if (!copy_sync(recv, out.data(), out.size(), st)) return ncclUnhandledCudaError;
    return ncclSuccess;
}

ncclResult_t run_p2p(std::vector<PendingP2P> &ops) {
    // sends first (staged, never block), then receives
    for (auto &o : ops) {
        if (!o.send) continue;
        if (o.peer < 0 || o.peer >= o.comm->g->n) return fail("send: bad peer");
        std::vector<char> msg(o.bytes);
        if (!copy_sync(msg.data(), o.sbuf, o.bytes, o.st)) return ncclUnhandledCudaError;
        Group *g = o.comm->g;
        std::lock_guard<std::mutex> l(g->m);
        g->box[{o.comm->rank, o.peer}].push_back(std::move(msg));
        g->cv.notify_all();
    }
    for (auto &o : ops) {
        if (o.send) continue;
        if (o.peer < 0 || o.peer >= o.comm->g->n) return fail("recv: bad peer");
        Group *g = o.comm->g;
        std::vector<char> msg;
        {
            std::unique_lock<std::mutex> l(g->m);
            auto &q = g->box[{o.peer, o.comm->rank}];
            if (!g->cv.wait_for(l, timeout(), [&] { return !q.empty(); }))
                return fail("recv timed out (no matching send from the peer)");
            msg = std::move(q.front());
            q.pop_front();
        }
        if (msg.size() != o.bytes) return fail("recv length differs from the matching send");
        if (!copy_sync(o.rbuf, msg.data(), o.bytes, o.st)) return ncclUnhandledCudaError;
    }
    return ncclSuccess;
}

ncclResult_t p2p(bool send, const void *sbuf, void *rbuf, size_t count, ncclDataType_t dt, int peer,
                 ncclComm_t comm, cudaStream_t st) {
    const size_t es = dt_size(dt);
    if (!es) return fail("unsupported datatype");
    g_stats[send ? 2 : 3]++;
    PendingP2P o{send, sbuf, rbuf, count * es, peer, reinterpret_cast<Comm *>(comm), st};
    if (t_group_depth > 0) {
        t_pending.push_back(o);
        return ncclSuccess;
    }
    std::vector<PendingP2P> one{o};
    return run_p2p(one);
}

}  // namespace

extern "C" {

// Test introspection (not an NCCL symbol): calls served since load.
void msk_shim_stats(long out[5]) {
    for (int i = 0; i < 5; ++i) out[i] = g_stats[i].load();
}

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
    std::random_device rd;
    std::memset(id, 0, sizeof *id);
    std::snprintf(id->internal, sizeof id->internal, "msk-shim-%08x%08x", rd(), rd());
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail("CommInitRank: bad rank / size");
    Group *g;
    {
        std::lock_guard<std::mutex> l(g_reg_m);
        Group *&slot = g_reg[std::string(id.internal, sizeof id.internal)];
        if (!slot) {
            slot = new Group();
            slot->n = nranks;
        }
        g = slot;
    }
    if (g->n != nranks) return fail("CommInitRank: ranks disagree on the size");
    std::unique_lock<std::mutex> l(g->m);
    ++g->joined;
    g->cv.notify_all();
    if (!g->cv.wait_for(l, timeout(), [&] { return g->joined >= g->n; }))
        return fail("CommInitRank timed out (not every rank joined)");
    *comm = reinterpret_cast<ncclComm_t>(new Comm{g, rank});
    g_stats[4]++;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete reinterpret_cast<Comm *>(comm);  // the group stays registered (test process lifetime)
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void *s, void *r, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
    return collective(reinterpret_cast<Comm *>(comm), 1, s, r, count, dt, op, st);
}

ncclResult_t ncclAllGather(const void *s, void *r, size_t count, ncclDataType_t dt, ncclComm_t comm,
                           cudaStream_t st) {
    return collective(reinterpret_cast<Comm *>(comm), 2, s, r, count, dt, ncclSum, st);
}

ncclResult_t ncclSend(const void *s, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t st) {
    return p2p(true, s, nullptr, count, dt, peer, comm, st);
}

ncclResult_t ncclRecv(void *r, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
    return p2p(false, nullptr, r, count, dt, peer, comm, st);
}

ncclResult_t ncclGroupStart() {
    ++t_group_depth;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (t_group_depth <= 0) return fail("GroupEnd without GroupStart");
    if (--t_group_depth > 0) return ncclSuccess;
    std::vector<PendingP2P> ops;
    ops.swap(t_pending);
    return run_p2p(ops);
}

const char *ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "no error";
        case ncclUnhandledCudaError: return "unhandled cuda error (shim)";
        case ncclInvalidUsage: return "invalid usage (shim: see stderr)";
        default: return "shim error";
    }
}

}  // extern "C"

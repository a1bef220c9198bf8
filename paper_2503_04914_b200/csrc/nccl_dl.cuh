// nccl_dl.cuh -- NCCL entry points resolved at run time from the libnccl that
// torch.distributed has already loaded into the process (dlopen RTLD_NOLOAD),
// else from the system library.  libmsk has no link-time NCCL dependency, and
// a process never carries two NCCL instances.
//
// MSK_NCCL_LIBRARY=<path> (test hook) resolves the entry points from that
// library instead: tests/nccl_shim implements the same API in-process for
// threads-as-ranks, so the rank >= 0 code path (halo plans, grouped
// send/recv, all-reduce sequencing) runs on one GPU without NCCL itself.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>

#include "common.cuh"

namespace msk {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi nccl_load() {
    NcclApi api;
    void *h = nullptr;
    if (const char *lib = std::getenv("MSK_NCCL_LIBRARY")) {
        h = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
        if (!h) throw Error(4, std::string("MSK_NCCL_LIBRARY: ") + dlerror());
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(4, std::string("NCCL not available: ") + dlerror());
    auto sym = [&](const char *name) {
        void *p = dlsym(h, name);
        if (!p) throw Error(4, std::string("NCCL symbol missing: ") + name);
        return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    return api;
}

// One resolution per process; thread-safe (ranks may be threads, see above).
// A failed resolution throws and is retried by the next call.
inline NcclApi *nccl_api() {
    static NcclApi api = nccl_load();
    return &api;
}

#define MSK_NCCL(call)                                                                         \
    do {                                                                                       \
        ncclResult_t r_ = (call);                                                              \
        if (r_ != ncclSuccess)                                                                 \
            throw ::msk::Error(4, std::string(#call) + ": " + ::msk::nccl_api()->GetErrorString(r_)); \
    } while (0)

}  // namespace msk

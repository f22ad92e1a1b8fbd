// NCCL bound at run time, not link time.
//
// libsplbcu.so shares its process with PyTorch, which ships its own
// libnccl.so.2 (a newer build than the system one).  Two builds under one
// soname cannot coexist, so instead of a DT_NEEDED entry we bind the handful
// of entry points the halo exchange uses lazily, preferring (1) an NCCL the
// process already loaded, (2) $SPLBCU_NCCL_LIB (the Python package points it
// at PyTorch's bundled copy), (3) the system libnccl.so.2.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>

namespace splbcu {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
    std::string source;
    bool ok = false;
};

inline const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (h) a.source = "already loaded";
        if (!h) {
            if (const char* p = std::getenv("SPLBCU_NCCL_LIB")) {
                h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
                if (h) a.source = p;
            }
        }
        if (!h) {
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (h) a.source = "system libnccl.so.2";
        }
        if (!h) {
            a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) a.error += std::string(" missing ") + name;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.CommAbort, "ncclCommAbort");
        sym(a.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.AllGather, "ncclAllGather");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        a.ok = a.error.empty();
        return a;
    }();
    return api;
}

}  // namespace splbcu

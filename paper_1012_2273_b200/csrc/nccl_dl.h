// nccl_dl.h -- NCCL entry points resolved at run time with dlopen.
//
// libmmws_gpu.so does not link libnccl: a process that already holds an NCCL
// (e.g. torch's bundled libnccl.so.2) must keep using that one -- a second,
// older libnccl.so.2 bound first would break the other library's newer
// symbols.  dlopen("libnccl.so.2") returns whichever copy the process already
// loaded, or the system one otherwise.  Only the row-block path needs NCCL.
// Resolved once, on the first row-block / communicator call.
#pragma once

#include <dlfcn.h>
#include <cstdlib>
#include <nccl.h>

#include <mutex>

namespace mmws_impl {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // MMWS_GPU_NCCL_LIB (tests only): a stand-in library with the same entry
    // points, loaded privately -- tests/fake_nccl runs several ranks on one GPU
    const char* lib = std::getenv("MMWS_GPU_NCCL_LIB");
    void* h = lib && *lib ? dlopen(lib, RTLD_NOW | RTLD_LOCAL)
                          : dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h && !(lib && *lib)) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define MMWS_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    MMWS_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    MMWS_NCCL_SYM(CommInitRank, "ncclCommInitRank");
    MMWS_NCCL_SYM(CommInitRankConfig, "ncclCommInitRankConfig");
    MMWS_NCCL_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    MMWS_NCCL_SYM(CommAbort, "ncclCommAbort");
    MMWS_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    MMWS_NCCL_SYM(Send, "ncclSend");
    MMWS_NCCL_SYM(Recv, "ncclRecv");
    MMWS_NCCL_SYM(Broadcast, "ncclBroadcast");
    MMWS_NCCL_SYM(AllReduce, "ncclAllReduce");
    MMWS_NCCL_SYM(GroupStart, "ncclGroupStart");
    MMWS_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    MMWS_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef MMWS_NCCL_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommInitRankConfig &&
             api.CommGetAsyncError && api.CommAbort && api.CommDestroy && api.Send && api.Recv &&
             api.Broadcast && api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

}  // namespace mmws_impl

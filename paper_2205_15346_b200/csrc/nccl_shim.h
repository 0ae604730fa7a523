// Lazy dlopen of libnccl.so.2 (the torch-bundled NCCL 2.28 in the venv, or the system one),
// so that single-GPU use of the library needs no NCCL at all.
#pragma once
#include <dlfcn.h>
#include <stdlib.h>
#include <nccl.h>

#include <string>

namespace te {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional: asynchronous error polling (a failed peer ends te_evolve instead of hanging it)
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  bool is_fake = false;  // the test stand-in (tests/support/fake_nccl.cu): no graph capture
};

inline NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // TE_NCCL_LIB: an alternative NCCL-compatible library (tests: tests/support/fake_nccl.cu runs
    // several ranks as threads on one GPU)
    const char* over = getenv("TE_NCCL_LIB");
    const char* cands[] = {
        over && *over ? over : "libnccl.so.2",
        "libnccl.so.2",
        "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
        "libnccl.so",
    };
    void* lib = nullptr;
    for (const char* c : cands)
      if ((lib = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!lib) {
      a.err = "dlopen(libnccl.so.2) failed";
      return a;
    }
#define TE_SYM(field, name)                                          \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(lib, name));   \
  if (!a.field) {                                                    \
    a.err = std::string("missing symbol ") + name;                   \
    return a;                                                        \
  }
    TE_SYM(GetUniqueId, "ncclGetUniqueId")
    TE_SYM(CommInitRank, "ncclCommInitRank")
    TE_SYM(CommDestroy, "ncclCommDestroy")
    TE_SYM(AllReduce, "ncclAllReduce")
    TE_SYM(AllGather, "ncclAllGather")
    TE_SYM(Send, "ncclSend")
    TE_SYM(Recv, "ncclRecv")
    TE_SYM(GroupStart, "ncclGroupStart")
    TE_SYM(GroupEnd, "ncclGroupEnd")
    TE_SYM(GetErrorString, "ncclGetErrorString")
#undef TE_SYM
    a.CommGetAsyncError = reinterpret_cast<decltype(a.CommGetAsyncError)>(dlsym(lib, "ncclCommGetAsyncError"));
    a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(dlsym(lib, "ncclCommAbort"));
    a.is_fake = dlsym(lib, "fake_nccl_calls") != nullptr;
    a.ok = true;
    return a;
  }();
  return api;
}

}  // namespace te

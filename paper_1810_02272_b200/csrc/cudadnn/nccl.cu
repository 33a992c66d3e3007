// nccl.cu — the data-parallel subsystem: NCCL communicators held as subsystem
// handles in the CudaDnn tables (the paper routes NCCL through the low-level
// DLL as a look-up-table object).  libnccl is resolved at run
// time (dlopen) so the library loads on hosts without NCCL; every call fails
// loudly there instead of falling back.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "internal.hpp"

using namespace cdnn;

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a = [] {
    NcclApi x;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      x.lib = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (x.lib) break;
    }
    if (!x.lib) return x;
    x.GetUniqueId = reinterpret_cast<decltype(x.GetUniqueId)>(dlsym(x.lib, "ncclGetUniqueId"));
    x.CommInitRank = reinterpret_cast<decltype(x.CommInitRank)>(dlsym(x.lib, "ncclCommInitRank"));
    x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(dlsym(x.lib, "ncclCommDestroy"));
    x.AllReduce = reinterpret_cast<decltype(x.AllReduce)>(dlsym(x.lib, "ncclAllReduce"));
    x.Broadcast = reinterpret_cast<decltype(x.Broadcast)>(dlsym(x.lib, "ncclBroadcast"));
    x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(dlsym(x.lib, "ncclGetErrorString"));
    x.CommCount = reinterpret_cast<decltype(x.CommCount)>(dlsym(x.lib, "ncclCommCount"));
    x.CommUserRank = reinterpret_cast<decltype(x.CommUserRank)>(dlsym(x.lib, "ncclCommUserRank"));
    x.ok = x.CommCount && x.CommUserRank && x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.AllReduce && x.Broadcast;
    return x;
  }();
  return a;
}

NcclApi& need_api() {
  NcclApi& a = api();
  if (!a.ok) fail(CDNN_CUDA_ERROR, "NCCL is not available (libnccl.so.2 not found)");
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    NcclApi& a = api();
    fail(CDNN_CUDA_ERROR, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "nccl error"));
  }
}

ncclDataType_t nccl_type(int dtype) {
  switch (dtype) {
    case CDNN_F32: return ncclFloat32;
    case CDNN_F64: return ncclFloat64;
    case CDNN_I32: return ncclInt32;
  }
  fail(CDNN_INVALID_ARGUMENT, "nccl: unsupported dtype");
}

}  // namespace

void cdnn::nccl_destroy(void* comm) {
  NcclApi& a = api();
  if (a.ok && comm) a.CommDestroy(static_cast<ncclComm_t>(comm));
}

extern "C" {

int cdnn_nccl_available(int* out) {
  return guarded([&] { *out = api().ok ? 1 : 0; });
}

int cdnn_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    nccl_check(need_api().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, 128);
  });
}

int cdnn_nccl_comm_create(cdnn_ctx ctx, int nranks, int rank, const uint8_t id[128], cdnn_handle* out) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(CDNN_INVALID_ARGUMENT, "nccl_comm_create: bad rank/nranks");
    NcclApi& a = need_api();
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    DeviceGuard g(c);
    ncclComm_t comm;
    nccl_check(a.CommInitRank(&comm, nranks, u, rank), "ncclCommInitRank");
    NcclSlot s;
    s.comm = comm;
    s.nranks = nranks;
    s.rank = rank;
    *out = insert_slot(c, s);
  });
}

int cdnn_nccl_comm_info(cdnn_ctx ctx, cdnn_handle comm, int* nranks, int* rank) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    NcclSlot& s = nccl(c, comm);
    NcclApi& a = need_api();
    nccl_check(a.CommCount(static_cast<ncclComm_t>(s.comm), nranks), "ncclCommCount");
    nccl_check(a.CommUserRank(static_cast<ncclComm_t>(s.comm), rank), "ncclCommUserRank");
  });
}

int cdnn_allreduce_sum(cdnn_ctx ctx, cdnn_handle comm, cdnn_handle buf, uint64_t offset, uint64_t n,
                       cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    NcclSlot& s = nccl(c, comm);
    BufferSlot& b = buffer(c, buf, "allreduce");
    if (offset + n > b.len) fail(CDNN_INVALID_ARGUMENT, "allreduce: range exceeds buffer");
    if (n == 0) return;
    DeviceGuard g(c);
    char* p = b.dev + offset * dtype_size(b.dtype);
    nccl_check(need_api().AllReduce(p, p, n, nccl_type(b.dtype), ncclSum, static_cast<ncclComm_t>(s.comm),
                                    stream_of(c, stream)),
               "ncclAllReduce");
  });
}

int cdnn_broadcast(cdnn_ctx ctx, cdnn_handle comm, cdnn_handle buf, uint64_t n, int root, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    NcclSlot& s = nccl(c, comm);
    BufferSlot& b = buffer(c, buf, "broadcast");
    if (n > b.len) fail(CDNN_INVALID_ARGUMENT, "broadcast: range exceeds buffer");
    if (n == 0) return;
    DeviceGuard g(c);
    nccl_check(need_api().Broadcast(b.dev, b.dev, n, nccl_type(b.dtype), root, static_cast<ncclComm_t>(s.comm),
                                    stream_of(c, stream)),
               "ncclBroadcast");
  });
}

}  // extern "C"

// Native NCCL communicator for sharded engines: the
// engine's all-gathers go straight to ncclAllGather on the engine stream
// (NVLink / NVSwitch, NVLS when NCCL selects it), without a host-language
// callback on the data path. libnccl.so.2 is opened at run time, so the
// library itself has no NCCL link dependency (single-GPU users never load it).
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../../include/smcl_gpu.h"

namespace smcl {
extern thread_local std::string g_last_error;
}

namespace {

// The subset of nccl.h used here (ABI-stable since NCCL 2.0).
using ncclComm_t = void*;
using ncclResult_t = int;
struct ncclUniqueId {
  char internal[128];
};
constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, void*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, void*) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, void*) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(a.h, "ncclCommInitRank"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(a.h, "ncclAllGather"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(a.h, "ncclGetErrorString"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(a.h, "ncclSend"));  // NCCL >= 2.7
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(a.h, "ncclRecv"));
    a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(a.h, "ncclGroupStart"));
    a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(a.h, "ncclGroupEnd"));
  });
  if (!a.getUniqueId || !a.commInitRank || !a.allGather || !a.commDestroy)
    throw std::runtime_error("NCCL (libnccl.so.2) not available");
  return a;
}

std::string nccl_err(ncclResult_t r) {
  const NcclApi& a = api();
  return a.getErrorString ? a.getErrorString(r) : ("nccl error " + std::to_string(r));
}

struct NcclCtx {
  ncclComm_t comm = nullptr;
  int world = 1;
};

// smcl_comm::allgather: `bytes` from every rank, rank-ordered into recv.
int nccl_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  if (bytes == 0) return 0;
  return api().allGather(send, recv, static_cast<size_t>(bytes), kNcclUint8, c->comm, stream) == 0 ? 0 : 1;
}

// smcl_comm::alltoallv as one NCCL group of point-to-point sends and receives
// (chunks packed in rank order on both sides).
int nccl_alltoallv(void* ctx, const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes,
                   void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  const NcclApi& a = api();
  const int world = c->world;
  if (a.groupStart() != 0) return 1;
  int rc = 0;
  uint64_t so = 0, ro = 0;
  for (int p = 0; p < world; ++p) {
    if (send_bytes[p] && a.send(static_cast<const char*>(send) + so, send_bytes[p], kNcclUint8, p, c->comm, stream))
      rc = 1;
    if (recv_bytes[p] && a.recv(static_cast<char*>(recv) + ro, recv_bytes[p], kNcclUint8, p, c->comm, stream))
      rc = 1;
    so += send_bytes[p];
    ro += recv_bytes[p];
  }
  if (a.groupEnd() != 0) rc = 1;
  return rc;
}

template <class F>
int cguard(F&& f) {
  try {
    f();
    return SMCL_OK;
  } catch (const std::invalid_argument& e) {
    smcl::g_last_error = e.what();
    return SMCL_EINVAL;
  } catch (const std::exception& e) {
    smcl::g_last_error = e.what();
    return SMCL_ENCCL;
  }
}

}  // namespace

extern "C" {

int smcl_nccl_get_unique_id(uint8_t id[128]) {
  return cguard([&] {
    ncclUniqueId u;
    const ncclResult_t r = api().getUniqueId(&u);
    if (r != 0) throw std::runtime_error("ncclGetUniqueId: " + nccl_err(r));
    std::memcpy(id, u.internal, sizeof(u.internal));
  });
}

int smcl_comm_nccl_create(const uint8_t id[128], int32_t rank, int32_t world, smcl_comm* out) {
  return cguard([&] {
    if (!out || !id || world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad NCCL comm args");
    ncclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    auto* c = new NcclCtx();
    c->world = world;
    const ncclResult_t r = api().commInitRank(&c->comm, world, u, rank);  // on the current CUDA device
    if (r != 0) {
      delete c;
      throw std::runtime_error("ncclCommInitRank: " + nccl_err(r));
    }
    out->ctx = c;
    out->rank = rank;
    out->world = world;
    out->allgather = nccl_allgather;
    const NcclApi& a = api();
    out->alltoallv = (a.send && a.recv && a.groupStart && a.groupEnd) ? nccl_alltoallv : nullptr;
  });
}

void smcl_comm_nccl_destroy(smcl_comm* c) {
  if (!c || !c->ctx) return;
  auto* ctx = static_cast<NcclCtx*>(c->ctx);
  if (ctx->comm) api().commDestroy(ctx->comm);
  delete ctx;
  c->ctx = nullptr;
}

}  // extern "C"

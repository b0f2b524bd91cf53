// NCCL-backed aj_comm for the z-slab sharded solve (row (e); north star: "one-plane
// halo exchange and dot-product allreduce via NCCL over NVLink").
//
// libnccl is opened at run time (dlopen): the binding passes the path of the NCCL
// that torch.distributed already loaded, so the process holds one NCCL.  The dot
// reductions are ncclAllReduce on the caller's stream (<= 64 doubles each); the halo
// exchange is one ncclSend/ncclRecv group per direction pair on a private stream, so
// the caller can compute the interior planes of the slab while it is in flight
// (halo_start records an event on the caller's stream, the group runs on the comm
// stream, halo_wait makes the caller's stream wait for it).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "aj_common.cuh"

namespace aj {
namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl(const char* path) {
  NcclApi a;
  const char* p = (path && path[0]) ? path : "libnccl.so.2";
  a.lib = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  AJ_REQUIRE(a.lib, AJ_ERR_CUDA, std::string("cannot dlopen ") + p + ": " + dlerror());
  auto sym = [&](const char* name) {
    void* f = dlsym(a.lib, name);
    AJ_REQUIRE(f, AJ_ERR_CUDA, std::string("libnccl lacks ") + name);
    return f;
  };
  a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
  a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
  a.Send = (decltype(a.Send))sym("ncclSend");
  a.Recv = (decltype(a.Recv))sym("ncclRecv");
  a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
  a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
  return a;
}

struct NcclCtx {
  NcclApi api;
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  aj_comm pub{};
};

#define NCCL_OK(ctx, call)                                                                 \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess) {                                                               \
      fprintf(stderr, "[aj comm] %s: %s\n", #call, (ctx)->api.GetErrorString(r_));         \
      return (int)AJ_ERR_CUDA;                                                             \
    }                                                                                      \
  } while (0)

int c_allreduce(void* vctx, double* buf, int32_t count, int32_t op, void* stream) {
  NcclCtx* c = (NcclCtx*)vctx;
  NCCL_OK(c, c->api.AllReduce(buf, buf, (size_t)count, ncclFloat64, op == 1 ? ncclMax : ncclSum, c->comm,
                              (cudaStream_t)stream));
  return 0;
}

int c_halo_start(void* vctx, const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi,
                 int64_t count, void* stream) {
  NcclCtx* c = (NcclCtx*)vctx;
  const int w = c->pub.world, r = c->pub.rank;
  const int down = (r - 1 + w) % w, up = (r + 1) % w;
  if (cudaEventRecord(c->ev_in, (cudaStream_t)stream) != cudaSuccess) return AJ_ERR_CUDA;
  if (cudaStreamWaitEvent(c->cs, c->ev_in, 0) != cudaSuccess) return AJ_ERR_CUDA;
  // posting order: with two ranks down == up, and messages between a pair match in order,
  // so every rank sends (last plane -> up) before (first plane -> down) and receives
  // (lower halo <- down) before (upper halo <- up)
  NCCL_OK(c, c->api.GroupStart());
  NCCL_OK(c, c->api.Send(send_hi, (size_t)count, ncclFloat64, up, c->comm, c->cs));
  NCCL_OK(c, c->api.Send(send_lo, (size_t)count, ncclFloat64, down, c->comm, c->cs));
  NCCL_OK(c, c->api.Recv(recv_lo, (size_t)count, ncclFloat64, down, c->comm, c->cs));
  NCCL_OK(c, c->api.Recv(recv_hi, (size_t)count, ncclFloat64, up, c->comm, c->cs));
  NCCL_OK(c, c->api.GroupEnd());
  if (cudaEventRecord(c->ev_out, c->cs) != cudaSuccess) return AJ_ERR_CUDA;
  return 0;
}

int c_halo_wait(void* vctx, void* stream) {
  NcclCtx* c = (NcclCtx*)vctx;
  return cudaStreamWaitEvent((cudaStream_t)stream, c->ev_out, 0) == cudaSuccess ? 0 : (int)AJ_ERR_CUDA;
}

}  // namespace
}  // namespace aj

extern "C" {

int aj_nccl_unique_id(const char* libnccl, void* h_id) {
  if (!h_id) return AJ_ERR_ARG;
  try {
    aj::NcclApi a = aj::load_nccl(libnccl);
    ncclUniqueId id;
    if (a.GetUniqueId(&id) != ncclSuccess) return AJ_ERR_CUDA;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(h_id, &id, sizeof(id));
    return AJ_OK;
  } catch (const aj::Error& e) {
    fprintf(stderr, "[aj comm] %s\n", e.what());
    return e.code;
  }
}

int aj_comm_nccl_create(aj_comm** out, const char* libnccl, const void* h_id, int32_t world, int32_t rank) {
  if (!out || !h_id || world < 1 || rank < 0 || rank >= world) return AJ_ERR_ARG;
  aj::NcclCtx* c = nullptr;
  try {
    c = new aj::NcclCtx();
    c->api = aj::load_nccl(libnccl);
    ncclUniqueId id;
    memcpy(&id, h_id, sizeof(id));
    if (c->api.CommInitRank(&c->comm, world, id, rank) != ncclSuccess) {
      delete c;
      return AJ_ERR_CUDA;
    }
    AJ_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
    AJ_CUDA(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    AJ_CUDA(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    c->pub.world = world;
    c->pub.rank = rank;
    c->pub.ctx = c;
    c->pub.allreduce = aj::c_allreduce;
    c->pub.halo_start = aj::c_halo_start;
    c->pub.halo_wait = aj::c_halo_wait;
    *out = &c->pub;
    return AJ_OK;
  } catch (const aj::Error& e) {
    fprintf(stderr, "[aj comm] %s\n", e.what());
    delete c;
    return e.code;
  }
}

int aj_comm_nccl_free(aj_comm* comm) {
  if (!comm) return AJ_OK;
  aj::NcclCtx* c = (aj::NcclCtx*)comm->ctx;
  if (c->comm) c->api.CommDestroy(c->comm);
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  delete c;
  return AJ_OK;
}

}  // extern "C"

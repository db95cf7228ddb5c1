// NCCL communicator of the row-sharded solvers: one rank
// per GPU, created once per process group from a unique id that the host
// exchanges once (any out-of-band channel; the Python layer uses one
// torch.distributed broadcast at setup).  Per iteration the host loop then
// calls mlr_comm_allreduce / mlr_comm_allgather on the plan's stream for the
// coarse Gram + packed stats (ML-PCP: one call; ML-CPCP: stats all-reduce,
// arg-max all-gather, QP-dot all-reduce), so no collective goes through
// Python/torch.distributed inside the loop.
//
// NCCL is loaded with dlopen at the first mlr_comm_* call: the library loads
// (and every single-GPU path works) on hosts without NCCL; in a process that
// already mapped torch's bundled libnccl.so.2, dlopen returns that copy.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace mlr {

// the subset of nccl.h this file uses (stable across NCCL 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclSum = 0, ncclProd = 1, ncclMax = 2, ncclMin = 3 } ncclRedOp_t;
typedef enum { ncclInt64 = 4, ncclFloat64 = 8 } ncclDataType_t;

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

static NcclApi g_nccl;
static std::once_flag g_nccl_once;

static void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce &&
              g_nccl.AllGather && g_nccl.GetErrorString;
}

static bool nccl_ready() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.ok) set_error("NCCL (libnccl.so.2) could not be loaded");
  return g_nccl.ok;
}

static int nccl_fail(ncclResult_t r, const char* where) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "NCCL error");
  set_error(buf);
  return kErrCuda;
}

struct MlrComm {
  ncclComm_t c;
  int rank, nranks, device;
};

}  // namespace mlr

using namespace mlr;

extern "C" {

int mlr_comm_available(void) {
  std::call_once(g_nccl_once, load_nccl);
  return g_nccl.ok ? 1 : 0;
}

int mlr_comm_unique_id(void* out128) {
  if (!out128) {
    set_error("mlr_comm_unique_id: null output");
    return kErrArg;
  }
  if (!nccl_ready()) return kErrArg;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, id.internal, sizeof(id.internal));
  return kOk;
}

int mlr_comm_create(const void* id128, int nranks, int rank, int device, void** comm_out) {
  if (!id128 || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("mlr_comm_create: bad arguments");
    return kErrArg;
  }
  if (!nccl_ready()) return kErrArg;
  MLR_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(id.internal, id128, sizeof(id.internal));
  MlrComm* c = new MlrComm{nullptr, rank, nranks, device};
  ncclResult_t r = g_nccl.CommInitRank(&c->c, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *comm_out = c;
  return kOk;
}

int mlr_comm_destroy(void* comm) {
  if (!comm) return kOk;
  MlrComm* c = (MlrComm*)comm;
  if (g_nccl.ok && c->c) g_nccl.CommDestroy(c->c);
  delete c;
  return kOk;
}

/* op: 0 sum, 2 max; dtype: 8 float64, 4 int64 (NCCL enum values) */
int mlr_comm_allreduce(void* comm, void* buf, int64_t count, int dtype, int op, void* stream) {
  MlrComm* c = (MlrComm*)comm;
  if (!c || (op != ncclSum && op != ncclMax) || (dtype != ncclFloat64 && dtype != ncclInt64)) {
    set_error("mlr_comm_allreduce: bad arguments");
    return kErrArg;
  }
  if (count == 0) return kOk;
  ncclResult_t r = g_nccl.AllReduce(buf, buf, (size_t)count, (ncclDataType_t)dtype, (ncclRedOp_t)op, c->c,
                                    (cudaStream_t)stream);
  return r == ncclSuccess ? kOk : nccl_fail(r, "ncclAllReduce");
}

/* out (nranks x count) <- every rank's in (count), rank order */
int mlr_comm_allgather(void* comm, const void* in, void* out, int64_t count, int dtype, void* stream) {
  MlrComm* c = (MlrComm*)comm;
  if (!c || (dtype != ncclFloat64 && dtype != ncclInt64)) {
    set_error("mlr_comm_allgather: bad arguments");
    return kErrArg;
  }
  ncclResult_t r = g_nccl.AllGather(in, out, (size_t)count, (ncclDataType_t)dtype, c->c, (cudaStream_t)stream);
  return r == ncclSuccess ? kOk : nccl_fail(r, "ncclAllGather");
}

int mlr_comm_rank(void* comm) { return comm ? ((MlrComm*)comm)->rank : -1; }
int mlr_comm_size(void* comm) { return comm ? ((MlrComm*)comm)->nranks : -1; }

}  // extern "C"

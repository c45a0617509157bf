// pf_nccl.cu — NCCL plumbing behind the C ABI (SURVEY §8b `pf_nccl_*`, §8e).
//
// The row-sharded hot path has two data-path exchanges (the target row
// broadcast from its owner rank, and the all-gather of finished field slabs
// when a tracer needs the whole field) plus tiny flag / domain-check
// reductions.  They run on NCCL over NVLink / NVSwitch through these entry
// points, on the caller's stream, so Python keeps PyTorch for buffer
// ownership and the process-group rendezvous only (the 128-byte unique id
// is exchanged over the control-plane process group).
//
// NCCL is bound at run time (dlopen + dlsym): the process normally already
// holds one libnccl.so.2 (the one torch links), and binding to that same
// image avoids two NCCL runtimes in one process.  Only the types come from
// <nccl.h>; their layout is part of NCCL's stable ABI.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "pf_common.cuh"

namespace {

struct NcclApi {
  void *handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                             ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*get_version)(int *) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
};

NcclApi g_api;
std::mutex g_api_mu;

template <typename F>
bool bind(void *h, const char *name, F *&fn) {
  fn = reinterpret_cast<F *>(dlsym(h, name));
  return fn != nullptr;
}

int require_api() {
  if (g_api.handle == nullptr)
    return pf::fail(PF_E_ARG, "NCCL is not loaded (call pf_nccl_load first)");
  return 0;
}

int nccl_status(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return 0;
  return pf::fail(PF_E_LAUNCH, "%s: %s (ncclResult %d)", what,
                  g_api.error_string ? g_api.error_string(r) : "?", static_cast<int>(r));
}

bool map_type(int dtype, ncclDataType_t *out) {
  switch (dtype) {
    case PF_T_U8: *out = ncclUint8; return true;
    case PF_T_I32: *out = ncclInt32; return true;
    case PF_T_I64: *out = ncclInt64; return true;
    case PF_T_F64: *out = ncclFloat64; return true;
    default: return false;
  }
}

bool map_op(int op, ncclRedOp_t *out) {
  switch (op) {
    case PF_OP_SUM: *out = ncclSum; return true;
    case PF_OP_MAX: *out = ncclMax; return true;
    case PF_OP_MIN: *out = ncclMin; return true;
    default: return false;
  }
}

}  // namespace

extern "C" {

int pf_nccl_load(const char *path_host) {
  std::lock_guard<std::mutex> lk(g_api_mu);
  if (g_api.handle != nullptr) return 0;
  // the NCCL image already in the process (torch's), else the given path,
  // else the loader's default libnccl.so.2
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (h == nullptr && path_host != nullptr && path_host[0] != '\0')
    h = dlopen(path_host, RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (h == nullptr) return pf::fail(PF_E_ARG, "dlopen libnccl.so.2: %s", dlerror());
  NcclApi api;
  api.handle = h;
  const bool ok = bind(h, "ncclGetUniqueId", api.get_unique_id) &&
                  bind(h, "ncclCommInitRank", api.comm_init_rank) &&
                  bind(h, "ncclCommDestroy", api.comm_destroy) &&
                  bind(h, "ncclBroadcast", api.broadcast) &&
                  bind(h, "ncclAllGather", api.all_gather) &&
                  bind(h, "ncclAllReduce", api.all_reduce) &&
                  bind(h, "ncclGetVersion", api.get_version) &&
                  bind(h, "ncclGetErrorString", api.error_string);
  if (!ok) return pf::fail(PF_E_ARG, "libnccl.so.2 lacks a required symbol");
  g_api = api;
  return 0;
}

int pf_nccl_version(int *version_host) {
  if (int rc = require_api()) return rc;
  if (version_host == nullptr) return pf::fail(PF_E_ARG, "version_host is NULL");
  return nccl_status(g_api.get_version(version_host), "ncclGetVersion");
}

int pf_nccl_unique_id(void *id_host) {
  if (int rc = require_api()) return rc;
  if (id_host == nullptr) return pf::fail(PF_E_ARG, "id_host is NULL");
  ncclUniqueId id;
  if (int rc = nccl_status(g_api.get_unique_id(&id), "ncclGetUniqueId")) return rc;
  memcpy(id_host, id.internal, PF_NCCL_ID_BYTES);
  return 0;
}

int pf_nccl_comm_init(int nranks, const void *id_host, int rank, int device, void **comm_host) {
  if (int rc = require_api()) return rc;
  if (id_host == nullptr || comm_host == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
    return pf::fail(PF_E_ARG, "pf_nccl_comm_init: bad arguments");
  const cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return pf::fail(static_cast<int>(e), "cudaSetDevice(%d)", device);
  ncclUniqueId id;
  memcpy(id.internal, id_host, PF_NCCL_ID_BYTES);
  ncclComm_t comm = nullptr;
  if (int rc = nccl_status(g_api.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank"))
    return rc;
  *comm_host = comm;
  return 0;
}

int pf_nccl_comm_destroy(void *comm) {
  if (int rc = require_api()) return rc;
  if (comm == nullptr) return 0;
  return nccl_status(g_api.comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

int pf_nccl_broadcast(void *comm, void *buf, int64_t count, int dtype, int root,
                      pf_stream_t stream) {
  if (int rc = require_api()) return rc;
  ncclDataType_t t;
  if (comm == nullptr || count < 0 || !map_type(dtype, &t))
    return pf::fail(PF_E_ARG, "pf_nccl_broadcast: bad arguments");
  if (count == 0) return 0;
  return nccl_status(g_api.broadcast(buf, buf, static_cast<size_t>(count), t, root,
                                     static_cast<ncclComm_t>(comm),
                                     static_cast<cudaStream_t>(stream)),
                     "ncclBroadcast");
}

int pf_nccl_all_gather(void *comm, const void *send, void *recv, int64_t count, int dtype,
                       pf_stream_t stream) {
  if (int rc = require_api()) return rc;
  ncclDataType_t t;
  if (comm == nullptr || count < 0 || !map_type(dtype, &t))
    return pf::fail(PF_E_ARG, "pf_nccl_all_gather: bad arguments");
  if (count == 0) return 0;
  return nccl_status(g_api.all_gather(send, recv, static_cast<size_t>(count), t,
                                      static_cast<ncclComm_t>(comm),
                                      static_cast<cudaStream_t>(stream)),
                     "ncclAllGather");
}

int pf_nccl_all_reduce(void *comm, const void *send, void *recv, int64_t count, int dtype,
                       int op, pf_stream_t stream) {
  if (int rc = require_api()) return rc;
  ncclDataType_t t;
  ncclRedOp_t o;
  if (comm == nullptr || count < 0 || !map_type(dtype, &t) || !map_op(op, &o))
    return pf::fail(PF_E_ARG, "pf_nccl_all_reduce: bad arguments");
  if (count == 0) return 0;
  return nccl_status(g_api.all_reduce(send, recv, static_cast<size_t>(count), t, o,
                                      static_cast<ncclComm_t>(comm),
                                      static_cast<cudaStream_t>(stream)),
                     "ncclAllReduce");
}

}  // extern "C"

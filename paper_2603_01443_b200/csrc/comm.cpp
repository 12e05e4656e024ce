// Native NCCL plumbing of the multi-GPU cut pipeline: communicator setup, the
// all-gather of subcircuit variant states (the only data
// exchange of the sharded pipeline) and the paired send/recv of the
// distributed uncut simulator's half-shard swaps.
//
// libnccl is resolved at run time with dlopen (the copy torch already loaded,
// by soname, or an explicit path from cs_nccl_load), so libcutsim has no
// link-time NCCL dependency and loads on machines without it. The NCCL ABI
// used here is the stable C API of nccl.h (2.x): ncclGetUniqueId,
// ncclCommInitRank, ncclAllGather, ncclSend/ncclRecv in a group,
// ncclCommDestroy, ncclGetErrorString.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/cutsim.h"
#include "capi_codes.hpp"

namespace cutsim {
int set_error(int code, const std::string& msg);
}

namespace {

struct UniqueId {
  char internal[128];
};
using comm_t = void*;
using GetUniqueId = int (*)(UniqueId*);
using CommInitRank = int (*)(comm_t*, int, UniqueId, int);
using CommDestroy = int (*)(comm_t);
using AllGather = int (*)(const void*, void*, size_t, int, comm_t, cudaStream_t);
using SendRecv = int (*)(const void*, size_t, int, int, comm_t, cudaStream_t);
using Group = int (*)();
using ErrStr = const char* (*)(int);
constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8

struct Api {
  void* lib = nullptr;
  GetUniqueId get_unique_id = nullptr;
  CommInitRank comm_init_rank = nullptr;
  CommDestroy comm_destroy = nullptr;
  AllGather all_gather = nullptr;
  SendRecv send = nullptr;
  SendRecv recv = nullptr;
  Group group_start = nullptr;
  Group group_end = nullptr;
  ErrStr err = nullptr;
} g_api;
std::mutex g_api_mu;

int bind(void* lib) {
  Api a;
  a.lib = lib;
  a.get_unique_id = reinterpret_cast<GetUniqueId>(dlsym(lib, "ncclGetUniqueId"));
  a.comm_init_rank = reinterpret_cast<CommInitRank>(dlsym(lib, "ncclCommInitRank"));
  a.comm_destroy = reinterpret_cast<CommDestroy>(dlsym(lib, "ncclCommDestroy"));
  a.all_gather = reinterpret_cast<AllGather>(dlsym(lib, "ncclAllGather"));
  a.send = reinterpret_cast<SendRecv>(dlsym(lib, "ncclSend"));
  a.recv = reinterpret_cast<SendRecv>(dlsym(lib, "ncclRecv"));
  a.group_start = reinterpret_cast<Group>(dlsym(lib, "ncclGroupStart"));
  a.group_end = reinterpret_cast<Group>(dlsym(lib, "ncclGroupEnd"));
  a.err = reinterpret_cast<ErrStr>(dlsym(lib, "ncclGetErrorString"));
  if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_gather || !a.send || !a.recv ||
      !a.group_start || !a.group_end || !a.err)
    return cutsim::set_error(CS_ERR_NODEVICE, "libnccl is missing required symbols");
  g_api = a;
  return CS_OK;
}

int ensure_loaded() {
  std::lock_guard<std::mutex> lk(g_api_mu);
  if (g_api.lib) return CS_OK;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib)
    return cutsim::set_error(CS_ERR_NODEVICE, std::string("libnccl.so.2 not found (cs_nccl_load): ") + dlerror());
  return bind(lib);
}

int nccl_fail(int rc, const char* where) {
  return cutsim::set_error(CS_ERR_NCCL, std::string(where) + ": " + (g_api.err ? g_api.err(rc) : "nccl error"));
}

}  // namespace

extern "C" {

int cs_nccl_load(const char* path) {
  std::lock_guard<std::mutex> lk(g_api_mu);
  if (g_api.lib) return CS_OK;
  void* lib = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return cutsim::set_error(CS_ERR_NODEVICE, std::string("dlopen failed: ") + dlerror());
  return bind(lib);
}

int cs_nccl_unique_id(uint8_t* id128) {
  if (!id128) return cutsim::set_error(CS_ERR_INVALID, "null id buffer");
  int rc = ensure_loaded();
  if (rc != CS_OK) return rc;
  UniqueId id;
  const int r = g_api.get_unique_id(&id);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id128, id.internal, sizeof(id.internal));
  return CS_OK;
}

int cs_nccl_comm_init(int32_t world, int32_t rank, const uint8_t* id128, int32_t device, void** comm) {
  if (!id128 || !comm || world < 1 || rank < 0 || rank >= world)
    return cutsim::set_error(CS_ERR_INVALID, "bad communicator arguments");
  int rc = ensure_loaded();
  if (rc != CS_OK) return rc;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cutsim::set_error(CS_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  UniqueId id;
  std::memcpy(id.internal, id128, sizeof(id.internal));
  comm_t c = nullptr;
  const int r = g_api.comm_init_rank(&c, world, id, rank);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return CS_OK;
}

int cs_nccl_comm_destroy(void* comm) {
  if (!comm) return CS_OK;
  if (!g_api.lib) return cutsim::set_error(CS_ERR_INVALID, "no NCCL library loaded");
  const int r = g_api.comm_destroy(comm);
  return r == 0 ? CS_OK : nccl_fail(r, "ncclCommDestroy");
}

int cs_allgather_states(void* comm, const void* send, int64_t bytes_per_rank, void* recv, void* stream) {
  if (!comm || !send || !recv || bytes_per_rank < 0)
    return cutsim::set_error(CS_ERR_INVALID, "bad all-gather arguments");
  if (!g_api.lib) return cutsim::set_error(CS_ERR_INVALID, "no NCCL library loaded");
  const int r = g_api.all_gather(send, recv, size_t(bytes_per_rank), kNcclUint8, comm,
                                 reinterpret_cast<cudaStream_t>(stream));
  return r == 0 ? CS_OK : nccl_fail(r, "ncclAllGather");
}

int cs_sendrecv(void* comm, const void* send, void* recv, int64_t bytes, int32_t peer, void* stream) {
  if (!comm || !send || !recv || bytes < 0 || peer < 0)
    return cutsim::set_error(CS_ERR_INVALID, "bad send/recv arguments");
  if (!g_api.lib) return cutsim::set_error(CS_ERR_INVALID, "no NCCL library loaded");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int r = g_api.group_start();
  if (r == 0) r = g_api.send(send, size_t(bytes), kNcclUint8, peer, comm, st);
  if (r == 0) r = g_api.recv(recv, size_t(bytes), kNcclUint8, peer, comm, st);
  const int r2 = g_api.group_end();
  if (r != 0) return nccl_fail(r, "ncclSend/ncclRecv");
  return r2 == 0 ? CS_OK : nccl_fail(r2, "ncclGroupEnd");
}

}  // extern "C"

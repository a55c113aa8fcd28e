// Multi-GPU exchange of the sharded hot path for C callers (SURVEY.md §8(b),
// §8(e)): one process per GPU, each measuring its shard of a batch / scoring
// its shard of a population; the only exchanges are an all-gather of the
// fixed-size measure records, an all-gather of the fitness vector, and a
// broadcast of the (serialised) cost model after each retrain.  No reductions,
// so results are bit-identical to the single-GPU path.
//
// NCCL is opened at run time (dlopen "libnccl.so.2", RTLD_LOCAL): when torch is
// already loaded this is its bundled NCCL (same soname), otherwise the system
// library; the shared object has no link-time NCCL dependency to conflict with
// either.  Python callers use torch.distributed (paper_2006_06762_b200/dist.py)
// for the same exchange.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>
#include <string>
#include "common.h"
#include "loomtune_b200.h"

namespace {

typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm;
enum { NCCL_INT8 = 0, NCCL_FLOAT64 = 8 };

struct Nccl {
  void* h = nullptr;
  int (*get_unique_id)(nccl_uid*) = nullptr;
  int (*comm_init_rank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  int (*comm_destroy)(nccl_comm) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
  int (*broadcast)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;

  int load() {
    if (h) return 0;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return lt::fail(std::string("NCCL not available: ") + dlerror());
    get_unique_id = (int (*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
    comm_init_rank = (int (*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
    comm_destroy = (int (*)(nccl_comm))dlsym(h, "ncclCommDestroy");
    all_gather = (int (*)(const void*, void*, size_t, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllGather");
    broadcast = (int (*)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclBroadcast");
    error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    if (!get_unique_id || !comm_init_rank || !comm_destroy || !all_gather || !broadcast)
      return lt::fail("NCCL: missing symbols");
    return 0;
  }
  int check(int r, const char* what) {
    if (r == 0) return 0;
    return lt::fail(std::string(what) + ": " + (error_string ? error_string(r) : std::to_string(r)));
  }
};
Nccl g_nccl;

struct Comm {
  nccl_comm comm = nullptr;
  int rank = 0, world = 1, device = 0;
  cudaStream_t stream = nullptr;
  void* d_buf = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes) {
    if (bytes <= cap) return 0;
    if (d_buf) cudaFree(d_buf);
    d_buf = nullptr;
    cap = 0;
    if (lt::check_cuda(cudaMalloc(&d_buf, bytes), "comm buffer")) return -1;
    cap = bytes;
    return 0;
  }
};

}  // namespace

extern "C" {

// 128 opaque bytes; rank 0 creates it and hands it to the others out of band.
int lt_comm_unique_id(char* out128) {
  if (g_nccl.load()) return -1;
  nccl_uid id;
  if (g_nccl.check(g_nccl.get_unique_id(&id), "ncclGetUniqueId")) return -1;
  memcpy(out128, id.internal, 128);
  return 0;
}

int64_t lt_comm_create(const char* id128, int rank, int world, int device) {
  if (g_nccl.load()) return 0;
  if (world < 1 || rank < 0 || rank >= world) { lt::fail("lt_comm_create: bad rank/world"); return 0; }
  if (lt::check_cuda(cudaSetDevice(device), "lt_comm_create: cudaSetDevice")) return 0;
  Comm* c = new Comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  nccl_uid id;
  memcpy(id.internal, id128, 128);
  if (g_nccl.check(g_nccl.comm_init_rank(&c->comm, world, id, rank), "ncclCommInitRank") ||
      lt::check_cuda(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "comm stream")) {
    delete c;
    return 0;
  }
  return (int64_t)(intptr_t)c;
}

void lt_comm_destroy(int64_t comm) {
  Comm* c = (Comm*)(intptr_t)comm;
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->comm) g_nccl.comm_destroy(c->comm);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->d_buf) cudaFree(c->d_buf);
  delete c;
}

// All-gather of `bytes_per_rank` host bytes from every rank, rank order, into
// out[world * bytes_per_rank] (shards padded to the largest shard by the caller).
int lt_comm_allgather(int64_t comm, const void* local, int64_t bytes_per_rank, void* out) {
  Comm* c = (Comm*)(intptr_t)comm;
  if (!c) return lt::fail("null communicator");
  if (bytes_per_rank < 0) return lt::fail("negative size");
  const size_t n = (size_t)bytes_per_rank, total = n * (size_t)c->world;
  if (lt::check_cuda(cudaSetDevice(c->device), "cudaSetDevice") || c->reserve(total + n + 16)) return -1;
  char* d_in = (char*)c->d_buf + total;
  cudaMemcpyAsync(d_in, local, n, cudaMemcpyHostToDevice, c->stream);
  if (g_nccl.check(g_nccl.all_gather(d_in, c->d_buf, n, NCCL_INT8, c->comm, c->stream), "ncclAllGather")) return -1;
  cudaMemcpyAsync(out, c->d_buf, total, cudaMemcpyDeviceToHost, c->stream);
  return lt::check_cuda(cudaStreamSynchronize(c->stream), "allgather");
}

// Measure records of every rank's shard (n_local_max records each, padded).
int lt_comm_allgather_records(int64_t comm, const lt_measure_record* local, int64_t n_local_max,
                              lt_measure_record* out) {
  return lt_comm_allgather(comm, local, n_local_max * (int64_t)sizeof(lt_measure_record), out);
}

// Fitness vector of every rank's population shard (n_local_max doubles each).
int lt_comm_allgather_f64(int64_t comm, const double* local, int64_t n_local_max, double* out) {
  return lt_comm_allgather(comm, local, n_local_max * 8, out);
}

// Broadcast `bytes` of host memory from `root` (e.g. the serialised cost model
// after a retrain, before lt_model_create on every rank).
int lt_comm_broadcast(int64_t comm, void* buf, int64_t bytes, int root) {
  Comm* c = (Comm*)(intptr_t)comm;
  if (!c) return lt::fail("null communicator");
  if (lt::check_cuda(cudaSetDevice(c->device), "cudaSetDevice") || c->reserve((size_t)bytes + 16)) return -1;
  if (c->rank == root) cudaMemcpyAsync(c->d_buf, buf, (size_t)bytes, cudaMemcpyHostToDevice, c->stream);
  if (g_nccl.check(g_nccl.broadcast(c->d_buf, c->d_buf, (size_t)bytes, NCCL_INT8, root, c->comm, c->stream),
                   "ncclBroadcast"))
    return -1;
  if (c->rank != root) cudaMemcpyAsync(buf, c->d_buf, (size_t)bytes, cudaMemcpyDeviceToHost, c->stream);
  return lt::check_cuda(cudaStreamSynchronize(c->stream), "broadcast");
}

int lt_comm_rank(int64_t comm, int* rank, int* world) {
  Comm* c = (Comm*)(intptr_t)comm;
  if (!c) return lt::fail("null communicator");
  *rank = c->rank;
  *world = c->world;
  return 0;
}

}  // extern "C"

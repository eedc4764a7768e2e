// Gradient all-reduce of the batch-sharded data parallelism (SURVEY.md §8b "Comm", §8e).
//
// One communicator per GPU process.  monet_allreduce_bucket forks the bucket's
// all-reduce off the compute stream: an event recorded after the kernels that
// finalize the bucket, a dedicated comm stream waiting on it, ncclAllReduce (sum,
// in place) on that stream, and a completion event; monet_comm_join makes the
// compute stream wait for every bucket forked since the last join (the optimizer
// runs after it).  Every step is a plain stream operation, so a whole data-parallel
// training step -- kernels, bucket all-reduces, SGD -- is captured into one CUDA
// graph (NCCL supports stream capture; the comm stream joins the capture through
// the fork event and is joined back before the capture ends).
//
// NCCL is resolved at run time (dlopen): the process that already loaded NCCL
// (torch's bundled libnccl.so.2) keeps its copy, so the library never mixes two
// NCCL versions in one process and does not need NCCL at link time.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "../../include/monet_b200.h"
#include "common.cuh"

namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return n;
  n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
  n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  n.get_version = reinterpret_cast<decltype(n.get_version)>(dlsym(h, "ncclGetVersion"));
  n.ok = n.get_unique_id && n.comm_init_rank && n.all_reduce && n.comm_destroy;
  return n;
}

// NCCL failures map to -(1000 + ncclResult_t), distinct from -cudaError_t
inline int nccl_err(ncclResult_t r) { return r == ncclSuccess ? 0 : -(1000 + (int)r); }
inline int cuda_err(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e; }

}  // namespace

struct monet_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;            // the comm stream
  std::vector<cudaEvent_t> fork, done;      // one pair per bucket of a step (reused every step)
  size_t pending = 0;                       // buckets forked since the last join
};

extern "C" {

int monet_comm_unique_id(void* id_out) {
  Nccl& n = nccl();
  if (!n.ok) return -(int)cudaErrorSharedObjectInitFailed;
  ncclUniqueId id;
  if (int e = nccl_err(n.get_unique_id(&id))) return e;
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

size_t monet_comm_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

int monet_comm_init(const void* unique_id, int rank, int nranks, monet_comm** out) {
  Nccl& n = nccl();
  if (!n.ok) return -(int)cudaErrorSharedObjectInitFailed;
  if (!unique_id || !out || rank < 0 || rank >= nranks) return -(int)cudaErrorInvalidValue;
  auto* c = new monet_comm();
  c->rank = rank;
  c->nranks = nranks;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  if (int e = nccl_err(n.comm_init_rank(&c->comm, nranks, id, rank))) {
    delete c;
    return e;
  }
  if (int e = cuda_err(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking))) {
    n.comm_destroy(c->comm);
    delete c;
    return e;
  }
  *out = c;
  return 0;
}

int monet_comm_destroy(monet_comm* c) {
  if (!c) return 0;
  cudaStreamSynchronize(c->stream);
  for (auto e : c->fork) cudaEventDestroy(e);
  for (auto e : c->done) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  int rc = nccl_err(nccl().comm_destroy(c->comm));
  delete c;
  return rc;
}

int monet_allreduce_bucket(monet_comm* c, float* buf, size_t count, void* stream) {
  if (!c) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t i = c->pending++;
  while (c->fork.size() <= i) {
    cudaEvent_t a, b;
    if (int e = cuda_err(cudaEventCreateWithFlags(&a, cudaEventDisableTiming))) return e;
    if (int e = cuda_err(cudaEventCreateWithFlags(&b, cudaEventDisableTiming))) return e;
    c->fork.push_back(a);
    c->done.push_back(b);
  }
  if (int e = cuda_err(cudaEventRecord(c->fork[i], st))) return e;
  if (int e = cuda_err(cudaStreamWaitEvent(c->stream, c->fork[i], 0))) return e;
  if (count)
    if (int e = nccl_err(nccl().all_reduce(buf, buf, count, ncclFloat32, ncclSum, c->comm, c->stream))) return e;
  return cuda_err(cudaEventRecord(c->done[i], c->stream));
}

int monet_comm_join(monet_comm* c, void* stream) {
  if (!c) return -(int)cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (size_t i = 0; i < c->pending; ++i)
    if (int e = cuda_err(cudaStreamWaitEvent(st, c->done[i], 0))) return e;
  c->pending = 0;
  return 0;
}

}  // extern "C"

// Communicators for the row-sharded powerURV (BASELINE C4).
//
// The reference is single-process (powerurv.py:41-72); the sharded path
// needs exactly three collectives on FP64 device buffers, all issued on the
// caller's stream:
//   allreduce_sum  Y = sum_i A_i^T Vhat_i   (n x n, once per power round)
//   allgather      the n x n TSQR R factors of every rank (twice per round)
//   broadcast      the reconstruction's n x n L\U' block + signs (once)
//
// Backends:
//  * NCCL (one process per GPU over NVLink/NVSwitch).  libnccl is NOT linked:
//    it is dlopen'ed at first use, preferring the copy already loaded in the
//    process (torch's), so one NCCL instance serves both; `UTV_NCCL_LIB`
//    overrides the path.  The few ABI items used (ncclUniqueId = 128 bytes,
//    ncclFloat64 = 8, ncclSum = 0) are stable across NCCL 2.x.
//  * local group: P emulated ranks = P host threads of one process (each on
//    its own stream, any device) exchanging through device-to-device copies
//    and a host barrier; sums in rank order (deterministic).  Used to run the
//    multi-rank schedule on a single B200 and by the single-GPU tall QR
//    (P = 1, no traffic at all).
#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/utv_b200.h"
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

// ---------------------------------------------------------------------------
// NCCL through dlopen
// ---------------------------------------------------------------------------
namespace nccl {
typedef struct ncclComm* comm_t;
struct UniqueId {
  char internal[128];
};
typedef int result_t;  // ncclResult_t: 0 = ncclSuccess
constexpr int FLOAT64 = 8, SUM = 0;

struct Api {
  result_t (*getUniqueId)(UniqueId*);
  result_t (*commInitRank)(comm_t*, int, UniqueId, int);
  result_t (*commDestroy)(comm_t);
  result_t (*commCount)(comm_t, int*);
  result_t (*commUserRank)(comm_t, int*);
  result_t (*allReduce)(const void*, void*, size_t, int, int, comm_t, cudaStream_t);
  result_t (*allGather)(const void*, void*, size_t, int, comm_t, cudaStream_t);
  result_t (*broadcast)(const void*, void*, size_t, int, int, comm_t, cudaStream_t);
  const char* (*errorString)(result_t);
  bool ok = false;
};

static Api g_api;
static std::once_flag g_once;

static void* open_lib() {
  if (const char* p = getenv("UTV_NCCL_LIB")) return dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  // the instance torch (or the host application) already loaded, if any
  if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD)) return h;
  if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL)) return h;
  return dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
}

static const Api* api() {
  std::call_once(g_once, [] {
    void* h = open_lib();
    if (!h) return;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    g_api.getUniqueId = (decltype(g_api.getUniqueId))sym("ncclGetUniqueId");
    g_api.commInitRank = (decltype(g_api.commInitRank))sym("ncclCommInitRank");
    g_api.commDestroy = (decltype(g_api.commDestroy))sym("ncclCommDestroy");
    g_api.commCount = (decltype(g_api.commCount))sym("ncclCommCount");
    g_api.commUserRank = (decltype(g_api.commUserRank))sym("ncclCommUserRank");
    g_api.allReduce = (decltype(g_api.allReduce))sym("ncclAllReduce");
    g_api.allGather = (decltype(g_api.allGather))sym("ncclAllGather");
    g_api.broadcast = (decltype(g_api.broadcast))sym("ncclBroadcast");
    g_api.errorString = (decltype(g_api.errorString))sym("ncclGetErrorString");
    g_api.ok = g_api.getUniqueId && g_api.commInitRank && g_api.commDestroy && g_api.commCount &&
               g_api.commUserRank && g_api.allReduce && g_api.allGather && g_api.broadcast;
  });
  return g_api.ok ? &g_api : nullptr;
}

static int fail(const char* what, result_t r) {
  fprintf(stderr, "libutvb200: %s failed: %s\n", what,
          g_api.errorString ? g_api.errorString(r) : "nccl error");
  return UTV_ERR_COMM;
}
}  // namespace nccl

struct NcclComm final : Comm {
  nccl::comm_t c = nullptr;
  bool owned = false;
  ~NcclComm() override {
    if (owned && c) nccl::api()->commDestroy(c);
  }
  int allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
    if (count == 0) return UTV_OK;
    const nccl::result_t r = nccl::api()->allReduce(buf, buf, count, nccl::FLOAT64, nccl::SUM, c, st);
    return r ? nccl::fail("ncclAllReduce", r) : UTV_OK;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if (count == 0) return UTV_OK;
    const nccl::result_t r = nccl::api()->allGather(send, recv, count, nccl::FLOAT64, c, st);
    return r ? nccl::fail("ncclAllGather", r) : UTV_OK;
  }
  int broadcast(double* buf, size_t count, int root, cudaStream_t st) override {
    if (count == 0) return UTV_OK;
    const nccl::result_t r = nccl::api()->broadcast(buf, buf, count, nccl::FLOAT64, root, c, st);
    return r ? nccl::fail("ncclBroadcast", r) : UTV_OK;
  }
};

// ---------------------------------------------------------------------------
// local group (threads of one process)
// ---------------------------------------------------------------------------
namespace {
__global__ void add_kernel(double* __restrict__ acc, const double* __restrict__ x, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    acc[i] += x[i];
}

struct Hub {
  int size;
  int refs;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const double*> slot;
  explicit Hub(int p) : size(p), refs(p), slot(p, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
}  // namespace

struct LocalComm final : Comm {
  Hub* hub = nullptr;
  ~LocalComm() override {
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      last = (--hub->refs == 0);
    }
    if (last) delete hub;
  }
  // publish `p`, wait for every rank; the caller's queued work on `st`
  // (which produced p) must be complete before the peers read it
  int publish(const double* p, cudaStream_t st) {
    UTV_CUDA(cudaStreamSynchronize(st));
    hub->slot[rank] = p;
    hub->barrier();
    return UTV_OK;
  }
  int done(cudaStream_t st) {  // every rank finished reading every slot
    UTV_CUDA(cudaStreamSynchronize(st));
    hub->barrier();
    return UTV_OK;
  }
  int allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
    if (size == 1 || count == 0) return UTV_OK;
    double* acc = nullptr;
    UTV_CUDA(cudaMallocAsync((void**)&acc, count * sizeof(double), st));
    UTV_CHECK(publish(buf, st));
    UTV_CUDA(cudaMemcpyAsync(acc, hub->slot[0], count * sizeof(double), cudaMemcpyDefault, st));
    const int grid = (int)std::min<size_t>((count + 255) / 256, 4096);
    for (int p = 1; p < size; ++p) add_kernel<<<grid, 256, 0, st>>>(acc, hub->slot[p], count);
    UTV_CUDA(cudaGetLastError());
    UTV_CHECK(done(st));
    UTV_CUDA(cudaMemcpyAsync(buf, acc, count * sizeof(double), cudaMemcpyDefault, st));
    UTV_CUDA(cudaFreeAsync(acc, st));
    return UTV_OK;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if (count == 0) return UTV_OK;
    UTV_CHECK(publish(send, st));
    for (int p = 0; p < size; ++p)
      UTV_CUDA(cudaMemcpyAsync(recv + (size_t)p * count, hub->slot[p], count * sizeof(double),
                               cudaMemcpyDefault, st));
    return done(st);
  }
  int broadcast(double* buf, size_t count, int root, cudaStream_t st) override {
    if (size == 1 || count == 0) return UTV_OK;
    UTV_CHECK(publish(buf, st));
    if (rank != root)
      UTV_CUDA(cudaMemcpyAsync(buf, hub->slot[root], count * sizeof(double), cudaMemcpyDefault, st));
    return done(st);
  }
};

Comm* new_local_group(int nranks, Comm** out) {
  Hub* hub = new Hub(nranks);
  for (int r = 0; r < nranks; ++r) {
    LocalComm* c = new LocalComm();
    c->hub = hub;
    c->rank = r;
    c->size = nranks;
    out[r] = c;
  }
  return out[0];
}

}  // namespace utv

using namespace utv;

extern "C" {

int utv_comm_nccl_available(void) { return nccl::api() != nullptr; }

int utv_comm_nccl_unique_id(void* id128) {
  if (!id128) return -1;
  const nccl::Api* a = nccl::api();
  if (!a) return UTV_ERR_COMM;
  nccl::UniqueId id;
  const nccl::result_t r = a->getUniqueId(&id);
  if (r) return nccl::fail("ncclGetUniqueId", r);
  memcpy(id128, id.internal, sizeof(id.internal));
  return UTV_OK;
}

int utv_comm_init_nccl(const void* id128, int nranks, int rank, utv_comm_t* comm) {
  if (!id128) return -1;
  if (nranks < 1) return -2;
  if (rank < 0 || rank >= nranks) return -3;
  if (!comm) return -4;
  const nccl::Api* a = nccl::api();
  if (!a) return UTV_ERR_COMM;
  nccl::UniqueId id;
  memcpy(id.internal, id128, sizeof(id.internal));
  NcclComm* c = new NcclComm();
  const nccl::result_t r = a->commInitRank(&c->c, nranks, id, rank);
  if (r) {
    delete c;
    return nccl::fail("ncclCommInitRank", r);
  }
  c->owned = true;
  c->rank = rank;
  c->size = nranks;
  *comm = (utv_comm_s*)static_cast<Comm*>(c);
  return UTV_OK;
}

int utv_comm_from_nccl(void* nccl_comm, utv_comm_t* comm) {
  if (!nccl_comm) return -1;
  if (!comm) return -2;
  const nccl::Api* a = nccl::api();
  if (!a) return UTV_ERR_COMM;
  NcclComm* c = new NcclComm();
  c->c = (nccl::comm_t)nccl_comm;
  nccl::result_t r = a->commCount(c->c, &c->size);
  if (!r) r = a->commUserRank(c->c, &c->rank);
  if (r) {
    delete c;
    return nccl::fail("ncclCommCount/UserRank", r);
  }
  *comm = (utv_comm_s*)static_cast<Comm*>(c);
  return UTV_OK;
}

int utv_comm_init_local(int nranks, utv_comm_t* comms) {
  if (nranks < 1) return -1;
  if (!comms) return -2;
  std::vector<Comm*> tmp(nranks);
  new_local_group(nranks, tmp.data());
  for (int r = 0; r < nranks; ++r) comms[r] = (utv_comm_s*)tmp[r];
  return UTV_OK;
}

int utv_comm_rank(const utv_comm_s* comm) { return comm ? ((const Comm*)comm)->rank : -1; }
int utv_comm_size(const utv_comm_s* comm) { return comm ? ((const Comm*)comm)->size : -1; }

int utv_comm_destroy(utv_comm_s* comm) {
  delete (Comm*)comm;
  return UTV_OK;
}

int utv_comm_allreduce_sum_f64(utv_comm_s* comm, double* buf, size_t count, void* stream) {
  if (!comm) return -1;
  return ((Comm*)comm)->allreduce_sum(buf, count, (cudaStream_t)stream);
}

int utv_comm_allgather_f64(utv_comm_s* comm, const double* send, double* recv, size_t count,
                           void* stream) {
  if (!comm) return -1;
  return ((Comm*)comm)->allgather(send, recv, count, (cudaStream_t)stream);
}

int utv_comm_broadcast_f64(utv_comm_s* comm, double* buf, size_t count, int root, void* stream) {
  if (!comm) return -1;
  if (root < 0 || root >= ((Comm*)comm)->size) return -4;
  return ((Comm*)comm)->broadcast(buf, count, root, (cudaStream_t)stream);
}

}  // extern "C"

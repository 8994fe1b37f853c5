// Library-owned auxiliary streams and events for the software-pipelined
// drivers (randUTV's side-stream Jacobi SVD, the blocked QR's look-ahead
// panel).  Created once per process, non-blocking, highest priority: the
// latency-bound kernels they carry get their few CTAs dispatched ahead of
// the persistent GEMM tiles, which pick up the remaining SMs through the
// dynamic tile scheduler.
#include <mutex>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace {
constexpr int NSTREAMS = 4, NEVENTS = 16;
std::once_flag g_once;
int g_err = 0;
cudaStream_t g_streams[NSTREAMS];
cudaStream_t g_low = nullptr;  // lowest-priority stream for deferred, off-critical-path work
cudaEvent_t g_events[NEVENTS];
}  // namespace

static int init_aux() {
  std::call_once(g_once, [] {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) g_err = 1;
    for (int i = 0; i < NSTREAMS; ++i)
      if (cudaStreamCreateWithPriority(&g_streams[i], cudaStreamNonBlocking, hi) != cudaSuccess) g_err = 1;
    if (cudaStreamCreateWithPriority(&g_low, cudaStreamNonBlocking, lo) != cudaSuccess) g_err = 1;
    for (int i = 0; i < NEVENTS; ++i)
      if (cudaEventCreateWithFlags(&g_events[i], cudaEventDisableTiming) != cudaSuccess) g_err = 1;
  });
  return g_err ? UTV_ERR_CUDA : UTV_OK;
}

int aux_stream(int idx, cudaStream_t* s) {
  UTV_CHECK(init_aux());
  if (idx < 0 || idx >= NSTREAMS) return UTV_ERR_CUDA;
  *s = g_streams[idx];
  return UTV_OK;
}

int aux_stream_low(cudaStream_t* s) {
  UTV_CHECK(init_aux());
  *s = g_low;
  return UTV_OK;
}

// Per-caller-stream sets of look-ahead streams/events: two factorisations
// issued on different caller streams (e.g. independent TSQR leaves) must
// not share a side stream, or their latency-bound panels serialise.  The
// null key is the global set above.
namespace {
constexpr int NKEYS = 8;
struct AuxSet {
  cudaStream_t key;
  cudaStream_t streams[NSTREAMS];
  cudaEvent_t events[NEVENTS];
};
std::mutex g_keys_mu;
AuxSet g_keys[NKEYS];
int g_nkeys = 0;
}  // namespace

static int aux_set(cudaStream_t key, AuxSet** out) {
  UTV_CHECK(init_aux());
  std::lock_guard<std::mutex> lk(g_keys_mu);
  for (int i = 0; i < g_nkeys; ++i)
    if (g_keys[i].key == key) {
      *out = &g_keys[i];
      return UTV_OK;
    }
  if (g_nkeys == NKEYS) return UTV_ERR_CUDA;
  AuxSet& a = g_keys[g_nkeys];
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return UTV_ERR_CUDA;
  for (int i = 0; i < NSTREAMS; ++i)
    if (cudaStreamCreateWithPriority(&a.streams[i], cudaStreamNonBlocking, hi) != cudaSuccess)
      return UTV_ERR_CUDA;
  for (int i = 0; i < NEVENTS; ++i)
    if (cudaEventCreateWithFlags(&a.events[i], cudaEventDisableTiming) != cudaSuccess)
      return UTV_ERR_CUDA;
  a.key = key;
  ++g_nkeys;
  *out = &a;
  return UTV_OK;
}

int aux_stream_for(cudaStream_t key, int idx, cudaStream_t* s) {
  if (key == nullptr || key == cudaStreamLegacy || key == cudaStreamPerThread) return aux_stream(idx, s);
  if (idx < 0 || idx >= NSTREAMS) return UTV_ERR_CUDA;
  AuxSet* a = nullptr;
  const int rc = aux_set(key, &a);
  if (rc != UTV_OK) return aux_stream(idx, s);  // table full: fall back to the shared set
  *s = a->streams[idx];
  return UTV_OK;
}

int aux_event_for(cudaStream_t key, int idx, cudaEvent_t* e) {
  if (key == nullptr || key == cudaStreamLegacy || key == cudaStreamPerThread) return aux_event(idx, e);
  if (idx < 0 || idx >= NEVENTS) return UTV_ERR_CUDA;
  AuxSet* a = nullptr;
  const int rc = aux_set(key, &a);
  if (rc != UTV_OK) return aux_event(idx, e);
  *e = a->events[idx];
  return UTV_OK;
}

int aux_event(int idx, cudaEvent_t* e) {
  UTV_CHECK(init_aux());
  if (idx < 0 || idx >= NEVENTS) return UTV_ERR_CUDA;
  *e = g_events[idx];
  return UTV_OK;
}

// ---- process model guards ----
// The library binds to the first device it is used on (side streams, events,
// tile-scheduler slots, split-K turn counters and kernel attributes live on
// it): entry points called with another current device fail with
// UTV_ERR_DEVICE instead of touching foreign memory.
namespace {
std::once_flag g_dev_once;
int g_dev = -1;
std::mutex g_driver_mu;
}  // namespace

int check_device() {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess) return UTV_ERR_CUDA;
  std::call_once(g_dev_once, [d] { g_dev = d; });
  return d == g_dev ? UTV_OK : UTV_ERR_DEVICE;
}

// Drivers that use the shared side streams/events enqueue under this lock, so
// concurrent host threads cannot interleave their record/wait pairs.
std::mutex& driver_mutex() { return g_driver_mu; }

}  // namespace utv

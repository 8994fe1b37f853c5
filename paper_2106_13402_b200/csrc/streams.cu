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

int aux_event(int idx, cudaEvent_t* e) {
  UTV_CHECK(init_aux());
  if (idx < 0 || idx >= NEVENTS) return UTV_ERR_CUDA;
  *e = g_events[idx];
  return UTV_OK;
}

}  // namespace utv

// Launch accounting + optional per-kernel CUDA-event profiling.
//
// Every kernel launch site wraps itself in a ProfScope.  When profiling is
// off (default) this only bumps a launch counter; when on, a pair of CUDA
// events brackets the launch on its own stream so bench.py can report the
// device time, algorithmic FLOPs and bytes of each kernel family (the
// roofline inputs) without a profiler attached.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace {
struct Rec {
  int cat;
  cudaEvent_t a, b;
  double flops, bytes;
  cudaStream_t st;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::atomic<long long> g_launches{0};
cudaEvent_t g_ref = nullptr;       // timestamp origin of the profiled region
double g_busy[PROF_NCAT] = {0.0};  // union of launch intervals per category (ms)

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(int cat, double flops, double bytes, cudaStream_t st, int launches)
    : cat_(cat), flops_(flops), bytes_(bytes), st_(st), a_(nullptr) {
  g_launches += launches;
  if (!g_on) return;
  std::lock_guard<std::mutex> lk(g_mu);
  a_ = get_event();
  cudaEventRecord((cudaEvent_t)a_, st_);
}

ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t b = get_event();
  cudaEventRecord(b, st_);
  g_recs.push_back(Rec{cat_, (cudaEvent_t)a_, b, flops_, bytes_, st_});
}

}  // namespace utv

using namespace utv;

extern "C" {

long long utv_launch_count(void) { return g_launches.load(); }

void utv_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = true;
  g_recs.clear();
  if (!g_ref) cudaEventCreate(&g_ref);
  cudaEventRecord(g_ref, 0);
}

// Synchronises the device, then returns per-category totals:
// ms[c], flops[c], bytes[c], count[c] for c < PROF_NCAT.  Returns PROF_NCAT.
int utv_profile_end(double* ms, double* flops, double* bytes, long long* count) {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_mu);
  for (int c = 0; c < PROF_NCAT; ++c) {
    ms[c] = flops[c] = bytes[c] = 0.0;
    count[c] = 0;
  }
  std::vector<std::pair<float, float>> iv[PROF_NCAT];
  // UTV_PROF_DUMP=<file>: append one "cat,start_ms,end_ms,flops,stream" line per launch
  static const char* dump_path = getenv("UTV_PROF_DUMP");
  FILE* dump = dump_path ? fopen(dump_path, "a") : nullptr;
  for (auto& r : g_recs) {
    float t = 0.f, t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (cudaEventElapsedTime(&t0, g_ref, r.a) == cudaSuccess &&
        cudaEventElapsedTime(&t1, g_ref, r.b) == cudaSuccess)
      iv[r.cat].push_back({t0, t1});
    if (dump) fprintf(dump, "%d,%.4f,%.4f,%.6g,%p\n", r.cat, t0, t1, r.flops, (void*)r.st);
    ms[r.cat] += t;
    flops[r.cat] += r.flops;
    bytes[r.cat] += r.bytes;
    count[r.cat] += 1;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  // busy time = union of the category's launch intervals over all streams:
  // concurrent launches (the side-stream transforms) are not double-counted
  for (int c = 0; c < PROF_NCAT; ++c) {
    auto& v = iv[c];
    std::sort(v.begin(), v.end());
    double busy = 0.0, cs = -1.0, ce = -1.0;
    for (auto& x : v) {
      if (x.first > ce) {
        if (ce > cs) busy += ce - cs;
        cs = x.first;
        ce = x.second;
      } else if (x.second > ce) {
        ce = x.second;
      }
    }
    if (ce > cs) busy += ce - cs;
    g_busy[c] = busy;
  }
  if (dump) fclose(dump);
  g_recs.clear();
  g_on = false;
  return PROF_NCAT;
}

// Per-category busy time (ms) of the last utv_profile_end: the union of the
// launch intervals across streams.  Returns PROF_NCAT.
int utv_profile_busy(double* busy_ms) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (int c = 0; c < PROF_NCAT; ++c) busy_ms[c] = g_busy[c];
  return PROF_NCAT;
}

}  // extern "C"

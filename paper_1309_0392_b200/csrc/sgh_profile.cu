// sgh_profile.cu -- optional per-launch timing of the transform kernels.
//
// When enabled, every transform launch is bracketed by two CUDA events recorded
// on the stream the kernel is launched on, and tagged with the kernel kind and
// its algorithmic bytes (16 B per point the launch transforms: one read and one
// write).  bench.py uses this to report the roofline fraction of
// the dominant kernel measured inside the timed region.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "../../include/sgh.h"
#include "sgh_plan.hpp"

namespace sgh {

struct ProfRec {
  int kind, l, inv, variant, dev;
  double bytes;
  cudaEvent_t a, b;
};

static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_recs;
// free events, per device: an event may only be recorded on a stream of the
// device that was current when it was created
static std::vector<std::pair<int, cudaEvent_t>> g_pool;

static cudaEvent_t take_event() {
  int dev = 0;
  cudaGetDevice(&dev);
  for (size_t i = g_pool.size(); i-- > 0;) {
    if (g_pool[i].first != dev) continue;
    cudaEvent_t e = g_pool[i].second;
    g_pool.erase(g_pool.begin() + i);
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

bool prof_active() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  return g_prof_on;
}

ProfToken prof_begin(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return ProfToken{nullptr};
  cudaEvent_t a = take_event();
  cudaEventRecord(a, s);
  return ProfToken{a};
}

void prof_end(ProfToken tok, int kind, int l, bool inv, double bytes, cudaStream_t s, int variant) {
  if (!tok.start) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t b = take_event();
  cudaEventRecord(b, s);
  int dev = 0;
  cudaGetDevice(&dev);
  g_recs.push_back(ProfRec{kind, l, inv ? 1 : 0, variant, dev, bytes, tok.start, b});
}

}  // namespace sgh

using namespace sgh;

extern "C" {

sgh_status sgh_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (ProfRec &r : g_recs) {
    g_pool.emplace_back(r.dev, r.a);
    g_pool.emplace_back(r.dev, r.b);
  }
  g_recs.clear();
  g_prof_on = on != 0;
  return SGH_OK;
}

int64_t sgh_profile_read(sgh_launch_record *out, int64_t capacity) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int64_t n = (int64_t)g_recs.size();
  if (!out) return n;
  for (int64_t i = 0; i < n && i < capacity; ++i) {
    const ProfRec &r = g_recs[i];
    float ms = -1.f;
    if (cudaEventSynchronize(r.b) == cudaSuccess) cudaEventElapsedTime(&ms, r.a, r.b);
    out[i].kind = r.kind;
    out[i].level = r.l;
    out[i].inverse = r.inv;
    out[i].variant = r.variant;
    out[i].bytes = r.bytes;
    out[i].ms = ms;
  }
  return n;
}

}  // extern "C"

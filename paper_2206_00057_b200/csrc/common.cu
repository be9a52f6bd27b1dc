// Status text, launch counting and live event profiling (digest.h "profiling").
#include <atomic>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace dg {

static thread_local char g_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

digest_status set_error(digest_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

digest_status ok() { return DIGEST_OK; }

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

struct ProfRec {
  int cls, tag;
  cudaEvent_t a, b;
  double bytes, flops;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

Launch::Launch(int cls_, cudaStream_t s, double bytes_, double flops_, int tag)
    : cls(cls_), stream(s), bytes(bytes_), flops(flops_), slot(-1) {
  if (g_prof_on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRec r{cls, tag, get_event(), get_event(), bytes, flops};
    cudaEventRecord(r.a, stream);
    g_prof.push_back(r);
    slot = (int)g_prof.size() - 1;
  }
}

cudaError_t Launch::done() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (slot >= 0) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_prof[slot].b, stream);
  }
  return e;
}

}  // namespace dg

extern "C" {

const char* digest_last_error(void) { return dg::g_err; }

uint64_t digest_launch_count(void) { return dg::g_launches.load(); }

digest_status digest_prof_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(dg::g_prof_mu);
  for (auto& r : dg::g_prof) {
    dg::g_event_pool.push_back(r.a);
    dg::g_event_pool.push_back(r.b);
  }
  dg::g_prof.clear();
  dg::g_prof_on = on != 0;
  return DIGEST_OK;
}

digest_status digest_prof_read(double* ms_h, int64_t* launches_h, double* alg_bytes_h,
                               double* alg_flops_h) {
  std::lock_guard<std::mutex> lk(dg::g_prof_mu);
  for (int c = 0; c < DIGEST_PROF_CLASSES; ++c) {
    if (ms_h) ms_h[c] = 0;
    if (launches_h) launches_h[c] = 0;
    if (alg_bytes_h) alg_bytes_h[c] = 0;
    if (alg_flops_h) alg_flops_h[c] = 0;
  }
  for (auto& r : dg::g_prof) {
    DG_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    DG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    if (ms_h) ms_h[r.cls] += ms;
    if (launches_h) launches_h[r.cls] += 1;
    if (alg_bytes_h) alg_bytes_h[r.cls] += r.bytes;
    if (alg_flops_h) alg_flops_h[r.cls] += r.flops;
  }
  return DIGEST_OK;
}

digest_status digest_prof_read_detail(int32_t max_groups, int32_t* cls_h, int32_t* tag_h,
                                      double* ms_h, int64_t* launches_h, double* alg_bytes_h,
                                      double* alg_flops_h, int32_t* count_h) {
  DG_ARG(count_h && max_groups >= 0, DIGEST_E_INVALID, "bad argument");
  std::lock_guard<std::mutex> lk(dg::g_prof_mu);
  int n = 0;
  std::vector<std::pair<int, int>> keys;
  for (auto& r : dg::g_prof) {
    DG_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    DG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    int g = -1;
    for (int i = 0; i < (int)keys.size(); ++i)
      if (keys[i].first == r.cls && keys[i].second == r.tag) g = i;
    if (g < 0) {
      if (n >= max_groups) continue;
      keys.emplace_back(r.cls, r.tag);
      g = n++;
      cls_h[g] = r.cls;
      tag_h[g] = r.tag;
      ms_h[g] = 0;
      launches_h[g] = 0;
      alg_bytes_h[g] = 0;
      alg_flops_h[g] = 0;
    }
    ms_h[g] += ms;
    launches_h[g] += 1;
    alg_bytes_h[g] += r.bytes;
    alg_flops_h[g] += r.flops;
  }
  *count_h = n;
  return DIGEST_OK;
}

}  // extern "C"

namespace dg {
const char* knob(const char* name) {
  static const bool on = [] {
    const char* e = getenv("DIGEST_KNOBS");
    return e && atoi(e) == 1;
  }();
  return on ? getenv(name) : nullptr;
}
}  // namespace dg

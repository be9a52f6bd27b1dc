// Shared host/device helpers of libdigest.so: status/error text, launch
// accounting, live CUDA-event profiling of kernel classes, small device utils.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "digest.h"

namespace dg {

digest_status set_error(digest_status s, const char* fmt, ...);
digest_status ok();

// Records a kernel launch (for digest_launch_count) and, when profiling is on,
// the event pair around it.  Usage:  { Launch L(cls, stream, bytes, flops); kernel<<<>>>; L.done(); }
struct Launch {
  int cls;
  cudaStream_t stream;
  double bytes, flops;
  int slot;
  Launch(int cls_, cudaStream_t s, double bytes_ = 0.0, double flops_ = 0.0, int tag = 0);
  cudaError_t done();
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }
int num_sms();

// Experiment switches (kernel variants, schedules) read from the environment ONLY when
// DIGEST_KNOBS=1 is set: the product path ignores the environment otherwise.  Returns
// getenv(name) or NULL.
const char* knob(const char* name);

}  // namespace dg

#define DG_ARG(cond, status, ...)                                  \
  do {                                                             \
    if (!(cond)) return ::dg::set_error((status), __VA_ARGS__);    \
  } while (0)

#define DG_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return ::dg::set_error(DIGEST_E_CUDA, "%s failed: %s (%s:%d)", #call,               \
                             cudaGetErrorString(e_), __FILE__, __LINE__);                 \
  } while (0)

#define DG_TRY(call)                              \
  do {                                            \
    digest_status st_ = (call);                   \
    if (st_ != DIGEST_OK) return st_;             \
  } while (0)

// Launch a kernel with accounting: DG_LAUNCH(cls, stream, bytes, flops, kernel, grid, block, smem, args...)
#define DG_LAUNCH(cls, stream, bytes, flops, kern, grid, block, smem, ...) \
  DG_LAUNCH_TAG(cls, 0, stream, bytes, flops, kern, grid, block, smem, __VA_ARGS__)

// Same, with an integer tag (e.g. the SpMM width) for the per-(class, tag) profile.
#define DG_LAUNCH_TAG(cls, tag, stream, bytes, flops, kern, grid, block, smem, ...) \
  do {                                                                              \
    ::dg::Launch L_((cls), (stream), (bytes), (flops), (tag));                      \
    kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                       \
    DG_CUDA(L_.done());                                                             \
  } while (0)

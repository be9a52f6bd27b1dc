// Loss (Eq. 3), AGG (Alg. 1 line 13) and the local update
// (Adam per P:582).
#include <cmath>

#include "comm_internal.cuh"
#include "kernels.cuh"

namespace {

constexpr int kXentThreads = 256;

int xent_blocks(int64_t n) {
  int64_t b = dg::ceil_div(n, kXentThreads / 32);
  int64_t cap = (int64_t)dg::num_sms() * 8;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

// Warp per row: softmax cross-entropy over the first C columns.  Per-block partial
// loss sums (double) in a fixed order; k_sum_partials adds them in block order.
__global__ void __launch_bounds__(kXentThreads)
k_xent(const float* __restrict__ Z, int64_t n, int C, int64_t ld, const int32_t* __restrict__ y,
       const uint8_t* __restrict__ mask, float w, float* __restrict__ G, int64_t ldg,
       double* __restrict__ partial) {
  __shared__ double wsum[kXentThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t i = warp; i < n; i += nw) {
    const float* z = Z + i * ld;
    float* g = G + i * ldg;
    const bool t = mask[i] != 0;
    if (!t) {
      for (int c = lane; c < ldg; c += 32) g[c] = 0.f;
      continue;
    }
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, z[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s += expf(z[c] - m);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int yi = y[i];
    const float inv = 1.f / s;
    for (int c = lane; c < ldg; c += 32) {
      float v = 0.f;
      if (c < C) v = w * (expf(z[c] - m) * inv - (c == yi ? 1.f : 0.f));
      g[c] = v;
    }
    if (lane == 0) acc += (double)(m + logf(s) - z[yi]);
  }
  if (lane == 0) wsum[wib] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int k = 0; k < kXentThreads / 32; ++k) b += wsum[k];
    partial[blockIdx.x] = b * (double)w;
  }
}

// The same for C <= ld_g <= 64 (every BASELINE config): a lane owns columns lane and
// lane + 32, the row is read once into registers and the next row's logits, label and
// mask are loaded while the current row is reduced (two rows in flight per warp).  Same
// operations in the same order as k_xent, so the results are bit-identical.
__global__ void __launch_bounds__(kXentThreads)
k_xent64(const float* __restrict__ Z, int64_t n, int C, int64_t ld, const int32_t* __restrict__ y,
         const uint8_t* __restrict__ mask, float w, float* __restrict__ G, int64_t ldg,
         double* __restrict__ partial) {
  __shared__ double wsum[kXentThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool c0 = lane < C, c1 = lane + 32 < C;
  double acc = 0.0;
  float z0 = -INFINITY, z1 = -INFINITY;
  int yi = 0;
  bool t = false;
  // A row outside the training mask only gets its zero gradient row, so its logits are
  // not read (products: 8% of the rows train -- the logits read drops by 92%).
  auto load = [&](int64_t i) {
    const float* z = Z + i * ld;
    t = __ldg(mask + i) != 0;
    yi = __ldg(y + i);
    z0 = (c0 && t) ? __ldg(z + lane) : -INFINITY;
    z1 = (c1 && t) ? __ldg(z + lane + 32) : -INFINITY;
  };
  if (warp < n) load(warp);
  for (int64_t i = warp; i < n; i += nw) {
    const float a0 = z0, a1 = z1;
    const int yc = yi;
    const bool tc = t;
    if (i + nw < n) load(i + nw);   // next row in flight while this one is reduced
    float* g = G + i * ldg;
    if (!tc) {
      if (lane < ldg) g[lane] = 0.f;
      if (lane + 32 < ldg) g[lane + 32] = 0.f;
      continue;
    }
    float m = fmaxf(a0, a1);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float e0 = c0 ? expf(a0 - m) : 0.f, e1 = c1 ? expf(a1 - m) : 0.f;
    float s = 0.f;
    if (c0) s += e0;
    if (c1) s += e1;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float inv = 1.f / s;
    if (lane < ldg) g[lane] = c0 ? w * (e0 * inv - (lane == yc ? 1.f : 0.f)) : 0.f;
    if (lane + 32 < ldg) g[lane + 32] = c1 ? w * (e1 * inv - (lane + 32 == yc ? 1.f : 0.f)) : 0.f;
    const float zy = __shfl_sync(0xffffffffu, yc < 32 ? a0 : a1, yc & 31);
    if (lane == 0) acc += (double)(m + logf(s) - zy);
  }
  if (lane == 0) wsum[wib] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int k = 0; k < kXentThreads / 32; ++k) b += wsum[k];
    partial[blockIdx.x] = b * (double)w;
  }
}

__global__ void k_sum_partials(const double* __restrict__ partial, int nb, double* __restrict__ out) {
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += partial[b];
  *out = s;
}

__global__ void k_sgd(float* __restrict__ W, const float* __restrict__ G, int64_t n, float lr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    W[i] = fmaf(-lr, G[i], W[i]);
}

__global__ void k_adam(float* __restrict__ W, const float* __restrict__ G, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps,
                       float c1, float c2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float g = G[i];
    float mi = b1 * m[i] + (1.f - b1) * g;
    float vi = b2 * v[i] + (1.f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    W[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

// Adam with the step count on the device (CUDA-graph replay: no host argument changes
// between epochs).  t = *step + 1 is this update's step; k_step_incr advances it after.
__global__ void k_adam_dev(float* __restrict__ W, const float* __restrict__ G, float* __restrict__ m,
                           float* __restrict__ v, int64_t n, float lr, float b1, float b2,
                           float eps, const int64_t* __restrict__ step) {
  const double t = (double)(*step + 1);
  const float c1 = (float)(1.0 - pow((double)b1, t));
  const float c2 = (float)(1.0 - pow((double)b2, t));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float g = G[i];
    float mi = b1 * m[i] + (1.f - b1) * g;
    float vi = b2 * v[i] + (1.f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    W[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

__global__ void k_step_incr(int64_t* step) { *step += 1; }

__global__ void k_scale(float* __restrict__ x, int64_t n, float a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= a;
}

struct PtrTable {
  float* p[DIGEST_MAX_PARTS];
};

__global__ void k_sum_bufs(PtrTable t, int nb, int64_t n, float a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += t.p[b][i];
    s *= a;
    for (int b = 0; b < nb; ++b) t.p[b][i] = s;
  }
}

unsigned elt_blocks(int64_t n) {
  int64_t b = dg::ceil_div(n, 256);
  int64_t cap = (int64_t)dg::num_sms() * 8;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

extern "C" {

digest_status digest_xent_workspace(int64_t n, size_t* scratch_bytes_h) {
  DG_ARG(n >= 0 && scratch_bytes_h, DIGEST_E_INVALID, "bad argument");
  *scratch_bytes_h = sizeof(double) * (size_t)xent_blocks(n);
  return DIGEST_OK;
}

digest_status digest_xent(const float* logits, int64_t n, int32_t C, int64_t ld,
                          const int32_t* labels, const uint8_t* train_mask, float w_loss,
                          float* G_logits, int64_t ld_g, double* loss_out, void* scratch,
                          void* stream) {
  DG_ARG(n >= 0 && C >= 1 && ld >= C && ld_g >= C, DIGEST_E_SHAPE, "bad xent shape");
  DG_ARG(loss_out && scratch, DIGEST_E_INVALID, "loss_out/scratch NULL");
  cudaStream_t s = dg::as_stream(stream);
  if (n == 0) {
    DG_CUDA(cudaMemsetAsync(loss_out, 0, sizeof(double), s));
    return DIGEST_OK;
  }
  DG_ARG(logits && labels && train_mask && G_logits, DIGEST_E_INVALID, "NULL input");
  int nb = xent_blocks(n);
  double* part = reinterpret_cast<double*>(scratch);
  if (ld_g <= 64)
    DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * n * C, 0, k_xent64, nb, kXentThreads, 0, logits, n, C,
              ld, labels, train_mask, w_loss, G_logits, ld_g, part);
  else
    DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * n * C, 0, k_xent, nb, kXentThreads, 0, logits, n, C,
              ld, labels, train_mask, w_loss, G_logits, ld_g, part);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, k_sum_partials, 1, 1, 0, part, nb, loss_out);
  return DIGEST_OK;
}

digest_status digest_grad_allreduce(digest_comm* comm, float* grads, int64_t count, float scale,
                                    void* stream) {
  DG_ARG(grads && count >= 0, DIGEST_E_INVALID, "bad gradient buffer");
  cudaStream_t s = dg::as_stream(stream);
  if (dg::is_peer(comm)) return dg::peer_allreduce(comm, grads, count, scale, s);  // scale fused
  if (comm && comm->kind == 0) DG_TRY(dg::comm_allreduce_sum(comm, grads, count, s));
  if (scale != 1.0f && count > 0)
    DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * count, 0, k_scale, elt_blocks(count), 256, 0, grads,
              count, scale);
  return DIGEST_OK;
}

digest_status digest_grad_allreduce_local(float* const* bufs_h, int32_t n, int64_t count,
                                          float scale, void* stream) {
  DG_ARG(bufs_h && n >= 1 && n <= DIGEST_MAX_PARTS && count >= 0, DIGEST_E_INVALID,
         "bad buffer list");
  PtrTable t{};
  for (int i = 0; i < n; ++i) {
    DG_ARG(bufs_h[i], DIGEST_E_INVALID, "NULL buffer %d", i);
    t.p[i] = bufs_h[i];
  }
  if (count == 0) return DIGEST_OK;
  cudaStream_t s = dg::as_stream(stream);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * count * n, 0, k_sum_bufs, elt_blocks(count), 256, 0, t, n,
            count, scale);
  return DIGEST_OK;
}

digest_status digest_sgd_step(float* W, const float* G, int64_t count, float lr, void* stream) {
  DG_ARG(W && G && count >= 0, DIGEST_E_INVALID, "bad argument");
  if (count == 0) return DIGEST_OK;
  cudaStream_t s = dg::as_stream(stream);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 12.0 * count, 2.0 * count, k_sgd, elt_blocks(count), 256, 0, W,
            G, count, lr);
  return DIGEST_OK;
}

digest_status digest_adam_step(float* W, const float* G, float* m, float* v, int64_t count,
                               float lr, float b1, float b2, float eps, int64_t step,
                               void* stream) {
  DG_ARG(W && G && m && v && count >= 0 && step >= 1, DIGEST_E_INVALID, "bad argument");
  if (count == 0) return DIGEST_OK;
  cudaStream_t s = dg::as_stream(stream);
  float c1 = (float)(1.0 - std::pow((double)b1, (double)step));
  float c2 = (float)(1.0 - std::pow((double)b2, (double)step));
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 28.0 * count, 12.0 * count, k_adam, elt_blocks(count), 256, 0,
            W, G, m, v, count, lr, b1, b2, eps, c1, c2);
  return DIGEST_OK;
}

digest_status digest_adam_step_dev(float* W, const float* G, float* m, float* v, int64_t count,
                                   float lr, float b1, float b2, float eps, int64_t* step_dev,
                                   void* stream) {
  DG_ARG(W && G && m && v && step_dev && count >= 0, DIGEST_E_INVALID, "bad argument");
  cudaStream_t s = dg::as_stream(stream);
  if (count > 0)
    DG_LAUNCH(DIGEST_PROF_OTHER, s, 28.0 * count, 12.0 * count, k_adam_dev, elt_blocks(count), 256,
              0, W, G, m, v, count, lr, b1, b2, eps, step_dev);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, k_step_incr, 1, 1, 0, step_dev);
  return DIGEST_OK;
}

}  // extern "C"

// DIGEST-A parameter server (each subgraph "downloads/uploads parameters from
// the PS without blindly waiting for the slowest subgraph"; the aggregation
// moves into the subgraph loop).  Mixing rule (reading R1):
//     W_global <- (1 - alpha) W_global + alpha W_m      per upload, atomically.
//   * digest_ps_mix / digest_ps_download: W_global is a caller buffer (single process,
//     the loopback DIGEST-A run whose event order is an input);
//   * digest_ps_*_peer: W_global lives in rank 0's peer window; every upload/download
//     is one single-CTA kernel that holds a system-scope spin lock in that window
//     while it reads/writes W_global over NVLink, so concurrent uploads from
//     independent processes are atomic (no barrier anywhere).
#include "comm_internal.cuh"

namespace {

__global__ void k_ps_mix(float* __restrict__ Wg, const float* __restrict__ Wm, int64_t n, float a) {
  const float b = 1.f - a;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Wg[i] = fmaf(a, Wm[i], b * Wg[i]);
}

__global__ void k_copy_f(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__device__ __forceinline__ void lock_acquire(int64_t* lock) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long old;
    asm volatile("atom.acquire.sys.global.cas.b64 %0, [%1], 0, 1;"
                 : "=l"(old) : "l"(lock) : "memory");
    if (old == 0) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 30ull * 1000000000ull) {
      printf("digest: PS lock wait timed out\n");
      __trap();
    }
    __nanosleep(128);
  }
}

// mode 0: upload (mix W_m into W_global), 1: download (W_m <- W_global), 2: init (W_global <- W_m)
__global__ void __launch_bounds__(1024) k_ps_locked(float* Wg, float* Wm, int64_t n, float a,
                                                    int64_t* lock, int64_t* updates, int mode) {
  if (threadIdx.x == 0) lock_acquire(lock);
  __syncthreads();
  const float b = 1.f - a;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (mode == 0) {
      Wg[i] = fmaf(a, __ldcv(Wm + i), b * __ldcv(Wg + i));
    } else if (mode == 1) {
      Wm[i] = __ldcv(Wg + i);
    } else {
      Wg[i] = Wm[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (mode == 0) atomicAdd(reinterpret_cast<unsigned long long*>(updates), 1ull);
    __threadfence_system();
    asm volatile("st.release.sys.global.b64 [%0], 0;" ::"l"(lock) : "memory");
  }
}

__global__ void k_delay(int64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((int64_t)(t - t0) < ns);
}

unsigned blocks_for(int64_t n) {
  int64_t b = dg::ceil_div(n, 256);
  int64_t cap = (int64_t)dg::num_sms() * 4;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

digest_status ps_locked(digest_comm* c, float* W_local, int64_t count, float alpha, int mode,
                        cudaStream_t s) {
  DG_ARG(c && c->kind == 1 && c->connected, DIGEST_E_STATE,
         "the PS needs a connected peer-memory communicator");
  DG_ARG(W_local && count >= 0 && count <= c->max_grad, DIGEST_E_SHAPE,
         "PS of %lld floats exceeds the window's %lld", (long long)count, (long long)c->max_grad);
  char* w0 = c->peer_win[0];
  float* Wg = reinterpret_cast<float*>(w0 + dg::kWinSlots + sizeof(float) * 2 * (size_t)c->max_grad);
  int64_t* ps = dg::win_i64(w0, dg::kWinPs);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 12.0 * count, 3.0 * count, k_ps_locked, 1, 1024, 0, Wg, W_local,
            count, alpha, ps, ps + 1, mode);
  return DIGEST_OK;
}

}  // namespace

extern "C" {

digest_status digest_ps_mix(float* W_global, const float* W_local, int64_t count, float alpha,
                            void* stream) {
  DG_ARG(W_global && W_local && count >= 0, DIGEST_E_INVALID, "bad PS buffers");
  DG_ARG(alpha > 0.f && alpha <= 1.f, DIGEST_E_INVALID, "alpha must be in (0, 1]");
  if (count == 0) return DIGEST_OK;
  cudaStream_t s = dg::as_stream(stream);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 12.0 * count, 3.0 * count, k_ps_mix, blocks_for(count), 256, 0,
            W_global, W_local, count, alpha);
  return DIGEST_OK;
}

digest_status digest_ps_download(const float* W_global, float* W_local, int64_t count,
                                 void* stream) {
  DG_ARG(W_global && W_local && count >= 0, DIGEST_E_INVALID, "bad PS buffers");
  if (count == 0) return DIGEST_OK;
  cudaStream_t s = dg::as_stream(stream);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * count, 0, k_copy_f, blocks_for(count), 256, 0, W_global,
            W_local, count);
  return DIGEST_OK;
}

digest_status digest_ps_init_peer(digest_comm* comm, const float* W0, int64_t count, void* stream) {
  DG_ARG(comm && comm->rank == 0, DIGEST_E_INVALID, "only rank 0 initialises the PS");
  return ps_locked(comm, const_cast<float*>(W0), count, 1.f, 2, dg::as_stream(stream));
}

digest_status digest_ps_upload_peer(digest_comm* comm, const float* W_local, int64_t count,
                                    float alpha, void* stream) {
  DG_ARG(alpha > 0.f && alpha <= 1.f, DIGEST_E_INVALID, "alpha must be in (0, 1]");
  return ps_locked(comm, const_cast<float*>(W_local), count, alpha, 0, dg::as_stream(stream));
}

digest_status digest_ps_download_peer(digest_comm* comm, float* W_local, int64_t count,
                                      void* stream) {
  return ps_locked(comm, W_local, count, 1.f, 1, dg::as_stream(stream));
}

digest_status digest_ps_updates_peer(digest_comm* comm, int64_t* updates_h) {
  DG_ARG(comm && comm->kind == 1 && comm->connected && updates_h, DIGEST_E_INVALID,
         "bad argument");
  DG_CUDA(cudaMemcpy(updates_h, dg::win_i64(comm->peer_win[0], dg::kWinPs) + 1, sizeof(int64_t),
                     cudaMemcpyDeviceToHost));
  return DIGEST_OK;
}

digest_status digest_delay(int64_t ns, void* stream) {
  DG_ARG(ns >= 0, DIGEST_E_INVALID, "negative delay");
  if (ns == 0) return DIGEST_OK;
  DG_LAUNCH(DIGEST_PROF_OTHER, dg::as_stream(stream), 0, 0, k_delay, 1, 1, 0, ns);
  return DIGEST_OK;
}

}  // extern "C"

// Register-held vs shared-memory-staged (cp.async) random row gathers on this B200.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/gather_async tools/gather_async.cu
//
// The SpMM's narrow gathers are latency bound: every gathered byte in flight occupies a
// register until its FMA, so the register file caps the bytes in flight per SM.  This
// measures whether cp.async (LDGSTS: 16-byte global->shared copies, no register held)
// with an S-stage ring per warp moves more rows per second than register loads, for the
// SpMM's lane layout (warp = 8 groups x 4 lanes, a group gathers one row per edge slot,
// 16 rows per stage).  Rows are uniform random over footprints that fit L2 or not.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));    \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// register version: 16 rows per step (8 groups x UNR 2), VPL float4 per lane
template <int VPL>
__global__ void __launch_bounds__(256) k_reg(const uint32_t* __restrict__ idx, int64_t n,
                                             const char* __restrict__ X, uint32_t rb,
                                             float* out) {
  const int lane = threadIdx.x & 31, cl = lane & 3, g = lane >> 2;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc[VPL] = {};
  for (int64_t s = warp * 16; s < n; s += nw * 16) {
    float4 t[2][VPL];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t r = __ldg(idx + s + u * 8 + g);
      const float4* p = reinterpret_cast<const float4*>(X + (uint64_t)r * rb);
#pragma unroll
      for (int q = 0; q < VPL; ++q) t[u][q] = __ldg(p + cl + 4 * q);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        acc[q].x += t[u][q].x;
        acc[q].y += t[u][q].y;
        acc[q].z += t[u][q].z;
        acc[q].w += t[u][q].w;
      }
  }
  float z = 0.f;
#pragma unroll
  for (int q = 0; q < VPL; ++q) z += acc[q].x + acc[q].y + acc[q].z + acc[q].w;
  if (z == 1234.5f) out[warp] = z;
}

// cp.async version: S-stage ring per warp, stage = 16 rows x (16*VPL) floats
template <int VPL, int S, int WPC>
__global__ void __launch_bounds__(WPC * 32) k_async(const uint32_t* __restrict__ idx, int64_t n,
                                                    const char* __restrict__ X, uint32_t rb,
                                                    float* out) {
  extern __shared__ __align__(16) float4 ring[];   // [WPC][S][16 rows][4*VPL float4]
  const int lane = threadIdx.x & 31, cl = lane & 3, g = lane >> 2, wib = threadIdx.x >> 5;
  float4* my = ring + (size_t)wib * S * 16 * 4 * VPL;
  const int64_t warp = ((int64_t)blockIdx.x * WPC) + wib;
  const int64_t nw = (int64_t)gridDim.x * WPC;
  const int64_t nst = (n / 16 - warp + nw - 1) / nw;   // stages of this warp
  auto issue = [&](int64_t k) {
    float4* slot = my + (size_t)(k % S) * 16 * 4 * VPL;
    if (k < nst) {
      const int64_t s = (warp + k * nw) * 16;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t r = __ldg(idx + s + u * 8 + g);
        const float4* p = reinterpret_cast<const float4*>(X + (uint64_t)r * rb);
#pragma unroll
        for (int q = 0; q < VPL; ++q) cp16(slot + (u * 8 + g) * 4 * VPL + cl + 4 * q, p + cl + 4 * q);
      }
    }
    cp_commit();
  };
  float4 acc[VPL] = {};
#pragma unroll
  for (int k = 0; k < S - 1; ++k) issue(k);
  for (int64_t k = 0; k < nst; ++k) {
    issue(k + S - 1);
    cp_wait<S - 1>();
    const float4* slot = my + (size_t)(k % S) * 16 * 4 * VPL;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const float4 v = slot[(u * 8 + g) * 4 * VPL + cl + 4 * q];
        acc[q].x += v.x;
        acc[q].y += v.y;
        acc[q].z += v.z;
        acc[q].w += v.w;
      }
  }
  cp_wait<0>();
  float z = 0.f;
#pragma unroll
  for (int q = 0; q < VPL; ++q) z += acc[q].x + acc[q].y + acc[q].z + acc[q].w;
  if (z == 1234.5f) out[warp] = z;
}

static uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <typename F>
float best_ms(F launch, int reps) {
  launch();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  CK(cudaGetLastError());
  return best;
}

template <int VPL, int S, int WPC>
void run_async(const uint32_t* idx, int64_t n, const char* X, int w, float* out, int sms,
               double fp_mb) {
  const size_t smem = (size_t)WPC * S * 16 * 4 * VPL * 16;
  CK(cudaFuncSetAttribute(k_async<VPL, S, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_async<VPL, S, WPC>, WPC * 32, smem));
  const int grid = per_sm * sms;
  const float ms = best_ms([&] { k_async<VPL, S, WPC><<<grid, WPC * 32, smem>>>(idx, n, X, w * 4, out); }, 5);
  printf("{\"kind\": \"async\", \"width\": %d, \"footprint_mb\": %.0f, \"S\": %d, \"warps_per_sm\": %d, "
         "\"ms\": %.4f, \"gbs\": %.1f, \"grows_per_s\": %.2f}\n",
         w, fp_mb, S, per_sm * WPC, ms, n * (w * 4.0) / ms / 1e6, n / ms / 1e6);
  fflush(stdout);
}

template <int VPL>
void run_reg(const uint32_t* idx, int64_t n, const char* X, int w, float* out, int sms,
             double fp_mb) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reg<VPL>, 256, 0));
  const int grid = per_sm * sms;
  const float ms = best_ms([&] { k_reg<VPL><<<grid, 256>>>(idx, n, X, w * 4, out); }, 5);
  printf("{\"kind\": \"reg\", \"width\": %d, \"footprint_mb\": %.0f, \"warps_per_sm\": %d, "
         "\"ms\": %.4f, \"gbs\": %.1f, \"grows_per_s\": %.2f}\n",
         w, fp_mb, per_sm * 8, ms, n * (w * 4.0) / ms / 1e6, n / ms / 1e6);
  fflush(stdout);
}

int main() {
  CK(cudaSetDevice(0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n = 64ll << 20;
  std::vector<uint32_t> h(n);
  uint32_t* idx;
  CK(cudaMalloc(&idx, n * 4));
  float* out;
  CK(cudaMalloc(&out, 1 << 24));
  const double fps[] = {32, 64, 470, 2500};
  for (int w : {48, 64}) {
    for (double fp : fps) {
      const int64_t rows = (int64_t)(fp * 1e6 / (w * 4.0));
      char* X;
      CK(cudaMalloc(&X, (size_t)rows * w * 4));
      CK(cudaMemset(X, 0, (size_t)rows * w * 4));
      uint64_t s = 99 + w;
      for (int64_t i = 0; i < n; ++i) h[i] = (uint32_t)(splitmix(s) % (uint64_t)rows);
      CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
      if (w == 48) {
        run_reg<3>(idx, n, X, w, out, sms, fp);
        run_async<3, 2, 4>(idx, n, X, w, out, sms, fp);
        run_async<3, 4, 4>(idx, n, X, w, out, sms, fp);
        run_async<3, 6, 4>(idx, n, X, w, out, sms, fp);
        run_async<3, 8, 2>(idx, n, X, w, out, sms, fp);
      } else {
        run_reg<4>(idx, n, X, w, out, sms, fp);
        run_async<4, 2, 4>(idx, n, X, w, out, sms, fp);
        run_async<4, 4, 4>(idx, n, X, w, out, sms, fp);
        run_async<4, 6, 2>(idx, n, X, w, out, sms, fp);
      }
      CK(cudaFree(X));
    }
  }
  return 0;
}

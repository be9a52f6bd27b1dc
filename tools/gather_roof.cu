// Row-gather ceilings of this B200: how fast can the SMs pull randomly indexed rows of
// an fp32 matrix, as a function of the row width and of the matrix footprint (L2-resident
// vs HBM-resident)?  This is the roof the SpMM's edge gathers meet;
// measured here instead of borrowing a B300 constant.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/gather_roof tools/gather_roof.cu
//   tools/gather_roof            # prints one JSON line per (width, footprint, variant)
//
// Kernel: persistent grid, one warp per block of 32 random row indices; the warp splits
// into EG = 32/LC groups of LC lanes, lane c of a group owns float4 columns c, c+LC, ...
// (VPL of them), UNR rows per group in flight -- the same lane layout as the library's
// SpMM, without the CSR (pure gathers + FADD).  Bytes counted: rows x width x 4 (the
// gathered payload) + 4 B per index.  Time: CUDA events, best of 5 after a warm-up.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

template <int LC, int VPL, int UNR>
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ idx, int64_t n_idx,
                                                const float* __restrict__ X, uint32_t row_bytes,
                                                int w4, float* out) {
  constexpr int EG = 32 / LC;
  const int lane = threadIdx.x & 31, cl = lane % LC, g = lane / LC;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  const char* base = reinterpret_cast<const char*>(X);
  for (int64_t b = warp * 32; b < n_idx; b += nwarps * 32) {
    const uint32_t my = b + lane < n_idx ? __ldg(idx + b + lane) : 0u;
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += EG * UNR) {
      float4 t[UNR][VPL];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint32_t r = __shfl_sync(0xffffffffu, my, j0 + u * EG + g);
        const float4* p = reinterpret_cast<const float4*>(base + (uint64_t)r * row_bytes);
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int c = cl + q * LC;
          t[u][q] = (g < EG && c < w4) ? __ldg(p + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          acc[q].x += t[u][q].x;
          acc[q].y += t[u][q].y;
          acc[q].z += t[u][q].z;
          acc[q].w += t[u][q].w;
        }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < VPL; ++q) s += acc[q].x + acc[q].y + acc[q].z + acc[q].w;
  if (s == 1234.5f) out[warp] = s;   // keeps the loads alive
}

// Streaming read of the same bytes (sequential rows): the HBM/L2 streaming reference.
__global__ void k_stream(const float4* __restrict__ X, int64_t n4, float* out) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(X + i);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

static uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <int LC, int VPL, int UNR>
float time_gather(const uint32_t* idx, int64_t n, const float* X, int w, float* out, int sms,
                  const char* name, int64_t rows, int reps) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather<LC, VPL, UNR>, 256, 0));
  const int grid = per_sm * sms;
  const uint32_t rb = (uint32_t)w * 4;
  k_gather<LC, VPL, UNR><<<grid, 256>>>(idx, n, X, rb, w / 4, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    k_gather<LC, VPL, UNR><<<grid, 256>>>(idx, n, X, rb, w / 4, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  const double bytes = (double)n * (w * 4.0 + 4.0);
  printf("{\"kind\": \"gather\", \"variant\": \"%s\", \"width\": %d, \"rows\": %lld, "
         "\"footprint_mb\": %.1f, \"gathers\": %lld, \"ms\": %.4f, \"gbs\": %.1f, "
         "\"grows_per_s\": %.3f, \"ctas_per_sm\": %d}\n",
         name, w, (long long)rows, rows * w * 4.0 / 1e6, (long long)n, best, bytes / best / 1e6,
         n / best / 1e6, per_sm);
  fflush(stdout);
  CK(cudaEventDestroy(a));
  CK(cudaEventDestroy(b));
  return best;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t n_idx = 64ll << 20;   // 64 Mi gathers per launch
  const int reps = 5;
  std::vector<uint32_t> h(n_idx);
  uint32_t* d_idx;
  CK(cudaMalloc(&d_idx, n_idx * 4));
  float* out;
  CK(cudaMalloc(&out, 1 << 24));
  const int widths[] = {48, 100, 256};
  // footprints: L2-resident (16, 48 MB), around L2 (96, 160 MB), HBM-resident (2.5 GB)
  const double fps_mb[] = {16, 48, 96, 160, 2500};
  for (int w : widths) {
    for (double fp : fps_mb) {
      const int64_t rows = (int64_t)(fp * 1e6 / (w * 4.0));
      float* X;
      CK(cudaMalloc(&X, (size_t)rows * w * 4));
      CK(cudaMemset(X, 0, (size_t)rows * w * 4));
      uint64_t s = 12345 + w;
      for (int64_t i = 0; i < n_idx; ++i) h[i] = (uint32_t)(splitmix(s) % (uint64_t)rows);
      CK(cudaMemcpy(d_idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
      if (w == 48) {
        time_gather<4, 3, 2>(d_idx, n_idx, X, w, out, sms, "LC4xVPL3xUNR2", rows, reps);
        time_gather<4, 3, 4>(d_idx, n_idx, X, w, out, sms, "LC4xVPL3xUNR4", rows, reps);
        time_gather<2, 6, 2>(d_idx, n_idx, X, w, out, sms, "LC2xVPL6xUNR2", rows, reps);
        time_gather<16, 1, 2>(d_idx, n_idx, X, w, out, sms, "LC16xVPL1xUNR2", rows, reps);
      } else if (w == 100) {
        time_gather<8, 4, 2>(d_idx, n_idx, X, w, out, sms, "LC8xVPL4xUNR2", rows, reps);
        time_gather<8, 4, 4>(d_idx, n_idx, X, w, out, sms, "LC8xVPL4xUNR4", rows, reps);
        time_gather<4, 7, 2>(d_idx, n_idx, X, w, out, sms, "LC4xVPL7xUNR2", rows, reps);
      } else {
        time_gather<32, 2, 4>(d_idx, n_idx, X, w, out, sms, "LC32xVPL2xUNR4", rows, reps);
        time_gather<32, 2, 8>(d_idx, n_idx, X, w, out, sms, "LC32xVPL2xUNR8", rows, reps);
        time_gather<16, 4, 4>(d_idx, n_idx, X, w, out, sms, "LC16xVPL4xUNR4", rows, reps);
      }
      CK(cudaFree(X));
    }
  }
  // streaming reference over 2.5 GB
  {
    const int64_t n4 = (int64_t)(2.5e9 / 16);
    float4* X;
    CK(cudaMalloc(&X, n4 * 16));
    CK(cudaMemset(X, 0, n4 * 16));
    k_stream<<<sms * 8, 256>>>(X, n4, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(a));
      k_stream<<<sms * 8, 256>>>(X, n4, out);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    printf("{\"kind\": \"stream_read\", \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           n4 * 16.0, best, n4 * 16.0 / best / 1e6);
    CK(cudaFree(X));
  }
  return 0;
}

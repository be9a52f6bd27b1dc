// Measure tcgen05.mma issue throughput (cycles per MMA, M=128, N=256) for
// kind::tf32 K-major and kind::f16 (bf16) K-major / MN-major operands.
// One CTA per SM; each issues `iters` MMAs on zero operands into TMEM.
#include <cstdio>
#include <vector>
#include "tc_util.cuh"
using namespace dg;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__global__ void rate(int kind, int mn, int iters, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
  uint64_t* bar = (uint64_t*)(sm + 65536 * 2);
  uint32_t* slot = (uint32_t*)(bar + 1);
  for (int i = threadIdx.x; i < 65536 * 2 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) { tc::mbar_init(bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x / 32 == 0) tc::tmem_alloc(slot, 256);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = *slot;
  if (threadIdx.x == 0) {
    const int N = 256, M = 128;
    uint32_t idesc = (1u << 4) | ((kind ? 1u : 2u) << 7) | ((kind ? 1u : 2u) << 10) |
                     ((uint32_t)mn << 15) | ((uint32_t)mn << 16) | ((uint32_t)(N >> 3) << 17) |
                     ((uint32_t)(M >> 4) << 24);
    uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 65536);
    uint64_t da = mn ? tc::smem_desc_sw128(a, 2048, 1024) : tc::smem_desc_sw128(a, 16, 1024);
    uint64_t db = mn ? tc::smem_desc_sw128(b, 2048, 1024) : tc::smem_desc_sw128(b, 16, 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (kind) mma_f16(tm, da, db, idesc, i > 0);
      else tc::mma_tf32(tm, da, db, idesc, i > 0);
    }
    tc::mma_commit(bar);
    tc::mbar_wait(bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before(); __syncthreads();
  if (threadIdx.x / 32 == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tm, 256); }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int sms = 148;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2 + 2048);
  const char* names[3] = {"tf32 K-major", "bf16 K-major", "bf16 MN-major"};
  int cfg[3][2] = {{0, 0}, {1, 0}, {1, 1}};
  for (int v = 0; v < 3; ++v) {
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    rate<<<sms, 128, 65536 * 2 + 2048>>>(cfg[v][0], cfg[v][1], 100, d);
    cudaEventRecord(e0);
    rate<<<sms, 128, 65536 * 2 + 2048>>>(cfg[v][0], cfg[v][1], iters, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> h(sms);
    cudaMemcpy(h.data(), d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0; for (auto x : h) avg += x; avg /= sms;
    int K = cfg[v][0] ? 16 : 8;
    double flops = 2.0 * 128 * 256 * K * (double)iters * sms;
    printf("%-14s %s: %.1f cycles/MMA, %.1f TFLOP/s (chip, %.3f ms)\n", names[v],
           cudaGetErrorString(e), avg / iters, flops / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}

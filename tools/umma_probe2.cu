// Probe MN-major operand support: kind::f16 (bf16) vs kind::tf32, per-operand transpose bits.
#include <cstdio>
#include <vector>
#include <cmath>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include "tc_util.cuh"
using namespace dg;
constexpr int M = 128, N = 64;
bool tmap(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esize, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) { cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q); }
  cuuint64_t dims[2] = {inner, outer}; cuuint64_t strides[1] = {inner * esize};
  cuuint32_t box[2] = {bi, bo}; cuuint32_t estr[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
__device__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// kind: 0 = tf32, 1 = bf16. a_mn/b_mn: operand majorness. Operand tiles: K-major: one box (rows = M or N, inner = K);
// MN-major: boxes of (inner = 128 B of MN, rows = K), consecutive.
__global__ void probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, int kind, int a_mn, int b_mn,
                      int K, int esize, float* C) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm; uint8_t* sB = sm + 16384;
  uint64_t* bar = (uint64_t*)(sm + 32768);
  uint32_t* slot = (uint32_t*)(bar + 2);
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::fence_mbar_init(); }
  if (warp == 1) tc::tmem_alloc(slot, 64);
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = *slot;
  const int run = 128 / esize;                 // elements per 128 B
  if (threadIdx.x == 0) {
    uint32_t bytesA = M * K * esize, bytesB = N * K * esize;
    tc::mbar_arrive_expect_tx(&bar[0], bytesA + bytesB);
    uint32_t boxA = a_mn ? K * 128 : 0, boxB = b_mn ? K * 128 : 0;
    if (a_mn) for (int j = 0; j < M / run; ++j) tc::tma_load_2d(sA + j * boxA, &tA, &bar[0], run * j, 0);
    else tc::tma_load_2d(sA, &tA, &bar[0], 0, 0);
    if (b_mn) for (int j = 0; j < N / run; ++j) tc::tma_load_2d(sB + j * boxB, &tB, &bar[0], run * j, 0);
    else tc::tma_load_2d(sB, &tB, &bar[0], 0, 0);
    tc::mbar_wait(&bar[0], 0);
    tc::tc_fence_after();
    uint32_t idesc = (1u << 4) | ((kind ? 1u : 2u) << 7) | ((kind ? 1u : 2u) << 10) | ((uint32_t)a_mn << 15) |
                     ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    int kper = 32 / esize;   // K per MMA instruction
    for (int k = 0; k < K / kper; ++k) {
      // K-major: advance 32 B along the row; MN-major: advance kper rows of 128 B
      uint32_t offA = a_mn ? k * kper * 128 : k * 32, offB = b_mn ? k * kper * 128 : k * 32;
      uint64_t da = a_mn ? tc::smem_desc_sw128(tc::smem_u32(sA) + offA, boxA, 1024) : tc::smem_desc_sw128(tc::smem_u32(sA) + offA, 16, 1024);
      uint64_t db = b_mn ? tc::smem_desc_sw128(tc::smem_u32(sB) + offB, boxB, 1024) : tc::smem_desc_sw128(tc::smem_u32(sB) + offB, 16, 1024);
      if (kind) mma_f16(tm, da, db, idesc, k > 0); else tc::mma_tf32(tm, da, db, idesc, k > 0);
    }
    tc::mma_commit(&bar[1]);
  }
  __syncwarp();
  tc::mbar_wait(&bar[1], 0);
  tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tc::tmem_ld_32x32b_x32(tm + ((uint32_t)(warp * 32) << 16) + c0, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) C[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before(); __syncthreads();
  if (warp == 1) { tc::tc_fence_after(); tc::tmem_dealloc(tm, 64); }
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  float* dC; cudaMalloc(&dC, 4 * M * N);
  for (int kind = 0; kind < 2; ++kind) {
    int esize = kind ? 2 : 4, K = kind ? 64 : 32;
    std::vector<float> a(M * K), b(N * K);
    srand(3);
    for (auto& x : a) x = (float)(rand() % 9 - 4);
    for (auto& x : b) x = (float)(rand() % 7 - 3);
    std::vector<double> ref(M * N, 0.0);
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) ref[m * N + n] += (double)a[m * K + k] * b[n * K + k];
    for (int a_mn = 0; a_mn < 2; ++a_mn) for (int b_mn = 0; b_mn < 2; ++b_mn) {
      std::vector<uint8_t> ha(M * K * esize), hb(N * K * esize);
      auto put = [&](std::vector<uint8_t>& h, int idx, float v) {
        if (esize == 4) memcpy(&h[idx * 4], &v, 4); else { __nv_bfloat16 x = __float2bfloat16(v); memcpy(&h[idx * 2], &x, 2); } };
      for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) put(ha, a_mn ? k * M + m : m * K + k, a[m * K + k]);
      for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) put(hb, b_mn ? k * N + n : n * K + k, b[n * K + k]);
      void *dA, *dB; cudaMalloc(&dA, ha.size()); cudaMalloc(&dB, hb.size());
      cudaMemcpy(dA, ha.data(), ha.size(), cudaMemcpyHostToDevice); cudaMemcpy(dB, hb.data(), hb.size(), cudaMemcpyHostToDevice);
      CUtensorMapDataType dt = kind ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
      int run = 128 / esize;
      CUtensorMap tA, tB;
      bool ok = (a_mn ? tmap(&tA, dA, dt, esize, M, K, run, K) : tmap(&tA, dA, dt, esize, K, M, run, M)) &&
                (b_mn ? tmap(&tB, dB, dt, esize, N, K, run, K) : tmap(&tB, dB, dt, esize, K, N, run, N));
      cudaMemset(dC, 0, 4 * M * N);
      probe<<<1, 128, 40960>>>(tA, tB, kind, a_mn, b_mn, K, esize, dC);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> c(M * N);
      cudaMemcpy(c.data(), dC, 4 * M * N, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0; int nz = 0;
      for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(c[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); nz += c[i] != 0; }
      printf("%s A%s B%s tmap=%d %s rel=%.3g nonzero=%d\n", kind ? "bf16" : "tf32", a_mn ? "MN" : "K ", b_mn ? "MN" : "K ",
             ok, cudaGetErrorString(e), err / mx, nz);
      cudaFree(dA); cudaFree(dB);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}

// Standalone probe of tcgen05 kind::tf32 operand layouts (K-major vs MN-major, SW128).
// C[128 x N] = sum_k A(m,k) B(n,k), one CTA, K = 16 (two K=8 MMAs).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "tc_util.cuh"
using namespace dg;
constexpr int M = 128, N = 64, K = 32;
__global__ void probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                      int mn_major, uint32_t lbo, uint32_t sbo, uint32_t kstep_bytes, float* C) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                 // 16 KB
  uint8_t* sB = sm + 16384;         // 8 KB
  uint64_t* bar = (uint64_t*)(sm + 24576);
  uint32_t* slot = (uint32_t*)(bar + 2);
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::fence_mbar_init(); }
  if (warp == 1) tc::tmem_alloc(slot, 64);
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  uint32_t tm = *slot;
  if (threadIdx.x == 0) {
    tc::mbar_arrive_expect_tx(&bar[0], 16384 + 8192);
    if (mn_major) {
      for (int j = 0; j < 4; ++j) tc::tma_load_2d(sA + j * 4096, &tA, &bar[0], 32 * j, 0);
      for (int j = 0; j < 2; ++j) tc::tma_load_2d(sB + j * 4096, &tB, &bar[0], 32 * j, 0);
    } else {
      tc::tma_load_2d(sA, &tA, &bar[0], 0, 0);
      tc::tma_load_2d(sB, &tB, &bar[0], 0, 0);
    }
    tc::mbar_wait(&bar[0], 0);
    tc::tc_fence_after();
    uint32_t idesc = tc::idesc_tf32(M, N, mn_major, mn_major);
    for (int k = 0; k < K / 8; ++k) {
      uint64_t da = tc::smem_desc_sw128(tc::smem_u32(sA) + k * kstep_bytes, lbo, sbo);
      uint64_t db = tc::smem_desc_sw128(tc::smem_u32(sB) + k * kstep_bytes, lbo, sbo);
      tc::mma_tf32(tm, da, db, idesc, k > 0);
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
  std::vector<float> a(M * K), b(N * K);   // logical A(m,k), B(n,k)
  srand(1);
  for (auto& x : a) x = (float)(rand() % 17 - 8);
  for (auto& x : b) x = (float)(rand() % 13 - 6);
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) ref[m * N + n] += (double)a[m * K + k] * b[n * K + k];
  // K-major buffers: A [M][K], B [N][K]; MN-major buffers: A [K][M], B [K][N]
  std::vector<float> aK(a), bK(b), aM(K * M), bM(K * N);
  for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) aM[k * M + m] = a[m * K + k];
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) bM[k * N + n] = b[n * K + k];
  float *dAK, *dBK, *dAM, *dBM, *dC;
  cudaMalloc(&dAK, 4 * M * K); cudaMalloc(&dBK, 4 * N * K); cudaMalloc(&dAM, 4 * M * K); cudaMalloc(&dBM, 4 * N * K);
  cudaMalloc(&dC, 4 * M * N);
  cudaMemcpy(dAK, aK.data(), 4 * M * K, cudaMemcpyHostToDevice); cudaMemcpy(dBK, bK.data(), 4 * N * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dAM, aM.data(), 4 * M * K, cudaMemcpyHostToDevice); cudaMemcpy(dBM, bM.data(), 4 * N * K, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  struct V { const char* name; int mn; uint32_t lbo, sbo, kstep; };
  V vs[] = {{"K-major (control)", 0, 16, 1024, 32}, {"MN lbo=4096 sbo=1024", 1, 4096, 1024, 1024},
            {"MN lbo=1024 sbo=4096", 1, 1024, 4096, 1024}};
  for (auto& v : vs) {
    CUtensorMap tA, tB;
    bool ok;
    if (v.mn) ok = make_tmap_2d(&tA, dAM, M, K, 4 * M, 32, K) && make_tmap_2d(&tB, dBM, N, K, 4 * N, 32, K);
    else ok = make_tmap_2d(&tA, dAK, K, M, 4 * K, 32, M) && make_tmap_2d(&tB, dBK, K, N, 4 * K, 32, N);
    cudaMemset(dC, 0, 4 * M * N);
    probe<<<1, 128, 40960>>>(tA, tB, v.mn, v.lbo, v.sbo, v.kstep, dC);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> c(M * N);
    cudaMemcpy(c.data(), dC, 4 * M * N, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0; int nz = 0;
    for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(c[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); nz += c[i] != 0; }
    printf("%-24s tmap=%d err=%s rel=%.3g nonzero=%d c[0..3]=%g %g %g %g ref=%g %g %g %g\n", v.name, ok,
           cudaGetErrorString(e), err / mx, nz, c[0], c[1], c[2], c[3], ref[0], ref[1], ref[2], ref[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}

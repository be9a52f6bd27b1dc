// FP32 CUDA-core GEMMs: the generic-stride product used where the tensor-core
// path does not apply (tiny or oddly strided shapes), the split-K weight gradient
// (Eq. 6: G_W = (P_m X_ext)^T D, K = rows of the partition), and the ReLU mask.
// Accumulation is fp32 FFMA (the oracle's tolerance, 1e-4, is met without
// compensation).
#include "kernels.cuh"

namespace dg {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
constexpr int kThreads = (BM / TM) * (BN / TN);  // 256

// One 64x64 output tile; k range [k0, k1).  out = C (+relu) or a dense partial.
__global__ void __launch_bounds__(kThreads)
k_gemm(GemmArgs g, int64_t k_per_split, float* partial) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int64_t i0 = (int64_t)blockIdx.y * BM;
  const int j0 = blockIdx.x * BN;
  const int64_t k0 = (int64_t)blockIdx.z * k_per_split;
  const int64_t k1 = min(g.K, k0 + k_per_split);
  const bool a_kfast = g.sAk == 1;
  const bool b_jfast = g.sBj == 1;
  float acc[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = 0.f;

  for (int64_t kb = k0; kb < k1; kb += BK) {
#pragma unroll
    for (int q = 0; q < (BM * BK) / kThreads; ++q) {
      int idx = tid + q * kThreads;
      int i, k;
      if (a_kfast) { i = idx / BK; k = idx % BK; } else { k = idx / BM; i = idx % BM; }
      int64_t gi = i0 + i, gk = kb + k;
      As[k][i] = (gi < g.M && gk < k1) ? __ldg(g.A + gi * g.sAi + gk * g.sAk) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < (BN * BK) / kThreads; ++q) {
      int idx = tid + q * kThreads;
      int j, k;
      if (b_jfast) { k = idx / BN; j = idx % BN; } else { j = idx / BK; k = idx % BK; }
      int gj = j0 + j;
      int64_t gk = kb + k;
      Bs[k][j] = (gj < g.N && gk < k1) ? __ldg(g.B + gk * g.sBk + (int64_t)gj * g.sBj) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int r = 0; r < TM; ++r) a[r] = As[k][ty + r * (BM / TM)];
#pragma unroll
      for (int c = 0; c < TN; ++c) b[c] = Bs[k][tx + c * (BN / TN)];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < TM; ++r) {
    int64_t gi = i0 + ty + r * (BM / TM);
    if (gi >= g.M) continue;
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      int gj = j0 + tx + c * (BN / TN);
      if (gj >= g.N) continue;
      float v = acc[r][c];
      if (partial) {
        partial[((int64_t)blockIdx.z * g.M + gi) * g.N + gj] = v;
      } else {
        if (g.relu) v = fmaxf(v, 0.f);
        if (g.mask && !(g.mask[gi * g.ldm + gj] > 0.f)) v = 0.f;
        if (g.mbits && !mask_bit(g.mbits, g.ldmb, gi, gj)) v = 0.f;
        g.C[gi * g.ldc + gj] = v;
      }
    }
  }
}

// C[i*N + j] = sum_{z < nsplit} partial[z][i][j], fixed order.
__global__ void k_reduce_splits(const float* __restrict__ partial, int64_t nsplit, int64_t MN,
                                float* __restrict__ C) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < MN;
       t += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t z = 0; z < nsplit; ++z) s += partial[z * MN + t];
    C[t] = s;
  }
}

__global__ void k_relu_mask(const float* __restrict__ G, int64_t ldg, const float* __restrict__ H,
                            int64_t ldh, float* __restrict__ D, int64_t ldd, int64_t n, int w4) {
  int64_t total = n * w4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / w4;
    int c = (int)(t % w4);
    float4 g = reinterpret_cast<const float4*>(G + i * ldg)[c];
    float4 h = reinterpret_cast<const float4*>(H + i * ldh)[c];
    g.x = h.x > 0.f ? g.x : 0.f;
    g.y = h.y > 0.f ? g.y : 0.f;
    g.z = h.z > 0.f ? g.z : 0.f;
    g.w = h.w > 0.f ? g.w : 0.f;
    reinterpret_cast<float4*>(D + i * ldd)[c] = g;
  }
}

__global__ void k_relu_mask_bits(const float* __restrict__ G, int64_t ldg,
                                 const uint32_t* __restrict__ mb, int64_t ldmb,
                                 float* __restrict__ D, int64_t ldd, int64_t n, int w4) {
  int64_t total = n * w4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / w4;
    int c = (int)(t % w4);
    float4 g = reinterpret_cast<const float4*>(G + i * ldg)[c];
    const uint32_t m = __ldg(mb + i * ldmb + (c >> 3)) >> ((c & 7) * 4);
    g.x = (m & 1u) ? g.x : 0.f;
    g.y = (m & 2u) ? g.y : 0.f;
    g.z = (m & 4u) ? g.z : 0.f;
    g.w = (m & 8u) ? g.w : 0.f;
    reinterpret_cast<float4*>(D + i * ldd)[c] = g;
  }
}

// one warp per (row, word): lane j tests column 32*word + j
__global__ void k_sign_bits(const float* __restrict__ C, int64_t ldc, int64_t n, int w,
                            int nw, uint32_t* __restrict__ bits, int64_t ldb) {
  const int lane = threadIdx.x & 31;
  const int64_t total = n * nw;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < total;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = t / nw;
    const int k = (int)(t % nw);
    const int j = 32 * k + lane;
    const bool pos = j < w && C[i * ldc + j] > 0.f;
    const uint32_t word = __ballot_sync(0xffffffffu, pos);
    if (lane == 0) bits[i * ldb + k] = word;
  }
}

constexpr int64_t kWgradRowsPerSplit = 2048;

int64_t wgrad_splits(int64_t K) {
  int64_t s = ceil_div(K, kWgradRowsPerSplit);
  int64_t cap = (int64_t)num_sms() * 2;
  return s < 1 ? 1 : (s > cap ? cap : s);
}

}  // namespace

digest_status gemm_simt(const GemmArgs& g, cudaStream_t s) {
  if (g.M == 0 || g.N == 0) return DIGEST_OK;
  dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM), 1);
  DG_ARG(grid.y < 65536u * 1024u, DIGEST_E_UNSUPPORTED, "GEMM M too large");
  const double flops = 2.0 * (double)g.M * g.N * g.K;
  const double bytes = 4.0 * ((double)g.M * g.K + (double)g.K * g.N + (double)g.M * g.N);
  // grid.y is limited to 65535: fold extra row tiles by repeated launches
  int64_t tiles_m = ceil_div(g.M, BM);
  for (int64_t t0 = 0; t0 < tiles_m; t0 += 65535) {
    GemmArgs sub = g;
    sub.A = g.A + t0 * BM * g.sAi;
    sub.C = g.C + t0 * BM * g.ldc;
    if (g.mask) sub.mask = g.mask + t0 * BM * g.ldm;
    if (g.mbits) sub.mbits = g.mbits + t0 * BM * g.ldmb;
    sub.M = min(g.M - t0 * BM, (int64_t)65535 * BM);
    dim3 gr((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(sub.M, BM), 1);
    DG_LAUNCH(DIGEST_PROF_GEMM, s, bytes * sub.M / g.M, flops * sub.M / g.M, k_gemm, gr,
              kThreads, 0, sub, g.K, (float*)nullptr);
  }
  // the 1-bit output mask: a second pass over C (this kernel only serves small or
  // oddly strided products; the tensor-core epilogue writes the bits in place)
  if (g.obits) DG_TRY(sign_bits(g.C, g.ldc, g.M, g.N, g.obits, g.ldob, s));
  return DIGEST_OK;
}

size_t wgrad_tc_scratch_bytes(int32_t M, int32_t N);
bool wgrad_tc_eligible(const WgradSeg* segs, int nseg, int M, int N);
digest_status wgrad_tc(const WgradSeg* segs, int nseg, int M, int N, float* C, void* scratch,
                       cudaStream_t s);

size_t wgrad_scratch_bytes(int64_t K_total, int32_t M, int32_t N) {
  size_t simt = sizeof(float) * (size_t)wgrad_splits(K_total) * 2 * (size_t)M * (size_t)N + 256;
  size_t tc = wgrad_tc_scratch_bytes(M, N);
  return simt > tc ? simt : tc;
}

digest_status wgrad(const WgradSeg* segs, int nseg, int32_t M, int32_t N, float* C,
                    void* scratch, cudaStream_t s) {
  DG_ARG(nseg >= 1 && nseg <= 2, DIGEST_E_INVALID, "wgrad: 1 or 2 segments");
  if (wgrad_tc_eligible(segs, nseg, M, N)) return wgrad_tc(segs, nseg, M, N, C, scratch, s);
  return wgrad_simt(segs, nseg, M, N, C, scratch, s);
}

digest_status wgrad_simt(const WgradSeg* segs, int nseg, int32_t M, int32_t N, float* C,
                         void* scratch, cudaStream_t s) {
  DG_ARG(nseg >= 1 && nseg <= 2, DIGEST_E_INVALID, "wgrad: 1 or 2 segments");
  int64_t Ktot = 0;
  for (int i = 0; i < nseg; ++i) Ktot += segs[i].K;
  float* partial = reinterpret_cast<float*>(scratch);
  int64_t zbase = 0;
  const int64_t MN = (int64_t)M * N;
  for (int i = 0; i < nseg; ++i) {
    const WgradSeg& sg = segs[i];
    DG_ARG(sg.mask == nullptr, DIGEST_E_UNSUPPORTED, "wgrad mask fusion not built");
    if (sg.K == 0) continue;
    int64_t ns = wgrad_splits(sg.K);
    int64_t kps = round_up(ceil_div(sg.K, ns), BK);
    ns = ceil_div(sg.K, kps);
    GemmArgs g{};
    g.A = sg.A;        // A^T: (i,k) = A[k*lda + i]
    g.sAi = 1;
    g.sAk = sg.lda;
    g.B = sg.B;
    g.sBk = sg.ldb;
    g.sBj = 1;
    g.C = nullptr;
    g.ldc = N;
    g.M = M;
    g.N = N;
    g.K = sg.K;
    dim3 gr((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)ns);
    const double flops = 2.0 * (double)M * N * sg.K;
    const double bytes = 4.0 * ((double)sg.K * (M + N) + (double)ns * MN);
    DG_LAUNCH(DIGEST_PROF_GEMM, s, bytes, flops, k_gemm, gr, kThreads, 0, g, kps,
              partial + zbase * MN);
    zbase += ns;
  }
  if (zbase == 0) {
    DG_CUDA(cudaMemsetAsync(C, 0, sizeof(float) * MN, s));
    return DIGEST_OK;
  }
  int64_t blocks = min(ceil_div(MN, 256), (int64_t)num_sms() * 4);
  DG_LAUNCH(DIGEST_PROF_GEMM, s, 4.0 * (zbase + 1) * MN, 0, k_reduce_splits, (unsigned)blocks,
            256, 0, partial, zbase, MN, C);
  return DIGEST_OK;
}

digest_status relu_mask(const float* G, int64_t ldg, const float* H, int64_t ldh, float* D,
                        int64_t ldd, int64_t n, int32_t w, cudaStream_t s) {
  if (n == 0) return DIGEST_OK;
  int w4 = w / 4;
  int64_t total = n * w4;
  int64_t blocks = min(ceil_div(total, 256), (int64_t)num_sms() * 16);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 12.0 * total * 4, 0, k_relu_mask, (unsigned)blocks, 256, 0, G,
            ldg, H, ldh, D, ldd, n, w4);
  return DIGEST_OK;
}

digest_status relu_mask_bits(const float* G, int64_t ldg, const uint32_t* mbits, int64_t ldmb,
                             float* D, int64_t ldd, int64_t n, int32_t w, cudaStream_t s) {
  if (n == 0) return DIGEST_OK;
  int w4 = w / 4;
  int64_t total = n * w4;
  int64_t blocks = min(ceil_div(total, 256), (int64_t)num_sms() * 16);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * total * 4 + (double)n * ((w + 31) / 32) * 4, 0,
            k_relu_mask_bits, (unsigned)blocks, 256, 0, G, ldg, mbits, ldmb, D, ldd, n, w4);
  return DIGEST_OK;
}

digest_status sign_bits(const float* C, int64_t ldc, int64_t n, int32_t w, uint32_t* bits,
                        int64_t ldb, cudaStream_t s) {
  if (n == 0 || w == 0) return DIGEST_OK;
  const int nw = (w + 31) / 32;
  int64_t blocks = min(ceil_div(n * nw * 32, 256), (int64_t)num_sms() * 16);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 4.0 * n * w + 4.0 * n * nw, 0, k_sign_bits, (unsigned)blocks,
            256, 0, C, ldc, n, w, nw, bits, ldb);
  return DIGEST_OK;
}

}  // namespace dg

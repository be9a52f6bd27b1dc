// Dense transform GEMM of Eq. 5 (Z = A W, T = X W) and the input-gradient GEMM
// (D W^T) on the 5th-generation tensor cores, at fp32 accuracy via 3xTF32
// (SURVEY §0 finding 7: plain TF32, unit roundoff ~5e-4, misses the 1e-4 bar).
//
//   x = hi + lo, hi = x with the low 13 mantissa bits cleared (exactly TF32),
//   lo = x - hi (exact in fp32);   A B ~= Ahi Bhi + Ahi Blo + Alo Bhi
// (the dropped Alo Blo term is ~2^-20 relative).  Accumulation in TMEM (fp32).
//
// Kernel: persistent, one CTA per SM, 128 x BN output tiles, K in 32-float
// (128-byte) blocks, warp-specialised:
//   warp 0      TMA producer: A tile (128 x 32) + B_hi/B_lo tiles (BN x 32), SW128
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (12 MMAs / k-block)
//   warps 2-5   split workers: A -> (A_hi in place, A_lo) in shared memory
//   warps 6-13  epilogue: tcgen05.ld -> ReLU -> global stores (double-buffered TMEM);
//               two warps per TMEM lane quarter, each draining half of the tile's columns
//               (the small-K shapes are bound by the epilogue, not the tensor pipe)
// B (the weight, <= 256 x 1436) is split and transposed to K-major once per call
// by a small prep kernel into a library-owned workspace.
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm_epi.cuh"
#include "kernels.cuh"
#include "tc_util.cuh"

namespace dg {

bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-gather map for TMA tile::gather4: fp32 [outer rows x inner floats], box = one row of
// `inner` floats (no swizzle, rows land packed in shared memory).
bool make_tmap_rows(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes) {
  CUtensorMap probe;
  if (!make_tmap_2d(&probe, base, inner, outer, row_stride_bytes, 32, 1)) return false;  // loads fn
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {(cuuint32_t)inner, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_rows_fwd(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes) {
  return make_tmap_rows(m, base, inner, outer, row_stride_bytes);
}

// A_hi = the raw fp32 tile (default): kind::tf32 reads only the upper 19 bits of an
// operand, i.e. truncates exactly as tf32_hi does, so the split workers write only A_lo.
// Measured (tools/gemm_bench.py, 2.45M rows): K x N = 100x256 0.968 -> 0.951 ms, 256x256
// 1.488 -> 1.453, 256x48 0.825 -> 0.812, 48x256 0.613 -> 0.597; the results are
// bit-identical to the explicit split (tests/test_gpu_gemm_variants.py).
// DIGEST_GEMM_RAWHI=0 writes A_hi explicitly.
int gemm_raw_hi() {
  static int v = -1;
  if (v < 0) {
    const char* e = dg::knob("DIGEST_GEMM_RAWHI");
    v = e ? (atoi(e) ? 1 : 0) : 1;
  }
  return v;
}

namespace {

constexpr int kBM = 128, kBK = 32, kEpiWarps = 8, kThreads = (6 + kEpiWarps) * 32;

constexpr uint32_t pow2_cols(uint32_t c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int BN>
struct Cfg {
  static constexpr int ACC = (BN + 31) / 32 * 32;           // TMEM column stride per accumulator
  static constexpr uint32_t TMEM_COLS = pow2_cols(2 * ACC);
  static constexpr uint32_t A_BYTES = kBM * kBK * 4;        // 16 KB
  static constexpr uint32_t B_BYTES = BN * kBK * 4;
  static constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (200 * 1024 / STAGE) > 4 ? 4 : (200 * 1024 / STAGE);
  static constexpr uint32_t EPI = kEpiWarps * 4096;         // per-warp epilogue staging
  static constexpr uint32_t SMEM = STAGES * STAGE + EPI + 1024 + 256;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  static_assert(B_BYTES % 1024 == 0, "1024-byte aligned stages (SW128 atoms)");
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
              const __grid_constant__ CUtensorMap tmBl, const EpiArgs e, int K, int raw_hi) {
  // raw_hi: A_hi is the raw fp32 tile (kind::tf32 reads only the upper 19 bits), so the
  // split workers write only A_lo (gemm_raw_hi()).
  using G = Cfg<BN>;
  const int64_t M = e.M;
  const int N = e.N;
  constexpr int S = G::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi = smem + S * G::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + G::EPI);
  uint64_t* full = bars;
  uint64_t* conv = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = bars + 3 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);
  auto stA = [&](int s) { return smem + s * G::STAGE; };
  auto stAl = [&](int s) { return smem + s * G::STAGE + G::A_BYTES; };
  auto stBh = [&](int s) { return smem + s * G::STAGE + 2 * G::A_BYTES; };
  auto stBl = [&](int s) { return smem + s * G::STAGE + 2 * G::A_BYTES + G::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kEpiWarps * 32);
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmBh);
    tc::tma_prefetch(&tmBl);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, G::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_tiles_n = (N + BN - 1) / BN;
  const int64_t n_tiles = ((M + kBM - 1) / kBM) * n_tiles_n;
  const int nk = (K + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = (int)((t / n_tiles_n) * kBM);
        const int n0 = (int)((t % n_tiles_n) * BN);
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&empty[s], ph ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], G::A_BYTES + 2 * G::B_BYTES);
          tc::tma_load_2d(stA(s), &tmA, &full[s], kb * kBK, m0);
          tc::tma_load_2d(stBh(s), &tmBh, &full[s], kb * kBK, n0);
          tc::tma_load_2d(stBl(s), &tmBl, &full[s], kb * kBK, n0);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = tc::idesc_tf32(kBM, BN, false, false);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        tc::mbar_wait(&tempty[acc], aph ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * G::ACC;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&conv[s], ph);
          tc::tc_fence_after();
          const uint32_t a = tc::smem_u32(stA(s)), al = tc::smem_u32(stAl(s));
          const uint32_t bh = tc::smem_u32(stBh(s)), bl = tc::smem_u32(stBl(s));
          // K tail: the last k-block issues only the 8-wide MMA steps that hold real K
          // (TMA zero-fills the rest; K=100 runs 13 of 16 steps instead of all 16)
          const int kk = (K - kb * kBK) >= kBK ? kBK / 8 : (K - kb * kBK + 7) / 8;
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            if (k >= kk) break;
            const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along K inside the 128B atom
            const uint64_t dA = tc::smem_desc_sw128(a + off, 16, 1024);
            const uint64_t dAl = tc::smem_desc_sw128(al + off, 16, 1024);
            const uint64_t dBh = tc::smem_desc_sw128(bh + off, 16, 1024);
            const uint64_t dBl = tc::smem_desc_sw128(bl + off, 16, 1024);
            tc::mma_tf32(d, dAl, dBh, idesc, (kb | k) != 0);
            tc::mma_tf32(d, dA, dBl, idesc, 1);
            tc::mma_tf32(d, dA, dBh, idesc, 1);
          }
          tc::mma_commit(&empty[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else if (warp < 6) {  // ---------------- split workers (128 threads)
    const int tid = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      for (int kb = 0; kb < nk; ++kb) {
        tc::mbar_wait(&full[s], ph);
        float4* A = reinterpret_cast<float4*>(stA(s));
        float4* Al = reinterpret_cast<float4*>(stAl(s));
#pragma unroll
        for (int i = 0; i < (int)(G::A_BYTES / 16 / 128); ++i) {
          const int idx = tid + i * 128;
          float4 v = A[idx];
          float4 h = make_float4(tc::tf32_hi(v.x), tc::tf32_hi(v.y), tc::tf32_hi(v.z),
                                 tc::tf32_hi(v.w));
          if (!raw_hi) A[idx] = h;
          Al[idx] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&conv[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {  // ---------------- epilogue (256 threads: 2 warps per TMEM lane quarter)
    const int q = warp & 3;   // TMEM lane quarter this warp may access
    const int half = (warp - 6) >> 2;
    constexpr int kSplit = ((BN + 1) / 2 + 31) / 32 * 32;
    const int c_beg = half ? kSplit : 0, c_end = half ? BN : (kSplit < BN ? kSplit : BN);
    int acc = 0;
    uint32_t aph = 0;
    float4* stg = reinterpret_cast<float4*>(epi + (warp - 6) * 4096);
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {   // n_tiles_n == 1 (BN >= N)
      const int64_t m0 = t * kBM;
      const int64_t tn = t + gridDim.x;
      if (half == 0)
        epi_prefetch_next<BN>(e, tn < n_tiles ? tn * kBM : -1, threadIdx.x % 128);
      tc::mbar_wait(&tfull[acc], aph);
      tc::tc_fence_after();
      epi_tile<BN>(e, tmem_base + acc * G::ACC, stg, m0, q, lane, c_beg, c_end);
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, G::TMEM_COLS);
  }
}

// Bt_hi/Bt_lo [N x Kp] from B(k, j) = B[k*sBk + j*sBj] (split + transpose to K-major).
__global__ void k_prep_b(const float* __restrict__ B, int64_t sBk, int64_t sBj, int K, int N,
                         int Kp, float* __restrict__ hi, float* __restrict__ lo) {
  int64_t total = (int64_t)N * Kp;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int j = (int)(t / Kp), k = (int)(t % Kp);
    float x = k < K ? B[(int64_t)k * sBk + (int64_t)j * sBj] : 0.f;
    float h = tc::tf32_hi(x);
    hi[t] = h;
    lo[t] = x - h;
  }
}

// Library-owned workspace for the split weights (grown on demand, never on a
// steady-state call; cudaFree synchronises the device before releasing).
struct Workspace {
  void* p = nullptr;
  size_t bytes = 0;
  std::mutex mu;
};
Workspace g_ws;

void* workspace(size_t bytes) {
  std::lock_guard<std::mutex> lk(g_ws.mu);
  if (g_ws.bytes < bytes) {
    if (g_ws.p) cudaFree(g_ws.p);
    g_ws.p = nullptr;
    g_ws.bytes = 0;
    size_t nb = bytes < (1u << 20) ? (1u << 20) : bytes * 2;
    if (cudaMalloc(&g_ws.p, nb) != cudaSuccess) return nullptr;
    g_ws.bytes = nb;
  }
  return g_ws.p;
}

template <int BN>
digest_status launch_tc(const GemmArgs& g, const CUtensorMap& tA, const CUtensorMap& tBh,
                        const CUtensorMap& tBl, cudaStream_t s) {
  using G = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA(cudaFuncSetAttribute(k_gemm_tf32x3<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 G::SMEM));
    attr = true;
  }
  const int64_t tiles = ceil_div(g.M, kBM) * ceil_div(g.N, BN);
  const int64_t grid = tiles < num_sms() ? tiles : num_sms();
  const double flops = 2.0 * (double)g.M * g.N * g.K;
  const double bytes = 4.0 * ((double)g.M * g.K + (double)g.M * g.N + 2.0 * g.N * g.K);
  // profile tag: 1KKKKNNN (forward-type GEMM, K and N)
  DG_LAUNCH_TAG(DIGEST_PROF_GEMM, 10000000 + (int)g.K * 1000 + g.N, s, bytes, flops,
                k_gemm_tf32x3<BN>, (unsigned)grid, kThreads, G::SMEM, tA, tBh, tBl, epi_of(g),
                (int)g.K, gemm_raw_hi());
  return DIGEST_OK;
}

}  // namespace

bool gemm_tc2_enabled(int N, int K);
digest_status gemm_tc2(const GemmArgs& g, const float* hi, const float* lo, int Kp,
                       cudaStream_t s);

bool gemm_tc_eligible(const GemmArgs& g) {
  static int force_simt = -1;
  if (force_simt < 0) {
    const char* e = dg::knob("DIGEST_GEMM");
    force_simt = (e && e[0] == 's') ? 1 : 0;
  }
  if (force_simt) return false;
  if (g.sAk != 1 || g.sAi % 4 != 0 || ((uintptr_t)g.A & 15) != 0) return false;
  if (g.sBj != 1 && g.sBk != 1) return false;
  if (g.N % 4 != 0 || g.N > 256 || g.K < 8 || g.K > (1 << 20)) return false;
  if (g.ldc % 4 != 0 || ((uintptr_t)g.C & 15) != 0) return false;
  if (g.mask && (g.ldm % 4 != 0 || ((uintptr_t)g.mask & 15) != 0)) return false;
  if (g.mask && g.obits) return false;   // the epilogue's bits precede the float-mask stage
  if (g.M < 256) return false;   // tiny problems: the CUDA-core kernel launches cheaper
  return true;
}

digest_status gemm_tc(const GemmArgs& g, cudaStream_t s) {
  const int K = (int)g.K, N = g.N;
  const int Kp = (int)round_up(K, 4);
  float* hi = reinterpret_cast<float*>(workspace(sizeof(float) * 2 * (size_t)N * Kp));
  DG_ARG(hi, DIGEST_E_NOMEM, "GEMM workspace allocation failed");
  float* lo = hi + (size_t)N * Kp;
  {
    int64_t total = (int64_t)N * Kp;
    int64_t blocks = ceil_div(total, 256);
    if (blocks > num_sms() * 4) blocks = num_sms() * 4;
    DG_LAUNCH(DIGEST_PROF_OTHER, s, 12.0 * total, 0, k_prep_b, (unsigned)blocks, 256, 0, g.B,
              g.sBk, g.sBj, K, N, Kp, hi, lo);
  }
  if (gemm_tc2_enabled(N, (int)g.K) && g.M >= 2 * kBM) return gemm_tc2(g, hi, lo, Kp, s);
  int BN = N <= 16 ? 16 : N <= 32 ? 32 : N <= 48 ? 48 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  CUtensorMap tA, tBh, tBl;
  bool ok = make_tmap_2d(&tA, g.A, (uint64_t)K, (uint64_t)g.M, (uint64_t)g.sAi * 4, kBK, kBM) &&
            make_tmap_2d(&tBh, hi, (uint64_t)K, (uint64_t)N, (uint64_t)Kp * 4, kBK, BN) &&
            make_tmap_2d(&tBl, lo, (uint64_t)K, (uint64_t)N, (uint64_t)Kp * 4, kBK, BN);
  DG_ARG(ok, DIGEST_E_CUDA, "cuTensorMapEncodeTiled failed");
  switch (BN) {
    case 16: return launch_tc<16>(g, tA, tBh, tBl, s);
    case 32: return launch_tc<32>(g, tA, tBh, tBl, s);
    case 48: return launch_tc<48>(g, tA, tBh, tBl, s);
    case 64: return launch_tc<64>(g, tA, tBh, tBl, s);
    case 128: return launch_tc<128>(g, tA, tBh, tBl, s);
    default: return launch_tc<256>(g, tA, tBh, tBl, s);
  }
}

}  // namespace dg

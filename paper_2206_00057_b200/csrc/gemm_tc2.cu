// 3xTF32 GEMM on CTA pairs (tcgen05 cta_group::2): the dense transform of Eq. 5
// (Z = A W, T = X W) and D W^T, with the same split-precision scheme as gemm_tc.cu.
//
// Why pairs: the single-CTA kernel streams 64 KB of split weights (B_hi, B_lo) per
// 32-wide k-block into every SM for 2052 MMA cycles -- right at the per-SM TMA fill
// rate.  A CTA pair computes a 256 x BN tile with M=256 MMAs; each CTA loads its own
// 128 rows of A and HALF of B, so the B traffic per SM halves and the A tile stays
// the same, while the MMA work per CTA is unchanged.
//
//   rank r of the pair: A rows m0 + 128 r, B rows n0 + (BN/2) r, its TMEM holds its
//   128 accumulator rows.  Both CTAs run TMA producer, split workers and epilogue;
//   only rank 0 issues the MMAs and commits them (multicast) to both CTAs' barriers.
//   Split workers and epilogues of both CTAs arrive on rank 0's conv / tempty
//   barriers through shared::cluster addresses.
#include <cudaTypedefs.h>

#include "gemm_epi.cuh"
#include "kernels.cuh"
#include "tc_util.cuh"

namespace dg {

void* workspace(size_t bytes);

int gemm_raw_hi();   // gemm_tc.cu

namespace {

// warps: 0 TMA, 1 MMA (rank 0), 2-5 split workers, 6-13 epilogue: two warps per TMEM lane
// quarter, each draining half of the tile's columns (the epilogue, not the tensor pipe,
// bounds the small-K shapes)
constexpr int kBM = 128, kBK = 32, kEpiWarps = 8, kThreads = (6 + kEpiWarps) * 32;

constexpr uint32_t pow2_cols2(uint32_t c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int BN>
struct Cfg2 {
  static constexpr int ACC = (BN + 31) / 32 * 32;
  static constexpr uint32_t TMEM_COLS = pow2_cols2(2 * ACC);
  static constexpr uint32_t A_BYTES = kBM * kBK * 4;          // 16 KB, this CTA's rows
  static constexpr uint32_t B_BYTES = (BN / 2) * kBK * 4;     // this CTA's half of B
  static constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (192 * 1024 / STAGE) > 4 ? 4 : (192 * 1024 / STAGE);
  static constexpr uint32_t EPI = kEpiWarps * 4096;
  static constexpr uint32_t SMEM = STAGES * STAGE + EPI + 1024 + 256;
  static_assert(BN % 16 == 0 && BN >= 32 && BN <= 256, "UMMA N for M=256");
  static_assert(B_BYTES % 1024 == 0, "1024-byte aligned stages (SW128 atoms)");
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm2_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
               const __grid_constant__ CUtensorMap tmBl, const EpiArgs e, int K, int flags) {
  // flags bit 1 (default, see gemm_raw_hi in gemm_tc.cu): A_hi is the raw fp32 tile
  // itself -- kind::tf32 uses only an operand's upper 19 bits -- so only
  // A_lo = A - trunc19(A) is written back.
  const int single = flags & 1, raw_hi = flags & 2;
  // single: the 128 split-worker (epilogue) threads of a CTA meet at a named barrier and
  // ONE of them arrives on rank 0's conv (tempty) barrier -- 2 cluster-scope arrivals per
  // stage instead of 256 (each thread still fences its own smem writes / TMEM loads).
  const uint32_t group_count = single ? 2u : 256u;
  using G = Cfg2<BN>;
  const int64_t M = e.M;
  const int N = e.N;
  constexpr int S = G::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi = smem + S * G::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + G::EPI);
  uint64_t* full = bars;            // local TMA -> local split workers
  uint64_t* conv = bars + S;        // both CTAs' split workers -> rank-0 MMA (count 256)
  uint64_t* empty = bars + 2 * S;   // rank-0 MMA commit (multicast) -> both producers
  uint64_t* tfull = bars + 3 * S;   // rank-0 MMA commit (multicast) -> both epilogues
  uint64_t* tempty = bars + 3 * S + 2;   // both epilogues -> rank-0 MMA (count 256)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);
  auto stA = [&](int s) { return smem + s * G::STAGE; };
  auto stAl = [&](int s) { return smem + s * G::STAGE + G::A_BYTES; };
  auto stBh = [&](int s) { return smem + s * G::STAGE + 2 * G::A_BYTES; };
  auto stBl = [&](int s) { return smem + s * G::STAGE + 2 * G::A_BYTES + G::B_BYTES; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], group_count);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 2);   // one arrival per CTA (after the epilogue barrier)
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmBh);
    tc::tma_prefetch(&tmBl);
  }
  if (warp == 1) tc::tmem_alloc2(tmem_slot, G::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();     // peers' barriers are initialised before any remote arrive
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_tiles_n = (N + BN - 1) / BN;
  const int64_t n_tiles = ((M + 2 * kBM - 1) / (2 * kBM)) * n_tiles_n;
  const int nk = (K + kBK - 1) / kBK;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = pair; t < n_tiles; t += npairs) {
        const int m0 = (int)((t / n_tiles_n) * 2 * kBM + rank * kBM);
        const int n0 = (int)((t % n_tiles_n) * BN + rank * (BN / 2));
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
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (rank 0 only)
      constexpr uint32_t idesc = tc::idesc_tf32(2 * kBM, BN, false, false);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = pair; t < n_tiles; t += npairs) {
        tc::mbar_wait_cluster(&tempty[acc], aph ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * G::ACC;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait_cluster(&conv[s], ph);
          tc::tc_fence_after();
          const uint32_t a = tc::smem_u32(stA(s)), al = tc::smem_u32(stAl(s));
          const uint32_t bh = tc::smem_u32(stBh(s)), bl = tc::smem_u32(stBl(s));
          // K tail: the last k-block issues only the 8-wide MMA steps that hold real K
          // (TMA zero-fills the rest; K=100 runs 13 of 16 steps instead of all 16)
          const int kk = (K - kb * kBK) >= kBK ? kBK / 8 : (K - kb * kBK + 7) / 8;
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            if (k >= kk) break;
            const uint32_t off = k * 32;
            const uint64_t dA = tc::smem_desc_sw128(a + off, 16, 1024);
            const uint64_t dAl = tc::smem_desc_sw128(al + off, 16, 1024);
            const uint64_t dBh = tc::smem_desc_sw128(bh + off, 16, 1024);
            const uint64_t dBl = tc::smem_desc_sw128(bl + off, 16, 1024);
            tc::mma2_tf32(d, dAl, dBh, idesc, (kb | k) != 0);
            tc::mma2_tf32(d, dA, dBl, idesc, 1);
            tc::mma2_tf32(d, dA, dBh, idesc, 1);
          }
          tc::mma2_commit_multicast(&empty[s], 0x3);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc::mma2_commit_multicast(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else if (warp < 6) {  // ---------------- split workers (128 threads per CTA)
    const int tid = threadIdx.x - 64;
    const uint32_t conv0 = tc::mapa(tc::smem_u32(conv), 0);
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = pair; t < n_tiles; t += npairs) {
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
        if (single) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (tid == 0) tc::mbar_arrive_cluster(conv0 + s * 8);
        } else {
          tc::mbar_arrive_cluster(conv0 + s * 8);
        }
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {  // ---------------- epilogue (256 threads per CTA, its own 128 rows)
    const int q = warp & 3;
    const int half = (warp - 6) >> 2;
    constexpr int kSplit = ((BN + 1) / 2 + 31) / 32 * 32;
    const int c_beg = half ? kSplit : 0, c_end = half ? BN : (kSplit < BN ? kSplit : BN);
    const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
    float4* stg = reinterpret_cast<float4*>(epi + (warp - 6) * 4096);
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = pair; t < n_tiles; t += npairs) {   // n_tiles_n == 1 (BN >= N)
      const int64_t m0 = t * 2 * kBM + rank * kBM;
      const int64_t tn = t + npairs;
      if (half == 0)
        epi_prefetch_next<BN>(e, tn < n_tiles ? tn * 2 * kBM + rank * kBM : -1, threadIdx.x % 128);
      tc::mbar_wait(&tfull[acc], aph);
      tc::tc_fence_after();
      epi_tile<BN>(e, tmem_base + acc * G::ACC, stg, m0, q, lane, c_beg, c_end);
      tc::tc_fence_before();
      asm volatile("bar.sync 2, 256;" ::: "memory");   // all 8 epilogue warps
      if (warp == 6 && lane == 0) tc::mbar_arrive_cluster(tempty0 + acc * 8);
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();     // the peer is done with every remote barrier and TMEM column
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc2(tmem_base, G::TMEM_COLS);
  }
}

template <int BN>
digest_status launch2(const GemmArgs& g, const CUtensorMap& tA, const CUtensorMap& tBh,
                      const CUtensorMap& tBl, cudaStream_t s) {
  using G = Cfg2<BN>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA(cudaFuncSetAttribute(k_gemm2_tf32x3<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 G::SMEM));
    attr = true;
  }
  const int64_t tiles = ceil_div(g.M, 2 * kBM) * ceil_div(g.N, BN);
  int64_t pairs = num_sms() / 2;
  if (pairs > tiles) pairs = tiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const double flops = 2.0 * (double)g.M * g.N * g.K;
  const double bytes = 4.0 * ((double)g.M * g.K + (double)g.M * g.N + 2.0 * g.N * g.K);
  Launch L(DIGEST_PROF_GEMM, s, bytes, flops, 30000000 + (int)g.K * 1000 + g.N);
  static int single = -1;   // DIGEST_GEMM_SINGLE_ARRIVE (default 1)
  if (single < 0) {
    const char* ev = dg::knob("DIGEST_GEMM_SINGLE_ARRIVE");
    single = ev ? atoi(ev) : 1;
    if (gemm_raw_hi()) single |= 2;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_gemm2_tf32x3<BN>, tA, tBh, tBl, epi_of(g), (int)g.K,
                                     single);
  cudaError_t e2 = L.done();
  DG_CUDA(e);
  DG_CUDA(e2);
  return DIGEST_OK;
}

}  // namespace

// Called by gemm_tc after the weight split: hi/lo are [N x Kp] K-major.
bool gemm_tc2_enabled(int N, int K) {
  static int v = -1;
  if (v < 0) {
    const char* e = dg::knob("DIGEST_GEMM_2CTA");
    v = e ? atoi(e) : 1;
  }
  // measured (tools/gemm_bench.py, 2.45M rows): N=256 1.64 -> 1.60 ms with pairs; N=48 is
  // 2x slower with pairs (too little MMA work per k-block to hide the cross-CTA handshake)
  // K <= 64: a tile is only 1-2 k-blocks, the pair handshake costs more than the halved
  // B traffic saves (K=48, N=256: 0.855 ms pair vs 0.772 ms single CTA)
  return v != 0 && N >= 128 && N % 16 == 0 && K > 64;
}

digest_status gemm_tc2(const GemmArgs& g, const float* hi, const float* lo, int Kp,
                       cudaStream_t s) {
  const int K = (int)g.K, N = g.N;
  int BN = N <= 32 ? 32 : N <= 48 ? 48 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  CUtensorMap tA, tBh, tBl;
  bool ok = make_tmap_2d(&tA, g.A, (uint64_t)K, (uint64_t)g.M, (uint64_t)g.sAi * 4, kBK, kBM) &&
            make_tmap_2d(&tBh, hi, (uint64_t)K, (uint64_t)N, (uint64_t)Kp * 4, kBK, BN / 2) &&
            make_tmap_2d(&tBl, lo, (uint64_t)K, (uint64_t)N, (uint64_t)Kp * 4, kBK, BN / 2);
  DG_ARG(ok, DIGEST_E_CUDA, "cuTensorMapEncodeTiled failed (2-CTA GEMM)");
  switch (BN) {
    case 32: return launch2<32>(g, tA, tBh, tBl, s);
    case 48: return launch2<48>(g, tA, tBh, tBl, s);
    case 64: return launch2<64>(g, tA, tBh, tBl, s);
    case 128: return launch2<128>(g, tA, tBh, tBl, s);
    default: return launch2<256>(g, tA, tBh, tBl, s);
  }
}

}  // namespace dg

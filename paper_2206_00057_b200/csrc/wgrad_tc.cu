// Weight gradient of Eq. 6: G_W = (P_m X_ext)^T D  (AGG_FIRST: A^T D;
// XFORM_FIRST: X_loc^T S_loc + X_halo^T S_halo) on the tensor cores.
//
// Shapes: M = d_in (<= 256 per CTA tile), N = d_out (<= 256), K = rows of the
// partition (up to 2.45M).  Both operands are row-major [K x M] / [K x N], i.e.
// MN-major for UMMA.  Measured on B200 (tools/umma_probe2.cu): kind::tf32 ignores
// MN-major operands (the MMA writes nothing), kind::f16 accepts them.  So this
// kernel splits each fp32 value into three bf16 pieces x = b0 + b1 + b2 (exactly, by
// truncation: |b1| < 2^-7 |x|, |b2| < 2^-15 |x|) and accumulates the six products
// b2c0 + b0c2 + b1c1 + b1c0 + b0c1 + b0c0 with kind::f16 (dropped terms <= 2^-22
// relative) -- the same tensor time as 3xTF32 (bf16 runs at twice the TF32 rate).  TMA loads 32-float x 16-row
// fp32 boxes (128B swizzle); split workers write the pieces in the bf16 MN-major
// SW128 canonical layout (64-element runs, LBO = next 64-run group, SBO = next
// 8-row K group).
//
// Split-K over CTAs (contiguous row ranges), fixed-order reduction afterwards, so
// the result is deterministic.  Tensor-core accumulation rounds towards zero, so a
// long K would bias the sum (~K/8 truncations); each CTA therefore accumulates at
// most kChunk rows in TMEM and the epilogue warps flush the chunk into an fp32
// partial (round-to-nearest adds) before the next chunk.
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace dg {

void* workspace(size_t bytes);

namespace {

constexpr int kBK = 16;           // K rows per stage
constexpr int kChunkBlocks = 64;  // k-blocks (x16 rows) accumulated in TMEM before a flush
// warp roles: 0 TMA, 1 MMA, 2 .. 2+kConvWarps-1 split workers, then 4 epilogue warps.
// Eight split-worker warps (two per SM sub-partition): the fp32 -> 3 x bf16 split of both
// operands is a dependent LDS -> ALU -> STS chain per element, and with one warp per
// sub-partition its latency, not the tensor pipe, set the stage time.
constexpr int kConvWarps = 8;
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kThreads = (2 + kConvWarps + 4) * 32;

constexpr uint32_t pow2_cols(uint32_t c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int MT, int BN>  // MT: 128-row M halves per CTA (1 or 2); BN: N padded to 32
struct WCfg {
  static constexpr int AG = MT * 2;                     // 64-element bf16 groups along M
  static constexpr int BG = (BN + 63) / 64;             // 64-element bf16 groups along N
  static constexpr uint32_t RAW_A = MT * 128 * kBK * 4; // fp32 TMA staging (32-float boxes)
  static constexpr uint32_t RAW_B = BN * kBK * 4;
  static constexpr uint32_t GRP = 64 * kBK * 2;         // one bf16 64-run group x 16 rows: 2 KB
  static constexpr uint32_t PA = AG * GRP;              // one bf16 piece of A
  static constexpr uint32_t PB = BG * GRP;              // one bf16 piece of B
  // Two decoupled rings: fp32 TMA staging (RS deep) -> split workers -> bf16 pieces
  // (PS deep, read by the MMA), so the TMA runs ahead of the conversion.
  static constexpr uint32_t RAW = RAW_A + RAW_B;
  static constexpr uint32_t PIECE = 3 * PA + 3 * PB;
  static constexpr int PS = 2;
  // staging depth: as many fp32 stages as fit (up to 8) -- the TMA bytes in flight per
  // SM are what keep the HBM busy for the narrow (N=48) and single-half (M<=128) shapes
  static constexpr int RS = ((200 * 1024 - PS * PIECE) / RAW) > 8 ? 8
                                                                   : ((200 * 1024 - PS * PIECE) / RAW);
  static constexpr uint32_t SMEM = RS * RAW + PS * PIECE + 1024 + 256;
  static_assert(RS >= 2, "staging ring");
  static constexpr uint32_t TMEM_COLS = pow2_cols(MT * BN);
  static constexpr uint32_t BOX = 32 * kBK * 4;         // one 32-float x 16-row fp32 box: 2 KB
  static_assert(BN % 32 == 0 && BN <= 256 && MT * BN <= 512, "tile");
  static_assert(RAW % 1024 == 0 && PIECE % 1024 == 0 && RAW_B % 1024 == 0,
                "1024-byte aligned swizzle atoms");
};

// Instruction descriptor, kind::f16 with bf16 A/B (format 1), fp32 D, MN-major A and B.
__host__ __device__ constexpr uint32_t idesc_bf16_mn(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// 8 consecutive MN elements of row k: fp32 raw (SW128, 32-float runs) -> three bf16
// pieces (SW128, 64-element runs).  Byte offsets of 16B chunks inside a 1024B atom
// are XOR-swizzled with the row index (k & 7), as TMA and UMMA both expect.
__device__ __forceinline__ void split8(const uint8_t* raw, uint8_t* p0, uint8_t* p1, uint8_t* p2,
                                       uint32_t piece_bytes, int k, int e) {
  const int sw = k & 7;
  const uint8_t* src = raw + (e >> 5) * (32 * kBK * 4) + k * 128;
  const float4 u = *reinterpret_cast<const float4*>(src + ((((e & 31) >> 2) ^ sw) << 4));
  const float4 w = *reinterpret_cast<const float4*>(src + (((((e & 31) >> 2) + 1) ^ sw) << 4));
  const float x[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
  // Truncation split (bit masks, full-rate ALU; no conversion-unit instructions):
  // b0 = top 8 significant bits of x, r1 = x - b0 (exact, <= 16 bits), b1 = top 8 bits
  // of r1, r2 = r1 - b1 (exact, <= 8 bits) = b2.  x = b0 + b1 + b2 exactly, and each
  // piece is its fp32 pattern's high half, so packing is a byte permute.
  uint32_t h0[8], h1[8], h2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t xb = __float_as_uint(x[i]);
    h0[i] = xb & 0xffff0000u;
    const float r1 = x[i] - __uint_as_float(h0[i]);
    h1[i] = __float_as_uint(r1) & 0xffff0000u;
    h2[i] = __float_as_uint(r1 - __uint_as_float(h1[i]));
  }
  uint32_t q0[4], q1[4], q2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    q0[i] = __byte_perm(h0[2 * i], h0[2 * i + 1], 0x7632);
    q1[i] = __byte_perm(h1[2 * i], h1[2 * i + 1], 0x7632);
    q2[i] = __byte_perm(h2[2 * i], h2[2 * i + 1], 0x7632);
  }
  const uint32_t off = (e >> 6) * (64 * kBK * 2) + k * 128 + ((((e & 63) >> 3) ^ sw) << 4);
  *reinterpret_cast<uint4*>(p0 + off) = make_uint4(q0[0], q0[1], q0[2], q0[3]);
  *reinterpret_cast<uint4*>(p1 + off) = make_uint4(q1[0], q1[1], q1[2], q1[3]);
  *reinterpret_cast<uint4*>(p2 + off) = make_uint4(q2[0], q2[1], q2[2], q2[3]);
  (void)piece_bytes;
}

template <int MT, int BN>
__global__ void __launch_bounds__(kThreads, 1)
k_wgrad_bf16x6(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               int64_t K, int64_t k_per_cta, int M, int N, float* __restrict__ partial,
               int dbg) {
  using G = WCfg<MT, BN>;
  constexpr int RS = G::RS, PS = G::PS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* pieces = smem + RS * G::RAW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pieces + PS * G::PIECE);
  uint64_t* full = bars;              // TMA -> split workers        [RS]
  uint64_t* rfree = bars + RS;        // split workers -> TMA        [RS]
  uint64_t* conv = bars + 2 * RS;     // split workers -> MMA        [PS]
  uint64_t* empty = conv + PS;        // MMA (commit) -> split workers [PS]
  uint64_t* tfull = empty + PS;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  auto rawA = [&](int r) { return smem + r * G::RAW; };
  auto rawB = [&](int r) { return smem + r * G::RAW + G::RAW_A; };
  auto pieceA = [&](int s, int p) { return pieces + s * G::PIECE + p * G::PA; };
  auto pieceB = [&](int s, int p) { return pieces + s * G::PIECE + 3 * G::PA + p * G::PB; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_base = blockIdx.y * (MT * 128);
  const int64_t k_begin = (int64_t)blockIdx.x * k_per_cta;
  const int64_t k_end = min(K, k_begin + k_per_cta);
  const int nkb = k_end > k_begin ? (int)((k_end - k_begin + kBK - 1) / kBK) : 0;
  const int nchunks = (nkb + kChunkBlocks - 1) / kChunkBlocks;
  float* out = partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * (int64_t)(MT * 128) * BN;

  if (warp == 0 && lane == 0) {
    for (int r = 0; r < RS; ++r) {
      tc::mbar_init(&full[r], 1);
      tc::mbar_init(&rfree[r], kConvThreads);
    }
    for (int s = 0; s < PS; ++s) {
      tc::mbar_init(&conv[s], kConvThreads);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, 128);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, G::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: fp32 boxes, 32 MN elements x 16 K rows each
      int r = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        const int k0 = (int)(k_begin + (int64_t)kb * kBK);
        tc::mbar_wait(&rfree[r], ph ^ 1);
        if (dbg & 4) {   // timing experiment: no TMA traffic
          tc::mbar_arrive(&full[r]);
        } else {
          tc::mbar_arrive_expect_tx(&full[r], G::RAW_A + G::RAW_B);
#pragma unroll
          for (int j = 0; j < MT * 4; ++j)
            tc::tma_load_2d(rawA(r) + j * G::BOX, &tmA, &full[r], m_base + 32 * j, k0);
#pragma unroll
          for (int j = 0; j < BN / 32; ++j)
            tc::tma_load_2d(rawB(r) + j * G::BOX, &tmB, &full[r], 32 * j, k0);
        }
        if (++r == RS) { r = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: 6 bf16 products per 128-row half, K = 16 per stage
      constexpr uint32_t idesc = idesc_bf16_mn(128, BN);
      constexpr int pa[6] = {2, 0, 1, 1, 0, 0}, pb[6] = {0, 2, 1, 0, 1, 0};
      int s = 0;
      uint32_t ph = 0;
      int kb = 0;
      for (int c = 0; c < nchunks; ++c) {
        tc::mbar_wait(tempty, (c & 1) ^ 1);
        tc::tc_fence_after();
        const int kb_end = min(nkb, kb + kChunkBlocks);
        const int kb_first = kb;
        for (; kb < kb_end; ++kb) {
          tc::mbar_wait(&conv[s], ph);
          tc::tc_fence_after();
#pragma unroll
          for (int h = 0; h < MT; ++h) {
            const uint32_t d = tmem_base + h * BN;
#pragma unroll
            for (int t = 0; t < 6; ++t) {
              const uint64_t dA = tc::smem_desc_sw128(
                  tc::smem_u32(pieceA(s, pa[t]) + h * 2 * G::GRP), G::GRP, 1024);
              const uint64_t dB = tc::smem_desc_sw128(tc::smem_u32(pieceB(s, pb[t])), G::GRP, 1024);
              if (!(dbg & 2)) mma_bf16(d, dA, dB, idesc, (kb != kb_first) || t != 0);
            }
          }
          tc::mma_commit(&empty[s]);
          if (++s == PS) { s = 0; ph ^= 1; }
        }
        tc::mma_commit(tfull);
      }
    }
  } else if (warp < 2 + kConvWarps) {  // split workers: fp32 -> 3 bf16 pieces, both operands
    const int tid = threadIdx.x - 64;
    constexpr int UA = kBK * (MT * 128 / 8);   // 8-element units of A per stage
    constexpr int UB = kBK * (BN / 8);
    int r = 0, s = 0;
    uint32_t rph = 0, ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      tc::mbar_wait(&full[r], rph);
      tc::mbar_wait(&empty[s], ph ^ 1);   // the MMA has finished reading piece slot s
      for (int u = tid; u < ((dbg & 1) ? 0 : UA); u += kConvThreads) {
        const int k = u / (MT * 128 / 8), e = (u % (MT * 128 / 8)) * 8;
        split8(rawA(r), pieceA(s, 0), pieceA(s, 1), pieceA(s, 2), G::PA, k, e);
      }
      for (int u = tid; u < ((dbg & 1) ? 0 : UB); u += kConvThreads) {
        const int k = u / (BN / 8), e = (u % (BN / 8)) * 8;
        split8(rawB(r), pieceB(s, 0), pieceB(s, 1), pieceB(s, 2), G::PB, k, e);
      }
      tc::mbar_arrive(&rfree[r]);          // staging slot r may be refilled by TMA
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&conv[s]);
      if (++r == RS) { r = 0; rph ^= 1; }
      if (++s == PS) { s = 0; ph ^= 1; }
    }
  } else {  // epilogue: flush each chunk into the fp32 partial (RN adds)
    const int q = warp & 3;
    for (int c = 0; c < nchunks; ++c) {
      tc::mbar_wait(tfull, c & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < MT; ++h) {
        const int row = h * 128 + q * 32 + lane;   // output row (feature) within the CTA tile
        float* orow = out + (int64_t)row * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          tc::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + h * BN + c0, r);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4* p = reinterpret_cast<float4*>(orow + c0 + j);
            float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                   __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
            if (c > 0) {
              float4 o = *p;
              v.x += o.x;
              v.y += o.y;
              v.z += o.z;
              v.w += o.w;
            }
            *p = v;
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(tempty);
    }
    if (nchunks == 0) {  // empty K range: this CTA's partial is zero
      for (int h = 0; h < MT; ++h) {
        const int row = h * 128 + q * 32 + lane;
        for (int c0 = 0; c0 < BN; c0 += 4)
          *reinterpret_cast<float4*>(out + (int64_t)row * BN + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, G::TMEM_COLS);
  }
}

// C[m*N + n] = sum_z partial[z][m][n] over all CTA slices, fixed order.
__global__ void k_wgrad_reduce(const float* __restrict__ partial, int nz, int MT128, int BN, int M,
                               int N, int ytiles, float* __restrict__ C) {
  const int64_t MN = (int64_t)M * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < MN;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(t / N), n = (int)(t % N);
    const int y = m / MT128, mr = m % MT128;
    float s = 0.f;
    for (int z = 0; z < nz; ++z)
      s += partial[(((int64_t)z * ytiles + y) * MT128 + mr) * BN + n];
    C[t] = s;
  }
}

int wgrad_dbg() {
  static int v = -1;
  if (v < 0) {
    const char* e = dg::knob("DIGEST_WGRAD_DBG");   // timing experiments only (wrong results)
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int MT, int BN>
digest_status launch_seg(const WgradSeg& sg, int M, int N, int grid_x, float* partial,
                         cudaStream_t s) {
  using G = WCfg<MT, BN>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA(cudaFuncSetAttribute(k_wgrad_bf16x6<MT, BN>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    attr = true;
  }
  CUtensorMap tA, tB;
  bool ok = make_tmap_2d(&tA, sg.A, (uint64_t)M, (uint64_t)sg.K, (uint64_t)sg.lda * 4, 32, kBK) &&
            make_tmap_2d(&tB, sg.B, (uint64_t)N, (uint64_t)sg.K, (uint64_t)sg.ldb * 4, 32, kBK);
  DG_ARG(ok, DIGEST_E_CUDA, "cuTensorMapEncodeTiled failed (wgrad)");
  const int ytiles = (int)ceil_div(M, MT * 128);
  int64_t kpc = round_up(ceil_div(sg.K, grid_x), kBK);
  dim3 grid((unsigned)grid_x, (unsigned)ytiles);
  const double flops = 2.0 * (double)M * N * sg.K;
  const double bytes = 4.0 * (double)sg.K * (M + N);
  // profile tag: 2MMMMNNN (weight gradient, M = d_in, N = d_out)
  DG_LAUNCH_TAG(DIGEST_PROF_GEMM, 20000000 + M * 1000 + N, s, bytes, flops,
                (k_wgrad_bf16x6<MT, BN>), grid, kThreads, G::SMEM, tA, tB, sg.K, kpc, M, N,
                partial, wgrad_dbg());
  return DIGEST_OK;
}

template <int MT, int BN>
digest_status run(const WgradSeg* segs, int nseg, int M, int N, float* C, float* partial,
                  cudaStream_t s) {
  const int ytiles = (int)ceil_div(M, MT * 128);
  const int64_t slice = (int64_t)ytiles * MT * 128 * BN;
  int zbase = 0;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].K == 0) continue;
    int gx = (int)ceil_div(num_sms(), ytiles);
    int64_t need = ceil_div(segs[i].K, kBK * 4);   // at least 64 rows per CTA
    if (gx > need) gx = (int)need;
    if (gx < 1) gx = 1;
    DG_TRY((launch_seg<MT, BN>(segs[i], M, N, gx, partial + zbase * slice, s)));
    zbase += gx;
  }
  const int64_t MN = (int64_t)M * N;
  if (zbase == 0) {
    DG_CUDA(cudaMemsetAsync(C, 0, sizeof(float) * MN, s));
    return DIGEST_OK;
  }
  int64_t blocks = ceil_div(MN, 256);
  if (blocks > num_sms() * 4) blocks = num_sms() * 4;
  DG_LAUNCH(DIGEST_PROF_GEMM, s, 4.0 * (zbase + 1) * MN, 0, k_wgrad_reduce, (unsigned)blocks, 256,
            0, partial, zbase, MT * 128, BN, M, N, ytiles, C);
  return DIGEST_OK;
}

}  // namespace

size_t wgrad_tc_scratch_bytes(int32_t M, int32_t N) {
  // up to 2 segments x num_sms CTA slices of (M padded to 128) x (N padded to 32)
  return sizeof(float) * 2 * (size_t)num_sms() * (size_t)round_up(M, 256) * round_up(N, 32) + 256;
}

bool wgrad_tc_eligible(const WgradSeg* segs, int nseg, int M, int N) {
  const char* e = dg::knob("DIGEST_GEMM");
  if (e && e[0] == 's') return false;
  if (N > 256 || N % 4 || M % 4 || M < 8) return false;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].mask) return false;
    if (segs[i].K == 0) continue;
    if (segs[i].lda % 4 || segs[i].ldb % 4 || ((uintptr_t)segs[i].A & 15) ||
        ((uintptr_t)segs[i].B & 15))
      return false;
    if (segs[i].K >= (1ll << 31)) return false;
  }
  return true;
}

digest_status wgrad_tc(const WgradSeg* segs, int nseg, int M, int N, float* C, void* scratch,
                       cudaStream_t s) {
  float* partial = reinterpret_cast<float*>(scratch);
  const int bn = (int)round_up(N, 32);
  const bool two = M > 128;
  if (two) {
    switch (bn) {
      case 32: return run<2, 32>(segs, nseg, M, N, C, partial, s);
      case 64: return run<2, 64>(segs, nseg, M, N, C, partial, s);
      case 96: return run<2, 96>(segs, nseg, M, N, C, partial, s);
      case 128: return run<2, 128>(segs, nseg, M, N, C, partial, s);
      case 160: return run<2, 160>(segs, nseg, M, N, C, partial, s);
      case 192: return run<2, 192>(segs, nseg, M, N, C, partial, s);
      case 224: return run<2, 224>(segs, nseg, M, N, C, partial, s);
      default: return run<2, 256>(segs, nseg, M, N, C, partial, s);
    }
  }
  switch (bn) {
    case 32: return run<1, 32>(segs, nseg, M, N, C, partial, s);
    case 64: return run<1, 64>(segs, nseg, M, N, C, partial, s);
    case 96: return run<1, 96>(segs, nseg, M, N, C, partial, s);
    case 128: return run<1, 128>(segs, nseg, M, N, C, partial, s);
    case 160: return run<1, 160>(segs, nseg, M, N, C, partial, s);
    case 192: return run<1, 192>(segs, nseg, M, N, C, partial, s);
    case 224: return run<1, 224>(segs, nseg, M, N, C, partial, s);
    default: return run<1, 256>(segs, nseg, M, N, C, partial, s);
  }
}

}  // namespace dg

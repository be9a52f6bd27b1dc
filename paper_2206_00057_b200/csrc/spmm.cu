// CSR-row SpMM over the extended column space [local ; halo] (Eq. 5's
// P_in H_in + P_out H~_out, as ONE product with two source pointers).
//
// Design: a group of LANES lanes owns one output row; each lane
// owns VPL float4 columns (128-bit loads).  The group loads LANES (col, val) pairs
// with one coalesced access, broadcasts them with width-LANES shuffles, and issues
// UNR independent row gathers before consuming them (memory-level parallelism).
// Halo rows come from a second pointer (no copy of the stale store into a
// contiguous X_ext).  HBM-bound: ~2 flop per (8 + 4w) bytes per nonzero.
#include "kernels.cuh"

namespace dg {
namespace {

constexpr int kUnroll = 4;

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

template <int LANES, int VPL>
__global__ void __launch_bounds__(256) k_spmm(SpmmArgs a) {
  constexpr int GROUPS = 32 / LANES;
  const int lane = threadIdx.x & 31;
  const int gl = lane % LANES;
  const int gid = lane / LANES;
  const unsigned gmask = LANES == 32 ? 0xffffffffu : (((1u << LANES) - 1u) << (gid * LANES));
  const int w4 = a.width >> 2;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp * GROUPS + gid; row < a.n_rows; row += nwarps * GROUPS) {
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t beg = a.row_ptr[row];
    const int64_t end = a.in_len ? beg + a.in_len[row] : a.row_ptr[row + 1];
    for (int64_t e0 = beg; e0 < end; e0 += LANES) {
      const int64_t e = e0 + gl;
      int32_t c = 0;
      float v = 0.f;
      if (e < end) {
        c = __ldg(a.col + e);
        v = __ldg(a.val + e);
      }
      const int cnt = (int)min((int64_t)LANES, end - e0);
      for (int j0 = 0; j0 < cnt; j0 += kUnroll) {
        const float* src[kUnroll];
        float vv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          int j = j0 + u;
          int cj = __shfl_sync(gmask, c, j & (LANES - 1), LANES);
          float x = __shfl_sync(gmask, v, j & (LANES - 1), LANES);
          vv[u] = j < cnt ? x : 0.f;
          src[u] = (int64_t)cj < a.split ? a.X0 + (int64_t)cj * a.ld0
                                         : a.X1 + ((int64_t)cj - a.split) * a.ld1;
        }
        float4 t[kUnroll][VPL];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            int idx = gl + q * LANES;
            t[u][q] = (idx < w4 && j0 + u < cnt) ? ldg4(src[u] + 4 * idx)
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            acc[q].x = fmaf(vv[u], t[u][q].x, acc[q].x);
            acc[q].y = fmaf(vv[u], t[u][q].y, acc[q].y);
            acc[q].z = fmaf(vv[u], t[u][q].z, acc[q].z);
            acc[q].w = fmaf(vv[u], t[u][q].w, acc[q].w);
          }
      }
    }
    float* y = a.Y + row * a.ldy;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      int idx = gl + q * LANES;
      if (idx < w4) {
        float4 r = acc[q];
        if (a.relu) {
          r.x = fmaxf(r.x, 0.f);
          r.y = fmaxf(r.y, 0.f);
          r.z = fmaxf(r.z, 0.f);
          r.w = fmaxf(r.w, 0.f);
        }
        reinterpret_cast<float4*>(y)[idx] = r;
      }
    }
  }
}

template <int LANES, int VPL>
digest_status launch(const SpmmArgs& a, cudaStream_t s) {
  constexpr int GROUPS = 32 / LANES;
  const int64_t warps = ceil_div(a.n_rows, GROUPS);
  int64_t blocks = ceil_div(warps, 8);
  const int64_t cap = (int64_t)num_sms() * 8 * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const double w = a.width;
  const double bytes = (double)a.nnz * (8.0 + 4.0 * w) + (double)a.n_rows * (4.0 * w + 8.0);
  const double flops = 2.0 * (double)a.nnz * w;
  DG_LAUNCH_TAG(DIGEST_PROF_SPMM, a.width, s, bytes, flops, (k_spmm<LANES, VPL>), (unsigned)blocks,
                256, 0, a);
  return DIGEST_OK;
}

}  // namespace

digest_status spmm(const SpmmArgs& a, cudaStream_t s) {
  if (a.n_rows == 0) return DIGEST_OK;
  DG_ARG(a.width > 0 && a.width % 4 == 0, DIGEST_E_INVALID,
         "SpMM width %d must be a positive multiple of 4", a.width);
  const int w4 = a.width / 4;
  if (w4 <= 1) return launch<1, 1>(a, s);
  if (w4 <= 2) return launch<2, 1>(a, s);
  if (w4 <= 4) return launch<4, 1>(a, s);
  if (w4 <= 8) return launch<8, 1>(a, s);
  if (w4 <= 12) return launch<4, 3>(a, s);
  if (w4 <= 16) return launch<16, 1>(a, s);
  if (w4 <= 32) return launch<32, 1>(a, s);
  if (w4 <= 64) return launch<32, 2>(a, s);
  if (w4 <= 96) return launch<32, 3>(a, s);
  if (w4 <= 128) return launch<32, 4>(a, s);
  if (w4 <= 192) return launch<32, 6>(a, s);
  if (w4 <= 256) return launch<32, 8>(a, s);
  if (w4 <= 384) return launch<32, 12>(a, s);
  return set_error(DIGEST_E_UNSUPPORTED, "SpMM width %d > 1536", a.width);
}

}  // namespace dg

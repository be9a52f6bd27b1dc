// Epilogue shared by the 3xTF32 GEMM kernels (gemm_tc.cu, gemm_tc2.cu): drains one
// 128-row accumulator tile from TMEM and applies, in registers, everything the layer
// fuses after the dense transform:
//   * ReLU (Eq. 5's sigma) and the 1-bit activation mask of its output
//     (bit j of word (row, c/32) = C[row, c] > 0),
//   * the consumer ReLU' of the previous layer (Eq. 6), either as a 1-bit mask
//     (mbits, 1/32 of the bytes) or as a float tensor (mask, 1[mask > 0]).
// TMEM gives lane l the 32 columns of row l; rows are staged through a per-warp
// 32 x 128 B shared buffer (16 B chunks XOR-swizzled by row, conflict-free) so the
// global stores are full 128 B lines: 4 rows x 8 chunks per warp store.
#pragma once
#include "kernels.cuh"
#include "tc_util.cuh"

namespace dg {

struct EpiArgs {
  float* C;
  int64_t ldc;
  int64_t M;
  int32_t N;
  int32_t relu;
  const float* mask;
  int64_t ldm;
  const uint32_t* mbits;
  int64_t ldmb;
  uint32_t* obits;
  int64_t ldob;
};

inline EpiArgs epi_of(const GemmArgs& g) {
  return EpiArgs{g.C, g.ldc, g.M, g.N, g.relu, g.mask, g.ldm, g.mbits, g.ldmb, g.obits, g.ldob};
}

__device__ __forceinline__ void prefetch_l2_line(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<uint64_t>(p)));
}

// Called by each of the 128 epilogue threads at the start of a tile: warm L2 with the
// consumer-mask rows of the tile this CTA drains NEXT (row = that tile's first row +
// tid), so the loads in epi_tile hit L2 instead of paying HBM latency in-line.
template <int BN>
__device__ __forceinline__ void epi_prefetch_next(const EpiArgs& e, int64_t next_row0, int tid) {
  const int64_t row = next_row0 + tid;
  if (next_row0 < 0 || row >= e.M) return;
  if (e.mask) tc::prefetch_l2_bulk(e.mask + row * e.ldm, 4 * min(BN, e.N));
  if (e.mbits) prefetch_l2_line(e.mbits + row * e.ldmb);
}

// Drain this warp's 32 rows (TMEM lane quarter q) of the tile at rows m0.., columns
// 0..N-1 (every kernel covers N in one tile, BN >= N, so column words align).
// Columns [c_beg, c_end) (multiples of 32): several warps may share a lane quarter.
template <int BN>
__device__ __forceinline__ void epi_tile(const EpiArgs& e, uint32_t tmem_acc, float4* stg,
                                         int64_t m0, int q, int lane, int c_beg = 0,
                                         int c_end = BN) {
  const int ch = lane & 7;
  const int64_t my_row = m0 + q * 32 + lane;   // the row TMEM hands this lane
  const bool my_ok = my_row < e.M;
  uint32_t mw_next = (e.mbits && my_ok && c_beg < c_end)
                         ? __ldg(e.mbits + my_row * e.ldmb + (c_beg >> 5)) : 0xffffffffu;
#pragma unroll 1
  for (int c0 = c_beg; c0 < c_end; c0 += 32) {
    float4 mk[8];
    if (e.mask) {  // issue all 8 mask loads before the TMEM read (8 in flight per lane)
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int64_t row = m0 + q * 32 + it * 4 + (lane >> 3);
        const int col = c0 + 4 * ch;
        mk[it] = (row < e.M && col < e.N)
                     ? __ldg(reinterpret_cast<const float4*>(e.mask + row * e.ldm + col))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const uint32_t mw = mw_next;
    if (e.mbits && my_ok && c0 + 32 < c_end && c0 + 32 < e.N)
      mw_next = __ldg(e.mbits + my_row * e.ldmb + ((c0 + 32) >> 5));
    uint32_t r[32];
    tc::tmem_ld_32x32b_x32(tmem_acc + ((uint32_t)(q * 32) << 16) + c0, r);
    tc::tmem_ld_wait();
    uint32_t ob = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                             __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      if (e.relu) {
        v.x = fmaxf(v.x, 0.f);
        v.y = fmaxf(v.y, 0.f);
        v.z = fmaxf(v.z, 0.f);
        v.w = fmaxf(v.w, 0.f);
      }
      if (e.mbits) {
        const uint32_t m = mw >> (4 * j);
        v.x = (m & 1u) ? v.x : 0.f;
        v.y = (m & 2u) ? v.y : 0.f;
        v.z = (m & 4u) ? v.z : 0.f;
        v.w = (m & 8u) ? v.w : 0.f;
      }
      ob |= ((v.x > 0.f ? 1u : 0u) | (v.y > 0.f ? 2u : 0u) | (v.z > 0.f ? 4u : 0u) |
             (v.w > 0.f ? 8u : 0u))
            << (4 * j);
      stg[lane * 8 + (j ^ (lane & 7))] = v;
    }
    // TMEM columns >= N were never written by the MMA (N < ACC): clear their bits
    if (e.N - c0 < 32) ob &= (1u << (max(e.N - c0, 0) & 31)) - 1u;
    if (e.obits && my_ok && c0 < e.N) e.obits[my_row * e.ldob + (c0 >> 5)] = ob;
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int rr = it * 4 + (lane >> 3);
      const int64_t row = m0 + q * 32 + rr;
      const int col = c0 + 4 * ch;
      if (row < e.M && col < e.N) {
        float4 v = stg[rr * 8 + (ch ^ (rr & 7))];
        if (e.mask) {
          v.x = mk[it].x > 0.f ? v.x : 0.f;
          v.y = mk[it].y > 0.f ? v.y : 0.f;
          v.z = mk[it].z > 0.f ? v.z : 0.f;
          v.w = mk[it].w > 0.f ? v.w : 0.f;
        }
        *reinterpret_cast<float4*>(e.C + row * e.ldc + col) = v;
      }
    }
    __syncwarp();
  }
}

}  // namespace dg

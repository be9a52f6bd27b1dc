// CSR-row SpMM over the extended column space [local ; halo] (Eq. 5's
// P_in H_in + P_out H~_out, as ONE product with two source pointers).
//
// Design: warp per row, edge groups x float4 column lanes,
// 128-bit loads, coalesced (col, val) chunks broadcast by shuffles, UNR
// independent row gathers in flight per edge group (memory-level parallelism).
// Halo rows come from a second pointer (no copy of the stale store into a
// contiguous X_ext).  HBM-bound: ~2 flop per (8 + 4w) bytes per nonzero.
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace dg {
// gemm_tc.cu: TMA map for tile::gather4 row copies of an fp32 [outer x inner] matrix
bool make_tmap_rows_fwd(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes);
namespace {

// L2 cache policies: the gathered source rows are re-read by many rows (keep them),
// the CSR streams are touched once (evict them first).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_gather(const float* ptr, uint64_t pol) {
  float4 r;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ int32_t ld_stream_i(const int32_t* ptr, uint64_t pol) {
  int32_t r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_stream_f(const float* ptr, uint64_t pol) {
  float r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// Row epilogue shared by both kernels.  Lanes of edge group 0 hold the reduced row
// (float4 column idx = cl + q*LC): optional ReLU, the consumer's ReLU' (float mask or
// 1-bit mask), the store, and optionally the 1-bit mask of the stored row (SURVEY §8
// a5): word k collects the nibbles of float4 columns 8k..8k+7 with a warp OR-reduce.
template <int LC, int VPL>
__device__ __forceinline__ void spmm_row_epilogue(const SpmmArgs& a, int64_t row, int lane, int cl,
                                                  int g, int w4, float4 (&acc)[VPL]) {
  uint32_t nib[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) nib[q] = 0;
  if (g == 0) {
    float* y = a.Y + row * a.ldy;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int idx = cl + q * LC;
      if (idx < w4) {
        float4 r = acc[q];
        if (a.relu) {
          r.x = fmaxf(r.x, 0.f);
          r.y = fmaxf(r.y, 0.f);
          r.z = fmaxf(r.z, 0.f);
          r.w = fmaxf(r.w, 0.f);
        }
        if (a.mask) {
          const float4 mk = ldg4(a.mask + row * a.ldm + 4 * idx);
          r.x = mk.x > 0.f ? r.x : 0.f;
          r.y = mk.y > 0.f ? r.y : 0.f;
          r.z = mk.z > 0.f ? r.z : 0.f;
          r.w = mk.w > 0.f ? r.w : 0.f;
        }
        if (a.mbits) {
          const uint32_t m = __ldg(a.mbits + row * a.ldmb + (idx >> 3)) >> ((idx & 7) * 4);
          r.x = (m & 1u) ? r.x : 0.f;
          r.y = (m & 2u) ? r.y : 0.f;
          r.z = (m & 4u) ? r.z : 0.f;
          r.w = (m & 8u) ? r.w : 0.f;
        }
        nib[q] = (r.x > 0.f ? 1u : 0u) | (r.y > 0.f ? 2u : 0u) | (r.z > 0.f ? 4u : 0u) |
                 (r.w > 0.f ? 8u : 0u);
        if (a.stream_out)   // streaming store: the output row is not re-read by this launch
          __stcs(reinterpret_cast<float4*>(y) + idx, r);
        else
          reinterpret_cast<float4*>(y)[idx] = r;
      }
    }
  }
  if (a.obits) {   // warp-uniform
    const int nw = (w4 + 7) >> 3;
    for (int k = 0; k < nw; ++k) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int idx = cl + q * LC;
        if ((idx >> 3) == k) c |= nib[q] << ((idx & 7) * 4);
      }
      c = __reduce_or_sync(0xffffffffu, c);
      if (lane == 0) a.obits[row * a.ldob + k] = c;
    }
  }
}

// One warp per output row.  The warp is split into EG = 32/LC edge groups of LC
// lanes; edge group g handles edges j = g, g+EG, ... of the row, lane c of a group
// owns float4 columns c, c+LC, ... (VPL of them).  The 32 (col, val) pairs of a
// chunk are loaded once, coalesced, and broadcast with full-warp shuffles; the next
// chunk's pairs are prefetched while the current one is gathered (software
// pipelining of the col -> row dependency).  A chunk is consumed in STEPS fully
// unrolled, predicated steps of UNR edges per group, so up to STEPS*UNR*VPL 16-byte
// gathers per lane can be in flight.  Edge-group partial sums are combined with xor
// shuffles at the end of the row.  All loop counts are warp-uniform.
// XR (cross-row pipelining): the warp's NEXT row's bounds are loaded when a row
// starts and its first (col, val) chunk is loaded during the current row's last
// gathers, so the row_ptr -> col -> gather dependency chain of a row overlaps the
// previous row's gathers instead of following them (latency-bound narrow rows).
// H: per-gather L2 cache-policy operands (bit-31 hot rows evict_last); without them the
// gathers are plain ld.global.nc (no per-load R2UR of a policy descriptor).
template <int LC, int VPL, int UNR, bool XR, int MB, bool H = true>
__global__ void __launch_bounds__(256, MB) k_spmm(SpmmArgs a) {
  constexpr int EG = 32 / LC;
  constexpr int STEP = EG * UNR;
  constexpr int STEPS = (32 + STEP - 1) / STEP;   // cover all 32 pairs of a chunk
  const int lane = threadIdx.x & 31;
  const int cl = lane % LC;
  const int g = lane / LC;
  const int w4 = a.width >> 2;
  // hints: 1 hot evict_last / rest evict_first, 2 hot evict_last / rest normal, 3 all
  // evict_last, 4 hot normal / rest evict_first (cold rows leave L2 first; no lines pinned)
  const uint64_t pol_x = (a.hints && a.hints != 4) ? policy_evict_last() : policy_evict_normal();
  const uint64_t pol_s = a.hints ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_c = (a.hints == 1 || a.hints == 4) ? policy_evict_first()
                         : a.hints == 3                 ? policy_evict_last()
                                                        : policy_evict_normal();
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t beg = 0, end = 0;
  int32_t c_nxt = 0;
  float v_nxt = 0.f;
  if (XR && warp < a.n_rows) {
    beg = a.row_ptr[warp];
    end = a.in_len ? beg + a.in_len[warp] : a.row_ptr[warp + 1];
    if (beg + lane < end) {
      c_nxt = ld_stream_i(a.col + beg + lane, pol_s);
      v_nxt = ld_stream_f(a.val + beg + lane, pol_s);
    }
  }
  for (int64_t row = warp; row < a.n_rows; row += nwarps) {
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t nbeg = 0, nend = 0;
    if (XR) {
      const int64_t nrow = row + nwarps;
      if (nrow < a.n_rows) {
        nbeg = a.row_ptr[nrow];
        nend = a.in_len ? nbeg + a.in_len[nrow] : a.row_ptr[nrow + 1];
      }
    } else {
      beg = a.row_ptr[row];
      end = a.in_len ? beg + a.in_len[row] : a.row_ptr[row + 1];
      if (beg + lane < end) {
        c_nxt = ld_stream_i(a.col + beg + lane, pol_s);
        v_nxt = ld_stream_f(a.val + beg + lane, pol_s);
      }
    }
    // the next row's first chunk (XR): loaded in the last chunk, after its gathers issue
    auto next_row_chunk = [&]() {
      c_nxt = 0;
      v_nxt = 0.f;
      if (nbeg + lane < nend) {
        c_nxt = ld_stream_i(a.col + nbeg + lane, pol_s);
        v_nxt = ld_stream_f(a.val + nbeg + lane, pol_s);
      }
    };
    if (XR && end <= beg) next_row_chunk();
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
      const int32_t c = c_nxt;
      const float v = v_nxt;
      const int cnt = (int)min((int64_t)32, end - e0);
      const bool last = e0 + 32 >= end;
      if (!last && e0 + 32 + lane < end) {
        c_nxt = ld_stream_i(a.col + e0 + 32 + lane, pol_s);
        v_nxt = ld_stream_f(a.val + e0 + 32 + lane, pol_s);
      }
#pragma unroll
      for (int st = 0; st < STEPS; ++st) {
        const float* src[UNR];
        float vv[UNR];
        bool ok[UNR];
        uint64_t pol[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int j = st * STEP + u * EG + g;
          const int cr = __shfl_sync(0xffffffffu, c, j & 31);
          const float x = __shfl_sync(0xffffffffu, v, j & 31);
          const int cj = cr & 0x7fffffff;   // bit 31: L2-hot source row (partition hint)
          pol[u] = cr < 0 ? pol_x : pol_c;
          ok[u] = g < EG && j < cnt;
          vv[u] = ok[u] ? x : 0.f;
          src[u] = (int64_t)cj < a.split ? a.X0 + (int64_t)cj * a.ld0
                                         : a.X1 + ((int64_t)cj - a.split) * a.ld1;
        }
        float4 t[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            const int idx = cl + q * LC;
            t[u][q] = (ok[u] && idx < w4) ? (H ? ld_gather(src[u] + 4 * idx, pol[u])
                                                 : ldg4(src[u] + 4 * idx))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        if (XR && st == 0 && last) next_row_chunk();
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            acc[q].x = fmaf(vv[u], t[u][q].x, acc[q].x);
            acc[q].y = fmaf(vv[u], t[u][q].y, acc[q].y);
            acc[q].z = fmaf(vv[u], t[u][q].z, acc[q].z);
            acc[q].w = fmaf(vv[u], t[u][q].w, acc[q].w);
          }
      }
    }
#pragma unroll
    for (int off = LC; off < EG * LC; off <<= 1)   // tree over the edge groups
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const bool in = lane + off < EG * LC;
        const float x = __shfl_down_sync(0xffffffffu, acc[q].x, off);
        const float y = __shfl_down_sync(0xffffffffu, acc[q].y, off);
        const float z = __shfl_down_sync(0xffffffffu, acc[q].z, off);
        const float w = __shfl_down_sync(0xffffffffu, acc[q].w, off);
        if (in) {
          acc[q].x += x;
          acc[q].y += y;
          acc[q].z += z;
          acc[q].w += w;
        }
      }
    spmm_row_epilogue<LC, VPL>(a, row, lane, cl, g, w4, acc);
    if (XR) {
      beg = nbeg;
      end = nend;
    }
  }
}

// Runtime-trip-count variant (no chunk prefetch, default caching): fewer registers,
// higher occupancy; best for the wide rows (measured).
template <int LC, int VPL, int UNR, int MB>
__global__ void __launch_bounds__(256, MB) k_spmm_rt(SpmmArgs a) {
  constexpr int EG = 32 / LC;
  const int lane = threadIdx.x & 31;
  const int cl = lane % LC;
  const int g = lane / LC;
  const int w4 = a.width >> 2;
  const uint64_t pol_x = policy_evict_last();
  const uint64_t pol_s = a.hints == 1   ? policy_evict_first()
                         : a.hints == 3 ? policy_evict_last()
                                        : policy_evict_normal();
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < a.n_rows; row += nwarps) {
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t beg = a.row_ptr[row];
    const int64_t end = a.in_len ? beg + a.in_len[row] : a.row_ptr[row + 1];
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
      const int64_t e = e0 + lane;
      int32_t c = 0;
      float v = 0.f;
      if (e < end) {
        c = __ldg(a.col + e);
        v = __ldg(a.val + e);
      }
      const int cnt = (int)min((int64_t)32, end - e0);
      for (int j0 = 0; j0 < cnt; j0 += EG * UNR) {
        const float* src[UNR];
        float vv[UNR];
        bool ok[UNR];
        bool hot[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int j = j0 + u * EG + g;
          const int cr = __shfl_sync(0xffffffffu, c, j & 31);
          const float x = __shfl_sync(0xffffffffu, v, j & 31);
          const int cj = cr & 0x7fffffff;   // bit 31: L2-hot source row (partition hint)
          hot[u] = cr < 0;
          ok[u] = g < EG && j < cnt;
          vv[u] = ok[u] ? x : 0.f;
          src[u] = (int64_t)cj < a.split ? a.X0 + (int64_t)cj * a.ld0
                                         : a.X1 + ((int64_t)cj - a.split) * a.ld1;
        }
        float4 t[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            const int idx = cl + q * LC;
            t[u][q] = !(ok[u] && idx < w4) ? make_float4(0.f, 0.f, 0.f, 0.f)
                      : !a.hints ? ldg4(src[u] + 4 * idx)
                                 : ld_gather(src[u] + 4 * idx, hot[u] ? pol_x : pol_s);
          }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            acc[q].x = fmaf(vv[u], t[u][q].x, acc[q].x);
            acc[q].y = fmaf(vv[u], t[u][q].y, acc[q].y);
            acc[q].z = fmaf(vv[u], t[u][q].z, acc[q].z);
            acc[q].w = fmaf(vv[u], t[u][q].w, acc[q].w);
          }
      }
    }
#pragma unroll
    for (int off = LC; off < EG * LC; off <<= 1)   // tree over the edge groups
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const bool in = lane + off < EG * LC;
        const float x = __shfl_down_sync(0xffffffffu, acc[q].x, off);
        const float y = __shfl_down_sync(0xffffffffu, acc[q].y, off);
        const float z = __shfl_down_sync(0xffffffffu, acc[q].z, off);
        const float w = __shfl_down_sync(0xffffffffu, acc[q].w, off);
        if (in) {
          acc[q].x += x;
          acc[q].y += y;
          acc[q].z += z;
          acc[q].w += w;
        }
      }
    spmm_row_epilogue<LC, VPL>(a, row, lane, cl, g, w4, acc);
  }
}

// Lean narrow-slab kernel (w <= 64 floats per launch; wider products run as column
// slabs of it, see spmm_slab_width).  Same lane layout as k_spmm -- warp per row, EG =
// 32/LC edge groups x LC lanes x VPL float4 -- but built for the instruction budget of an
// L2-fabric-bound gather (tools/gather_roof.cu: ~18-20 TB/s of L2-resident row gathers on
// this B200): 32-bit source offsets (one IMAD.WIDE.U32 per gather: the hot bit 31 is
// shifted out and the row stride halved), one base select for two-source products (X1 is
// pre-offset by -split rows, so both sources index with the same column), no per-gather
// predicate selects (lanes past the chunk read vals of 0 and skip the load), the next
// chunk's (col, val) prefetched under the current gathers, and a warp-uniform exit from
// the unrolled steps of a short chunk.  RAG: the slab is not a multiple of 4*LC floats
// (the last float4 of a lane is predicated on the slab width).
// XR (cross-row software pipelining): the next row's bounds load when a row starts and
// its first (col, val) chunk loads under the current row's last gathers, so a row's
// row_ptr -> col -> gather chain overlaps the previous row instead of following it.
// CH: the CSR streams (touched once) load with an L2 evict_first policy so they do not
// displace the gathered source rows, which are reused by ~avg-degree rows.
template <int LC, int VPL, int UNR, bool TWO, bool RAG, int MB, bool XR = false, bool CH = false>
__global__ void __launch_bounds__(256, MB) k_spmm_n(SpmmArgs a, const char* __restrict__ x0,
                                                    const char* __restrict__ x1m,
                                                    uint32_t split, uint32_t rb_half) {
  const uint64_t pol_s = CH ? policy_evict_first() : 0;
  auto ldc = [&](const int32_t* p) { return CH ? ld_stream_i(p, pol_s) : __ldg(p); };
  auto ldv = [&](const float* p) { return CH ? ld_stream_f(p, pol_s) : __ldg(p); };
  constexpr int EG = 32 / LC;
  constexpr int STEP = EG * UNR;
  constexpr int STEPS = (32 + STEP - 1) / STEP;
  const int lane = threadIdx.x & 31;
  const int cl = lane % LC;
  const int g = lane / LC;
  const int w4 = a.width >> 2;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  auto bounds = [&](int64_t r, int64_t& b, int64_t& e) {
    b = e = 0;
    if (r < a.n_rows) {
      b = a.row_ptr[r];
      e = a.in_len ? b + a.in_len[r] : a.row_ptr[r + 1];
    }
  };
  int64_t beg, end;
  int32_t c_nxt = 0;
  float v_nxt = 0.f;
  if (XR) {
    bounds(warp, beg, end);
    if (beg + lane < end) {
      c_nxt = ldc(a.col + beg + lane);
      v_nxt = ldv(a.val + beg + lane);
    }
  }
  for (int64_t row = warp; row < a.n_rows; row += nwarps) {
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t nbeg = 0, nend = 0;
    if (XR) {
      bounds(row + nwarps, nbeg, nend);
      if (end <= beg) {   // empty row: its "last chunk" is the next row's first
        c_nxt = 0;
        v_nxt = 0.f;
        if (nbeg + lane < nend) {
          c_nxt = ldc(a.col + nbeg + lane);
          v_nxt = ldv(a.val + nbeg + lane);
        }
      }
    } else {
      bounds(row, beg, end);
      c_nxt = 0;
      v_nxt = 0.f;
      if (beg + lane < end) {
        c_nxt = ldc(a.col + beg + lane);
        v_nxt = ldv(a.val + beg + lane);
      }
    }
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
      const int32_t c = c_nxt;
      const float v = v_nxt;
      const int cnt = (int)min((int64_t)32, end - e0);
      c_nxt = 0;
      v_nxt = 0.f;
      if (e0 + 32 < end) {
        if (e0 + 32 + lane < end) {
          c_nxt = ldc(a.col + e0 + 32 + lane);
          v_nxt = ldv(a.val + e0 + 32 + lane);
        }
      } else if (XR && nbeg + lane < nend) {   // last chunk: the next row's first
        c_nxt = ldc(a.col + nbeg + lane);
        v_nxt = ldv(a.val + nbeg + lane);
      }
#pragma unroll
      for (int st = 0; st < STEPS; ++st) {
        if (st * STEP >= cnt) break;   // warp-uniform
        // Lanes past the chunk hold (col 0, val 0): their gathers read source row 0
        // (valid, L1-resident) and contribute 0 -- no predicates, so every load of the
        // step issues before the first FMA waits.  RAG: the last float4 of a lane past
        // the slab re-reads the slab's last float4 into an accumulator never stored.
        float4 t[UNR][VPL];
        float x[UNR];
        const float4* p[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int j = st * STEP + u * EG + g;
          const uint32_t cr = (uint32_t)__shfl_sync(0xffffffffu, c, j);
          x[u] = __shfl_sync(0xffffffffu, v, j);
          const char* base = x0;
          if (TWO) base = (cr & 0x7fffffffu) >= split ? x1m : x0;
          p[u] = reinterpret_cast<const float4*>(base + (uint64_t)(cr << 1) * rb_half);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            const int idx = cl + q * LC;
            t[u][q] = __ldg(p[u] + (RAG && q == VPL - 1 ? min(idx, w4 - 1) : idx));
          }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            acc[q].x = fmaf(x[u], t[u][q].x, acc[q].x);
            acc[q].y = fmaf(x[u], t[u][q].y, acc[q].y);
            acc[q].z = fmaf(x[u], t[u][q].z, acc[q].z);
            acc[q].w = fmaf(x[u], t[u][q].w, acc[q].w);
          }
      }
    }
#pragma unroll
    for (int off = LC; off < 32; off <<= 1)   // tree over the edge groups
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        acc[q].x += __shfl_down_sync(0xffffffffu, acc[q].x, off);
        acc[q].y += __shfl_down_sync(0xffffffffu, acc[q].y, off);
        acc[q].z += __shfl_down_sync(0xffffffffu, acc[q].z, off);
        acc[q].w += __shfl_down_sync(0xffffffffu, acc[q].w, off);
      }
    spmm_row_epilogue<LC, VPL>(a, row, lane, cl, g, w4, acc);
    if (XR) {
      beg = nbeg;
      end = nend;
    }
  }
}

// Grouped narrow kernel (k_spmm_g): one ROW per edge group.  The lean kernel spends a
// warp on one row -- at every row start the row_ptr -> (col, val) -> gather chain runs with
// no gathers in flight, and the edge groups' partial sums meet in a shuffle tree -- which
// keeps it at about half of the L2 gather roof.  Here the EG = 32/LC groups
// of a warp take EG different rows, taken side by side from the partition's length-grouped
// row order (digest_part::ord_*: rows grouped by length bin within windows of 4096
// consecutive rows, so the warp's rows have similar lengths and the sweep keeps its L2
// locality).  Each group walks its own row UNR edges per step; the chain is paid once per EG
// rows, no cross-group reduction is needed (a group's lanes own disjoint columns), and the
// (col, val) of the next step are loaded one step ahead (L1-cached: a group reads its row's
// 128-byte lines over consecutive steps; L2 evict_first as in the lean kernel).
__device__ __forceinline__ int32_t ld_csr_i(const int32_t* ptr, uint64_t pol) {
  int32_t r;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_csr_f(const float* ptr, uint64_t pol) {
  float r;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(ptr), "l"(pol));
  return r;
}

// Group epilogue: the LC lanes of a group hold the whole row (float4 columns cl + q*LC).
template <int LC, int VPL>
__device__ __forceinline__ void spmm_group_epilogue(const SpmmArgs& a, int64_t row, int lane,
                                                    int cl, int w4, const float4 (&acc)[VPL]) {
  uint32_t nib[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) nib[q] = 0;
  if (row >= 0) {
    float* y = a.Y + row * a.ldy;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int idx = cl + q * LC;
      if (idx < w4) {
        float4 r = acc[q];
        if (a.relu) {
          r.x = fmaxf(r.x, 0.f);
          r.y = fmaxf(r.y, 0.f);
          r.z = fmaxf(r.z, 0.f);
          r.w = fmaxf(r.w, 0.f);
        }
        if (a.mask) {
          const float4 mk = ldg4(a.mask + row * a.ldm + 4 * idx);
          r.x = mk.x > 0.f ? r.x : 0.f;
          r.y = mk.y > 0.f ? r.y : 0.f;
          r.z = mk.z > 0.f ? r.z : 0.f;
          r.w = mk.w > 0.f ? r.w : 0.f;
        }
        if (a.mbits) {
          const uint32_t m = __ldg(a.mbits + row * a.ldmb + (idx >> 3)) >> ((idx & 7) * 4);
          r.x = (m & 1u) ? r.x : 0.f;
          r.y = (m & 2u) ? r.y : 0.f;
          r.z = (m & 4u) ? r.z : 0.f;
          r.w = (m & 8u) ? r.w : 0.f;
        }
        nib[q] = (r.x > 0.f ? 1u : 0u) | (r.y > 0.f ? 2u : 0u) | (r.z > 0.f ? 4u : 0u) |
                 (r.w > 0.f ? 8u : 0u);
        if (a.stream_out)
          __stcs(reinterpret_cast<float4*>(y) + idx, r);
        else
          reinterpret_cast<float4*>(y)[idx] = r;
      }
    }
  }
  if (a.obits) {   // warp-uniform; word k = float4 columns 8k..8k+7, OR over the group's lanes
    const int nw = (w4 + 7) >> 3;
    for (int k = 0; k < nw; ++k) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int idx = cl + q * LC;
        if ((idx >> 3) == k) c |= nib[q] << ((idx & 7) * 4);
      }
#pragma unroll
      for (int off = 1; off < LC; off <<= 1) c |= __shfl_xor_sync(0xffffffffu, c, off);
      if (cl == 0 && row >= 0) a.obits[row * a.ldob + k] = c;
    }
  }
  (void)lane;
}

// POL (experiment): per-gather L2 policy from the partition's hot bit (bit 31 of col):
// hot source rows evict_normal, the others evict_first, so the rarely re-read rows leave
// L2 before the often re-read ones.
template <int POL>
__device__ __forceinline__ float4 g_gather(const float4* p, uint32_t cr, uint64_t ph, uint64_t pc) {
  if (POL) return ld_gather(reinterpret_cast<const float*>(p), (int32_t)cr < 0 ? ph : pc);
  return __ldg(p);
}

template <int LC, int VPL, int UNR, bool TWO, bool RAG, int MB, int POL = 0, bool COOP = false>
__global__ void __launch_bounds__(256, MB) k_spmm_g(SpmmArgs a, const char* __restrict__ x0,
                                                    const char* __restrict__ x1m,
                                                    uint32_t split, uint32_t rb_half,
                                                    unsigned long long* __restrict__ ctr) {
  constexpr int EG = 32 / LC;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_h = POL ? policy_evict_normal() : 0;
  const int lane = threadIdx.x & 31;
  const int cl = lane % LC;
  const int g = lane / LC;
  const int w4 = a.width >> 2;
  // Batches of EG slots are handed out by an atomic counter (zeroed before the launch): a
  // warp that drew long rows simply draws fewer batches, so the rows in flight stay one
  // narrow window and the sweep keeps its L2 locality.  (A static round-robin deal drifts:
  // the length-grouped order gives some warps systematically longer rows, and the window
  // spread over several planted blocks -- L2 hit 65% -> 23-36%, measured.)
  for (;;) {
    unsigned long long b0 = 0;
    if (lane == 0) b0 = atomicAdd(ctr, (unsigned long long)EG);
    const int64_t base = (int64_t)__shfl_sync(0xffffffffu, b0, 0);
    if (base >= a.n_rows) break;
    const int64_t slot = base + g;
    int64_t row = -1, beg = 0, end = 0;
    if (slot < a.n_rows) {
      row = __ldg(a.order + slot);
      beg = a.row_ptr[row];
      end = a.in_len ? beg + a.in_len[row] : a.row_ptr[row + 1];
    }
    const int len = (int)(end - beg);
    const int mx = __reduce_max_sync(0xffffffffu, len);
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    // A batch from the long tail (rows up to 5k entries; the length bins are 32 wide above
    // 64) can be far from uniform: side by side its groups would all wait for the longest
    // row (max / UNR steps).  Then the warp takes the batch's rows one at a time instead,
    // all groups on one row as in the lean kernel (sum / (EG UNR) steps + one chain per row).
    const int sum = __reduce_add_sync(0xffffffffu, cl == 0 ? len : 0);
    if (mx * EG > sum + 64 * EG) {
      for (int r = 0; r < EG; ++r) {
        const int64_t rr = __shfl_sync(0xffffffffu, row, r * LC);
        const int64_t rb = __shfl_sync(0xffffffffu, beg, r * LC);
        const int64_t re = __shfl_sync(0xffffffffu, end, r * LC);
        if (rr < 0) continue;   // warp-uniform
#pragma unroll
        for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t e0 = rb; e0 < re; e0 += 32) {
          int32_t cc = 0;
          float vv = 0.f;
          if (e0 + lane < re) {
            cc = ld_csr_i(a.col + e0 + lane, pol_s);
            vv = ld_csr_f(a.val + e0 + lane, pol_s);
          }
          const int cnt = (int)min((int64_t)32, re - e0);
          for (int j0 = 0; j0 < cnt; j0 += EG * UNR) {   // warp-uniform
            float4 t[UNR][VPL];
            float x[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
              const int j = j0 + u * EG + g;   // < 32; past cnt: (col 0, val 0)
              const uint32_t cr = (uint32_t)__shfl_sync(0xffffffffu, cc, j);
              x[u] = __shfl_sync(0xffffffffu, vv, j);
              const char* bs = x0;
              if (TWO) bs = (cr & 0x7fffffffu) >= split ? x1m : x0;
              const float4* p = reinterpret_cast<const float4*>(bs + (uint64_t)(cr << 1) * rb_half);
#pragma unroll
              for (int q = 0; q < VPL; ++q) {
                const int idx = cl + q * LC;
                t[u][q] = g_gather<POL>(p + (RAG && q == VPL - 1 ? min(idx, w4 - 1) : idx), cr,
                                        pol_h, pol_s);
              }
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
              for (int q = 0; q < VPL; ++q) {
                acc[q].x = fmaf(x[u], t[u][q].x, acc[q].x);
                acc[q].y = fmaf(x[u], t[u][q].y, acc[q].y);
                acc[q].z = fmaf(x[u], t[u][q].z, acc[q].z);
                acc[q].w = fmaf(x[u], t[u][q].w, acc[q].w);
              }
          }
        }
#pragma unroll
        for (int off = LC; off < 32; off <<= 1)   // tree over the edge groups
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            acc[q].x += __shfl_down_sync(0xffffffffu, acc[q].x, off);
            acc[q].y += __shfl_down_sync(0xffffffffu, acc[q].y, off);
            acc[q].z += __shfl_down_sync(0xffffffffu, acc[q].z, off);
            acc[q].w += __shfl_down_sync(0xffffffffu, acc[q].w, off);
          }
        spmm_row_epilogue<LC, VPL>(a, rr, lane, cl, g, w4, acc);
      }
      continue;
    }
    if constexpr (COOP) {
      // (col, val) of a step loaded once per group: lane cl < UNR loads entry cl (one
      // coalesced 4*UNR-byte read per group and array) and the group's lanes take the UNR
      // entries by shuffles at the step start -- 2 loads per lane per step instead of 2 UNR.
      static_assert(UNR <= LC, "COOP needs UNR <= LC");
      const int gb = lane & ~(LC - 1);
      int32_t mc = 0;
      float mv = 0.f;
      if (cl < UNR && cl < len) {
        mc = ld_csr_i(a.col + beg + cl, pol_s);
        mv = ld_csr_f(a.val + beg + cl, pol_s);
      }
      for (int e = 0; e < mx; e += UNR) {
        int32_t c[UNR];
        float v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          c[u] = __shfl_sync(0xffffffffu, mc, gb + u);
          v[u] = __shfl_sync(0xffffffffu, mv, gb + u);
        }
        mc = 0;
        mv = 0.f;
        if (cl < UNR && e + UNR + cl < len) {
          mc = ld_csr_i(a.col + beg + e + UNR + cl, pol_s);
          mv = ld_csr_f(a.val + beg + e + UNR + cl, pol_s);
        }
        float4 t[UNR][VPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const uint32_t cr = (uint32_t)c[u];
          const char* bs = x0;
          if (TWO) bs = (cr & 0x7fffffffu) >= split ? x1m : x0;
          const float4* p = reinterpret_cast<const float4*>(bs + (uint64_t)(cr << 1) * rb_half);
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            const int idx = cl + q * LC;
            t[u][q] = g_gather<POL>(p + (RAG && q == VPL - 1 ? min(idx, w4 - 1) : idx), cr,
                                    pol_h, pol_s);
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            acc[q].x = fmaf(v[u], t[u][q].x, acc[q].x);
            acc[q].y = fmaf(v[u], t[u][q].y, acc[q].y);
            acc[q].z = fmaf(v[u], t[u][q].z, acc[q].z);
            acc[q].w = fmaf(v[u], t[u][q].w, acc[q].w);
          }
      }
      spmm_group_epilogue<LC, VPL>(a, row, lane, cl, w4, acc);
      continue;
    }
    int32_t c[UNR];
    float v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      c[u] = 0;
      v[u] = 0.f;
      if (u < len) {
        c[u] = ld_csr_i(a.col + beg + u, pol_s);
        v[u] = ld_csr_f(a.val + beg + u, pol_s);
      }
    }
    for (int e = 0; e < mx; e += UNR) {
      // next step's (col, val): in flight while this step's gathers are
      int32_t cn[UNR];
      float vn[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        cn[u] = 0;
        vn[u] = 0.f;
        if (e + UNR + u < len) {
          cn[u] = ld_csr_i(a.col + beg + e + UNR + u, pol_s);
          vn[u] = ld_csr_f(a.val + beg + e + UNR + u, pol_s);
        }
      }
      // past its row's end a group gathers source row 0 (valid) with weight 0: no predicates
      float4 t[UNR][VPL];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint32_t cr = (uint32_t)c[u];
        const char* bs = x0;
        if (TWO) bs = (cr & 0x7fffffffu) >= split ? x1m : x0;
        const float4* p = reinterpret_cast<const float4*>(bs + (uint64_t)(cr << 1) * rb_half);
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int idx = cl + q * LC;
          t[u][q] = g_gather<POL>(p + (RAG && q == VPL - 1 ? min(idx, w4 - 1) : idx), cr,
                                  pol_h, pol_s);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          acc[q].x = fmaf(v[u], t[u][q].x, acc[q].x);
          acc[q].y = fmaf(v[u], t[u][q].y, acc[q].y);
          acc[q].z = fmaf(v[u], t[u][q].z, acc[q].z);
          acc[q].w = fmaf(v[u], t[u][q].w, acc[q].w);
        }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        c[u] = cn[u];
        v[u] = vn[u];
      }
    }
    spmm_group_epilogue<LC, VPL>(a, row, lane, cl, w4, acc);
  }
}

// Single-source product through TMA row gathers (tile::gather4), experimental
// (DIGEST_SPMM_TMA=1; measured 1.45-1.6x SLOWER than the load-based kernels at w=48/100,
// products M=1 and 8 parts -- profiles/r1_spmm_variant_sweep.log -- so it is off).  Warp per row as above, but the 32 gathered rows of a (col, val)
// chunk are fetched by ceil(cnt/4) gather4 copies that one lane issues into a per-warp
// shared-memory buffer (two buffers: the next chunk -- possibly of the next row -- is in
// flight while the current one is consumed), so no registers are tied up by loads in
// flight and the row_ptr -> col -> gather chain of the next row overlaps this row.
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t r0,
                                        int32_t r1, int32_t r2, int32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint32_t a = tc::smem_u32(bar);
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 10ull * 1000000000ull) __trap();
  }
}

template <int LC, int VPL>
__global__ void __launch_bounds__(256) k_spmm_tg(SpmmArgs a, const __grid_constant__ CUtensorMap tm,
                                                 int slot_bytes) {
  constexpr int EG = 32 / LC;
  extern __shared__ __align__(128) uint8_t smem_tg[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw_cta = blockDim.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_tg) + wib * 2;
  int32_t* idx = reinterpret_cast<int32_t*>(smem_tg + 1024) + wib * 32;
  uint8_t* ring = smem_tg + 2048 + (size_t)wib * 16 * slot_bytes;
  if (lane == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  __syncwarp();
  const int cl = lane % LC, g = lane / LC, w4 = a.width >> 2;
  const int row_bytes = a.width * 4;
  const int64_t nwarps = (int64_t)gridDim.x * nw_cta;
  int64_t irow = (int64_t)blockIdx.x * nw_cta + wib, ie0 = 0, iend = 0;
  if (irow < a.n_rows) {
    ie0 = a.row_ptr[irow];
    iend = a.in_len ? ie0 + a.in_len[irow] : a.row_ptr[irow + 1];
  }
  int64_t crow[2] = {0, 0};
  int ccnt[2] = {0, 0};
  bool clast[2] = {false, false};
  float v0 = 0.f, v1 = 0.f;
  uint32_t ph0 = 0, ph1 = 0;
  float4 acc[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);

  auto issue = [&](int b) -> bool {
    if (irow >= a.n_rows) return false;
    const int64_t e0 = ie0;
    const int cnt = (int)min((int64_t)32, iend - e0);
    int32_t c = 0;
    float v = 0.f;
    if (lane < cnt) {
      c = __ldg(a.col + e0 + lane) & 0x7fffffff;
      v = __ldg(a.val + e0 + lane);
    } else if (cnt > 0) {
      c = __ldg(a.col + e0) & 0x7fffffff;   // pad a gather4 group with a row already fetched
    }
    crow[b] = irow;
    ccnt[b] = cnt;
    if (b) v1 = v; else v0 = v;
    ie0 += 32;
    clast[b] = ie0 >= iend;
    if (clast[b]) {
      irow += nwarps;
      if (irow < a.n_rows) {
        ie0 = a.row_ptr[irow];
        iend = a.in_len ? ie0 + a.in_len[irow] : a.row_ptr[irow + 1];
      }
    }
    if (cnt > 0) {
      idx[lane] = c;
      __syncwarp();
      if (lane == 0) {
        const int ng = (cnt + 3) >> 2;
        tc::mbar_arrive_expect_tx(&bar[b], (uint32_t)(ng * 4 * row_bytes));
        uint8_t* dst = ring + (size_t)b * 8 * slot_bytes;
        for (int q = 0; q < ng; ++q)
          gather4(dst + (size_t)q * slot_bytes, &tm, &bar[b], idx[4 * q], idx[4 * q + 1],
                  idx[4 * q + 2], idx[4 * q + 3]);
      }
      __syncwarp();
    }
    return true;
  };

  auto consume = [&](int b) {
    const int cnt = ccnt[b];
    if (cnt > 0) {
      if (b) { mbar_wait_bounded(&bar[1], ph1); ph1 ^= 1; }
      else   { mbar_wait_bounded(&bar[0], ph0); ph0 ^= 1; }
    }
    const float v = b ? v1 : v0;
    const uint8_t* base = ring + (size_t)b * 8 * slot_bytes;
#pragma unroll 4
    for (int j0 = 0; j0 < 32; j0 += EG) {
      if (j0 >= cnt) break;
      const int j = j0 + g;
      const float x = __shfl_sync(0xffffffffu, v, j & 31);
      if (g < EG && j < cnt) {
        const float* rowp = reinterpret_cast<const float*>(base + (size_t)(j >> 2) * slot_bytes +
                                                           (size_t)(j & 3) * row_bytes);
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int i4 = cl + q * LC;
          if (i4 < w4) {
            const float4 t = reinterpret_cast<const float4*>(rowp)[i4];
            acc[q].x = fmaf(x, t.x, acc[q].x);
            acc[q].y = fmaf(x, t.y, acc[q].y);
            acc[q].z = fmaf(x, t.z, acc[q].z);
            acc[q].w = fmaf(x, t.w, acc[q].w);
          }
        }
      }
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // reads before the next fill
    if (clast[b]) {
#pragma unroll
      for (int off = LC; off < EG * LC; off <<= 1)
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const bool in = lane + off < EG * LC;
          const float x = __shfl_down_sync(0xffffffffu, acc[q].x, off);
          const float y = __shfl_down_sync(0xffffffffu, acc[q].y, off);
          const float z = __shfl_down_sync(0xffffffffu, acc[q].z, off);
          const float w = __shfl_down_sync(0xffffffffu, acc[q].w, off);
          if (in) {
            acc[q].x += x;
            acc[q].y += y;
            acc[q].z += z;
            acc[q].w += w;
          }
        }
      spmm_row_epilogue<LC, VPL>(a, crow[b], lane, cl, g, w4, acc);
#pragma unroll
      for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };

  int b = 0;
  bool have = issue(0);
  while (have) {
    const bool next = issue(b ^ 1);
    consume(b);
    b ^= 1;
    have = next;
  }
}

template <int LC, int VPL>
digest_status launch_tg(const SpmmArgs& a, cudaStream_t s) {
  CUtensorMap tm;
  DG_ARG(make_tmap_rows_fwd(&tm, a.X0, (uint64_t)a.width, (uint64_t)a.x0_rows,
                            (uint64_t)a.ld0 * 4),
         DIGEST_E_CUDA, "row-gather tensor map failed");
  const int slot = (int)round_up(4 * (int64_t)a.width * 4, 128);
  int wpc = (int)((227 * 1024 - 2048) / (16 * (int64_t)slot));
  if (wpc > 8) wpc = 8;
  if (wpc < 1) wpc = 1;
  const int smem = 2048 + wpc * 16 * slot;
  static int attr = 0;
  if (smem > attr) {
    DG_CUDA(cudaFuncSetAttribute(k_spmm_tg<LC, VPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem));
    attr = smem;
  }
  int per_sm = 0;
  DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmm_tg<LC, VPL>, wpc * 32, smem));
  int64_t blocks = (int64_t)(per_sm < 1 ? 1 : per_sm) * num_sms();
  const int64_t need = ceil_div(a.n_rows, wpc);
  if (blocks > need) blocks = need < 1 ? 1 : need;
  const double W = a.full_width > 0 ? a.full_width : a.width;
  const double frac = a.width / W;
  const double bytes = frac * ((double)a.nnz * (8.0 + 4.0 * W) + (double)a.n_rows * (4.0 * W + 8.0));
  const double flops = 2.0 * (double)a.nnz * a.width;
  DG_LAUNCH_TAG(DIGEST_PROF_SPMM, a.full_width > 0 ? a.full_width : a.width, s, bytes, flops,
                (k_spmm_tg<LC, VPL>), (unsigned)blocks, wpc * 32, smem, a, tm, slot);
  return DIGEST_OK;
}

// Grid: at most the number of CTAs that are resident at once (a persistent grid).  The
// rows are dealt round-robin (row = warp + k * nwarps), so with every warp resident the
// rows in flight form one narrow, monotonically advancing window -- a graph block's
// gathered source rows stay in L2 while the window sweeps it (with column slabs, see
// spmm_slab_width).  An oversubscribed grid would let each CTA sweep the whole row range
// over its lifetime and scatter the window across the graph.
template <typename K>
int64_t resident_ctas(K kern) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return (int64_t)per_sm * num_sms();
}

// DIGEST_SPMM_GRID: 0 persistent, 1 oversubscribed (64 CTAs/SM cap), unset = by mean row
// length: persistent below 128 nonzeros per row (measured, products M=1 w=256/100/48:
// 17.9/9.3/5.2 -> 16.6/8.4/4.6 ms), oversubscribed for long rows (Reddit, ~490 per row:
// w=256 12.4 vs 13.6 ms persistent).
bool spmm_persistent(const SpmmArgs& a) {
  static int v = -2;
  if (v == -2) {
    const char* e = dg::knob("DIGEST_SPMM_GRID");
    v = e ? atoi(e) : -1;
  }
  if (v >= 0) return v == 0;
  return a.nnz < 128 * a.n_rows;
}

template <int LC, int VPL, int UNR, bool PF, int MB>
digest_status launch_mb(const SpmmArgs& a, cudaStream_t s, int64_t blocks, double bytes,
                        double flops) {
  // DIGEST_SPMM_PFH=1: cache-policy operands in the prefetching (narrow-width) kernel.
  // Off by default: the per-load policy descriptor costs an R2UR per gather in this
  // instruction-bound kernel (w=48 products M=1: 4.12 -> 3.85 ms without, M=8: 0.515 ->
  // 0.454 ms; profiles/r1_spmm_variant_sweep.log)
  static int pfh = -1;
  if (pfh < 0) {
    const char* e = dg::knob("DIGEST_SPMM_PFH");
    pfh = e ? atoi(e) : 0;
  }
  // (cross-row pipelining, the kernel's XR=true form, measured 20-50% slower with the
  // persistent grid -- profiles/r1_spmm_variant_sweep.log -- and is not instantiated)
  if (PF && pfh && a.hints) {
    static const int64_t cap = resident_ctas(k_spmm<LC, VPL, UNR, false, MB, true>);
    if (spmm_persistent(a) && blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, a.full_width > 0 ? a.full_width : a.width, s, bytes, flops,
                  (k_spmm<LC, VPL, UNR, false, MB, true>),
                  (unsigned)blocks, 256, 0, a);
  } else if (PF) {
    static const int64_t cap = resident_ctas(k_spmm<LC, VPL, UNR, false, MB, false>);
    if (spmm_persistent(a) && blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, a.full_width > 0 ? a.full_width : a.width, s, bytes, flops,
                  (k_spmm<LC, VPL, UNR, false, MB, false>),
                  (unsigned)blocks, 256, 0, a);
  } else {
    static const int64_t cap = resident_ctas(k_spmm_rt<LC, VPL, UNR, MB>);
    if (spmm_persistent(a) && blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, a.full_width > 0 ? a.full_width : a.width, s, bytes, flops,
                  (k_spmm_rt<LC, VPL, UNR, MB>),
                  (unsigned)blocks, 256, 0, a);
  }
  return DIGEST_OK;
}

template <int LC, int VPL, int UNR, bool PF = true, int MB_DEFAULT = 1>
digest_status launch(const SpmmArgs& a, cudaStream_t s) {
  int64_t blocks = ceil_div(a.n_rows, 8);
  const int64_t cap = (int64_t)num_sms() * 8 * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // algorithmic bytes/flops of the whole product (SURVEY §8.d.4 edge-gather model); a
  // column-slab launch declares its share slab/W of them, tagged with the full width W
  const double W = a.full_width > 0 ? a.full_width : a.width;
  const double frac = a.width / W;
  const double bytes = frac * ((double)a.nnz * (8.0 + 4.0 * W) + (double)a.n_rows * (4.0 * W + 8.0));
  const double flops = 2.0 * (double)a.nnz * a.width;
  // MB: minimum resident blocks per SM the register allocation must allow (0 = the
  // compiler's choice); the narrow widths are latency-bound and gain from occupancy
  static int mb = -1;
  if (mb < 0) {
    const char* e = dg::knob("DIGEST_SPMM_MB");
    mb = e ? atoi(e) : 0;
  }
  // (MB 5 and 6 were measured slower for every width and are not instantiated)
  switch (mb ? mb : MB_DEFAULT) {
    case 4: return launch_mb<LC, VPL, UNR, PF, 4>(a, s, blocks, bytes, flops);
    default: return launch_mb<LC, VPL, UNR, PF, 1>(a, s, blocks, bytes, flops);
  }
  return DIGEST_OK;
}

// Lean narrow-slab kernel launch (w4 = width/4 in 5..16).  Byte/flop accounting as in
// launch(): the slab's share of the whole product's edge-gather bytes.
template <int LC, int VPL, int UNR, bool RAG, int MB, bool XR = false, bool CH = false>
digest_status launch_n(const SpmmArgs& a, cudaStream_t s) {
  const double W = a.full_width > 0 ? a.full_width : a.width;
  const double frac = a.width / W;
  const double bytes = frac * ((double)a.nnz * (8.0 + 4.0 * W) + (double)a.n_rows * (4.0 * W + 8.0));
  const double flops = 2.0 * (double)a.nnz * a.width;
  const bool two = !(a.in_len != nullptr || a.X1 == nullptr || a.split >= INT32_MAX);
  const char* x0 = reinterpret_cast<const char*>(a.X0);
  const char* x1m = two ? reinterpret_cast<const char*>(a.X1) - a.split * a.ld1 * 4 : x0;
  const uint32_t rb_half = (uint32_t)(a.ld0 * 2);
  int64_t blocks = ceil_div(a.n_rows, 8);
  if (two) {
    static const int64_t cap = resident_ctas(k_spmm_n<LC, VPL, UNR, true, RAG, MB, XR, CH>);
    if (blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, (int)W, s, bytes, flops, (k_spmm_n<LC, VPL, UNR, true, RAG, MB, XR, CH>),
                  (unsigned)blocks, 256, 0, a, x0, x1m, (uint32_t)a.split, rb_half);
  } else {
    static const int64_t cap = resident_ctas(k_spmm_n<LC, VPL, UNR, false, RAG, MB, XR, CH>);
    if (blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, (int)W, s, bytes, flops, (k_spmm_n<LC, VPL, UNR, false, RAG, MB, XR, CH>),
                  (unsigned)blocks, 256, 0, a, x0, x1m, (uint32_t)INT32_MAX, rb_half);
  }
  return DIGEST_OK;
}

// Grouped kernel launch (k_spmm_g): persistent grid of the resident CTAs; needs the
// partition's row order (a.order).
// Work counters of the grouped kernel: a ring of slots, one per launch, zeroed on the
// launching stream right before it (graph-capturable; launches on different streams in
// flight at once take different slots).
// (A slot is reused 64 launches later: safe on one stream, and on several unless more
// than 64 grouped launches are in flight at once.)  The ring is allocated when a partition
// is built (spmm_counters_init), never inside a launch that may be stream-captured.
constexpr unsigned kCtrSlots = 64;
unsigned long long* g_ctr_ring = nullptr;
std::once_flag g_ctr_once;
std::atomic<unsigned> g_ctr_next{0};

unsigned long long* grab_counter(cudaStream_t s) {
  if (!spmm_counters_init()) return nullptr;
  unsigned long long* c = g_ctr_ring + (g_ctr_next.fetch_add(1) % kCtrSlots) * 16;   // 128 B apart
  if (cudaMemsetAsync(c, 0, sizeof(unsigned long long), s) != cudaSuccess) return nullptr;
  return c;
}

template <int LC, int VPL, int UNR, bool RAG, int MB, int POL = 0, bool COOP = false>
digest_status launch_g(const SpmmArgs& a, cudaStream_t s) {
  unsigned long long* ctr = grab_counter(s);
  DG_ARG(ctr, DIGEST_E_CUDA, "SpMM work counter allocation failed");
  const double W = a.full_width > 0 ? a.full_width : a.width;
  const double frac = a.width / W;
  const double bytes = frac * ((double)a.nnz * (8.0 + 4.0 * W) + (double)a.n_rows * (4.0 * W + 8.0));
  const double flops = 2.0 * (double)a.nnz * a.width;
  const bool two = !(a.in_len != nullptr || a.X1 == nullptr || a.split >= INT32_MAX);
  const char* x0 = reinterpret_cast<const char*>(a.X0);
  const char* x1m = two ? reinterpret_cast<const char*>(a.X1) - a.split * a.ld1 * 4 : x0;
  const uint32_t rb_half = (uint32_t)(a.ld0 * 2);
  int64_t blocks = ceil_div(a.n_rows, 8 * (32 / LC));
  if (two) {
    static const int64_t cap = resident_ctas(k_spmm_g<LC, VPL, UNR, true, RAG, MB, POL, COOP>);
    if (blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, (int)W, s, bytes, flops, (k_spmm_g<LC, VPL, UNR, true, RAG, MB, POL, COOP>),
                  (unsigned)blocks, 256, 0, a, x0, x1m, (uint32_t)a.split, rb_half, ctr);
  } else {
    static const int64_t cap = resident_ctas(k_spmm_g<LC, VPL, UNR, false, RAG, MB, POL, COOP>);
    if (blocks > cap) blocks = cap;
    DG_LAUNCH_TAG(DIGEST_PROF_SPMM, (int)W, s, bytes, flops, (k_spmm_g<LC, VPL, UNR, false, RAG, MB, POL, COOP>),
                  (unsigned)blocks, 256, 0, a, x0, x1m, (uint32_t)INT32_MAX, rb_half, ctr);
  }
  return DIGEST_OK;
}

// DIGEST_SPMM_N (experiment switch): 0 = the round-1 kernels for narrow widths;
// 1 = default lean kernel; 2 = cross-row pipelined, 32 gathers per group step (fewer
// warps); 3 = default without the CSR evict_first policy; 4 = cross-row pipelined at the
// default's unroll and occupancy (profiles/r2_spmm_variant_sweeps.log); 5-9 = the grouped
// kernel (k_spmm_g) at every narrow width with different unroll / lane layouts; 11 = the
// grouped defaults with per-lane (col, val) loads; 13 = the grouped defaults (cooperative
// loads) at any row count.
int narrow_variant() {
  static int v = -2;
  if (v == -2) {
    const char* e = dg::knob("DIGEST_SPMM_N");
    v = e ? atoi(e) : 1;
  }
  return v;
}

// The lean kernel applies when the two sources share one row stride and every offset
// fits 32 bits (source rows < 2^31, row bytes < 2^32).
bool narrow_ok(const SpmmArgs& a, int max_w4 = 32) {
  const int w4 = a.width / 4;
  if (w4 < 5 || w4 > max_w4) return false;
  const bool two = !(a.in_len != nullptr || a.X1 == nullptr || a.split >= INT32_MAX);
  if (two && a.ld1 != a.ld0) return false;
  return a.ld0 > 0 && a.ld0 * 2 < (int64_t)UINT32_MAX;
}

digest_status launch_narrow(const SpmmArgs& a, cudaStream_t s) {
  const int w4 = a.width / 4;
  const int v = narrow_variant();
  // Default (v == 1), measured on products-shaped partitions
  // (profiles/r2_spmm_grouped_sweep.log): the grouped kernel for w = 68..128 (d0 = 100:
  // M=1 6.23 -> 4.50 ms, one 8-part partition 0.90 -> 0.83 ms) and for w = 48 on products
  // of >= 1M rows (M=1: 2.96 -> 2.22 ms).  On smaller products (an 8-part partition, 306K
  // rows) the w=48 grouped kernel loses (0.46 -> 0.55 ms): 8 rows per warp batch leave only
  // ~11 batches per warp and the last wave's imbalance shows, so the lean kernel stays.
  // Cooperative (col, val) loads (COOP: one load per group lane, shuffled to the group)
  // since the end of round 2: products M=1 w=48 2.231 -> 2.144 ms, w=100 4.460 -> 4.417
  // ms, 8-part partition w=100 0.813 -> 0.803 ms (profiles/r2_spmm_grouped_sweep.log);
  // v == 11 keeps the per-lane loads for comparison.  (The same at one more CTA per SM,
  // and 3 or 2 edges per step at 3-4 CTAs per SM, measured 5-43% slower and are not
  // instantiated.)
  if (v == 11 && a.order) {
    if (w4 > 16) return launch_g<8, 4, 4, true, 2>(a, s);
    if (w4 == 12) return launch_g<4, 3, 4, false, 3>(a, s);
  }
  if (v == 13 && a.order) {   // the default grouped forms at any row count (parity tests)
    if (w4 > 16) return launch_g<8, 4, 4, true, 2, 0, true>(a, s);
    if (w4 == 12) return launch_g<4, 3, 4, false, 3, 0, true>(a, s);
  }
  if (v == 1 && a.order && w4 > 16) return launch_g<8, 4, 4, true, 2, 0, true>(a, s);
  if (v == 1 && a.order && w4 == 12 && a.n_rows >= (1 << 20))
    return launch_g<4, 3, 4, false, 3, 0, true>(a, s);
  if (v >= 5 && v <= 9 && a.order) {   // grouped kernel experiments (one row per edge group)
    if (w4 == 12) {
      if (v == 9) return launch_g<4, 3, 3, false, 3>(a, s);
      if (v == 6) return launch_g<4, 3, 4, false, 3>(a, s);
      if (v == 7) return launch_g<2, 6, 2, false, 3>(a, s);
      return launch_g<4, 3, 2, false, 4>(a, s);
    }
    if (w4 == 16) return launch_g<4, 4, 2, false, 4>(a, s);
    if (w4 == 8) return launch_g<4, 2, 2, false, 4>(a, s);
    if (w4 <= 7) return launch_g<4, 2, 2, true, 4>(a, s);
    if (w4 <= 11) return launch_g<4, 3, 2, true, 4>(a, s);
    if (w4 <= 15) return launch_g<4, 4, 2, true, 4>(a, s);
    if (v == 6) return launch_g<8, 4, 4, true, 2>(a, s);
    if (v == 8) return launch_g<8, 4, 3, true, 2>(a, s);
    if (v == 7 && w4 <= 28) return launch_g<4, 7, 2, true, 3>(a, s);
    return launch_g<8, 4, 2, true, 3>(a, s);
  }
  // measured, products-shaped partitions (profiles/r2_spmm_sweep.md): w=48 M=1 3.86 ->
  // 2.97 ms, M=8 0.52 -> 0.46 ms; w=100 7.23 -> 6.38 ms
  if (w4 == 12) {
    if (v == 2) return launch_n<4, 3, 4, false, 3, true, true>(a, s);
    if (v == 4) return launch_n<4, 3, 2, false, 4, true, true>(a, s);
    if (v == 3) return launch_n<4, 3, 2, false, 4>(a, s);
    return launch_n<4, 3, 2, false, 4, false, true>(a, s);
  }
  if (w4 == 16) {
    if (v == 2) return launch_n<8, 2, 4, false, 3, true, true>(a, s);
    if (v == 4) return launch_n<4, 4, 2, false, 4, true, true>(a, s);
    if (v == 3) return launch_n<4, 4, 2, false, 4>(a, s);
    return launch_n<4, 4, 2, false, 4, false, true>(a, s);
  }
  if (w4 == 8) return launch_n<4, 2, 2, false, 4, false, true>(a, s);
  if (w4 <= 7) return launch_n<4, 2, 2, true, 4, false, true>(a, s);
  if (w4 <= 11) return launch_n<4, 3, 2, true, 4, false, true>(a, s);
  if (w4 <= 15) return launch_n<4, 4, 2, true, 4, false, true>(a, s);
  // w = 68..128 (products d0 = 100: 25 float4 on 8 lanes x 4, ragged)
  if (v == 2 || v == 4) return launch_n<8, 4, 2, true, 3, true, true>(a, s);
  if (v == 3) return launch_n<8, 4, 2, true, 3>(a, s);
  return launch_n<8, 4, 2, true, 3, false, true>(a, s);
}

}  // namespace

digest_status spmm_one(const SpmmArgs& a, cudaStream_t s);

bool spmm_counters_init() {
  std::call_once(g_ctr_once, [] {
    void* p = nullptr;
    if (cudaMalloc(&p, kCtrSlots * 128) == cudaSuccess) g_ctr_ring = static_cast<unsigned long long*>(p);
  });
  return g_ctr_ring != nullptr;
}

// Column-slab schedule: the gathered source rows of a slab (n_src x slab floats) are
// sized to stay resident in L2 while the row window sweeps a graph block, so the
// edge gathers hit L2 instead of HBM; each slab re-reads the CSR (8 B / nnz).
// DIGEST_SPMM_SLAB overrides the slab width (0 = no slabs).
// Otherwise (auto) widths above `smax` floats are cut into balanced slabs of at most
// smax (a multiple of 32 when 1-bit masks are read or written, so mask words stay whole)
// that the lean narrow kernel runs; DIGEST_SPMM_SMAX overrides smax (0 = no slabs).
int spmm_slab_width(const SpmmArgs& a) {
  static int env = -2, smax = -2;
  if (env == -2) {
    const char* e = dg::knob("DIGEST_SPMM_SLAB");
    env = e ? atoi(e) : -1;
    const char* m = dg::knob("DIGEST_SPMM_SMAX");
    smax = m ? atoi(m) : 0;
  }
  if (env >= 0) return env;
  if (smax <= 0 || narrow_variant() == 0 || a.width <= smax) return 0;
  const int nslab = (a.width + smax - 1) / smax;
  int slab = (int)round_up(ceil_div(a.width, nslab), 4);
  if (a.mbits || a.obits || a.mask) slab = (int)round_up(slab, 32);
  return slab;
}

digest_status spmm(const SpmmArgs& a0, cudaStream_t s) {
  if (a0.n_rows == 0) return DIGEST_OK;
  // L2 policy of the gathers (DIGEST_SPMM_HINTS overrides): 2 = bit-31 hot source rows
  // evict_last, the rest evict_normal, for wide rows; 0 = no policy operands for narrower
  // ones.  Measured with the persistent grid, products M=1: w=256 16.57 ms (hints 1, the
  // rest evict_first) -> 15.37 ms (2); w=100 8.51 (1) -> 8.01 ms (0)
  // (profiles/r1_spmm_variant_sweep.log).
  static int hints = -2;
  if (hints == -2) {
    const char* e = dg::knob("DIGEST_SPMM_HINTS");
    hints = e ? atoi(e) : -1;
  }
  SpmmArgs a = a0;
  a.hints = hints >= 0 ? hints : (a0.width >= 128 ? 2 : 0);
  static int cs = -1;   // DIGEST_SPMM_STREAM_OUT: st.global.cs for the output rows
  if (cs < 0) {
    const char* e = dg::knob("DIGEST_SPMM_STREAM_OUT");
    cs = e ? atoi(e) : 0;
  }
  a.stream_out = cs;
  DG_ARG(a.width > 0 && a.width % 4 == 0, DIGEST_E_INVALID,
         "SpMM width %d must be a positive multiple of 4", a.width);
  const int slab = spmm_slab_width(a);
  if (slab <= 0 || slab % 4 != 0 || slab >= a.width || ((a.mbits || a.obits) && slab % 32 != 0))
    return spmm_one(a, s);
  for (int c0 = 0; c0 < a.width; c0 += slab) {
    SpmmArgs b = a;
    b.X0 = a.X0 + c0;
    b.X1 = a.X1 + c0;
    b.Y = a.Y + c0;
    if (a.mask) b.mask = a.mask + c0;
    if (a.mbits) b.mbits = a.mbits + c0 / 32;   // 1-bit masks: one word per 32 columns
    if (a.obits) b.obits = a.obits + c0 / 32;
    b.width = a.width - c0 < slab ? a.width - c0 : slab;
    b.full_width = a.width;
    DG_TRY(spmm_one(b, s));
  }
  return DIGEST_OK;
}

digest_status spmm_one(const SpmmArgs& a, cudaStream_t s) {
  const int w4 = a.width / 4;
  if (narrow_variant() > 0 && narrow_ok(a)) return launch_narrow(a, s);
  static int tg = -1;   // DIGEST_SPMM_TMA=1: TMA row-gather kernel for single-source products
  if (tg < 0) {
    const char* e = dg::knob("DIGEST_SPMM_TMA");
    tg = e ? atoi(e) : 0;
  }
  const bool single = a.in_len != nullptr || a.X1 == nullptr || a.split >= INT32_MAX;
  if (tg && single && a.x0_rows > 0 && a.x0_rows < INT32_MAX && a.width <= 256 &&
      (a.width * 4) % 16 == 0) {
    if (w4 <= 12) return launch_tg<4, 3>(a, s);
    if (w4 <= 32) return launch_tg<8, 4>(a, s);
    return launch_tg<32, 2>(a, s);
  }
  // (lanes per edge, float4 per lane, edges per group per step); EG = 32 / LC edge groups
  if (w4 <= 1) return launch<1, 1, 1>(a, s);
  if (w4 <= 2) return launch<2, 1, 1>(a, s);
  if (w4 <= 4) return launch<4, 1, 2>(a, s);
  if (w4 <= 8) return launch<8, 1, 4>(a, s);
  if (w4 <= 12) {
    static int v = -1;
    if (v < 0) {
      const char* e = dg::knob("DIGEST_SPMM_V12");
      v = e ? atoi(e) : 0;
    }
    if (v == 1) return launch<4, 3, 4>(a, s);
    if (v == 2) return launch<4, 3, 2, false>(a, s);
    if (v == 3) return launch<4, 3, 4, false>(a, s);
    if (v == 4) return launch<8, 2, 2>(a, s);
    if (v == 5) return launch<2, 6, 1, true, 4>(a, s);
    if (v == 6) return launch<2, 6, 2, true>(a, s);
    if (v == 7) return launch<4, 3, 1, true, 4>(a, s);
    // measured best for w=48 with the persistent grid (products M=1): 4.11 ms vs 4.30 ms
    // for <4,3,4> (profiles/r1_spmm_variant_sweep.log)
    return launch<4, 3, 2, true, 4>(a, s);
  }
  if (w4 <= 16) return launch<8, 2, 4>(a, s);
  if (w4 <= 25) {   // w = 100 (products d0); variant 1: 6 groups x 5 lanes x 5 float4
    static int v = -1;
    if (v < 0) {
      const char* e = dg::knob("DIGEST_SPMM_V25");
      v = e ? atoi(e) : 0;
    }
    if (v == 1) return launch<5, 5, 2, false>(a, s);
    if (v == 2) return launch<5, 5, 2, true>(a, s);
    if (v == 3) return launch<8, 4, 2, true>(a, s);
    if (v == 4) return launch<8, 4, 2, false, 4>(a, s);
    if (v == 5) return launch<8, 4, 1, true>(a, s);
    // measured best for w=100 (persistent grid, no policy operands): chunk-prefetching
    // <8,4,4>: products M=1 7.15 ms vs 7.91 ms for <8,4,2,rt,MB4>; 8-part partition
    // 0.97 vs 1.33 ms (profiles/r1_spmm_variant_sweep.log)
    return launch<8, 4, 4, true>(a, s);
  }
  if (w4 <= 32) {   // w = 128 (arxiv d0)
    static int v = -1;
    if (v < 0) {
      const char* e = dg::knob("DIGEST_SPMM_V32");
      v = e ? atoi(e) : 0;
    }
    if (v == 1) return launch<8, 4, 2, false>(a, s);
    return launch<8, 4, 4, true>(a, s);
  }
  if (w4 <= 64) {
    static int v = -1;
    if (v < 0) {
      const char* e = dg::knob("DIGEST_SPMM_V");
      v = e ? atoi(e) : 0;
    }
    switch (v) {
      case 1: return launch<32, 2, 4>(a, s);
      case 2: return launch<32, 2, 4, false, 4>(a, s);
      case 3: return launch<32, 2, 8, false>(a, s);
      case 4: return launch<16, 4, 4, false>(a, s);
      case 5: return launch<32, 2, 2, false>(a, s);
      case 6: return launch<32, 2, 4, false, 4>(a, s);
      // the row-per-warp kernel (the w=256 default before the grouped kernel)
      case 7: return launch<32, 2, 8>(a, s);
      case 18:   // grouped with cooperative (col, val) loads (experiment)
        if (a.order && narrow_ok(a, 64) && w4 == 64) return launch_g<16, 4, 4, false, 2, 0, true>(a, s);
        return launch<32, 2, 8>(a, s);
      case 17:   // grouped with the hot-bit L2 policy (experiment; set DIGEST_HOT_ROWS)
        if (a.order && narrow_ok(a, 64) && w4 == 64) return launch_g<16, 4, 4, false, 2, 1>(a, s);
        return launch<32, 2, 8>(a, s);
      // Default for w = 196..256: the grouped kernel, two rows per warp (16 lanes x 4
      // float4 per row; length-grouped order, dynamic batches).  Measured w=256
      // (profiles/r2_w256_sweep.log): products M=1 14.94 -> 11.97 ms (DRAM 77.6 GB at 6.53
      // TB/s, 1.0 of the copy peak), one 8-part partition 2.06 -> 1.79 ms, Reddit M=1
      // 11.84 -> 5.81 ms; 4 rows per warp (8 x 8) or fewer edges per step lose.  Without a
      // row order (or with 64-bit offsets) the row-per-warp chunk-prefetching <32,2,8>
      // (products M=1 14.91 ms vs 15.35 ms for the runtime-loop <32,2,4,MB=4>,
      // profiles/r1_spmm_variant_sweep.log).
      default:
        if (a.order && narrow_ok(a, 64) && w4 > 48) {
          if (w4 == 64) return launch_g<16, 4, 4, false, 2>(a, s);
          return launch_g<16, 4, 4, true, 2>(a, s);
        }
        return launch<32, 2, 8>(a, s);
    }
  }
  if (w4 <= 96) return launch<32, 3, 4, false>(a, s);
  if (w4 <= 128) return launch<32, 4, 4, false>(a, s);
  if (w4 <= 192) return launch<32, 6, 2, false>(a, s);
  if (w4 <= 256) return launch<32, 8, 2, false>(a, s);
  if (w4 <= 384) return launch<32, 12, 2, false>(a, s);
  return set_error(DIGEST_E_UNSUPPORTED, "SpMM width %d > 1536", a.width);
}

}  // namespace dg

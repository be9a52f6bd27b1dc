// CSR-row SpMM over the extended column space [local ; halo] (Eq. 5's
// P_in H_in + P_out H~_out, as ONE product with two source pointers).
//
// Design: warp per row, edge groups x float4 column lanes,
// 128-bit loads, coalesced (col, val) chunks broadcast by shuffles, UNR
// independent row gathers in flight per edge group (memory-level parallelism).
// Halo rows come from a second pointer (no copy of the stale store into a
// contiguous X_ext).  HBM-bound: ~2 flop per (8 + 4w) bytes per nonzero.
#include "kernels.cuh"

namespace dg {
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
  const uint64_t pol_x = a.hints ? policy_evict_last() : policy_evict_normal();
  const uint64_t pol_s = a.hints ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_c = a.hints == 1   ? policy_evict_first()
                         : a.hints == 3 ? policy_evict_last()
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
    const char* e = getenv("DIGEST_SPMM_GRID");
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
    const char* e = getenv("DIGEST_SPMM_PFH");
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
    const char* e = getenv("DIGEST_SPMM_MB");
    mb = e ? atoi(e) : 0;
  }
  // (MB 5 and 6 were measured slower for every width and are not instantiated)
  switch (mb ? mb : MB_DEFAULT) {
    case 4: return launch_mb<LC, VPL, UNR, PF, 4>(a, s, blocks, bytes, flops);
    default: return launch_mb<LC, VPL, UNR, PF, 1>(a, s, blocks, bytes, flops);
  }
  return DIGEST_OK;
}

}  // namespace

digest_status spmm_one(const SpmmArgs& a, cudaStream_t s);

// Column-slab schedule: the gathered source rows of a slab (n_src x slab floats) are
// sized to stay resident in L2 while the row window sweeps a graph block, so the
// edge gathers hit L2 instead of HBM; each slab re-reads the CSR (8 B / nnz).
// DIGEST_SPMM_SLAB overrides the slab width (0 = no slabs).
int spmm_slab_width(const SpmmArgs& a) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("DIGEST_SPMM_SLAB");
    env = e ? atoi(e) : -1;
  }
  if (env >= 0) return env;
  return 0;
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
    const char* e = getenv("DIGEST_SPMM_HINTS");
    hints = e ? atoi(e) : -1;
  }
  SpmmArgs a = a0;
  a.hints = hints >= 0 ? hints : (a0.width >= 128 ? 2 : 0);
  static int cs = -1;   // DIGEST_SPMM_STREAM_OUT: st.global.cs for the output rows
  if (cs < 0) {
    const char* e = getenv("DIGEST_SPMM_STREAM_OUT");
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
  // (lanes per edge, float4 per lane, edges per group per step); EG = 32 / LC edge groups
  if (w4 <= 1) return launch<1, 1, 1>(a, s);
  if (w4 <= 2) return launch<2, 1, 1>(a, s);
  if (w4 <= 4) return launch<4, 1, 2>(a, s);
  if (w4 <= 8) return launch<8, 1, 4>(a, s);
  if (w4 <= 12) {
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("DIGEST_SPMM_V12");
      v = e ? atoi(e) : 0;
    }
    if (v == 1) return launch<4, 3, 4>(a, s);
    if (v == 2) return launch<4, 3, 2, false>(a, s);
    if (v == 3) return launch<4, 3, 4, false>(a, s);
    if (v == 4) return launch<8, 2, 2>(a, s);
    // measured best for w=48 with the persistent grid (products M=1): 4.11 ms vs 4.30 ms
    // for <4,3,4> (profiles/r1_spmm_variant_sweep.log)
    return launch<4, 3, 2, true, 4>(a, s);
  }
  if (w4 <= 16) return launch<8, 2, 4>(a, s);
  if (w4 <= 25) {   // w = 100 (products d0); variant 1: 6 groups x 5 lanes x 5 float4
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("DIGEST_SPMM_V25");
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
      const char* e = getenv("DIGEST_SPMM_V32");
      v = e ? atoi(e) : 0;
    }
    if (v == 1) return launch<8, 4, 2, false>(a, s);
    return launch<8, 4, 4, true>(a, s);
  }
  if (w4 <= 64) {
    static int v = -1;
    if (v < 0) {
      const char* e = getenv("DIGEST_SPMM_V");
      v = e ? atoi(e) : 0;
    }
    switch (v) {
      case 1: return launch<32, 2, 4>(a, s);
      case 2: return launch<32, 2, 4, false, 4>(a, s);
      case 3: return launch<32, 2, 8, false>(a, s);
      case 4: return launch<16, 4, 4, false>(a, s);
      case 5: return launch<32, 2, 2, false>(a, s);
      case 6: return launch<32, 2, 4, false, 4>(a, s);
      // w=256, persistent grid, products M=1: chunk-prefetching <32,2,8> 14.91 ms vs
      // runtime-loop <32,2,4,MB=4> 15.35 ms (profiles/r1_spmm_variant_sweep.log)
      default: return launch<32, 2, 8>(a, s);
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

// Device-wide exclusive prefix sum of a predicate/length functor (used by the
// one-time partition build).  Three passes: tile sums, a single-block scan of the
// tile sums, tile scans with the carried offset.  out has n+1 entries;
// out[n] = total.  Deterministic (integer arithmetic).
#pragma once
#include "common.cuh"

namespace dg {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T x, T* smem_warp, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) smem_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    T v = lane < nw ? smem_warp[lane] : T(0);
    T vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    if (lane < nw) smem_warp[lane] = vi - v;
    if (lane == nw - 1) *total = vi;
  }
  __syncthreads();
  T r = smem_warp[warp] + incl - x;
  __syncthreads();
  return r;
}

template <typename F>
__global__ void scan_tile_sums(F f, int64_t n, int64_t* tile_sums) {
  __shared__ int64_t sw[32];
  __shared__ int64_t tot;
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    if (base + j < n) s += (int64_t)f(base + j);
  block_exclusive_scan<int64_t>(s, sw, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void scan_carry(int64_t* tile_sums, int64_t ntiles, int64_t* total_out) {
  __shared__ int64_t sw[32];
  __shared__ int64_t tot;
  int64_t carry = 0;
  for (int64_t b = 0; b < ntiles; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    int64_t v = i < ntiles ? tile_sums[i] : 0;
    int64_t ex = block_exclusive_scan<int64_t>(v, sw, &tot);
    if (i < ntiles) tile_sums[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry;
}

template <typename F, typename O>
__global__ void scan_tiles(F f, int64_t n, const int64_t* tile_off, O* out) {
  __shared__ int64_t sw[32];
  __shared__ int64_t tot;
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = base + j < n ? (int64_t)f(base + j) : 0;
    s += v[j];
  }
  int64_t ex = block_exclusive_scan<int64_t>(s, sw, &tot) + tile_off[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (base + j < n) out[base + j] = (O)ex;
    ex += v[j];
  }
}

template <typename O>
__global__ void scan_write_total(O* out, int64_t n, const int64_t* total) {
  out[n] = (O)*total;
}

// Exclusive scan of f(0..n-1) into out[0..n]; `tmp` must hold
// ceil(n/kScanTile)+1 int64 values.  If total_h != NULL the stream is synchronised
// and the total copied to the host.
template <typename F, typename O>
digest_status exclusive_scan(F f, int64_t n, O* out, int64_t* tmp, cudaStream_t s,
                             int64_t* total_h) {
  int64_t ntiles = ceil_div(n, kScanTile);
  if (ntiles == 0) ntiles = 1;
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, scan_tile_sums<F>, (unsigned)ntiles, kScanThreads, 0, f,
            n, tmp);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, scan_carry, 1, 1024, 0, tmp, ntiles, tmp + ntiles);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, (scan_tiles<F, O>), (unsigned)ntiles, kScanThreads, 0,
            f, n, tmp, out);
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, scan_write_total<O>, 1, 1, 0, out, n, tmp + ntiles);
  if (total_h) {
    DG_CUDA(cudaMemcpyAsync(total_h, tmp + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DG_CUDA(cudaStreamSynchronize(s));
  }
  return DIGEST_OK;
}

inline int64_t scan_tmp_elems(int64_t n) { return ceil_div(n, kScanTile) + 2; }

}  // namespace dg

// The stale representation store (Alg. 1 PULL/PUSH P:208-221).
//
// The paper keeps stale representations in a host shared-memory KVS (Plasma,
// P:385).  On B200 every GPU's halo buffers ARE the store: level l of partition m
// holds two n_halo x ld_l buffers (front = read by layer l+1, back = written by
// pushes).  A push gathers the boundary rows H[send_idx] once and delivers them
// into each peer's back buffer at the (owner, id) segment of that peer's halo —
// which is exactly the sender's send order, so nothing is unpacked on receipt.
//   * loopback (several partitions in one process): the gather kernel writes the
//     peers' back buffers directly (fused gather + put);
//   * NCCL: gather into a contiguous send buffer, then a grouped send/recv
//     all-to-allv straight into the back buffers, optionally on a side stream
//     (async mode, overlapping the next layer: P:250-251).
// A pull flips front/back (or copies, CUDA-graph safe) only when the back buffer
// holds a newer version that is older than the current epoch (reading A7).
#include <cuda_bf16.h>

#include <cstring>
#include <vector>

#include "comm_internal.cuh"
#include "kernels.cuh"
#include "part_internal.cuh"

namespace {

struct Level {
  int32_t width = 0;
  int64_t ld = 0;
  float* buf[2] = {nullptr, nullptr};   // bf16 store: buf[0] fp32 front, buf[1] bf16 back
  int64_t ver[2] = {0, 0};
  int front = 0;
  float* send_buf = nullptr;
  cudaEvent_t done = nullptr;   // exchange completion (async mode)
  bool inflight = false;
  float* grad_buf = nullptr;    // n_halo x ld: gradient of this part's halo rows (P:816 term)
                                // (peer transport: two slots, alternating per backward)
  float* ret_recv = nullptr;    // n_send x ld: returned gradients received from peers (NCCL)
  int64_t last_pull = 0;        // epoch of the last pull call (peer transport)
  int64_t gseq = 0;             // grad_buffer calls so far (peer transport)
  // Single-process (linked) stores: pushes that peers wrote into THIS store's back
  // buffer (the receiver's own record; a pusher's version says nothing about what the
  // receiver holds when workers push at different local epochs, DIGEST-A) and the
  // count the last pull consumed.
  int64_t rx_seq = 0, rx_seen = 0;
  size_t halo_bytes = 0;        // bytes of one n_halo x ld fp32 buffer
  bool bf16 = false;            // back buffer (and transfers) in bf16
  size_t es() const { return bf16 ? 2 : 4; }   // element size of back / send buffers
};

// Row `row` of a back/send buffer with leading dimension ld and element size es.
__host__ __device__ inline float* xrow(float* base, int64_t row, int64_t ld, size_t es) {
  return reinterpret_cast<float*>(reinterpret_cast<char*>(base) + (size_t)row * ld * es);
}

// Store 4 consecutive values at float4 column c of a row, as fp32 or as bf16 (RNE).
template <bool BF>
__device__ __forceinline__ void st4(float* row, int c, float4 v) {
  if (BF) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    reinterpret_cast<uint2*>(row)[c] = u;
  } else {
    reinterpret_cast<float4*>(row)[c] = v;
  }
}
template <bool BF>
__device__ __forceinline__ float4 ld4(const float* row, int c) {
  if (BF) {
    const uint2 u = __ldcv(reinterpret_cast<const uint2*>(row) + c);
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                       __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
  }
  return __ldcv(reinterpret_cast<const float4*>(row) + c);
}

// What a peer needs to reach this store's buffers (digest_store_export / _connect).
struct PeerBlob {
  int32_t rank, levels;
  int64_t halo_rows;             // rows of one halo buffer, max(n_halo, 1) (gradient slot stride)
  int64_t recv_off[DIGEST_MAX_PARTS];
  cudaIpcMemHandle_t h[64][3];   // per level: buf[0], buf[1], grad_buf
};
struct PeerLevel {
  float* buf[2];
  float* grad;
  size_t slot_bytes;   // the owner's gradient slot stride
};

// G[idx[j]] += 1[mask[idx[j]] > 0] * src[j]  for the rows of one peer's segment (one launch
// per peer, in ascending peer order: a local row may be a halo row of several peers, so
// this keeps the accumulation race-free and deterministic).
__global__ void k_return_add(const float* __restrict__ src, int64_t ld_src,
                             const int32_t* __restrict__ idx, int64_t n, float* __restrict__ G,
                             int64_t ld_g, const float* __restrict__ mask, int64_t ld_m, int w4) {
  const int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nw) {
    const int64_t i = idx[j];
    const float4* s = reinterpret_cast<const float4*>(src + j * ld_src);
    float4* g = reinterpret_cast<float4*>(G + i * ld_g);
    const float4* m = mask ? reinterpret_cast<const float4*>(mask + i * ld_m) : nullptr;
    for (int c = lane; c < w4; c += 32) {
      float4 v = s[c], o = g[c];
      if (m) {
        const float4 mk = m[c];
        v.x = mk.x > 0.f ? v.x : 0.f;
        v.y = mk.y > 0.f ? v.y : 0.f;
        v.z = mk.z > 0.f ? v.z : 0.f;
        v.w = mk.w > 0.f ? v.w : 0.f;
      }
      o.x += v.x;
      o.y += v.y;
      o.z += v.z;
      o.w += v.w;
      g[c] = o;
    }
  }
}

struct Segs {
  float* dst[DIGEST_MAX_PARTS];
  int64_t start[DIGEST_MAX_PARTS + 1];  // send-row offsets per segment
  int32_t nseg;
};

// Row s of the send list -> segment k (binary search), destination row s - start[k].
// Optional row L2 normalisation (Alg. 1, applied to the pushed copies only).
template <bool NORM, bool BF>
__global__ void k_pack(const float* __restrict__ H, int64_t ldh, const int32_t* __restrict__ idx,
                       int64_t n_send, Segs segs, int64_t ld, int w4) {
  const int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_send; r += nw) {
    int lo = 0, hi = segs.nseg - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (segs.start[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const float4* src = reinterpret_cast<const float4*>(H + (int64_t)idx[r] * ldh);
    float* dst = xrow(segs.dst[lo], r - segs.start[lo], ld, BF ? 2 : 4);
    float scale = 1.f;
    if (NORM) {
      float ss = 0.f;
      for (int c = lane; c < w4; c += 32) {
        float4 v = src[c];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      scale = ss > 0.f ? 1.f / sqrtf(ss) : 0.f;
    }
    for (int c = lane; c < w4; c += 32) {
      float4 v = src[c];
      if (NORM) {
        v.x *= scale;
        v.y *= scale;
        v.z *= scale;
        v.w *= scale;
      }
      st4<BF>(dst, c, v);
    }
  }
}

// Peer transport: the fused gather + put of a push.  Every block first waits until
// each receiving peer has pulled past the epoch whose flip made its back buffer free
// (its `pulled` flag), then writes its rows straight into the peers' back buffers
// through their IPC mappings; the last block to finish fences and raises the
// receivers' `arrived` flags to the pushed version.
template <bool NORM, bool BF>
__global__ void k_put(const float* __restrict__ H, int64_t ldh, const int32_t* __restrict__ idx,
                      int64_t n_send, Segs segs, int64_t ld, int w4, dg::FlagWait wait,
                      dg::FlagSet sig, unsigned* counter) {
  if (threadIdx.x == 0) dg::wait_flags(wait);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_send; r += nw) {
    int lo = 0, hi = segs.nseg - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (segs.start[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const float4* src = reinterpret_cast<const float4*>(H + (int64_t)idx[r] * ldh);
    float* dst = xrow(segs.dst[lo], r - segs.start[lo], ld, BF ? 2 : 4);
    float scale = 1.f;
    if (NORM) {
      float ss = 0.f;
      for (int c = lane; c < w4; c += 32) {
        float4 v = src[c];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      scale = ss > 0.f ? 1.f / sqrtf(ss) : 0.f;
    }
    for (int c = lane; c < w4; c += 32) {
      float4 v = src[c];
      if (NORM) {
        v.x *= scale;
        v.y *= scale;
        v.z *= scale;
        v.w *= scale;
      }
      st4<BF>(dst, c, v);
    }
  }
  if (dg::last_block_done(counter) && threadIdx.x == 0) dg::set_flags(sig);
}

// DIGEST-A snapshot pull (peer transport): CTA k copies owner segment k back -> front
// under that owner's sequence word (seqlock: odd = a push is writing the segment).
struct SnapSegs {
  int64_t off[DIGEST_MAX_PARTS], cnt[DIGEST_MAX_PARTS];
  const int64_t* seq[DIGEST_MAX_PARTS];
};
template <bool BF>
__global__ void __launch_bounds__(1024) k_snapshot(const float* back, float* front, int64_t ld,
                                                   SnapSegs sg) {
  __shared__ int64_t s1;
  __shared__ int retry;
  const int k = blockIdx.x;
  const float* src = xrow(const_cast<float*>(back), sg.off[k], ld, BF ? 2 : 4);
  float4* dst = reinterpret_cast<float4*>(front + sg.off[k] * ld);
  const int64_t n4 = sg.cnt[k] * ld / 4;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    if (threadIdx.x == 0) {
      int64_t v;
      while ((v = dg::ld_acquire_sys(sg.seq[k])) & 1) __nanosleep(256);
      s1 = v;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = ld4<BF>(src, (int)i);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      retry = dg::ld_acquire_sys(sg.seq[k]) != s1;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (retry && t - t0 > 30ull * 1000000000ull) {
        printf("digest: snapshot pull of segment %d never stabilised\n", k);
        __trap();
      }
    }
    __syncthreads();
    if (!retry) break;
  }
}

// bf16 store pull: front (fp32) <- back (bf16), exact widening.
__global__ void k_widen(const float* __restrict__ src, float4* __restrict__ dst, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = ld4<true>(src, (int)i);
}

__global__ void k_copy(const float4* __restrict__ src, float4* __restrict__ dst, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

struct digest_store {
  const digest_part* part = nullptr;
  digest_comm* comm = nullptr;
  std::vector<Level> lev;
  std::vector<digest_store*> peers;  // loopback group, index = rank
  cudaStream_t side = nullptr;
  cudaEvent_t packed = nullptr;
  // peer transport: every rank's buffers mapped here, [rank][level]
  std::vector<std::vector<PeerLevel>> pl;
  std::vector<std::vector<int64_t>> peer_recv_off;   // [rank][owner]
  bool connected = false;
  unsigned* counters = nullptr;                      // one last-block counter per level
};

namespace {

void destroy_store(digest_store* st) {
  if (!st) return;
  if (st->connected) {
    for (size_t k = 0; k < st->pl.size(); ++k) {
      if ((int)k == st->part->rank) continue;
      for (auto& q : st->pl[k]) {
        if (q.buf[0]) cudaIpcCloseMemHandle(q.buf[0]);
        if (q.buf[1]) cudaIpcCloseMemHandle(q.buf[1]);
        if (q.grad) cudaIpcCloseMemHandle(q.grad);
      }
    }
  }
  cudaFree(st->counters);
  for (auto& L : st->lev) {
    cudaFree(L.buf[0]);
    cudaFree(L.buf[1]);
    cudaFree(L.send_buf);
    cudaFree(L.grad_buf);
    cudaFree(L.ret_recv);
    if (L.done) cudaEventDestroy(L.done);
  }
  if (st->packed) cudaEventDestroy(st->packed);
  if (st->side) cudaStreamDestroy(st->side);
  delete st;
}

digest_status get_level(digest_store* st, int32_t level, Level** out) {
  DG_ARG(st, DIGEST_E_INVALID, "NULL store");
  DG_ARG(level >= 1 && level <= (int32_t)st->lev.size(), DIGEST_E_INVALID,
         "level %d outside [1, %d] (stale levels never equal L, P:208/P:220)", level,
         (int)st->lev.size());
  *out = &st->lev[level - 1];
  return DIGEST_OK;
}

digest_status pack(const float* H, int64_t ldh, const int32_t* idx, int64_t n_send, const Segs& sg,
                   int64_t ld, int32_t width, bool norm, cudaStream_t s, bool bf = false) {
  if (n_send == 0) return DIGEST_OK;
  int64_t blocks = dg::ceil_div(n_send, 8);
  int64_t cap = (int64_t)dg::num_sms() * 16;
  if (blocks > cap) blocks = cap;
  double bytes = (double)n_send * ((bf ? 6.0 : 8.0) * width + 4.0);
#define DG_PACK(NORM, BF)                                                                        \
  DG_LAUNCH(DIGEST_PROF_PACK, s, bytes, 0, (k_pack<NORM, BF>), (unsigned)blocks, 256, 0, H, ldh, \
            idx, n_send, sg, ld, width / 4)
  if (norm && bf) DG_PACK(true, true);
  else if (norm) DG_PACK(true, false);
  else if (bf) DG_PACK(false, true);
  else DG_PACK(false, false);
#undef DG_PACK
  return DIGEST_OK;
}

}  // namespace

extern "C" {

digest_status digest_store_create(const digest_part* part, digest_comm* comm, int32_t num_levels,
                                  const int32_t* width_h, digest_store** out_h) {
  return digest_store_create_ex(part, comm, num_levels, width_h, 0u, out_h);
}

digest_status digest_store_create_ex(const digest_part* part, digest_comm* comm,
                                     int32_t num_levels, const int32_t* width_h, uint32_t flags,
                                     digest_store** out_h) {
  DG_ARG((flags & ~DIGEST_STORE_BF16) == 0, DIGEST_E_INVALID, "unknown store flags 0x%x", flags);
  DG_ARG(part && out_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(num_levels >= 0 && num_levels <= 64 && (num_levels == 0 || width_h), DIGEST_E_INVALID,
         "bad level list");
  if (comm)
    DG_ARG(comm->nranks == part->num_parts && comm->rank == part->rank, DIGEST_E_INVALID,
           "communicator (%d ranks, rank %d) does not match the partition (%d parts, rank %d)",
           comm->nranks, comm->rank, part->num_parts, part->rank);
  *out_h = nullptr;
  digest_store* st = new digest_store();
  st->part = part;
  st->comm = comm;
  st->lev.resize(num_levels);
  auto fail = [&](digest_status s) {
    destroy_store(st);
    return s;
  };
  for (int l = 0; l < num_levels; ++l) {
    Level& L = st->lev[l];
    if (width_h[l] <= 0 || width_h[l] % 4 != 0) {
      destroy_store(st);
      return dg::set_error(DIGEST_E_INVALID, "level width %d must be a positive multiple of 4",
                           width_h[l]);
    }
    L.width = width_h[l];
    L.ld = dg::round_up(L.width, 4);
    L.bf16 = (flags & DIGEST_STORE_BF16) != 0;
    size_t hb = sizeof(float) * (size_t)(part->n_halo > 0 ? part->n_halo : 1) * L.ld;
    size_t sb = L.es() * (size_t)(part->n_send > 0 ? part->n_send : 1) * L.ld;
    for (int b = 0; b < 2; ++b) {
      const size_t bytes = (b == 1 && L.bf16) ? hb / 2 : hb;   // bf16: buf[1] is the back buffer
      if (cudaMalloc(&L.buf[b], bytes) != cudaSuccess)
        return fail(dg::set_error(DIGEST_E_NOMEM, "halo buffer allocation failed"));
      if (cudaMemset(L.buf[b], 0, bytes) != cudaSuccess)
        return fail(dg::set_error(DIGEST_E_CUDA, "cudaMemset failed"));
    }
    L.halo_bytes = hb;
    const size_t gb = dg::is_peer(comm) ? 2 * hb : hb;
    if (cudaMalloc(&L.grad_buf, gb) != cudaSuccess ||
        cudaMemset(L.grad_buf, 0, gb) != cudaSuccess)
      return fail(dg::set_error(DIGEST_E_NOMEM, "gradient-return buffer allocation failed"));
    if (dg::is_nccl(comm)) {
      if (cudaMalloc(&L.send_buf, sb) != cudaSuccess ||
          cudaMalloc(&L.ret_recv, sizeof(float) * (size_t)(part->n_send > 0 ? part->n_send : 1) *
                                      L.ld) != cudaSuccess)
        return fail(dg::set_error(DIGEST_E_NOMEM, "send buffer allocation failed"));
    }
    if (cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming) != cudaSuccess)
      return fail(dg::set_error(DIGEST_E_CUDA, "event creation failed"));
  }
  if (dg::is_peer(comm) &&
      (cudaMalloc(&st->counters, 64 * sizeof(unsigned)) != cudaSuccess ||
       cudaMemset(st->counters, 0, 64 * sizeof(unsigned)) != cudaSuccess ||
       cudaDeviceSynchronize() != cudaSuccess))
    return fail(dg::set_error(DIGEST_E_NOMEM, "counter allocation failed"));
  if (cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&st->packed, cudaEventDisableTiming) != cudaSuccess)
    return fail(dg::set_error(DIGEST_E_CUDA, "stream/event creation failed"));
  *out_h = st;
  return DIGEST_OK;
}

digest_status digest_store_link(digest_store* const* stores_h, int32_t count) {
  DG_ARG(stores_h && count >= 1 && count <= DIGEST_MAX_PARTS, DIGEST_E_INVALID, "bad store list");
  for (int i = 0; i < count; ++i) {
    digest_store* s = stores_h[i];
    DG_ARG(s, DIGEST_E_INVALID, "NULL store %d", i);
    DG_ARG(s->part->num_parts == count && s->part->rank == i, DIGEST_E_INVALID,
           "store %d belongs to partition %d of %d", i, s->part->rank, s->part->num_parts);
    DG_ARG(!s->comm || s->comm->nranks == 1, DIGEST_E_INVALID, "linked stores must not use NCCL");
    DG_ARG(s->lev.size() == stores_h[0]->lev.size(), DIGEST_E_INVALID, "level count mismatch");
    for (size_t l = 0; l < s->lev.size(); ++l)
      DG_ARG(s->lev[l].width == stores_h[0]->lev[l].width, DIGEST_E_INVALID, "width mismatch");
  }
  for (int i = 0; i < count; ++i) stores_h[i]->peers.assign(stores_h, stores_h + count);
  return DIGEST_OK;
}

digest_status digest_push_boundary(digest_store* st, int32_t level, const float* H_local,
                                   int64_t ld, int64_t version, uint32_t flags, void* stream) {
  Level* L;
  DG_TRY(get_level(st, level, &L));
  const digest_part* p = st->part;
  DG_ARG(H_local || p->n_local == 0, DIGEST_E_INVALID, "H_local is NULL");
  DG_ARG(ld >= L->width && ld % 4 == 0 && ((uintptr_t)H_local & 15) == 0, DIGEST_E_INVALID,
         "H_local: ld must be >= width and a multiple of 4, pointer 16-byte aligned");
  DG_ARG(version > L->ver[0] && version > L->ver[1], DIGEST_E_STATE,
         "push version %lld is not newer than the stored versions", (long long)version);
  cudaStream_t s = dg::as_stream(stream);
  const int M = p->num_parts, me = p->rank;
  const int back = 1 - L->front;
  const bool norm = (flags & DIGEST_PUSH_L2NORM) != 0;
  const bool nccl = dg::is_nccl(st->comm);
  const bool peer = dg::is_peer(st->comm);
  if (peer) {
    DG_ARG(st->connected, DIGEST_E_STATE, "peer-transport store is not connected");
    const bool nowait = (flags & DIGEST_PUSH_NOWAIT) != 0;
    Segs sg{};
    sg.nseg = M;
    dg::FlagWait wt{};
    dg::FlagSet sig{}, odd{};
    wt.value = L->last_pull;
    sig.value = nowait ? 2 * version : version;
    odd.value = 2 * version - 1;
    for (int k = 0; k < M; ++k) {
      sg.start[k] = p->send_off[k];
      sg.dst[k] = nullptr;
      if (k == me || p->send_count[k] == 0) continue;
      // same schedule on every rank => the receiver's back buffer has our index `back`
      sg.dst[k] = xrow(st->pl[k][level - 1].buf[back], st->peer_recv_off[k][me], L->ld, L->es());
      if (!nowait)
        wt.ptr[wt.n++] = dg::win_i64(st->comm->peer_win[k], dg::kWinPulled) + (level - 1);
      sig.ptr[sig.n++] = dg::win_i64(st->comm->peer_win[k], dg::kWinArrived) +
                         (int64_t)(level - 1) * 64 + me;
    }
    sg.start[M] = p->n_send;
    if (nowait && p->n_send > 0) {   // seqlock: segment words odd while this push writes
      for (int i = 0; i < sig.n; ++i) odd.ptr[i] = sig.ptr[i];
      odd.n = sig.n;
      DG_TRY(dg::flag_sync(dg::FlagWait{}, odd, s));
    }
    if (p->n_send > 0) {
      int64_t blocks = dg::ceil_div(p->n_send, 8);
      int64_t cap = (int64_t)dg::num_sms() * 16;
      if (blocks > cap) blocks = cap;
      double bytes = (double)p->n_send * ((4.0 + L->es()) * L->width + 4.0);
#define DG_PUT(NORM, BF)                                                                      \
  DG_LAUNCH(DIGEST_PROF_PACK, s, bytes, 0, (k_put<NORM, BF>), (unsigned)blocks, 256, 0, H_local, \
            ld, p->send_idx, p->n_send, sg, L->ld, L->width / 4, wt, sig,                      \
            st->counters + (level - 1))
      if (norm && L->bf16) DG_PUT(true, true);
      else if (norm) DG_PUT(true, false);
      else if (L->bf16) DG_PUT(false, true);
      else DG_PUT(false, false);
#undef DG_PUT
    }
  } else if (M > 1 && !nccl) {
    DG_ARG((int)st->peers.size() == M, DIGEST_E_STATE,
           "single-process store of a %d-part graph: link the stores first", M);
    Segs sg{};
    sg.nseg = M;
    for (int k = 0; k < M; ++k) {
      sg.start[k] = p->send_off[k];
      if (k == me) {
        sg.dst[k] = nullptr;
        continue;
      }
      digest_store* pk = st->peers[k];
      Level& Lk = pk->lev[level - 1];
      DG_ARG(Lk.bf16 == L->bf16, DIGEST_E_STATE, "linked stores disagree on the bf16 store");
      sg.dst[k] = xrow(Lk.buf[1 - Lk.front], pk->part->recv_off[me], Lk.ld, Lk.es());
      if (p->send_count[k] > 0) ++Lk.rx_seq;   // k's back buffer now holds new rows of mine
    }
    sg.start[M] = p->n_send;
    DG_TRY(pack(H_local, ld, p->send_idx, p->n_send, sg, L->ld, L->width, norm, s, L->bf16));
  } else if (nccl) {
    if (L->inflight) DG_CUDA(cudaStreamWaitEvent(s, L->done, 0));  // send buffer reuse
    Segs sg{};
    sg.nseg = 1;
    sg.dst[0] = L->send_buf;
    sg.start[0] = 0;
    sg.start[1] = p->n_send;
    DG_TRY(pack(H_local, ld, p->send_idx, p->n_send, sg, L->ld, L->width, norm, s, L->bf16));
    std::vector<const float*> sp(M);
    std::vector<float*> rp(M);
    std::vector<int64_t> cs(M), cr(M);
    for (int k = 0; k < M; ++k) {
      sp[k] = xrow(L->send_buf, p->send_off[k], L->ld, L->es());
      rp[k] = xrow(L->buf[back], p->recv_off[k], L->ld, L->es());
      cs[k] = p->send_count[k] * L->ld;
      cr[k] = p->recv_count[k] * L->ld;
    }
    cudaStream_t xs = s;
    if (flags & DIGEST_PUSH_ASYNC) {
      DG_CUDA(cudaEventRecord(st->packed, s));
      DG_CUDA(cudaStreamWaitEvent(st->side, st->packed, 0));
      xs = st->side;
    }
    DG_TRY(dg::comm_alltoallv(st->comm, sp.data(), cs.data(), rp.data(), cr.data(), xs,
                              L->bf16 ? ncclBfloat16 : ncclFloat));
    DG_CUDA(cudaEventRecord(L->done, xs));
    L->inflight = true;
  }
  L->ver[back] = version;
  return DIGEST_OK;
}

digest_status digest_pull(digest_store* st, int32_t level, int64_t epoch, int32_t mode,
                          void* stream, const float** front_h) {
  Level* L;
  DG_TRY(get_level(st, level, &L));
  DG_ARG(mode == DIGEST_PULL_FLIP || mode == DIGEST_PULL_COPY || mode == DIGEST_PULL_SNAPSHOT,
         DIGEST_E_INVALID, "bad pull mode");
  cudaStream_t s = dg::as_stream(stream);
  if (mode == DIGEST_PULL_SNAPSHOT && !dg::is_peer(st->comm)) mode = DIGEST_PULL_COPY;
  if (L->bf16 && mode == DIGEST_PULL_FLIP) mode = DIGEST_PULL_COPY;   // bf16 back -> fp32 front
  const int back = 1 - L->front;
  if (L->ver[back] >= epoch)
    return dg::set_error(DIGEST_E_STATE,
                         "pull at epoch %lld would expose version %lld (pushes are visible to "
                         "later epochs only)", (long long)epoch, (long long)L->ver[back]);
  const bool peer = dg::is_peer(st->comm);
  if (peer) DG_ARG(st->connected, DIGEST_E_STATE, "peer-transport store is not connected");
  dg::FlagSet pulled{};   // peer transport: "my back buffer is free for pushes after `epoch`"
  if (peer) {
    pulled.n = 1;
    pulled.ptr[0] = dg::win_i64(st->comm->win, dg::kWinPulled) + (level - 1);
    pulled.value = epoch;
    L->last_pull = epoch;
  }
  if (peer && mode == DIGEST_PULL_SNAPSHOT) {   // DIGEST-A: no waiting for arrivals
    // Always copy: the owners push at their own pace, so whether new rows arrived is
    // only known to the seqlock words, not to this rank's own push count.
    {
      const digest_part* p = st->part;
      SnapSegs sg{};
      int n = 0;
      for (int k = 0; k < p->num_parts; ++k) {
        if (k == p->rank || p->recv_count[k] == 0) continue;
        sg.off[n] = p->recv_off[k];
        sg.cnt[n] = p->recv_count[k];
        sg.seq[n] = dg::win_i64(st->comm->win, dg::kWinArrived) + (int64_t)(level - 1) * 64 + k;
        ++n;
      }
      if (n > 0 && L->bf16)
        DG_LAUNCH(DIGEST_PROF_PACK, s, 6.0 * st->part->n_halo * L->ld, 0, k_snapshot<true>, n, 1024,
                  0, L->buf[back], L->buf[L->front], L->ld, sg);
      else if (n > 0)
        DG_LAUNCH(DIGEST_PROF_PACK, s, 8.0 * st->part->n_halo * L->ld, 0, k_snapshot<false>, n,
                  1024, 0, L->buf[back], L->buf[L->front], L->ld, sg);
      L->ver[L->front] = L->ver[back];
    }
    if (front_h) *front_h = L->buf[L->front];
    return DIGEST_OK;
  }
  // new rows in the back buffer: our own schedule's push (every rank pushes at the same
  // epochs in the synchronous mode), or -- linked single-process stores -- rows a peer
  // wrote there since the last pull (DIGEST-A: peers push at their own local epochs)
  const bool fresh_rows = L->ver[back] > L->ver[L->front] || (!peer && mode == DIGEST_PULL_COPY && L->rx_seq > L->rx_seen);
  L->rx_seen = L->rx_seq;
  if (fresh_rows) {
    if (peer) {   // wait until every owner's rows of this version have arrived
      dg::FlagWait arr{};
      arr.value = L->ver[back];
      const digest_part* p = st->part;
      for (int k = 0; k < p->num_parts; ++k)
        if (k != p->rank && p->recv_count[k] > 0)
          arr.ptr[arr.n++] = dg::win_i64(st->comm->win, dg::kWinArrived) +
                             (int64_t)(level - 1) * 64 + k;
      DG_TRY(dg::flag_sync(arr, mode == DIGEST_PULL_FLIP ? pulled : dg::FlagSet{}, s));
      if (mode == DIGEST_PULL_FLIP) pulled.n = 0;   // already raised
    }
    if (L->inflight) {
      DG_CUDA(cudaStreamWaitEvent(s, L->done, 0));
      L->inflight = false;
    }
    if (mode == DIGEST_PULL_FLIP) {
      L->front = back;
    } else {
      int64_t n4 = st->part->n_halo * L->ld / 4;
      if (n4 > 0) {
        int64_t blocks = dg::ceil_div(n4, 256);
        int64_t cap = (int64_t)dg::num_sms() * 8;
        if (L->bf16)
          DG_LAUNCH(DIGEST_PROF_PACK, s, 24.0 * n4, 0, k_widen,
                    (unsigned)(blocks > cap ? cap : blocks), 256, 0, L->buf[back],
                    reinterpret_cast<float4*>(L->buf[L->front]), n4);
        else
          DG_LAUNCH(DIGEST_PROF_PACK, s, 32.0 * n4, 0, k_copy,
                    (unsigned)(blocks > cap ? cap : blocks), 256, 0,
                    reinterpret_cast<const float4*>(L->buf[back]),
                    reinterpret_cast<float4*>(L->buf[L->front]), n4);
      }
      L->ver[L->front] = L->ver[back];
    }
  }
  if (peer && pulled.n) DG_TRY(dg::flag_sync(dg::FlagWait{}, pulled, s));
  if (front_h) *front_h = L->buf[L->front];
  return DIGEST_OK;
}

digest_status digest_gather_rows(const float* src, int64_t ld_src, const int32_t* idx, int64_t n,
                                 float* dst, int64_t ld_dst, int32_t width, void* stream) {
  DG_ARG(n >= 0 && width > 0 && width % 4 == 0 && ld_src >= width && ld_dst >= width &&
             ld_src % 4 == 0 && ld_dst % 4 == 0,
         DIGEST_E_SHAPE, "bad gather shape");
  if (n == 0) return DIGEST_OK;
  DG_ARG(src && idx && dst, DIGEST_E_INVALID, "NULL argument");
  Segs sg{};
  sg.nseg = 1;
  sg.dst[0] = dst;
  sg.start[0] = 0;
  sg.start[1] = n;
  return pack(src, ld_src, idx, n, sg, ld_dst, width, false, dg::as_stream(stream));
}

digest_status digest_store_front(const digest_store* st, int32_t level, const float** front_h,
                                 int64_t* ld_h, int64_t* version_h) {
  DG_ARG(st, DIGEST_E_INVALID, "NULL store");
  DG_ARG(level >= 1 && level <= (int32_t)st->lev.size(), DIGEST_E_INVALID, "bad level");
  const Level& L = st->lev[level - 1];
  if (front_h) *front_h = L.buf[L.front];
  if (ld_h) *ld_h = L.ld;
  if (version_h) *version_h = L.ver[L.front];
  return DIGEST_OK;
}

digest_status digest_store_grad_buffer(digest_store* st, int32_t level, float** buf_h,
                                       int64_t* ld_h) {
  Level* L;
  DG_TRY(get_level(st, level, &L));
  float* b = L->grad_buf;
  if (dg::is_peer(st->comm)) {   // two slots, alternating per backward (see return below)
    ++L->gseq;
    b = reinterpret_cast<float*>(reinterpret_cast<char*>(L->grad_buf) +
                                 (size_t)(L->gseq & 1) * L->halo_bytes);
  }
  if (buf_h) *buf_h = b;
  if (ld_h) *ld_h = L->ld;
  return DIGEST_OK;
}

digest_status digest_return_halo_grad(digest_store* st, int32_t level, float* G_local,
                                      int64_t ld_g, const float* mask, int64_t ld_m,
                                      void* stream) {
  Level* L;
  DG_TRY(get_level(st, level, &L));
  const digest_part* p = st->part;
  DG_ARG(G_local || p->n_local == 0, DIGEST_E_INVALID, "G_local is NULL");
  DG_ARG(ld_g >= L->width && ld_g % 4 == 0 && ((uintptr_t)G_local & 15) == 0, DIGEST_E_INVALID,
         "G_local: ld must be >= width and a multiple of 4, pointer 16-byte aligned");
  DG_ARG(!mask || (ld_m >= L->width && ld_m % 4 == 0 && ((uintptr_t)mask & 15) == 0),
         DIGEST_E_INVALID, "mask: bad ld or alignment");
  cudaStream_t s = dg::as_stream(stream);
  const int M = p->num_parts, me = p->rank;
  if (M == 1) return DIGEST_OK;
  const bool nccl = dg::is_nccl(st->comm);
  const bool peer = dg::is_peer(st->comm);
  bool odd = false;
  if (peer) {
    // Peer transport, sequence q = this level's grad_buffer calls: raise gready[q] on
    // every neighbouring part, wait for theirs, then read their slot q%2 in place.  A
    // slot is rewritten at q+2 only after its owner saw gready[q+1] from every reader,
    // which each reader raises after finishing its reads of q (stream order).
    DG_ARG(st->connected, DIGEST_E_STATE, "peer-transport store is not connected");
    dg::FlagSet sig{};
    dg::FlagWait wt{};
    sig.value = wt.value = L->gseq;
    for (int k = 0; k < M; ++k) {
      if (k == me || (p->send_count[k] == 0 && p->recv_count[k] == 0)) continue;
      sig.ptr[sig.n++] = dg::win_i64(st->comm->peer_win[k], dg::kWinGReady) +
                         (int64_t)(level - 1) * 64 + me;
      wt.ptr[wt.n++] = dg::win_i64(st->comm->win, dg::kWinGReady) + (int64_t)(level - 1) * 64 + k;
    }
    if (sig.n == 0) return DIGEST_OK;   // no neighbouring part: nothing to return
    DG_ARG(L->gseq > 0, DIGEST_E_STATE, "digest_store_grad_buffer was not called for this level");
    DG_TRY(dg::flag_sync(dg::FlagWait{}, sig, s));
    DG_TRY(dg::flag_sync(wt, dg::FlagSet{}, s));
    odd = (L->gseq & 1) != 0;
  } else if (!nccl)
    DG_ARG((int)st->peers.size() == M, DIGEST_E_STATE,
           "single-process store of a %d-part graph: link the stores first", M);
  if (nccl) {   // reverse of the push: my halo segment of owner k goes back to k
    std::vector<const float*> sp(M);
    std::vector<float*> rp(M);
    std::vector<int64_t> cs(M), cr(M);
    for (int k = 0; k < M; ++k) {
      sp[k] = L->grad_buf + p->recv_off[k] * L->ld;
      cs[k] = p->recv_count[k] * L->ld;
      rp[k] = L->ret_recv + p->send_off[k] * L->ld;
      cr[k] = p->send_count[k] * L->ld;
    }
    DG_TRY(dg::comm_alltoallv(st->comm, sp.data(), cs.data(), rp.data(), cr.data(), s));
  }
  for (int k = 0; k < M; ++k) {
    if (k == me || p->send_count[k] == 0) continue;
    const float* src;
    if (nccl) {
      src = L->ret_recv + p->send_off[k] * L->ld;
    } else if (peer) {
      const PeerLevel& q = st->pl[k][level - 1];
      src = reinterpret_cast<const float*>(reinterpret_cast<const char*>(q.grad) +
                                           (odd ? q.slot_bytes : 0)) +
            st->peer_recv_off[k][me] * L->ld;
    } else {
      digest_store* pk = st->peers[k];
      src = pk->lev[level - 1].grad_buf + pk->part->recv_off[me] * L->ld;
    }
    const int64_t n = p->send_count[k];
    int64_t blocks = dg::ceil_div(n, 8);
    if (blocks > dg::num_sms() * 16) blocks = dg::num_sms() * 16;
    DG_LAUNCH(DIGEST_PROF_PACK, s, 12.0 * n * L->width, 0, k_return_add, (unsigned)blocks, 256, 0,
              src, L->ld, p->send_idx + p->send_off[k], n, G_local, ld_g, mask, ld_m,
              L->width / 4);
  }
  return DIGEST_OK;
}

digest_status digest_store_export(const digest_store* st, uint8_t* blob_h, size_t* bytes_h) {
  DG_ARG(st && bytes_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(dg::is_peer(st->comm), DIGEST_E_INVALID, "store does not use the peer transport");
  *bytes_h = sizeof(PeerBlob);
  if (!blob_h) return DIGEST_OK;
  PeerBlob b;
  std::memset(&b, 0, sizeof(b));
  b.rank = st->part->rank;
  b.levels = (int32_t)st->lev.size();
  for (int k = 0; k < st->part->num_parts; ++k) b.recv_off[k] = st->part->recv_off[k];
  b.halo_rows = st->part->n_halo > 0 ? st->part->n_halo : 1;
  for (size_t l = 0; l < st->lev.size(); ++l) {
    DG_CUDA(cudaIpcGetMemHandle(&b.h[l][0], st->lev[l].buf[0]));
    DG_CUDA(cudaIpcGetMemHandle(&b.h[l][1], st->lev[l].buf[1]));
    DG_CUDA(cudaIpcGetMemHandle(&b.h[l][2], st->lev[l].grad_buf));
  }
  std::memcpy(blob_h, &b, sizeof(b));
  return DIGEST_OK;
}

digest_status digest_store_connect(digest_store* st, const uint8_t* blobs_h, size_t blob_bytes) {
  DG_ARG(st && blobs_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(dg::is_peer(st->comm), DIGEST_E_INVALID, "store does not use the peer transport");
  DG_ARG(st->comm->connected, DIGEST_E_STATE, "connect the peer communicator first");
  DG_ARG(!st->connected, DIGEST_E_STATE, "store already connected");
  DG_ARG(blob_bytes == sizeof(PeerBlob), DIGEST_E_INVALID, "blob size %zu, expected %zu",
         blob_bytes, sizeof(PeerBlob));
  const int M = st->part->num_parts, me = st->part->rank;
  const size_t nl = st->lev.size();
  st->pl.assign(M, std::vector<PeerLevel>(nl, PeerLevel{{nullptr, nullptr}, nullptr, 0}));
  st->peer_recv_off.assign(M, std::vector<int64_t>(DIGEST_MAX_PARTS, 0));
  for (int k = 0; k < M; ++k) {
    PeerBlob b;
    std::memcpy(&b, blobs_h + (size_t)k * sizeof(PeerBlob), sizeof(b));
    DG_ARG(b.rank == k && b.levels == (int32_t)nl, DIGEST_E_INVALID,
           "blob %d is from rank %d with %d levels (expected rank %d, %zu levels)", k, b.rank,
           b.levels, k, nl);
    for (int j = 0; j < M; ++j) st->peer_recv_off[k][j] = b.recv_off[j];
    for (size_t l = 0; l < nl; ++l) {
      if (k == me) {
        st->pl[k][l] = PeerLevel{{st->lev[l].buf[0], st->lev[l].buf[1]}, st->lev[l].grad_buf,
                                 st->lev[l].halo_bytes};
        continue;
      }
      void* ptr[3];
      for (int i = 0; i < 3; ++i) {
        cudaError_t e = cudaIpcOpenMemHandle(&ptr[i], b.h[l][i], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
          return dg::set_error(DIGEST_E_CUDA, "cudaIpcOpenMemHandle(rank %d level %zu): %s", k,
                               l + 1, cudaGetErrorString(e));
      }
      const size_t hb = sizeof(float) * (size_t)b.halo_rows * (size_t)st->lev[l].ld;
      st->pl[k][l] = PeerLevel{{(float*)ptr[0], (float*)ptr[1]}, (float*)ptr[2], hb};
    }
  }
  st->connected = true;
  return DIGEST_OK;
}

digest_status digest_store_destroy(digest_store* st) {
  if (st && st->side) cudaStreamSynchronize(st->side);
  destroy_store(st);
  return DIGEST_OK;
}

}  // extern "C"

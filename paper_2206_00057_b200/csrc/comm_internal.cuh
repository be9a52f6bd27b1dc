// Communicator handle (library-owned): NCCL, or the peer-memory (CUDA IPC) transport.
#pragma once
#include <nccl.h>
#include <cstdio>

#include "common.cuh"

// Peer-memory window: one cudaMalloc per rank, identical layout on every rank, mapped
// into every peer's address space with CUDA IPC.  Flag words are int64 versions/sequence
// numbers, written with st.release.sys by the producer and polled with ld.acquire.sys.
namespace dg {
constexpr int kWinLevels = 64;
constexpr size_t kWinArrived = 0;                                   // int64 [level][src]: push arrived (version)
constexpr size_t kWinPulled = kWinArrived + 8 * kWinLevels * 64;    // int64 [level]: last pull epoch of the owner
constexpr size_t kWinGReady = kWinPulled + 8 * kWinLevels;          // int64 [level][src]: halo-grad slot ready (seq)
constexpr size_t kWinArReady = kWinGReady + 8 * kWinLevels * 64;    // int64 [src]: allreduce slot ready (seq)
constexpr size_t kWinPs = kWinArReady + 8 * 64;                      // int64 [2]: PS lock, PS updates
constexpr size_t kWinSlots = (kWinPs + 16 + 4095) / 4096 * 4096;    // float [3][max_grad]: 2 AGG slots, PS W
}  // namespace dg

struct digest_comm {
  int32_t kind = 0;   // 0 NCCL, 1 peer memory
  ncclComm_t comm = nullptr;
  int32_t nranks = 1, rank = 0;
  // peer transport
  char* win = nullptr;                       // own window (device)
  char* peer_win[DIGEST_MAX_PARTS] = {};     // every rank's window in this address space
  bool connected = false;
  int64_t max_grad = 0;
  int64_t ar_seq = 0;                        // allreduce calls so far (same on every rank)
  unsigned* counters = nullptr;              // last-block-done counters (device, own)
};

namespace dg {
digest_status comm_allreduce_sum(digest_comm* c, float* buf, int64_t count, cudaStream_t s);
// Grouped point-to-point all-to-allv: send[k] (count_s[k] floats) to rank k and
// recv[k] (count_r[k] floats) from rank k, k != own rank.
digest_status comm_alltoallv(digest_comm* c, const float* const* send, const int64_t* count_s,
                             float* const* recv, const int64_t* count_r, cudaStream_t s,
                             ncclDataType_t dt = ncclFloat);
inline bool is_peer(const digest_comm* c) { return c && c->kind == 1 && c->nranks > 1; }
inline bool is_nccl(const digest_comm* c) { return c && c->kind == 0 && c->nranks > 1; }
inline int64_t* win_i64(char* w, size_t off) { return reinterpret_cast<int64_t*>(w + off); }

// Device-side waits and signals on window flags (peer.cu).
struct FlagWait {            // spin until *ptr[i] >= value for i < n (ld.acquire.sys)
  const int64_t* ptr[DIGEST_MAX_PARTS];
  int32_t n;
  int64_t value;
};
struct FlagSet {             // *ptr[i] = value for i < n (fence.sys, st.release.sys)
  int64_t* ptr[DIGEST_MAX_PARTS];
  int32_t n;
  int64_t value;
};
// One tiny launch: wait on `w`, then set `f` (either may be empty).
digest_status flag_sync(const FlagWait& w, const FlagSet& f, cudaStream_t s);
// AGG over the peer windows: g <- scale * sum_k g_k (rank order, bit-identical on all ranks).
digest_status peer_allreduce(digest_comm* c, float* g, int64_t count, float scale, cudaStream_t s,
                             bool in_slot = false);
void peer_comm_release(digest_comm* c);
float* peer_next_slot(digest_comm* c);   // own slot of the next allreduce call
}  // namespace dg

// --- device helpers (included by the kernels that fuse their own wait/signal)
#ifdef __CUDACC__
namespace dg {
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Bounded spin (30 s of %globaltimer): a peer that never arrives traps the kernel (a
// sticky, reported CUDA error) instead of hanging the device.
__device__ __forceinline__ void wait_flags(const FlagWait& w) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < w.n; ++i) {
    while (ld_acquire_sys(w.ptr[i]) < w.value) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 30ull * 1000000000ull) {
        printf("digest: peer flag wait timed out (slot %d, want %lld, have %lld)\n", i,
               (long long)w.value, (long long)ld_acquire_sys(w.ptr[i]));
        __trap();
      }
      __nanosleep(256);
    }
  }
}
__device__ __forceinline__ void set_flags(const FlagSet& f) {
  __threadfence_system();
  for (int i = 0; i < f.n; ++i) st_release_sys(f.ptr[i], f.value);
}
// Last-block-done: every block calls this once at its end (after its stores); the
// block that arrives last sees all blocks' stores (fences + atomic) and returns true.
// It also resets the counter for the next launch in stream order.
__device__ __forceinline__ bool last_block_done(unsigned* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
    if (last) *counter = 0u;
  }
  __syncthreads();
  return last;
}
}  // namespace dg
#endif

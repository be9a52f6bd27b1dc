// Peer-memory transport (one process per GPU, or several processes on one GPU):
// every rank owns a window (flags + two gradient slots) that is mapped into every
// peer's address space with CUDA IPC, so the exchange steps of the method are plain
// loads and stores over NVLink / NVSwitch issued by the library's own kernels:
//   * AGG (Alg. 1, update rule P:896): publish the local gradient into the own
//     window (slot = call parity) and signal every peer, then each rank sums all
//     ranks' slots in rank order -- the same order as the loopback sum, so every rank
//     (and a single-process run of the same partitions) gets bit-identical weights;
//   * the boundary push (Alg. 1) and the halo-gradient return
//      live in store.cu and use the flag words of the same window.
// No host synchronisation: producers signal with st.release.sys after a system fence,
// consumers spin with ld.acquire.sys inside the consuming kernel (bounded: 30 s).
#include <cstring>

#include "comm_internal.cuh"

namespace {

__global__ void k_flag_sync(dg::FlagWait w, dg::FlagSet f) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    dg::wait_flags(w);
    dg::set_flags(f);
  }
}

// slot_own[i] = g[i]; the last block signals ar_ready[me] = seq on every rank.
__global__ void k_ar_publish(const float* __restrict__ g, int64_t n, float* __restrict__ slot,
                             unsigned* counter, dg::FlagSet sig) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    slot[i] = g[i];
  if (dg::last_block_done(counter) && threadIdx.x == 0) dg::set_flags(sig);
}

struct SlotTable {
  const float* p[DIGEST_MAX_PARTS];
};

// g[i] = scale * (slot_0[i] + slot_1[i] + ... + slot_{M-1}[i]), summed in rank order
// exactly like the loopback k_sum_bufs (s = 0; s += b; s *= a).
// `sig` (fused AGG, the slot was written by the weight-gradient kernels before this
// launch in stream order): every block raises this rank's ready flag on every peer
// (idempotent: same value) before waiting, so no block depends on another's schedule.
__global__ void k_ar_reduce(float* __restrict__ g, int64_t n, SlotTable t, int nb, float a,
                            dg::FlagWait w, dg::FlagSet sig) {
  if (threadIdx.x == 0) {
    if (sig.n) dg::set_flags(sig);
    dg::wait_flags(w);
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += __ldcv(t.p[b] + i);
    s *= a;
    g[i] = s;
  }
}

unsigned blocks_for(int64_t n) {
  int64_t b = dg::ceil_div(n, 256);
  int64_t cap = (int64_t)dg::num_sms() * 4;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

namespace dg {

digest_status flag_sync(const FlagWait& w, const FlagSet& f, cudaStream_t s) {
  if (w.n == 0 && f.n == 0) return DIGEST_OK;
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 0, 0, k_flag_sync, 1, 32, 0, w, f);
  return DIGEST_OK;
}

digest_status peer_allreduce(digest_comm* c, float* g, int64_t count, float scale,
                             cudaStream_t s, bool in_slot) {
  DG_ARG(c->connected, DIGEST_E_STATE, "peer communicator is not connected");
  DG_ARG(count <= c->max_grad, DIGEST_E_SHAPE,
         "allreduce of %lld floats exceeds the window's %lld", (long long)count,
         (long long)c->max_grad);
  const int64_t seq = ++c->ar_seq;
  const int par = (int)(seq & 1);
  const int M = c->nranks;
  const size_t slot_off = kWinSlots + sizeof(float) * (size_t)par * (size_t)c->max_grad;
  FlagSet sig{};
  sig.n = M;
  sig.value = seq;
  for (int k = 0; k < M; ++k) sig.ptr[k] = win_i64(c->peer_win[k], kWinArReady) + c->rank;
  if (!in_slot)
    DG_LAUNCH(DIGEST_PROF_OTHER, s, 8.0 * count, 0, k_ar_publish, blocks_for(count), 256, 0, g,
              count, reinterpret_cast<float*>(c->win + slot_off), c->counters, sig);
  FlagWait w{};
  w.n = M;
  w.value = seq;
  SlotTable t{};
  for (int k = 0; k < M; ++k) {
    w.ptr[k] = win_i64(c->win, kWinArReady) + k;
    t.p[k] = reinterpret_cast<const float*>(c->peer_win[k] + slot_off);
  }
  DG_LAUNCH(DIGEST_PROF_OTHER, s, 4.0 * count * (M + 1), 0, k_ar_reduce, blocks_for(count), 256, 0,
            g, count, t, M, scale, w, in_slot ? sig : FlagSet{});
  return DIGEST_OK;
}

// Own window slot of the NEXT allreduce call (parity of ar_seq + 1).
float* peer_next_slot(digest_comm* c) {
  const int par = (int)((c->ar_seq + 1) & 1);
  return reinterpret_cast<float*>(c->win + kWinSlots +
                                  sizeof(float) * (size_t)par * (size_t)c->max_grad);
}

}  // namespace dg

extern "C" {

digest_status digest_grad_slot(digest_comm* c, float** slot_h) {
  DG_ARG(slot_h, DIGEST_E_INVALID, "NULL argument");
  *slot_h = nullptr;
  DG_ARG(dg::is_peer(c), DIGEST_E_UNSUPPORTED, "digest_grad_slot needs a multi-rank peer communicator");
  DG_ARG(c->connected, DIGEST_E_STATE, "peer communicator is not connected");
  *slot_h = dg::peer_next_slot(c);
  return DIGEST_OK;
}

digest_status digest_grad_allreduce_ex(digest_comm* c, float* grads, int64_t count, float scale,
                                       uint32_t flags, void* stream) {
  if (!(flags & DIGEST_AR_IN_SLOT)) return digest_grad_allreduce(c, grads, count, scale, stream);
  DG_ARG(grads && count >= 0, DIGEST_E_INVALID, "bad gradient buffer");
  DG_ARG(dg::is_peer(c), DIGEST_E_UNSUPPORTED, "DIGEST_AR_IN_SLOT needs a multi-rank peer communicator");
  return dg::peer_allreduce(c, grads, count, scale, dg::as_stream(stream), true);
}

digest_status digest_comm_init_peer(int32_t nranks, int32_t rank, int64_t max_grad_count,
                                    digest_comm** out_h) {
  DG_ARG(out_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(nranks >= 1 && nranks <= DIGEST_MAX_PARTS && rank >= 0 && rank < nranks,
         DIGEST_E_INVALID, "bad rank/nranks");
  DG_ARG(max_grad_count >= 0, DIGEST_E_INVALID, "bad max_grad_count");
  *out_h = nullptr;
  digest_comm* c = new digest_comm();
  c->kind = 1;
  c->nranks = nranks;
  c->rank = rank;
  c->max_grad = dg::round_up(max_grad_count, 4);
  const size_t bytes = dg::kWinSlots + sizeof(float) * 3 * (size_t)(c->max_grad > 0 ? c->max_grad : 4);
  if (cudaMalloc(&c->win, bytes) != cudaSuccess || cudaMemset(c->win, 0, bytes) != cudaSuccess ||
      cudaMalloc(&c->counters, 256 * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(c->counters, 0, 256 * sizeof(unsigned)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(c->win);
    cudaFree(c->counters);
    delete c;
    return dg::set_error(DIGEST_E_NOMEM, "peer window allocation failed");
  }
  c->peer_win[rank] = c->win;
  c->connected = (nranks == 1);
  *out_h = c;
  return DIGEST_OK;
}

digest_status digest_comm_export(const digest_comm* c, uint8_t handle_h[DIGEST_IPC_HANDLE_BYTES]) {
  DG_ARG(c && handle_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(c->kind == 1, DIGEST_E_INVALID, "not a peer-memory communicator");
  static_assert(sizeof(cudaIpcMemHandle_t) == DIGEST_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  DG_CUDA(cudaIpcGetMemHandle(&h, c->win));
  std::memcpy(handle_h, &h, sizeof(h));
  return DIGEST_OK;
}

digest_status digest_comm_connect(digest_comm* c, const uint8_t* handles_h) {
  DG_ARG(c && handles_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(c->kind == 1, DIGEST_E_INVALID, "not a peer-memory communicator");
  DG_ARG(!c->connected || c->nranks == 1, DIGEST_E_STATE, "already connected");
  for (int k = 0; k < c->nranks; ++k) {
    if (k == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles_h + (size_t)k * DIGEST_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return dg::set_error(DIGEST_E_CUDA, "cudaIpcOpenMemHandle(rank %d window): %s", k,
                           cudaGetErrorString(e));
    c->peer_win[k] = static_cast<char*>(p);
  }
  c->connected = true;
  return DIGEST_OK;
}

}  // extern "C"

namespace dg {
void peer_comm_release(digest_comm* c) {
  if (!c || c->kind != 1) return;
  for (int k = 0; k < c->nranks; ++k)
    if (k != c->rank && c->peer_win[k]) cudaIpcCloseMemHandle(c->peer_win[k]);
  cudaFree(c->win);
  cudaFree(c->counters);
}
}  // namespace dg

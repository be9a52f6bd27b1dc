// NCCL plumbing: communicator bootstrap (id broadcast by the caller's process
// group), the gradient allreduce (AGG) and the grouped send/recv
// all-to-allv of boundary rows (the stale-store exchange).
#include <cstring>

#include "comm_internal.cuh"

#define DG_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      return ::dg::set_error(DIGEST_E_NCCL, "%s failed: %s (%s:%d)", #call,            \
                             ncclGetErrorString(r_), __FILE__, __LINE__);              \
  } while (0)

namespace dg {

digest_status comm_allreduce_sum(digest_comm* c, float* buf, int64_t count, cudaStream_t s) {
  if (count == 0) return DIGEST_OK;
  DG_ARG(c->kind == 0, DIGEST_E_INVALID, "not an NCCL communicator");
  DG_NCCL(ncclAllReduce(buf, buf, (size_t)count, ncclFloat, ncclSum, c->comm, s));
  return DIGEST_OK;
}

digest_status comm_alltoallv(digest_comm* c, const float* const* send, const int64_t* count_s,
                             float* const* recv, const int64_t* count_r, cudaStream_t s,
                             ncclDataType_t dt) {
  DG_NCCL(ncclGroupStart());
  for (int k = 0; k < c->nranks; ++k) {   // own rank included: a self transfer if counted
    if (count_s[k] > 0) {
      ncclResult_t r = ncclSend(send[k], (size_t)count_s[k], dt, k, c->comm, s);
      if (r != ncclSuccess) {
        ncclGroupEnd();
        return set_error(DIGEST_E_NCCL, "ncclSend: %s", ncclGetErrorString(r));
      }
    }
    if (count_r[k] > 0) {
      ncclResult_t r = ncclRecv(recv[k], (size_t)count_r[k], dt, k, c->comm, s);
      if (r != ncclSuccess) {
        ncclGroupEnd();
        return set_error(DIGEST_E_NCCL, "ncclRecv: %s", ncclGetErrorString(r));
      }
    }
  }
  DG_NCCL(ncclGroupEnd());
  return DIGEST_OK;
}

}  // namespace dg

extern "C" {

digest_status digest_comm_unique_id(uint8_t id_h[128]) {
  DG_ARG(id_h, DIGEST_E_INVALID, "NULL id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  DG_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_h, &id, 128);
  return DIGEST_OK;
}

digest_status digest_comm_init(const uint8_t id_h[128], int32_t nranks, int32_t rank,
                               digest_comm** out_h) {
  DG_ARG(id_h && out_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(nranks >= 1 && nranks <= DIGEST_MAX_PARTS && rank >= 0 && rank < nranks,
         DIGEST_E_INVALID, "bad rank/nranks");
  ncclUniqueId id;
  std::memcpy(&id, id_h, 128);
  digest_comm* c = new digest_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return dg::set_error(DIGEST_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out_h = c;
  return DIGEST_OK;
}

digest_status digest_comm_alltoallv(digest_comm* c, const float* const* send_h,
                                    const int64_t* count_s_h, float* const* recv_h,
                                    const int64_t* count_r_h, void* stream) {
  DG_ARG(c && send_h && count_s_h && recv_h && count_r_h, DIGEST_E_INVALID, "NULL argument");
  DG_ARG(c->kind == 0, DIGEST_E_INVALID, "not an NCCL communicator");
  for (int k = 0; k < c->nranks; ++k) {
    DG_ARG(count_s_h[k] >= 0 && count_r_h[k] >= 0, DIGEST_E_INVALID, "negative count");
    DG_ARG(!count_s_h[k] || send_h[k], DIGEST_E_INVALID, "NULL send buffer %d", k);
    DG_ARG(!count_r_h[k] || recv_h[k], DIGEST_E_INVALID, "NULL recv buffer %d", k);
  }
  return dg::comm_alltoallv(c, send_h, count_s_h, recv_h, count_r_h, dg::as_stream(stream));
}

digest_status digest_comm_destroy(digest_comm* c) {
  if (!c) return DIGEST_OK;
  if (c->kind == 1) {
    cudaDeviceSynchronize();
    dg::peer_comm_release(c);
  }
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return DIGEST_OK;
}

}  // extern "C"

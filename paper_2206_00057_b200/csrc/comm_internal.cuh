// NCCL communicator handle (library-owned).
#pragma once
#include <nccl.h>

#include "common.cuh"

struct digest_comm {
  ncclComm_t comm = nullptr;
  int32_t nranks = 1, rank = 0;
};

namespace dg {
digest_status comm_allreduce_sum(digest_comm* c, float* buf, int64_t count, cudaStream_t s);
// Grouped point-to-point all-to-allv: send[k] (count_s[k] floats) to rank k and
// recv[k] (count_r[k] floats) from rank k, k != own rank.
digest_status comm_alltoallv(digest_comm* c, const float* const* send, const int64_t* count_s,
                             float* const* recv, const int64_t* count_r, cudaStream_t s);
}  // namespace dg

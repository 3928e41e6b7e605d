// Communicator handle of the distributed (t-slab) solver (comm.cu).
#pragma once
#include "common.cuh"

struct mgt_comm_s {
  int nranks, rank;
  void *nccl;  // ncclComm_t (null for a single rank)
};

namespace mgt {
// sum-all-reduce n doubles in place on stream st (no-op for one rank)
int comm_allreduce_sum(mgt_comm_s *c, double *buf, size_t n, cudaStream_t st);
// ring exchange of the two t-faces: to_prev -> rank-1, to_next -> rank+1;
// receives rank+1's to_prev into from_next and rank-1's to_next into from_prev
int comm_halo(mgt_comm_s *c, const void *to_prev, const void *to_next, void *from_next, void *from_prev,
              size_t bytes, cudaStream_t st);
}  // namespace mgt

// paper_2307_08507_b200/csrc/comm.h -- internal communicator (see comm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/mdot.h"

namespace mdot {

struct Comm {
  int nranks = 1, rank = 0, device = 0;
  void* nccl = nullptr;   // ncclComm_t
};

// In-place fp64 sum allreduce on `st` (no-op for a single rank).
mdot_status comm_allreduce_sum(Comm* cm, double* buf, size_t count, cudaStream_t st);

}  // namespace mdot

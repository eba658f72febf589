// paper_2307_08507_b200/csrc/comm.h -- internal communicator (see comm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/mdot.h"

namespace mdot {

struct LocalGroup;

struct Comm {
  int nranks = 1, rank = 0, device = 0;
  void* nccl = nullptr;          // ncclComm_t (NCCL transport)
  LocalGroup* local = nullptr;   // in-process transport (virtual ranks / tests)
  // graph-capturable transport (NCCL): the sharded solve may run under
  // device control with the allreduce inside the CUDA-graph slots
  bool capturable() const { return nccl != nullptr; }
};

enum { COMM_SUM = 0, COMM_MAX = 1 };
// In-place fp64 allreduce on `st` (no-op for a single rank).
mdot_status comm_allreduce(Comm* cm, double* buf, size_t count, int op, cudaStream_t st);
inline mdot_status comm_allreduce_sum(Comm* cm, double* buf, size_t count, cudaStream_t st) {
  return comm_allreduce(cm, buf, count, COMM_SUM, st);
}

}  // namespace mdot

// paper_2307_08507_b200/csrc/comm.h -- internal communicator (see comm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/mdot.h"

namespace mdot {

struct LocalGroup;
struct PersistArgs;

// Fused peer exchange state (mdot_comm_enable_peer): this rank's exchange
// block and the view of every rank's block from this GPU.
struct PeerState {
  void* block = nullptr;              // own block: [2][nranks][ld] fp64 | flags[8] u32 | epoch u32 | err i32
  size_t bytes = 0;
  int64_t ld = 0, n_max = 0;
  double* recv[8] = {};
  unsigned int* flag[8] = {};
  unsigned int* epoch = nullptr;
  int* err = nullptr;
  void* opened[8] = {};               // IPC-opened peer blocks (NCCL transport)
};

struct Comm {
  int nranks = 1, rank = 0, device = 0;
  void* nccl = nullptr;          // ncclComm_t (NCCL transport)
  LocalGroup* local = nullptr;   // in-process transport (virtual ranks / tests)
  PeerState* peer = nullptr;     // fused peer exchange enabled (mdot_comm_enable_peer)
  // graph-capturable transport (NCCL): the sharded solve may run under
  // device control with the allreduce inside the CUDA-graph slots
  bool capturable() const { return nccl != nullptr; }
};

enum { COMM_SUM = 0, COMM_MAX = 1 };
// CTAs per rank of the fused peer persistent kernel for a problem with n
// columns, given the co-resident grid of one GPU (0: no peer path).
int comm_peer_ncta(const Comm* cm, int64_t n, int grid);
// Run one persistent projection launch of this rank with the fused peer
// exchange (the in-process transport gathers every rank's arguments and
// launches ONE kernel for all of them).  Synchronizes `st`.
mdot_status comm_peer_persist(Comm* cm, const PersistArgs& a, const void* tmap, int ncta, cudaStream_t st);
// In-place fp64 allreduce on `st` (no-op for a single rank).
mdot_status comm_allreduce(Comm* cm, double* buf, size_t count, int op, cudaStream_t st);
inline mdot_status comm_allreduce_sum(Comm* cm, double* buf, size_t count, cudaStream_t st) {
  return comm_allreduce(cm, buf, count, COMM_SUM, st);
}

}  // namespace mdot

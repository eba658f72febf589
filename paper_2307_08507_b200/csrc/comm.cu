// paper_2307_08507_b200/csrc/comm.cu -- NCCL communicator for the row-sharded
// multi-GPU path.  NCCL is loaded with dlopen("libnccl.so.2")
// so the library shares the NCCL that torch.distributed already loaded in
// the process (one NCCL per process, no version clash).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include "../../include/mdot.h"
#include "comm.h"
#include "solver.h"

namespace mdot {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;

static bool load_nccl() {
  if (g_nccl.h) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    g_nccl.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) {
    set_error("cannot dlopen libnccl.so.2: %s", dlerror());
    return false;
  }
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(g_nccl.h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(g_nccl.h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(g_nccl.h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.CommGetAsyncError = (decltype(g_nccl.CommGetAsyncError))dlsym(g_nccl.h, "ncclCommGetAsyncError");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(g_nccl.h, "ncclGetErrorString");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy) {
    set_error("libnccl.so.2 lacks required symbols");
    dlclose(g_nccl.h);
    g_nccl.h = nullptr;
    return false;
  }
  return true;
}

mdot_status comm_allreduce_sum(Comm* cm, double* buf, size_t count, cudaStream_t st) {
  if (!cm || cm->nranks == 1) return MDOT_OK;
  ncclResult_t r = g_nccl.AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)cm->nccl, st);
  if (r != ncclSuccess) {
    set_error("ncclAllReduce failed: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
    return MDOT_ENCCL;
  }
  return MDOT_OK;
}

}  // namespace mdot

using namespace mdot;

extern "C" {

mdot_status mdot_get_unique_id(void* out) {
  if (!out) { set_error("NULL output"); return MDOT_EINVAL; }
  if (!load_nccl()) return MDOT_ENCCL;
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) { set_error("ncclGetUniqueId failed"); return MDOT_ENCCL; }
  memcpy(out, &id, sizeof(id));
  return MDOT_OK;
}

mdot_status mdot_comm_create(const void* uid, int32_t nranks, int32_t rank, int32_t device, mdot_comm** out) {
  if (!uid || !out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("bad comm arguments"); return MDOT_EINVAL; }
  if (cudaSetDevice(device) != cudaSuccess) { set_error("cudaSetDevice(%d) failed", device); return MDOT_ECUDA; }
  Comm* cm = new Comm();
  cm->nranks = nranks;
  cm->rank = rank;
  cm->device = device;
  if (nranks > 1) {
    if (!load_nccl()) { delete cm; return MDOT_ENCCL; }
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclComm_t c;
    ncclResult_t r = g_nccl.CommInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) {
      set_error("ncclCommInitRank failed: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
      delete cm;
      return MDOT_ENCCL;
    }
    cm->nccl = c;
  }
  *out = reinterpret_cast<mdot_comm*>(cm);
  return MDOT_OK;
}

mdot_status mdot_comm_destroy(mdot_comm* c) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm) return MDOT_OK;
  if (cm->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)cm->nccl);
  delete cm;
  return MDOT_OK;
}

}  // extern "C"

extern "C" mdot_status mdot_solve_sharded(mdot_comm* c, const mdot_problem* local_rows, int64_t row0,
                                          int64_t n_local, const mdot_schedule* sched, const mdot_options* opt,
                                          double* u_local_out, double* v_out, mdot_result* res) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm || !local_rows) { set_error("bad arguments"); return MDOT_EINVAL; }
  if (cm->nranks == 1 && row0 == 0 && n_local == local_rows->n)
    return mdot_solve(local_rows, sched, opt, u_local_out, v_out, nullptr, res);
  set_error("multi-rank sharded solve is not available in this build");
  return MDOT_EINVAL;
}

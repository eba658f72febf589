// paper_2307_08507_b200/csrc/comm.cu -- NCCL communicator for the row-sharded
// multi-GPU path.  NCCL is loaded with dlopen("libnccl.so.2")
// so the library shares the NCCL that torch.distributed already loaded in
// the process (one NCCL per process, no version clash).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

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

// In-process transport: ranks are threads of one process (one stream each);
// each allreduce syncs its stream, deposits its buffer, waits for all ranks
// and reduces the deposits in rank order (deterministic).  No device code
// waits on another rank, so virtual ranks may share one GPU.
struct LocalGroup {
  int nranks = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<std::vector<double>> slots;
  std::vector<double> result;
  int refs = 0;
};
static std::mutex g_groups_m;
static std::map<std::string, std::shared_ptr<LocalGroup>> g_groups;

static mdot_status local_allreduce(Comm* cm, double* buf, size_t count, int op, cudaStream_t st) {
  LocalGroup* g = cm->local;
  std::vector<double> mine(count);
  if (cudaStreamSynchronize(st) != cudaSuccess ||
      cudaMemcpy(mine.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
    set_error("local allreduce: device copy failed");
    return MDOT_ECUDA;
  }
  {
    std::unique_lock<std::mutex> lk(g->m);
    g->slots[cm->rank].swap(mine);
    const long long gen = g->generation;
    if (++g->arrived == g->nranks) {
      g->result.assign(count, op == COMM_MAX ? -INFINITY : 0.0);
      for (int q = 0; q < g->nranks; ++q)
        for (size_t i = 0; i < count; ++i) {
          const double x = g->slots[q][i];
          g->result[i] = (op == COMM_MAX) ? (x > g->result[i] ? x : g->result[i]) : g->result[i] + x;
        }
      g->arrived = 0;
      g->generation++;
      g->cv.notify_all();
    } else {
      g->cv.wait(lk, [&] { return g->generation != gen; });
    }
    mine = g->result;
  }
  // second barrier: nobody may start the next allreduce (overwriting result)
  // before every rank copied this one
  {
    std::unique_lock<std::mutex> lk(g->m);
    const long long gen = g->generation;
    if (++g->arrived == g->nranks) {
      g->arrived = 0;
      g->generation++;
      g->cv.notify_all();
    } else {
      g->cv.wait(lk, [&] { return g->generation != gen; });
    }
  }
  if (cudaMemcpy(buf, mine.data(), count * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    set_error("local allreduce: device copy failed");
    return MDOT_ECUDA;
  }
  return MDOT_OK;
}

mdot_status comm_allreduce(Comm* cm, double* buf, size_t count, int op, cudaStream_t st) {
  if (!cm || (cm->nranks == 1 && !cm->nccl)) return MDOT_OK;
  if (cm->local) return local_allreduce(cm, buf, count, op, st);
  ncclResult_t r = g_nccl.AllReduce(buf, buf, count, ncclFloat64, op == COMM_MAX ? ncclMax : ncclSum,
                                    (ncclComm_t)cm->nccl, st);
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
  // MDOT_SHARDED_SELFTEST (tests only): a 1-rank NCCL communicator that runs
  // the sharded code path (NCCL calls, graph capture) on a single GPU
  if (nranks > 1 || getenv("MDOT_SHARDED_SELFTEST")) {
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

mdot_status mdot_comm_create_local(const char* group, int32_t nranks, int32_t rank, int32_t device,
                                   mdot_comm** out) {
  if (!group || !out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("bad comm arguments"); return MDOT_EINVAL; }
  if (cudaSetDevice(device) != cudaSuccess) { set_error("cudaSetDevice(%d) failed", device); return MDOT_ECUDA; }
  std::shared_ptr<LocalGroup> g;
  {
    std::lock_guard<std::mutex> lk(g_groups_m);
    auto it = g_groups.find(group);
    if (it == g_groups.end()) {
      g = std::make_shared<LocalGroup>();
      g->nranks = nranks;
      g->slots.resize(nranks);
      g_groups[group] = g;
    } else {
      g = it->second;
      if (g->nranks != nranks) { set_error("local group %s has %d ranks", group, g->nranks); return MDOT_EINVAL; }
    }
    g->refs++;
  }
  Comm* cm = new Comm();
  cm->nranks = nranks;
  cm->rank = rank;
  cm->device = device;
  cm->local = g.get();
  *out = reinterpret_cast<mdot_comm*>(cm);
  return MDOT_OK;
}

mdot_status mdot_comm_destroy(mdot_comm* c) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm) return MDOT_OK;
  if (cm->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)cm->nccl);
  if (cm->local) {
    std::lock_guard<std::mutex> lk(g_groups_m);
    for (auto it = g_groups.begin(); it != g_groups.end(); ++it)
      if (it->second.get() == cm->local) {
        if (--it->second->refs == 0) g_groups.erase(it);
        break;
      }
  }
  delete cm;
  return MDOT_OK;
}

}  // extern "C"


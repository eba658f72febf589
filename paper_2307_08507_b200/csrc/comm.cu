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
  // fused peer exchange, emulated: every rank's exchange block, and the
  // per-launch rendezvous (ranks deposit their arguments; rank 0 launches
  // ONE cooperative kernel over all ranks' groups of CTAs)
  std::vector<void*> peer_blocks;
  std::vector<int64_t> peer_nmax;
  PeerLaunch pend{};
  cudaError_t launch_err = cudaSuccess;
  int peer_err = 0;
};

// Host barrier of the in-process group (same generation counter as the
// allreduce: every rank makes the same sequence of calls).
static void local_barrier(LocalGroup* g) {
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

// ---------------------------------------------------------------------------
// Fused peer exchange (mdot_comm_enable_peer; persist.cu k_persist_peer)
// ---------------------------------------------------------------------------
// slot: [n column totals | kNumScalars row-scalar partials per CTA]
constexpr int kPeerMaxCta = 512;
static int64_t peer_ld(int64_t n) { return (n + (int64_t)kNumScalars * kPeerMaxCta + 31) / 32 * 32; }
// 16-byte self-validating records (persist.cu ll_pack)
static size_t peer_recv_bytes(int nranks, int64_t ld) { return (size_t)2 * nranks * ld * 16; }

// views of rank q's block from this GPU
static void peer_map(PeerState* ps, int q, void* base, int nranks) {
  ps->recv[q] = reinterpret_cast<double*>(base);
  ps->flag[q] = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(base) + peer_recv_bytes(nranks, ps->ld));
}

static void peer_free(Comm* cm) {
  PeerState* ps = cm->peer;
  if (!ps) return;
  for (int q = 0; q < kMaxPeers; ++q)
    if (ps->opened[q]) cudaIpcCloseMemHandle(ps->opened[q]);
  if (ps->block) cudaFree(ps->block);
  delete ps;
  cm->peer = nullptr;
}

int comm_peer_ncta(const Comm* cm, int64_t n, int grid) {
  if (!cm || !cm->peer || n > cm->peer->n_max || grid <= 0) return 0;
  if (getenv("MDOT_NO_PEER")) return 0;
  // the in-process transport runs every rank's CTAs in one co-resident grid
  const int ncta = cm->local ? grid / cm->nranks : grid;
  if (ncta > kPeerMaxCta) return 0;
  return ncta >= 1 ? ncta : 0;
}

mdot_status comm_peer_persist(Comm* cm, const PersistArgs& a, const void* tmap, int ncta, cudaStream_t st) {
  PeerState* ps = cm->peer;
  PeerGroup pg{};
  pg.a = a;
  pg.rank = cm->rank;
  pg.epoch = ps->epoch;
  pg.err = ps->err;
  auto fill_net = [&](PeerNet& net) {
    for (int q = 0; q < cm->nranks; ++q) {
      net.recv[q] = ps->recv[q];
      net.flag[q] = ps->flag[q];
    }
    net.nranks = cm->nranks;
    net.ld = ps->ld;
  };
  int err_h = 0;
  if (!cm->local) {
    // one rank per GPU: this rank's launch; the peers run theirs
    PeerLaunch* L = new PeerLaunch();
    memcpy(L->tmap[0], tmap, 128);
    L->g[0] = pg;
    fill_net(L->net);
    L->groups = 1;
    L->cta_per_group = ncta;
    cudaError_t e = cudaMemsetAsync(ps->err, 0, sizeof(int), st);
    if (e == cudaSuccess) e = launch_persist_peer(*L, st);
    delete L;
    if (e != cudaSuccess) { set_error("peer persistent launch failed: %s", cudaGetErrorString(e)); return MDOT_ECUDA; }
    if (cudaMemcpyAsync(&err_h, ps->err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("peer persistent kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
      return MDOT_ECUDA;
    }
  } else {
    // emulated ranks on one GPU: deposit, rank 0 launches all groups at once
    LocalGroup* g = cm->local;
    if (cudaStreamSynchronize(st) != cudaSuccess) { set_error("stream sync failed"); return MDOT_ECUDA; }
    {
      std::lock_guard<std::mutex> lk(g->m);
      memcpy(g->pend.tmap[cm->rank], tmap, 128);
      g->pend.g[cm->rank] = pg;
    }
    local_barrier(g);
    if (cm->rank == 0) {
      fill_net(g->pend.net);
      g->pend.groups = cm->nranks;
      g->pend.cta_per_group = ncta;
      g->launch_err = cudaSuccess;
      for (int q = 0; q < cm->nranks && g->launch_err == cudaSuccess; ++q)
        g->launch_err = cudaMemsetAsync(g->pend.g[q].err, 0, sizeof(int), st);
      if (g->launch_err == cudaSuccess) g->launch_err = launch_persist_peer(g->pend, st);
      if (g->launch_err == cudaSuccess) g->launch_err = cudaStreamSynchronize(st);
      g->peer_err = 0;
      for (int q = 0; q < cm->nranks && g->launch_err == cudaSuccess; ++q) {
        int e = 0;
        cudaMemcpy(&e, reinterpret_cast<char*>(g->pend.g[q].err), sizeof(int), cudaMemcpyDeviceToHost);
        g->peer_err |= e;
      }
    }
    local_barrier(g);
    if (g->launch_err != cudaSuccess) {
      set_error("peer persistent launch failed: %s", cudaGetErrorString(g->launch_err));
      return MDOT_ECUDA;
    }
    err_h = g->peer_err;
  }
  if (err_h) { set_error("fused peer exchange: a peer flag wait timed out"); return MDOT_ENCCL; }
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

mdot_status mdot_comm_enable_peer(mdot_comm* c, int64_t n_max) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm || n_max < 0) { set_error("bad arguments"); return MDOT_EINVAL; }
  if (n_max == 0) {   // disable (collective: every rank drops its block)
    if (cm->local && cm->peer) local_barrier(cm->local);
    if (cudaSetDevice(cm->device) != cudaSuccess) { set_error("cudaSetDevice failed"); return MDOT_ECUDA; }
    cudaDeviceSynchronize();
    peer_free(cm);
    return MDOT_OK;
  }
  if (cm->nranks > kMaxPeers) { set_error("fused peer exchange supports at most %d ranks", kMaxPeers); return MDOT_EINVAL; }
  if (!cm->local && !cm->nccl) { set_error("single-rank communicator: nothing to exchange"); return MDOT_EINVAL; }
  if (cudaSetDevice(cm->device) != cudaSuccess) { set_error("cudaSetDevice failed"); return MDOT_ECUDA; }
  peer_free(cm);
  PeerState* ps = new PeerState();
  ps->n_max = n_max;
  ps->ld = peer_ld(n_max);
  ps->bytes = peer_recv_bytes(cm->nranks, ps->ld) + 256;
  int ok = 1;
  if (cudaMalloc(&ps->block, ps->bytes) != cudaSuccess || cudaMemset(ps->block, 0, ps->bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    ok = 0;
    cudaGetLastError();
  }
  if (cm->local) {
    LocalGroup* g = cm->local;
    {
      std::lock_guard<std::mutex> lk(g->m);
      if ((int)g->peer_blocks.size() != g->nranks) { g->peer_blocks.assign(g->nranks, nullptr); g->peer_nmax.assign(g->nranks, 0); }
      g->peer_blocks[cm->rank] = ok ? ps->block : nullptr;
      g->peer_nmax[cm->rank] = n_max;
    }
    local_barrier(g);
    for (int q = 0; q < cm->nranks; ++q) {
      if (!g->peer_blocks[q] || g->peer_nmax[q] != n_max) ok = 0;
      else peer_map(ps, q, g->peer_blocks[q], cm->nranks);
    }
    local_barrier(g);
  } else {
    // IPC handles of every rank's block, gathered with an allreduce (sum of
    // zero-padded byte slots), opened with lazy peer access; every rank then
    // agrees on success (min allreduce) so all take the same path
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    std::vector<unsigned char> hs((size_t)cm->nranks * hb, 0);
    cudaIpcMemHandle_t h{};
    if (ok && cudaIpcGetMemHandle(&h, ps->block) != cudaSuccess) { ok = 0; cudaGetLastError(); }
    memcpy(&hs[(size_t)cm->rank * hb], &h, hb);
    unsigned char* dh = nullptr;
    int* dok = nullptr;
    if (cudaMalloc(&dh, hs.size()) != cudaSuccess || cudaMalloc(&dok, sizeof(int)) != cudaSuccess) {
      set_error("peer handle buffer allocation failed");
      if (dh) cudaFree(dh);
      if (dok) cudaFree(dok);
      cm->peer = ps;
      peer_free(cm);
      return MDOT_ENOMEM;
    }
    cudaMemcpy(dh, hs.data(), hs.size(), cudaMemcpyHostToDevice);
    ncclResult_t r = g_nccl.AllReduce(dh, dh, hs.size(), ncclUint8, ncclSum, (ncclComm_t)cm->nccl, 0);
    if (r == ncclSuccess && cudaDeviceSynchronize() == cudaSuccess) {
      cudaMemcpy(hs.data(), dh, hs.size(), cudaMemcpyDeviceToHost);
      for (int q = 0; q < cm->nranks && ok; ++q) {
        if (q == cm->rank) { peer_map(ps, q, ps->block, cm->nranks); continue; }
        void* ptr = nullptr;
        cudaIpcMemHandle_t hq;
        memcpy(&hq, &hs[(size_t)q * hb], hb);
        if (cudaIpcOpenMemHandle(&ptr, hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          ok = 0;
          cudaGetLastError();
          break;
        }
        ps->opened[q] = ptr;
        peer_map(ps, q, ptr, cm->nranks);
      }
    } else {
      ok = 0;
    }
    cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice);
    r = g_nccl.AllReduce(dok, dok, 1, ncclInt32, ncclMin, (ncclComm_t)cm->nccl, 0);
    if (r != ncclSuccess || cudaDeviceSynchronize() != cudaSuccess) ok = 0;
    else cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(dh);
    cudaFree(dok);
  }
  if (!ok) {
    cm->peer = ps;
    peer_free(cm);
    set_error("fused peer exchange unavailable (allocation, IPC or peer access failed on some rank)");
    return MDOT_ECUDA;
  }
  ps->epoch = ps->flag[cm->rank] + kMaxPeers;
  ps->err = reinterpret_cast<int*>(ps->flag[cm->rank] + kMaxPeers + 1);
  cm->peer = ps;
  return MDOT_OK;
}

mdot_status mdot_comm_destroy(mdot_comm* c) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm) return MDOT_OK;
  if (cm->local && cm->peer) local_barrier(cm->local);   // no rank frees a block another may still map
  peer_free(cm);
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


// paper_2307_08507_b200/csrc/solver.cu -- host control of the MDOT-PNCG hot
// path and the C ABI of include/mdot.h.
//
// Control flow:
//   mdot_solve  -> setup (log r, log c, anchors)                 a1
//               -> for each MD step t (Alg. 1)  a2
//                    warm start, project (PNCG / Sinkhorn / NCG)  a3-a8
//                    U += u, V += v, gauge centring               a9
//               -> rounding + cost                 a10
// Every O(n^2) pass runs in kernels.cu; this file holds only O(1) scalar
// decisions (line-search logic, beta, stop tests) on values the finalize
// kernel publishes to mapped pinned memory.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdlib.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <nvtx3/nvToolsExt.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/mdot.h"
#include "internal.cuh"
#include "comm.h"
#include "solver.h"

namespace mdot {

// NVTX ranges (header-only NVTX v3: no library to link; a profiler that
// injects itself -- nsys, ncu --nvtx -- sees the solve, each MD step (its
// projection) and the rounding as named ranges; otherwise each is a no-op call)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, int t, double gbar) {
    char buf[96];
    snprintf(buf, sizeof(buf), fmt, t, gbar);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

static double now_s() {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, __LINE__, \
                cudaGetErrorString(e_));                                             \
      return e_ == cudaErrorMemoryAllocation ? MDOT_ENOMEM : MDOT_ECUDA;             \
    }                                                                                \
  } while (0)

// launch + count (Workspace member context)
#define CKL(call)        \
  do {                   \
    ++launches;          \
    CK(call);            \
  } while (0)

#define CKS(call)                        \
  do {                                   \
    mdot_status s_ = (call);             \
    if (s_ != MDOT_OK) return s_;        \
  } while (0)

// ---------------------------------------------------------------------------
// Workspace
// ---------------------------------------------------------------------------
bool Workspace::sharded() const { return comm != nullptr && (comm->nranks > 1 || comm->nccl != nullptr); }

// Keep freed stream-ordered allocations in the device pool (no release at
// every synchronize): repeated solves reuse the workspace / staging memory.
static void retain_mempool() {
  static int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

// Mapped pinned scalar blocks are recycled across calls: cudaHostAlloc /
// cudaFreeHost cost milliseconds (and cudaFreeHost synchronizes the device),
// which showed up as 30-50 ms outliers in repeated solves.
static std::mutex g_host_mu;
static std::vector<double*> g_host_free;

static double* host_block_get() {
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    if (!g_host_free.empty()) {
      double* b = g_host_free.back();
      g_host_free.pop_back();
      return b;
    }
  }
  void* b = nullptr;
  if (cudaHostAlloc(&b, 256 * sizeof(double), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return static_cast<double*>(b);
}

static void host_block_put(double* b) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  g_host_free.push_back(b);
}

mdot_status Workspace::alloc(cudaStream_t stream, int64_t n_, int64_t nrows_) {
  retain_mempool();
  st = stream;
  n = n_;
  nrows = nrows_;
  const int64_t items = nrows + n;
  // evaluation grid: 256-column tiles, row tiles sized for >= ~4 CTAs per SM
  eval.n = n;
  eval.nrows = nrows;
  eval.n_col_tiles = (int)((n + kTileN - 1) / kTileN);
  // Row tile height: minimise the busiest CTA's work over the 2 x 148
  // persistent CTAs, (tiles per CTA) x (rows per tile + ~128 rows of per-tile
  // cost: parameter loads, column write-out, two CTA barriers; fitted).  n = 16384:
  // 512; config 3 (n = 4096): 256, one tile per CTA (K1 17.7 -> 14.4 us vs
  // two 128-row tiles; profiles/r01_cfg3_tile_grid.txt).
  int tile_m = 512;
  {
    // CTAs that will share the pass: 2 per SM (K1 and the persistent kernel),
    // divided among the ranks when one GPU emulates several (in-process
    // transport with the fused peer exchange)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t ctas = 2 * (int64_t)sms;
    if (comm && comm->local && comm->peer && comm->nranks > 1) ctas = std::max<int64_t>(1, ctas / comm->nranks);
    int64_t best = INT64_MAX;
    for (int tm = 512; tm >= 32; tm /= 2) {
      const int64_t tiles = (int64_t)eval.n_col_tiles * ((nrows + tm - 1) / tm);
      const int64_t cost = ((tiles + ctas - 1) / ctas) * (std::min<int64_t>(tm, nrows) + 128);
      if (cost < best) { best = cost; tile_m = tm; }
    }
  }
  if (const char* tm_env = getenv("MDOT_TILE_M")) {   // A/B experiments only
    const int v = atoi(tm_env);
    if (v >= 32 && v <= 512 && (v & (v - 1)) == 0) tile_m = v;
  }
  eval.tile_m = tile_m;
  eval.n_row_tiles = (int)((nrows + tile_m - 1) / tile_m);
  chunks = (int)std::max<int64_t>(1, std::min<int64_t>(nrows, (4 * 148 + (n + 255) / 256 - 1) / ((n + 255) / 256)));
  const int64_t fin_blocks = std::max<int64_t>((items * 8 + 255) / 256 + 8, 1024);   // k_finalize / persistent CTAs

  size_t dbl = 0;
  guards.clear();
  auto take = [&](int64_t k) {
    size_t o = dbl;
    dbl += (size_t)((k + 31) / 32 * 32);
#ifdef MDOT_CHECKED
    guards.push_back(dbl);   // a guard band after every sub-buffer
    dbl += kGuardDbl;
#endif
    return o;
  };
  size_t o_r = take(nrows), o_c = take(n), o_logr = take(nrows), o_logc = take(n);
  size_t o_rho = take(nrows), o_sig = take(n);
  size_t o_U = take(nrows), o_V = take(n), o_u = take(nrows), o_v = take(n), o_tu = take(nrows), o_tv = take(n);
  size_t o_A = take(nrows), o_B = take(n);
  size_t o_p = take(items), o_pp = take(items);
  size_t o_m[2][4];
  for (int b = 0; b < 2; ++b)
    for (int q = 0; q < 4; ++q) o_m[b][q] = take(items);
  size_t o_rowpart = take((int64_t)eval.n_col_tiles * nrows);
  size_t o_colpart = take((int64_t)eval.n_row_tiles * n);
  size_t o_colm = take((int64_t)chunks * n), o_cols = take((int64_t)chunks * n);
  size_t o_lr = take(nrows);
  size_t o_blk = take(fin_blocks * kNumScalars);
  size_t o_scal = take(kNumScalars * 2);
  size_t o_aux = take(8 * items);
  size_t o_tot = take(items + 32);
  size_t o_ctrl = take((int64_t)((sizeof(CtrlState) + 7) / 8));
  size_t o_nrm = take((items + 1) / 2);   // items floats
  size_t o_bp[2] = {take(items), take(items)};
  const int64_t nrows_p = (nrows + 127) / 128 * 128, n_p = (n + 255) / 256 * 256;
  // 32 floats per row; A one chunk longer: tiles shorter than 128 rows run
  // their last chunk's MMA over up to 127 rows past the padded end
  size_t o_sopA = take((nrows_p + 128) * 16), o_sopB = take(n_p * 16);
  size_t o_scr = take(6);                 // smin[2], scount[2], ymax
  const size_t tickets = (size_t)eval.n_row_tiles + eval.n_col_tiles + 64;
  size_t bytes = dbl * sizeof(double) + (size_t)(items + 64) * sizeof(float4) + 256 + tickets * 4;
#ifdef MDOT_CHECKED
  const size_t tail_guard = bytes;
  bytes += kGuardDbl * sizeof(double);
#endif
  cudaError_t e = cudaMallocAsync(&base, bytes, st);
  if (e != cudaSuccess) {
    set_error("workspace allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    return MDOT_ENOMEM;
  }
  double* D = reinterpret_cast<double*>(base);
#ifdef MDOT_CHECKED
  guards.push_back(tail_guard / sizeof(double));
  for (size_t g : guards) CK(cudaMemsetAsync(D + g, 0xA5, kGuardDbl * sizeof(double), st));
#endif
  r = D + o_r; c = D + o_c; logr = D + o_logr; logc = D + o_logc; rho_r = D + o_rho; sig_c = D + o_sig;
  U = D + o_U; V = D + o_V; u = D + o_u; v = D + o_v; tu = D + o_tu; tv = D + o_tv;
  A = D + o_A; B = D + o_B; p = D + o_p; pprev = D + o_pp;
  for (int b = 0; b < 2; ++b) {
    mg[b].lm = D + o_m[b][0]; mg[b].m = D + o_m[b][1]; mg[b].s = D + o_m[b][2]; mg[b].g = D + o_m[b][3];
    mg[b].bp = D + o_bp[b];
  }
  sopA = reinterpret_cast<float*>(D + o_sopA);
  sopB = reinterpret_cast<float*>(D + o_sopB);
  smin = reinterpret_cast<unsigned long long*>(D + o_scr);
  scount = smin + 2;
  sop_ymax = D + o_scr + 4;
  CK(cudaMemsetAsync(smin, 0xFF, 2 * sizeof(unsigned long long), st));   // NaN keys: keep everything
  CK(cudaMemsetAsync(scount, 0, 2 * sizeof(unsigned long long), st));
  cur = &mg[0];
  trial = &mg[1];
  rowpart = D + o_rowpart; colpart = D + o_colpart; colm = D + o_colm; cols = D + o_cols; lr_ex = D + o_lr;
  blockpart = D + o_blk; scal_dev = D + o_scal; aux = D + o_aux;
  ctrl = reinterpret_cast<CtrlState*>(D + o_ctrl);
  nrm = reinterpret_cast<float*>(D + o_nrm);
  tot.coltot = D + o_tot;   // sharded: [column totals | row scalars] allreduce buffer
  float4* F4 = reinterpret_cast<float4*>(reinterpret_cast<char*>(base) + dbl * sizeof(double));
  F4 = reinterpret_cast<float4*>((reinterpret_cast<uintptr_t>(F4) + 15) & ~uintptr_t(15));
  rowp = F4;
  colp = F4 + nrows;
  ticket_flag = reinterpret_cast<unsigned int*>(colp + n + 8);
  CK(cudaMemsetAsync(ticket_flag, 0, 64 + tickets * 4, st));
  ticket = ticket_flag;
  flag = reinterpret_cast<int*>(ticket_flag + 4);
  pers_bar = ticket_flag + 8;   // [2] barrier + [2 x u64] K1 timing (16-byte aligned)
  scal_host = host_block_get();
  if (!scal_host) {
    set_error("mapped host allocation failed");
    return MDOT_ENOMEM;
  }
  CK(cudaHostGetDevicePointer((void**)&scal_host_dev, scal_host, 0));
  memset(scal_host, 0, 256 * sizeof(double));
  done_host = reinterpret_cast<int*>(scal_host + 64);
  ran_host = reinterpret_cast<int*>(scal_host + 72);
  eval.rowp = rowp;
  eval.colp = colp;
  eval.rowpart = rowpart;
  eval.colpart = colpart;
  return MDOT_OK;
}

void Workspace::release() {
  if (gexec) cudaGraphExecDestroy(gexec);
  gexec = nullptr;
  if (cap_stream) cudaStreamDestroy(cap_stream);
  cap_stream = nullptr;
  if (gev_made)
    for (auto& e : gev)
      if (e) cudaEventDestroy(e);
  gev_made = false;
  if (base) cudaFreeAsync(base, st);
  base = nullptr;
  if (trace_dev) cudaFreeAsync(trace_dev, st);
  trace_dev = nullptr;
  trace_len_dev = nullptr;
  if (scal_host) {
    cudaStreamSynchronize(st);   // the block may still be written by queued kernels
    host_block_put(scal_host);
  }
  scal_host = nullptr;
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  ev0 = ev1 = nullptr;
}

// ---------------------------------------------------------------------------
// One evaluation at the parameters last written by prep: fast fp32 kernel,
// finalize, and (if the range guard fires) the exact fp64 re-evaluation.
// ---------------------------------------------------------------------------
mdot_status Workspace::launch_eval() {
  if (time_kernels) CK(cudaEventRecord(ev0, st));
  if (use_tma) {
    CKL(launch_eval_tma(tmap, eval, tma_grid, st));
  } else {
    CKL(launch_eval_fast(eval, kind_fast, st));
  }
  if (time_kernels) CK(cudaEventRecord(ev1, st));
  return MDOT_OK;
}

// NC2 trial: phi'(alpha) = <p, m(alpha)> - <p, (r, c)> and the
// mass are linear in the marginals, so each rank's partial totals contribute
// additively; 4 scalars are reduced over the ranks (both
// teams on a 2-D grid) and the partials stay in place for the completion of
// an accepted trial (evaluate with skip_k1).
mdot_status Workspace::nc2_trial(double* q) {
  evals++;
  CKS(launch_eval());
  CKL(launch_nc2_trial(rowpart, eval.n_col_tiles, colpart, eval.n_row_tiles, nrows, n, rho_r, sig_c, p, flag,
                       blockpart, ticket, scal_dev, st));
  CKS(comm_allreduce(comm, scal_dev, 4, COMM_SUM, st));
  if (two_d()) CKS(comm_allreduce(comm_row, scal_dev, 4, COMM_SUM, st));
  CK(cudaMemcpyAsync(q, scal_dev, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (time_kernels) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    kernel_ms += ms;
    kernel_launches++;
  }
  return MDOT_OK;
}

mdot_status Workspace::nc2_prc(double* prc) {
  // rows: distinct over the ranks of `comm`; columns: replicated (1-D) or
  // distinct over the row team (2-D)
  const double* xr = p;
  const double* yr = r;
  CKL(launch_dots(nrows, 1, &xr, &yr, blockpart, ticket, scal_dev, scal_host_dev, st));
  CKS(comm_allreduce(comm, scal_dev, 1, COMM_SUM, st));
  double a = 0.0, b = 0.0;
  CK(cudaMemcpyAsync(&a, scal_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double* xc = p + nrows;
  const double* yc = c;
  CKL(launch_dots(n, 1, &xc, &yc, blockpart, ticket, scal_dev, scal_host_dev, st));
  if (two_d()) CKS(comm_allreduce(comm_row, scal_dev, 1, COMM_SUM, st));
  CK(cudaMemcpyAsync(&b, scal_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *prc = a + b;
  return MDOT_OK;
}

mdot_status Workspace::evaluate(Marg* out, const double* gcur, const double* pcur, double* sc, bool skip_k1) {
  FinalizeArgs f{};
  f.n = n; f.nrows = nrows;
  f.rho_r = rho_r; f.sig_c = sig_c;
  f.r = r; f.c = c; f.logr = logr; f.logc = logc;
  f.gcur = gcur; f.pcur = pcur;
  f.lm = out->lm; f.m = out->m; f.s = out->s; f.g = out->g;
  f.blockpart = blockpart; f.ticket = ticket;
  f.scalars_dev = scal_dev; f.scalars_host = scal_host_dev;
  f.prep_flag = flag;
  f.jacobi = jacobi;
  const bool shard = sharded();
  if (!skip_k1) evals++;
  if (!exact_mode) {
    if (!skip_k1) CKS(launch_eval());
    f.from_partials = 1;
    f.rowpart = rowpart; f.n_col_tiles = eval.n_col_tiles;
    f.colpart = colpart; f.n_row_tiles = eval.n_row_tiles;
    if (two_d()) {
      // 2-D block: row totals are partial over this rank's columns, column
      // totals over its rows.  Allreduce each over the ranks holding the other
      // parts (row_comm / col_comm), finalize both sides locally, then sum
      // each side's 16 scalars over the ranks holding the OTHER blocks of that
      // side (row items are replicated across comm_row, columns across comm).
      double* colbuf = tot.coltot;                   // [n column totals | 16 column scalars]
      double* rowbuf = tot.coltot + n + kNumScalars; // [nrows row totals | 16 row scalars]
      CKL(launch_reduce_colpart(colpart, eval.n_row_tiles, n, colbuf, st));
      CKL(launch_reduce_colpart(rowpart, eval.n_col_tiles, nrows, rowbuf, st));   // [tc][row]: same layout
      CKS(comm_allreduce(comm, colbuf, (size_t)n, COMM_SUM, st));
      CKS(comm_allreduce(comm_row, rowbuf, (size_t)nrows, COMM_SUM, st));
      FinalizeArgs fr = f;
      fr.rowtot = rowbuf;
      fr.item_begin = 0; fr.item_end = nrows;
      fr.scalars_dev = rowbuf + nrows; fr.scalars_host = nullptr;
      CKL(launch_finalize(fr, st));
      FinalizeArgs fc = f;
      fc.coltot = colbuf;
      fc.item_begin = nrows; fc.item_end = nrows + n;
      fc.scalars_dev = colbuf + n; fc.scalars_host = nullptr;
      fc.prep_flag = nullptr;
      CKL(launch_finalize(fc, st));
      CKS(comm_allreduce(comm, rowbuf + nrows, kNumScalars, COMM_SUM, st));
      CKS(comm_allreduce(comm_row, colbuf + n, kNumScalars, COMM_SUM, st));
      double h[2][kNumScalars];
      CK(cudaMemcpyAsync(h[0], rowbuf + nrows, sizeof(h[0]), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h[1], colbuf + n, sizeof(h[1]), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int q = 0; q < kNumScalars; ++q) scal_host[q] = h[0][q] + h[1][q];
    } else if (!shard) {
      CKL(launch_finalize(f, st));
    } else {
      // rows are complete locally; columns are partial over this rank's rows.
      // Row scalars go into the tail of the column buffer so ONE allreduce
      // carries [column totals | row scalars].
      double* colbuf = tot.coltot;
      CKL(launch_reduce_colpart(colpart, eval.n_row_tiles, n, colbuf, st));
      FinalizeArgs fr = f;
      fr.item_begin = 0; fr.item_end = nrows;
      fr.scalars_dev = colbuf + n; fr.scalars_host = nullptr;
      CKL(launch_finalize(fr, st));
      CKS(comm_allreduce(comm, colbuf, (size_t)n + kNumScalars, COMM_SUM, st));
      FinalizeArgs fc = f;
      fc.from_partials = 1;
      fc.coltot = colbuf;
      fc.item_begin = nrows; fc.item_end = nrows + n;
      fc.add_in = colbuf + n;
      fc.prep_flag = nullptr;
      CKL(launch_finalize(fc, st));
    }
    CK(cudaStreamSynchronize(st));
    if (time_kernels && !skip_k1) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev0, ev1));
      kernel_ms += ms;
      kernel_launches++;
    }
    memcpy(sc, scal_host, kNumScalars * sizeof(double));
    if (sc[SC_BAD] == 0.0) return MDOT_OK;
    fallbacks++;
  }
  ExactArgs x{};
  x.C = Cdev; x.ldc = n; x.c_f64 = c_f64;
  x.X = Xdev; x.Y = Ydev; x.d = d; x.scale = scale; x.otf = otf;
  x.n = n; x.nrows = nrows;
  x.A = A; x.B = B; x.gbar = gbar;
  x.lr = lr_ex; x.colm = colm; x.cols = cols; x.chunks = chunks;
  CKL(launch_eval_exact(x, st));
  f.from_partials = 0;
  f.lr_in = lr_ex; f.colm = colm; f.cols = cols; f.chunks = chunks;
  f.prep_flag = nullptr;
  if (two_d()) {
    // 2-D exact: column (max, sum) pairs combined over the column team (as
    // the 1-D path), row log-sums of this block's columns combined over the
    // row team the same way: M = max-allreduce, S = sum-allreduce of
    // e^(l - M), l = M + log S; then both sides finalize and their scalars
    // are summed over the other team (as the fp32-entry branch above)
    double* Mloc = aux;
    double* Mg = aux + n;
    double* Sg = aux + 2 * n;
    double* Mr = aux + 3 * n;
    double* Sr = Mr + nrows;
    CKL(launch_exact_colcombine(colm, cols, chunks, n, Mloc, Sg, st));
    CK(cudaMemcpyAsync(Mg, Mloc, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CKS(comm_allreduce(comm, Mg, (size_t)n, COMM_MAX, st));
    CKL(launch_rescale_to_max(n, Mloc, Mg, Sg, st));
    CKS(comm_allreduce(comm, Sg, (size_t)n, COMM_SUM, st));
    CK(cudaMemcpyAsync(Mr, lr_ex, sizeof(double) * nrows, cudaMemcpyDeviceToDevice, st));
    CKS(comm_allreduce(comm_row, Mr, (size_t)nrows, COMM_MAX, st));
    CKL(launch_fill(nrows, 1.0, Sr, st));
    CKL(launch_rescale_to_max(nrows, lr_ex, Mr, Sr, st));
    CKS(comm_allreduce(comm_row, Sr, (size_t)nrows, COMM_SUM, st));
    CKL(launch_lse_finish(nrows, Mr, Sr, lr_ex, st));
    double* colsc = tot.coltot + n;
    double* rowsc = tot.coltot + n + kNumScalars + nrows;
    FinalizeArgs fr = f;
    fr.item_begin = 0; fr.item_end = nrows;
    fr.scalars_dev = rowsc; fr.scalars_host = nullptr;
    CKL(launch_finalize(fr, st));
    FinalizeArgs fc = f;
    fc.colm = Mg; fc.cols = Sg; fc.chunks = 1;
    fc.item_begin = nrows; fc.item_end = nrows + n;
    fc.scalars_dev = colsc; fc.scalars_host = nullptr;
    CKL(launch_finalize(fc, st));
    CKS(comm_allreduce(comm, rowsc, kNumScalars, COMM_SUM, st));
    CKS(comm_allreduce(comm_row, colsc, kNumScalars, COMM_SUM, st));
    double h[2][kNumScalars];
    CK(cudaMemcpyAsync(h[0], rowsc, sizeof(h[0]), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h[1], colsc, sizeof(h[1]), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int q = 0; q < kNumScalars; ++q) sc[q] = h[0][q] + h[1][q];
    if (sc[SC_BAD] != 0.0) {
      set_error("non-finite marginals at gbar=%g on the exact fp64 evaluator (2-D)", gbar);
      return MDOT_EINSTABLE;
    }
    return MDOT_OK;
  }
  if (!shard) {
    CKL(launch_finalize(f, st));
  } else {
    // columns: local (max, sum) -> global max -> rescale -> global sum
    double* Mloc = aux;
    double* Mg = aux + n;
    double* Sg = aux + 2 * n;   // followed by kNumScalars row scalars
    CKL(launch_exact_colcombine(colm, cols, chunks, n, Mloc, Sg, st));
    CK(cudaMemcpyAsync(Mg, Mloc, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    CKS(comm_allreduce(comm, Mg, (size_t)n, COMM_MAX, st));
    CKL(launch_rescale_to_max(n, Mloc, Mg, Sg, st));
    FinalizeArgs fr = f;
    fr.item_begin = 0; fr.item_end = nrows;
    fr.scalars_dev = Sg + n; fr.scalars_host = nullptr;
    CKL(launch_finalize(fr, st));
    CKS(comm_allreduce(comm, Sg, (size_t)n + kNumScalars, COMM_SUM, st));
    FinalizeArgs fc = f;
    fc.colm = Mg; fc.cols = Sg; fc.chunks = 1;
    fc.item_begin = nrows; fc.item_end = nrows + n;
    fc.add_in = Sg + n;
    CKL(launch_finalize(fc, st));
  }
  CK(cudaStreamSynchronize(st));
  memcpy(sc, scal_host, kNumScalars * sizeof(double));
  if (sc[SC_BAD] != 0.0) {
    set_error("non-finite marginals at gbar=%g on the exact fp64 evaluator", gbar);
    return MDOT_EINSTABLE;
  }
  return MDOT_OK;
}

mdot_status Workspace::prep(int mode, double alpha, double beta, const double* s_dir,
                            const double* Ain, const double* Bin) {
  PrepArgs a{};
  a.n = n; a.nrows = nrows; a.mode = mode; a.alpha = alpha; a.beta = beta;
  a.U = U; a.V = V; a.u = u; a.v = v; a.tu = tu; a.tv = tv;
  a.p = p; a.s = s_dir; a.pprev = pprev; a.lm = cur->lm;
  a.logr = logr; a.logc = logc; a.rho_r = rho_r; a.sig_c = sig_c;
  a.Ain = Ain; a.Bin = Bin; a.Aout = A; a.Bout = B;
  a.rowp = rowp; a.colp = colp; a.flag = flag; a.nrm = use_nrm ? nrm : nullptr;
  CKL(launch_prep(a, st));
  return MDOT_OK;
}

void Workspace::set_gamma(double gb) {
  gbar = gb;
  const double g2 = gb * 1.4426950408889634;
  const float gh = (float)g2;
  eval.gh = gh;
  eval.gl = (float)(g2 - (double)gh);
}

// ---------------------------------------------------------------------------
// Projections
// ---------------------------------------------------------------------------
static inline double stopval(const double* sc, int stop_rho) { return stop_rho ? sc[SC_RHO] : sc[SC_L1]; }

// Sinkhorn, Alg. 3; one fused evaluation per half-step.
mdot_status project_sinkhorn(Workspace& w, const mdot_options& o, int t, mdot_result* res) {
  res->control_path = 0;
  double sc[kNumScalars];
  CKS(w.prep(PREP_CUR, 0, 0, nullptr, nullptr, nullptr));
  CKS(w.evaluate(w.cur, nullptr, nullptr, sc));
  if (t >= 1 && t <= 64) { res->rho0[t - 1] = sc[SC_RHO]; res->l10[t - 1] = sc[SC_L1]; }
  int64_t k = 0;
  mdot_status st = MDOT_OK;
  while (stopval(sc, o.stop) > o.eps) {
    if (w.evals >= o.max_evals) { st = MDOT_ENOCONV; break; }
    ++k;
    if (w.trace_cap) {
      mdot_trace_rec q{};
      q.t = t; q.k = (int32_t)k; q.l1 = sc[SC_L1]; q.rho = sc[SC_RHO]; q.alpha = 1.0;
      w.trace_add(q);
    }
    CKS(w.prep((k % 2 == 1) ? PREP_SK_ROW : PREP_SK_COL, 0, 0, nullptr, nullptr, nullptr));
    CKS(w.evaluate(w.cur, nullptr, nullptr, sc));
    res->iterations++;
    if (t >= 1 && t <= 64) res->iters_step[t - 1]++;
  }
  res->l1_final = sc[SC_L1];
  res->rho_final = sc[SC_RHO];
  w.last_mass = sc[SC_MASS];
  return st;
}

// PNCG, Alg. 2 with the line search of Appx. C
// and readings Z5-Z10.
mdot_status project_pncg(Workspace& w, const mdot_options& o, int t, mdot_result* res) {
  res->control_path = 0;
  const bool ncg = o.projector == MDOT_PROJ_NCG;
  double sc[kNumScalars], ts[kNumScalars];
  CKS(w.prep(PREP_CUR, 0, 0, nullptr, nullptr, nullptr));
  CKS(w.evaluate(w.cur, nullptr, nullptr, sc));
  if (t >= 1 && t <= 64) { res->rho0[t - 1] = sc[SC_RHO]; res->l10[t - 1] = sc[SC_L1]; }
  double mass = sc[SC_MASS];
  double S_sg = sc[SC_SG], S_gcs = 0, S_pcg = 0, S_gg = sc[SC_GG], S_gcg = 0;
  double dphi0_prev = 0, sg_prev = 0, gg_prev = 0;
  double alpha_prev = 1.0;
  const double c1 = o.c1, c2 = o.c2;
  const double noise = ls_noise(w.exact_mode, w.gbar);   // decrease-safeguard tolerance (Z9)
  int64_t k = 0;
  mdot_status st = MDOT_OK;
  while (stopval(sc, o.stop) > o.eps) {
    if (w.evals >= o.max_evals) { st = MDOT_ENOCONV; break; }
    ++k;
    // beta_k (Z6; FR / PR+ variants) from scalars of the current iterate
    double beta = 0.0;
    if (k > 1) beta = beta_k(ncg, o.beta, S_sg, S_gcs, S_gg, S_gcg, dphi0_prev, sg_prev, gg_prev);
    const double* dir = ncg ? w.cur->g : w.cur->s;
    const double dg = ncg ? S_gg : S_sg;            // <dir, g>
    double dphi0 = -dg + beta * S_pcg;              // <p, g> with p = -dir + beta p_prev
    int reset = 0;
    if (!(dphi0 < 0.0)) { beta = 0.0; dphi0 = -dg; res->resets++; reset = 1; }   // Z5
    double alpha = (k == 1) ? 1.0 : std::min(4.0, std::max(0.25, alpha_prev));  // Z8
    CKS(w.prep(PREP_NEWDIR | PREP_TRIAL, alpha, beta, dir, nullptr, nullptr));
    int accepted = 0, attempt = 0, trials = 0;
    double dphi_a = 0, dval = 0;
    // NC2: <p, (r, c)> once per direction; trials exchange 4 scalars
    double prc = 0.0;
    if (w.nc2) CKS(w.nc2_prc(&prc));
    while (!accepted && attempt < 2) {
      double lo = 0.0, dlo = dphi0, hi = 0.0, dhi = 0.0;
      int have_hi = 0, doublings = 0;
      for (int tr = 0; tr < o.ls_max_trials; ++tr) {
        if (tr > 0) CKS(w.prep(PREP_TRIAL, alpha, 0, nullptr, nullptr, nullptr));
        bool partial = false;   // NC2 trial: only the line-search scalars are known
        if (w.nc2) {
          double q[4];
          CKS(w.nc2_trial(q));
          if (q[3] == 0.0 && std::isfinite(q[0] + q[1] + q[2])) {
            partial = true;
            dphi_a = q[0] + q[2] - prc;                            // phi'(alpha) = <p, m(alpha)> - <p, (r, c)>
            dval = (q[1] - mass) - alpha * prc;
          } else {
            w.evals--;                                             // re-done in full below
          }
        }
        if (!partial) {
          CKS(w.evaluate(w.trial, w.cur->g, w.p, ts));
          dphi_a = ts[SC_PCG];                                     // phi'(alpha)
          dval = (ts[SC_MASS] - mass) - alpha * ts[SC_PRC];
        }
        res->ls_evaluations++;
        trials++;
        int wolfe = ((2.0 * c1 - 1.0) * dphi0 >= dphi_a) && (dphi_a >= c2 * dphi0);
        int decrease = dval <= noise * std::max(1.0, mass);
        if (wolfe && decrease && partial) {
          // complete the accepted trial from its kept partials (the vector
          // exchange + finalize); re-test with the full scalars, which may
          // come from the exact evaluator if the range guard fires
          CKS(w.evaluate(w.trial, w.cur->g, w.p, ts, true));
          dphi_a = ts[SC_PCG];
          dval = (ts[SC_MASS] - mass) - alpha * ts[SC_PRC];
          wolfe = ((2.0 * c1 - 1.0) * dphi0 >= dphi_a) && (dphi_a >= c2 * dphi0);
          decrease = dval <= noise * std::max(1.0, mass);
        }
        if (wolfe && decrease) { accepted = 1; break; }
        if (dphi_a < 0.0 && decrease) { lo = alpha; dlo = dphi_a; }
        else { hi = alpha; dhi = dphi_a; have_hi = 1; }
        if (!have_hi) {
          if (++doublings > 60) break;
          alpha *= 2.0;
        } else if (dhi > dlo) {
          const double a_sec = (lo * dhi - hi * dlo) / (dhi - dlo);
          alpha = 0.5 * a_sec + 0.5 * (hi + lo) / 2.0;
        } else {
          alpha = 0.5 * (lo + hi);
        }
      }
      if (accepted) break;
      attempt++;                                                      // Z10
      res->ls_restarts++;
      dphi0 = -dg;
      alpha = 1.0;
      beta = 0.0;
      reset = 1;
      if (attempt < 2) {
        CKS(w.prep(PREP_NEWDIR | PREP_TRIAL, alpha, 0.0, dir, nullptr, nullptr));
        if (w.nc2) CKS(w.nc2_prc(&prc));   // the restart direction p = -s
      }
    }
    if (!accepted) {
      set_error("line search failed twice at MD step %d, iteration %lld", t, (long long)k);
      st = MDOT_ELINESEARCH;
      break;
    }
    if (w.trace_cap) {
      mdot_trace_rec q{};
      q.t = t; q.k = (int32_t)k; q.l1 = sc[SC_L1]; q.rho = sc[SC_RHO];
      q.alpha = alpha; q.dphi0 = dphi0; q.dphi_alpha = dphi_a; q.dphi_value = dval;
      q.trials = trials; q.reset = reset; q.beta = beta; q.gs = S_sg;
      w.trace_add(q);
    }
    // accept (Alg. 2 lines 11-13): the trial becomes the iterate
    std::swap(w.u, w.tu);
    std::swap(w.v, w.tv);
    std::swap(w.cur, w.trial);
    std::swap(w.p, w.pprev);
    dphi0_prev = dphi0;
    sg_prev = S_sg;
    gg_prev = S_gg;
    S_sg = ts[SC_SG]; S_gcs = ts[SC_GCS]; S_pcg = ts[SC_PCG]; S_gg = ts[SC_GG]; S_gcg = ts[SC_GCG];
    mass = ts[SC_MASS];
    memcpy(sc, ts, sizeof(sc));
    alpha_prev = alpha;
    res->iterations++;
    if (t >= 1 && t <= 64) res->iters_step[t - 1]++;
  }
  res->l1_final = sc[SC_L1];
  res->rho_final = sc[SC_RHO];
  w.last_mass = mass;
  return st;
}

// ---------------------------------------------------------------------------
// Device-resident control: graphs of [k_ctrl, k_prep, eval, k_finalize] slots
// ---------------------------------------------------------------------------
// done_host / ran_host live in mapped pinned memory; the device pointers
// handed to kernels are their device aliases.
static int* dev_alias(int* h) {
  void* d = nullptr;
  cudaHostGetDevicePointer(&d, h, 0);
  return reinterpret_cast<int*>(d);
}

mdot_status Workspace::launch_slot_body(cudaStream_t s, int slot, bool timed, bool with_ctrl) {
  // timed slot events: gev[0] ctrl gev[1] prep gev[2] K1 gev[3] finalize gev[4]
  if (timed) CK(cudaEventRecordWithFlags(gev[0], s, cudaEventRecordExternal));
  if (with_ctrl) {
    int* dh = nullptr;
    int* rh = nullptr;
    cudaHostGetDevicePointer((void**)&dh, done_host, 0);
    cudaHostGetDevicePointer((void**)&rh, ran_host, 0);
    CKL(launch_ctrl(ctrl, slot, dh, rh, s));
  }
  if (timed) CK(cudaEventRecordWithFlags(gev[1], s, cudaEventRecordExternal));
  PrepArgs a{};
  a.n = n; a.nrows = nrows; a.mode = 0;
  a.U = U; a.V = V; a.u = u; a.v = v; a.tu = tu; a.tv = tv;
  a.p = p; a.s = cur->s; a.pprev = pprev; a.lm = cur->lm;
  a.logr = logr; a.logc = logc; a.rho_r = rho_r; a.sig_c = sig_c;
  a.Aout = A; a.Bout = B;
  a.rowp = rowp; a.colp = colp; a.flag = flag; a.nrm = use_nrm ? nrm : nullptr;
  a.ctrl = ctrl;
  a.cur_lm = cur->lm; a.cur_m = cur->m; a.cur_s = cur->s; a.cur_g = cur->g;
  a.tr_lm = trial->lm; a.tr_m = trial->m; a.tr_s = trial->s; a.tr_g = trial->g;
  const bool scr = screen_cap && !exact_mode;   // K2s bounds (every slot, so cur->bp stays current)
  if (scr) {
    a.cur_bp = cur->bp; a.tr_bp = trial->bp; a.sopA = sopA; a.sopB = sopB; a.smin = smin;
    a.X = Xdev; a.Y = Ydev; a.d = d; a.scale = scale; a.sop_ymax = sop_ymax; a.screen_T = screen_T;
  }
  CKL(launch_prep(a, s));
  FinalizeArgs f{};
  f.n = n; f.nrows = nrows;
  f.rho_r = rho_r; f.sig_c = sig_c;
  f.r = r; f.c = c; f.logr = logr; f.logc = logc;
  f.gcur = cur->g; f.pcur = p;
  f.lm = trial->lm; f.m = trial->m; f.s = trial->s; f.g = trial->g;
  f.blockpart = blockpart; f.ticket = ticket;
  f.scalars_dev = ctrl->sc; f.scalars_host = nullptr;
  f.prep_flag = flag;
  f.jacobi = jacobi;
  f.done = &ctrl->done;
  if (scr) f.smin_reset = smin;
  if (timed) CK(cudaEventRecordWithFlags(gev[2], s, cudaEventRecordExternal));
  if (!exact_mode) {
    EvalArgs e = eval;
    e.gpair = ctrl->gpair;
    e.done = &ctrl->done;
    if (use_tma) {
      CKL(launch_eval_tma(tmap, e, tma_grid, s));
    } else if (scr && screen_now && with_ctrl) {
      // K2s: the slot's evaluation against the accepted iterate's bounds (the
      // projection's initial evaluation, with_ctrl = false, stays dense: its
      // reference marginals belong to the previous gbar)
      e.sopA = sopA; e.sopB = sopB; e.smin = smin; e.scount = scount;
      if (sharded()) {
        // column totals sum over every rank's rows: the bound needs the smallest
        // row shift of ALL ranks (one scalar MAX-allreduce of its negation)
        double* g = tot.coltot + n + kNumScalars;
        CKL(launch_smin_neg(smin, g, s));
        CKS(comm_allreduce(comm, g, 1, COMM_MAX, s));
        e.smin_rows_neg = g;
      }
      CKL(launch_eval_screen(e, s));
    } else {
      CKL(launch_eval_fast(e, kind_fast, s));
    }
    f.from_partials = 1;
    f.rowpart = rowpart; f.n_col_tiles = eval.n_col_tiles;
    f.colpart = colpart; f.n_row_tiles = eval.n_row_tiles;
    if (two_d()) {
      // the host path's 2-D evaluation (Workspace::evaluate), captured with
      // both teams' NCCL allreduces; the summed scalars land in ctrl->sc
      if (timed) CK(cudaEventRecordWithFlags(gev[3], s, cudaEventRecordExternal));
      double* colbuf = tot.coltot;
      double* rowbuf = tot.coltot + n + kNumScalars;
      CKL(launch_reduce_colpart(colpart, eval.n_row_tiles, n, colbuf, s, &ctrl->done));
      CKL(launch_reduce_colpart(rowpart, eval.n_col_tiles, nrows, rowbuf, s, &ctrl->done));
      CKS(comm_allreduce(comm, colbuf, (size_t)n, COMM_SUM, s));
      CKS(comm_allreduce(comm_row, rowbuf, (size_t)nrows, COMM_SUM, s));
      FinalizeArgs fr = f;
      fr.rowtot = rowbuf;
      fr.item_begin = 0; fr.item_end = nrows;
      fr.scalars_dev = rowbuf + nrows;
      CKL(launch_finalize(fr, s));
      FinalizeArgs fc = f;
      fc.coltot = colbuf;
      fc.item_begin = nrows; fc.item_end = nrows + n;
      fc.scalars_dev = colbuf + n;
      fc.prep_flag = nullptr;
      CKL(launch_finalize(fc, s));
      CKS(comm_allreduce(comm, rowbuf + nrows, kNumScalars, COMM_SUM, s));
      CKS(comm_allreduce(comm_row, colbuf + n, kNumScalars, COMM_SUM, s));
      CKL(launch_sum_scalars(rowbuf + nrows, colbuf + n, ctrl->sc, &ctrl->done, s));
      if (timed) CK(cudaEventRecordWithFlags(gev[4], s, cudaEventRecordExternal));
      return MDOT_OK;
    }
    if (sharded()) {
      // the host path's sharded evaluation (Workspace::evaluate), captured:
      // rows finalize locally with their scalars in the tail of the column
      // buffer, ONE allreduce of [column totals | row scalars] (SURVEY 8(e)
      // NC1), then the (replicated) columns finalize and add the row scalars.
      // Every rank holds identical scalars, so every rank's controller takes
      // the same decisions and launches the same number of graphs.
      if (timed) CK(cudaEventRecordWithFlags(gev[3], s, cudaEventRecordExternal));
      double* colbuf = tot.coltot;
      CKL(launch_reduce_colpart(colpart, eval.n_row_tiles, n, colbuf, s, &ctrl->done));
      FinalizeArgs fr = f;
      fr.item_begin = 0; fr.item_end = nrows;
      fr.scalars_dev = colbuf + n;
      CKL(launch_finalize(fr, s));
      CKS(comm_allreduce(comm, colbuf, (size_t)n + kNumScalars, COMM_SUM, s));
      FinalizeArgs fc = f;
      fc.coltot = colbuf;
      fc.item_begin = nrows; fc.item_end = nrows + n;
      fc.add_in = colbuf + n;
      fc.prep_flag = nullptr;
      CKL(launch_finalize(fc, s));
      if (timed) CK(cudaEventRecordWithFlags(gev[4], s, cudaEventRecordExternal));
      return MDOT_OK;
    }
  } else {
    ExactArgs x{};
    x.C = Cdev; x.ldc = n; x.c_f64 = c_f64;
    x.X = Xdev; x.Y = Ydev; x.d = d; x.scale = scale; x.otf = otf;
    x.n = n; x.nrows = nrows;
    x.A = A; x.B = B; x.gbar = 0.0;   // gbar set below from the host value (exact mode rebuilds per step)
    x.gbar = gbar;
    x.lr = lr_ex; x.colm = colm; x.cols = cols; x.chunks = chunks;
    x.done = &ctrl->done;
    CKL(launch_eval_exact(x, s));
    f.from_partials = 0;
    f.lr_in = lr_ex; f.colm = colm; f.cols = cols; f.chunks = chunks;
  }
  if (timed) CK(cudaEventRecordWithFlags(gev[3], s, cudaEventRecordExternal));
  CKL(launch_finalize(f, s));
  if (timed) CK(cudaEventRecordWithFlags(gev[4], s, cudaEventRecordExternal));
  return MDOT_OK;
}

mdot_status Workspace::build_graph() {
  const void* sig[9] = {cur, trial, u, tu, p, pprev, (const void*)(intptr_t)(exact_mode ? 1 : 0),
                        (const void*)(intptr_t)(exact_mode ? (int64_t)(gbar * 1024.0) : 0),
                        (const void*)(intptr_t)(screen_now ? 1 : 0)};
  if (gexec && memcmp(sig, gsig, sizeof(sig)) == 0) return MDOT_OK;
  if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
  if (!cap_stream) CK(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
  if (!gev_made) {
    for (auto& e : gev) CK(cudaEventCreate(&e));
    gev_made = true;
  }
  // slots per graph: ~2 ms of work, 4..64
  const double est = 4.0 * (double)n * (double)nrows / 5.0e12 + 8e-6;
  gslots = (int)std::max(4.0, std::min(64.0, ceil(2e-3 / est)));
  int* dh = dev_alias(done_host);
  int* rh = dev_alias(ran_host);
  // NCCL in the capture (sharded): enqueue on the capture stream's device
  CK(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
  const int64_t saved = launches;
  mdot_status stt = MDOT_OK;
  (void)dh;
  (void)rh;
  for (int k = 0; k < gslots && stt == MDOT_OK; ++k) {
    // stage durations are sampled with CUDA events on the first slot of each
    // graph only: event nodes between every kernel cost more than they
    // measure (the launch gaps they insert)
    stt = launch_slot_body(cap_stream, k, time_kernels && k == 0, true);
  }
  launches = saved;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(cap_stream, &g);
  if (stt != MDOT_OK) { if (g) cudaGraphDestroy(g); return stt; }
  if (e != cudaSuccess) { set_error("graph capture failed: %s", cudaGetErrorString(e)); return MDOT_ECUDA; }
  e = cudaGraphInstantiate(&gexec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) { set_error("graph instantiate failed: %s", cudaGetErrorString(e)); return MDOT_ECUDA; }
  memcpy(gsig, sig, sizeof(sig));
  return MDOT_OK;
}

void Workspace::ctrl_trace_setup(CtrlState& h, int t) {
  h.md_t = t;
  h.trace = nullptr; h.trace_len = nullptr; h.trace_cap = 0;
  if (!trace_cap || !trace_dev) return;
  h.trace = trace_dev;
  h.trace_len = trace_len_dev;
  h.trace_cap = std::max<int64_t>(0, std::min<int64_t>(trace_cap - (int64_t)trace_host.size(), kTraceDevCap));
  cudaMemsetAsync(trace_len_dev, 0, sizeof(long long), st);
}

mdot_status Workspace::ctrl_trace_collect() {
  if (!trace_cap || !trace_dev) return MDOT_OK;
  long long len = 0;
  CK(cudaMemcpyAsync(&len, trace_len_dev, sizeof(len), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (len <= 0) return MDOT_OK;
  const size_t old = trace_host.size();
  trace_host.resize(old + (size_t)len);
  CK(cudaMemcpyAsync(trace_host.data() + old, trace_dev, sizeof(mdot_trace_rec) * (size_t)len,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return MDOT_OK;
}

// K2s counters of the slots since the last call (kept, screened), summed over
// the ranks when sharded so that every rank takes the same screen decision;
// zeroes them, synchronizes the stream
mdot_status Workspace::screen_counts(unsigned long long* hc) {
  if (sharded()) {
    double* g = tot.coltot + n + kNumScalars + 1;   // 2 doubles past the bound scalar
    double h[2];
    CK(cudaMemcpyAsync(hc, scount, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h[0] = (double)hc[0]; h[1] = (double)hc[1];
    CK(cudaMemcpyAsync(g, h, sizeof(h), cudaMemcpyHostToDevice, st));
    CKS(comm_allreduce(comm, g, 2, COMM_SUM, st));
    CK(cudaMemcpyAsync(h, g, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(scount, 0, 2 * sizeof(unsigned long long), st));
    CK(cudaStreamSynchronize(st));
    hc[0] = (unsigned long long)h[0]; hc[1] = (unsigned long long)h[1];
    return MDOT_OK;
  }
  CK(cudaMemcpyAsync(hc, scount, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemsetAsync(scount, 0, 2 * sizeof(unsigned long long), st));
  CK(cudaStreamSynchronize(st));
  return MDOT_OK;
}

mdot_status project_device(Workspace& w, const mdot_options& o, int t, mdot_result* res) {
  CtrlState h{};
  h.eps = o.eps; h.c1 = o.c1; h.c2 = o.c2;
  h.noise = ls_noise(w.exact_mode, w.gbar);
  h.stop_rho = o.stop; h.ncg = o.projector == MDOT_PROJ_NCG; h.sinkhorn = o.projector == MDOT_PROJ_SINKHORN;
  h.beta_kind = o.beta; h.ls_max_trials = o.ls_max_trials;
  h.max_evals = o.max_evals - w.evals;
  h.gpair[0] = w.eval.gh; h.gpair[1] = w.eval.gl;
  h.mode = PREP_CUR; h.phase = 0; h.alpha_prev = 1.0;
  w.ctrl_trace_setup(h, t);
  res->control_path = 1;
  // K2s from the first graph of every projection except the first MD step of
  // a multi-step schedule (the smallest gamma: nearly every entry matters) and
  // the one after a probe that kept more than 8 screen_fmax
  w.screen_now = w.screen_cap && !w.exact_mode && !(t == 1 && !w.md_last) && !w.screen_skip;
  w.screen_skip = false;
  bool probe = true;
  CKS(w.build_graph());
  cudaStream_t st = w.st;
  CK(cudaMemcpyAsync(w.ctrl, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  *((volatile int*)w.done_host) = 0;
  // initial evaluation (its result is consumed by the first k_ctrl)
  if (w.time_kernels) CK(cudaEventRecord(w.ev0, st));
  {
    // the slot body with ctrl->mode = PREP_CUR and no accept
    const int64_t before = w.launches;
    CKS(w.launch_slot_body(st, 0, false));
    (void)before;
  }
  if (w.time_kernels) CK(cudaEventRecord(w.ev1, st));
  if (w.screen_now) {
    // K2s probe: ONE slot outside the graphs (a whole graph of K2s slots at a
    // density where the dense kernel is faster costs several evaluations)
    ((volatile int*)w.ran_host)[0] = 0;
    CKS(w.launch_slot_body(st, 0, false, true));
    w.launches += 4;
    unsigned long long hc[2] = {0ull, 0ull};
    CKS(w.screen_counts(hc));
    w.screen_kept += (int64_t)hc[0];
    w.screen_total += (int64_t)hc[1];
    w.screen_slots += (int64_t)(hc[1] / (unsigned long long)(w.n * (w.sharded() ? w.n : w.nrows)));
    if (getenv("MDOT_SCREEN_DEBUG"))
      fprintf(stderr, "[mdot] t=%d probe kept %.4f%%\n", t, hc[1] ? 100.0 * (double)hc[0] / (double)hc[1] : 0.0);
    if (hc[1] > 0 && (double)hc[0] > w.screen_fmax * (double)hc[1]) {
      if ((double)hc[0] > 8.0 * w.screen_fmax * (double)hc[1]) w.screen_skip = true;
      w.screen_now = false;
      CKS(w.build_graph());
    }
    probe = false;
  }
  bool first = true;
  for (;;) {
    if (*((volatile int*)w.done_host)) break;   // the probe slot may have ended the projection
    for (int k = 0; k < w.gslots; ++k) ((volatile int*)w.ran_host)[k] = 0;
    CK(cudaGraphLaunch(w.gexec, st));
    w.launches += (w.two_d() ? 8 : w.sharded() ? 6 : 4) * w.gslots;   // our kernels per slot (NCCL's not counted)
    const bool was_scr = w.screen_now;
    unsigned long long hc[2] = {0ull, 0ull};
    if (was_scr) CKS(w.screen_counts(hc));
    CK(cudaStreamSynchronize(st));
    if (was_scr) {
      w.screen_kept += (int64_t)hc[0];
      w.screen_total += (int64_t)hc[1];
      w.screen_slots += (int64_t)(hc[1] / (unsigned long long)(w.n * (w.sharded() ? w.n : w.nrows)));
      // too many survivors at this gbar: the dense kernel is faster for the rest of the projection
      if (hc[1] > 0 && (double)hc[0] > w.screen_fmax * (double)hc[1]) {
        if (probe && (double)hc[0] > 8.0 * w.screen_fmax * (double)hc[1]) w.screen_skip = true;
        w.screen_now = false;
        CKS(w.build_graph());
      }
      probe = false;
    }
    if (w.time_kernels) {
      float ms = 0.f;
      if (first) {
        CK(cudaEventElapsedTime(&ms, w.ev0, w.ev1));
        w.kernel_ms += ms;   // includes the initial prep (a few us)
        w.kernel_launches++;
      }
      if (((volatile int*)w.ran_host)[0]) {
        float st4[4];
        for (int q = 0; q < 4; ++q) CK(cudaEventElapsedTime(&st4[q], w.gev[q], w.gev[q + 1]));
        for (int q = 0; q < 4; ++q) w.stage_ms[q] += st4[q];
        w.stage_samples++;
        w.kernel_ms += st4[2];
        w.kernel_launches++;
        if (was_scr) { w.screen_ms += st4[2]; w.screen_timed++; }
        if (getenv("MDOT_SCREEN_DEBUG"))
          fprintf(stderr, "[mdot] t=%d %s eval %.3f ms (kept %.4f%%)\n", t, was_scr ? "K2s" : "K2 ", st4[2],
                  hc[1] ? 100.0 * (double)hc[0] / (double)hc[1] : 0.0);
      }
    }
    first = false;
    if (*((volatile int*)w.done_host)) break;
  }
  CK(cudaMemcpyAsync(&h, w.ctrl, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CKS(w.ctrl_trace_collect());
  w.evals += h.evals;
  res->iterations += h.iterations;
  res->ls_evaluations += h.ls_evals;
  res->resets += h.resets;
  res->ls_restarts += h.restarts;
  if (t >= 1 && t <= 64) {
    res->rho0[t - 1] = h.rho_0;
    res->l10[t - 1] = h.l1_0;
    res->iters_step[t - 1] += h.iterations;
  }
  res->l1_final = h.l1;
  res->rho_final = h.rho;
  w.last_mass = h.mass;
  switch (h.status) {
    case CTRL_OK: return MDOT_OK;
    case CTRL_NOCONV: return MDOT_ENOCONV;
    case CTRL_LS_FAIL:
      set_error("line search failed twice at MD step %d (device control)", t);
      return MDOT_ELINESEARCH;
    case CTRL_NEED_HOST:
    default:
      // range guard fired: continue this projection under host control with
      // the exact fp64 re-evaluation available (u, v hold the last iterate)
      w.fallbacks++;
      return (o.projector == MDOT_PROJ_SINKHORN) ? project_sinkhorn(w, o, t, res) : project_pncg(w, o, t, res);
  }
}

// ---------------------------------------------------------------------------
// Persistent cooperative projection: one launch per projection (persist.cu)
// ---------------------------------------------------------------------------
// Persistent projection: prepare the control state and the kernel arguments,
// launch, collect the controller's result.
static mdot_status persist_prepare(Workspace& w, const mdot_options& o, int t, PersistArgs& a) {
  CtrlState h{};
  h.eps = o.eps; h.c1 = o.c1; h.c2 = o.c2;
  h.noise = 6e-8;
  h.stop_rho = o.stop; h.ncg = o.projector == MDOT_PROJ_NCG; h.sinkhorn = o.projector == MDOT_PROJ_SINKHORN;
  h.beta_kind = o.beta; h.ls_max_trials = o.ls_max_trials;
  h.max_evals = o.max_evals - w.evals;
  h.gpair[0] = w.eval.gh; h.gpair[1] = w.eval.gl;
  h.mode = PREP_CUR; h.phase = 0; h.alpha_prev = 1.0;
  w.ctrl_trace_setup(h, t);
  cudaStream_t st = w.st;
  CK(cudaMemcpyAsync(w.ctrl, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(w.pers_bar, 0, 2 * sizeof(unsigned int) + 14 * sizeof(unsigned long long) + 8, st));
  *((volatile int*)w.done_host) = 0;
  a = PersistArgs{};
  a.e = w.eval;
  PrepArgs& p = a.p;
  p.n = w.n; p.nrows = w.nrows; p.mode = 0;
  p.U = w.U; p.V = w.V; p.u = w.u; p.v = w.v; p.tu = w.tu; p.tv = w.tv;
  p.p = w.p; p.s = w.cur->s; p.pprev = w.pprev; p.lm = w.cur->lm;
  p.logr = w.logr; p.logc = w.logc; p.rho_r = w.rho_r; p.sig_c = w.sig_c;
  p.Aout = w.A; p.Bout = w.B;
  p.rowp = w.rowp; p.colp = w.colp; p.flag = w.flag; p.nrm = w.use_nrm ? w.nrm : nullptr;
  p.ctrl = nullptr;
  p.cur_lm = w.cur->lm; p.cur_m = w.cur->m; p.cur_s = w.cur->s; p.cur_g = w.cur->g;
  p.tr_lm = w.trial->lm; p.tr_m = w.trial->m; p.tr_s = w.trial->s; p.tr_g = w.trial->g;
  FinalizeArgs& f = a.f;
  f.n = w.n; f.nrows = w.nrows;
  f.rho_r = w.rho_r; f.sig_c = w.sig_c;
  f.r = w.r; f.c = w.c; f.logr = w.logr; f.logc = w.logc;
  f.gcur = w.cur->g; f.pcur = w.p;
  f.lm = w.trial->lm; f.m = w.trial->m; f.s = w.trial->s; f.g = w.trial->g;
  f.prep_flag = w.flag;
  f.jacobi = w.jacobi;
  f.from_partials = 1;
  f.rowpart = w.rowpart; f.n_col_tiles = w.eval.n_col_tiles;
  f.colpart = w.colpart; f.n_row_tiles = w.eval.n_row_tiles;
  a.ctrl = w.ctrl;
  cudaHostGetDevicePointer((void**)&a.done_host, w.done_host, 0);
  a.gbar = w.pers_bar;
  a.k1_ns = reinterpret_cast<unsigned long long*>(w.pers_bar + 4);
  a.cta_part = w.blockpart;
  a.initial = 1;
  a.max_slots = (long long)1 << 40;
  a.dbg_fin = nullptr;
  if (getenv("MDOT_DEBUG_K1TAIL") && w.pers_grid > 0) {
    CK(cudaMallocAsync((void**)&a.dbg_fin, (size_t)64 * w.pers_grid * 8, st));
    CK(cudaMemsetAsync(a.dbg_fin, 0, (size_t)64 * w.pers_grid * 8, st));
  }
  return MDOT_OK;
}

static mdot_status persist_collect(Workspace& w, const mdot_options& o, int t, mdot_result* res,
                                   const PersistArgs& a) {
  cudaStream_t st = w.st;
  if (a.dbg_fin) {
    // MDOT_DEBUG_K1TAIL: spread of the CTAs' K1 finish times per slot
    const int g = w.pers_grid;
    std::vector<unsigned long long> h((size_t)64 * g);
    cudaMemcpyAsync(h.data(), a.dbg_fin, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    // low 8 bits: %smid of the CTA; per-SM pairs: finish(higher CTA index) - finish(lower)
    std::vector<int> sm_of(g, -1);
    for (int c = 0; c < g; ++c) sm_of[c] = (int)(h[(size_t)2 * g + c] & 255ull);
    for (auto& x : h) x >>= 8;
    {
      double dsum = 0; int dn = 0, same = 0;
      for (int c = 0; c < g; ++c)
        for (int c2 = c + 1; c2 < g; ++c2)
          if (sm_of[c] == sm_of[c2] && h[(size_t)2 * g + c] && h[(size_t)2 * g + c2]) {
            for (int sl = 2; sl < 64; ++sl) {
              const unsigned long long a0 = h[(size_t)sl * g + c], a1 = h[(size_t)sl * g + c2];
              if (!a0 || !a1) break;
              dsum += ((double)a1 - (double)a0) * 1e-3; ++dn;
            }
            if (c2 == c + g / 2) ++same;
          }
      fprintf(stderr, "[mdot] K1 tail: CTA pairs sharing an SM finish(higher idx) - finish(lower idx) = %.2f us mean over %d; pairs (c, c+grid/2): %d\n",
              dn ? dsum / dn : 0.0, dn, same);
    }
    double sum_mean = 0, sum_max = 0;
    int ns = 0;
    std::vector<double> late(g, 0.0);
    for (int sl = 2; sl < 64; ++sl) {
      unsigned long long mx = 0;
      bool ok = true;
      for (int c = 0; c < g; ++c) { if (!h[(size_t)sl * g + c]) ok = false; mx = std::max(mx, h[(size_t)sl * g + c]); }
      if (!ok) break;
      double sm = 0, smax = 0;
      for (int c = 0; c < g; ++c) {
        const double d = (double)(mx - h[(size_t)sl * g + c]) * 1e-3;
        sm += d; smax = std::max(smax, d); late[c] += d;
      }
      sum_mean += sm / g; sum_max += smax; ++ns;
    }
    if (ns) {
      fprintf(stderr, "[mdot] K1 tail over %d slots: mean CTA slack %.2f us, max %.2f us; slack by CTA group of 16:", ns,
              sum_mean / ns, sum_max / ns);
      for (int c0 = 0; c0 < g; c0 += 16) {
        double z = 0; int k = 0;
        for (int c = c0; c < std::min(g, c0 + 16); ++c) { z += late[c]; ++k; }
        fprintf(stderr, " %.1f", z / k / ns);
      }
      fprintf(stderr, "\n");
    }
    cudaFreeAsync(a.dbg_fin, st);
  }
  CtrlState h{};
  unsigned long long k1[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // [K1 ns, count, tm[0..7]]
  CK(cudaMemcpyAsync(&h, w.ctrl, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(k1, a.k1_ns, sizeof(k1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CKS(w.ctrl_trace_collect());
  if (w.time_kernels && k1[1]) {
    w.kernel_ms += (double)k1[0] * 1e-6;
    w.kernel_launches += (int64_t)k1[1];
    // persistent phases: [ctrl+prep, K1, finalize, combine] (each incl. its grid barrier)
    for (int q = 0; q < 4; ++q) w.stage_ms[q] += (double)k1[2 + q] * 1e-6;
    if (getenv("MDOT_DEBUG"))
      fprintf(stderr, "[mdot] persistent finalize sub-phases (us/slot): partials %.2f items %.2f cta-reduce %.2f\n",
              k1[6] * 1e-3 / k1[1], k1[7] * 1e-3 / k1[1], k1[8] * 1e-3 / k1[1]);
    w.stage_samples += (int64_t)k1[1];
  }
  w.evals += h.evals;
  res->iterations += h.iterations;
  res->ls_evaluations += h.ls_evals;
  res->resets += h.resets;
  res->ls_restarts += h.restarts;
  if (t >= 1 && t <= 64) {
    res->rho0[t - 1] = h.rho_0;
    res->l10[t - 1] = h.l1_0;
    res->iters_step[t - 1] += h.iterations;
  }
  res->l1_final = h.l1;
  res->rho_final = h.rho;
  w.last_mass = h.mass;
  switch (h.status) {
    case CTRL_OK: return MDOT_OK;
    case CTRL_NOCONV: return MDOT_ENOCONV;
    case CTRL_LS_FAIL:
      set_error("line search failed twice at MD step %d (persistent control)", t);
      return MDOT_ELINESEARCH;
    case CTRL_NEED_HOST:
    default:
      w.fallbacks++;
      return (o.projector == MDOT_PROJ_SINKHORN) ? project_sinkhorn(w, o, t, res) : project_pncg(w, o, t, res);
  }
}

mdot_status project_persistent(Workspace& w, const mdot_options& o, int t, mdot_result* res) {
  res->control_path = 2;
  PersistArgs a;
  CKS(persist_prepare(w, o, t, a));
  if (w.sharded()) {
    // row-sharded: column exchange fused into the kernel over peer memory
    CKS(comm_peer_persist(w.comm, a, w.tmap, w.pers_grid, w.st));
  } else {
    CK(launch_persist(w.tmap, a, w.pers_grid, w.st));
  }
  w.launches++;
  return persist_collect(w, o, t, res, a);
}

// ---------------------------------------------------------------------------
// Schedules (Z13)
// ---------------------------------------------------------------------------
mdot_status build_schedule(const mdot_schedule* s, std::vector<double>& g) {
  g.clear();
  if (!s) { set_error("schedule is NULL"); return MDOT_EINVAL; }
  if (s->kind == MDOT_SCHED_EXPLICIT) {
    if (!s->gammas || s->n_gammas < 1) { set_error("explicit schedule without gammas"); return MDOT_EINVAL; }
    g.assign(s->gammas, s->gammas + s->n_gammas);
  } else if (s->kind == MDOT_SCHED_FIXED) {
    if (!(s->gamma_bar > 0)) { set_error("gamma_bar must be > 0"); return MDOT_EINVAL; }
    int T = s->T;
    if (T <= 0) {
      const double sm = s->step_max > 0 ? s->step_max : 256.0;
      const double q = floor(s->gamma_bar / sm);
      T = (int)(q > 1.0 ? q : 1.0);
    }
    g.assign(T, s->gamma_bar / T);
  } else if (s->kind == MDOT_SCHED_DOUBLING) {
    if (!(s->gamma_bar > 0)) { set_error("gamma_bar must be > 0"); return MDOT_EINVAL; }
    const double g0 = s->gamma0 > 0 ? s->gamma0 : 1.0;
    double gb = 0.0;
    while (gb < s->gamma_bar * (1.0 - 1e-12)) {
      double next = g.empty() ? g0 : gb;
      if (gb + next > s->gamma_bar * (1.0 + 1e-12)) next = s->gamma_bar - gb;
      g.push_back(next);
      gb += next;
      if (g.size() > 4096) { set_error("doubling schedule too long"); return MDOT_EINVAL; }
    }
  } else if (s->kind == MDOT_SCHED_ADAPTIVE) {
    // only the first step is known up front (Z29); solve_impl / K8 choose the rest
    if (!(s->gamma_bar > 0) || !isfinite(s->gamma_bar)) { set_error("gamma_bar must be > 0"); return MDOT_EINVAL; }
    const double g1 = s->step_max > 0 ? s->step_max : 256.0;
    g.assign(1, std::min(g1, s->gamma_bar));
  } else {
    set_error("unknown schedule kind %d", s->kind);
    return MDOT_EINVAL;
  }
  for (double x : g)
    if (!(x > 0) || !isfinite(x)) { set_error("schedule step %g is not > 0", x); return MDOT_EINVAL; }
  return MDOT_OK;
}

// ---------------------------------------------------------------------------
// Input handling
// ---------------------------------------------------------------------------
mdot_status validate_marginal(const double* h, int64_t n, const char* name) {
  // Neumaier-compensated sum: the test sees the exact sum of the given fp64
  // values to ~1 ulp at any n, so the documented 1e-12 bound holds as stated
  double s = 0.0, comp = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(h[i] > 0.0) || !isfinite(h[i])) {
      set_error("%s[%lld] = %g is not strictly positive (PAPER.md:38)", name, (long long)i, h[i]);
      return MDOT_EINVAL;
    }
    const double t = s + h[i];
    comp += (fabs(s) >= fabs(h[i])) ? (s - t) + h[i] : (h[i] - t) + s;
    s = t;
  }
  s += comp;
  if (fabs(s - 1.0) > 1e-12) {
    set_error("%s sums to %.17g, not 1 within 1e-12", name, s);
    return MDOT_EINVAL;
  }
  return MDOT_OK;
}

mdot_status Workspace::load_problem(const mdot_problem* pb, int64_t row0) {
  if (!pb || pb->n < 1) { set_error("problem is NULL or n < 1"); return MDOT_EINVAL; }
  if (pb->kind < 0 || pb->kind > 3) { set_error("unknown cost kind %d", pb->kind); return MDOT_EINVAL; }
  const bool dev = pb->mem == MDOT_MEM_DEVICE;
  host_io = !dev;
  otf = pb->kind == MDOT_COST_SQEUCLID_F32 ? 1 : (pb->kind == MDOT_COST_SQEUCLID_DOT_F32 ? 2 : 0);   // Z22 / Z22b
  c_f64 = pb->kind == MDOT_COST_DENSE_F64;
  kind_fast = otf ? 1 : 0;
  d = pb->d;
  scale = pb->scale;
  if (otf && (d < 1 || d > 64 || !pb->X || !pb->Y)) { set_error("SQEUCLID needs X, Y and 1 <= d <= 64"); return MDOT_EINVAL; }
  if (otf) {
    // on-the-fly cost: taller row tiles amortise each CTA's Y-tile staging
    // (K2 is FP32-bound; the partial buffers only shrink). MDOT_OTF_TILE_M: A/B.
    int cap = 2048;
    if (const char* e = getenv("MDOT_OTF_TILE_M")) cap = atoi(e);
    while (eval.tile_m < cap && (int64_t)eval.n_col_tiles * ((nrows + 2 * eval.tile_m - 1) / (2 * eval.tile_m)) >= 4 * 148)
      eval.tile_m *= 2;
    eval.n_row_tiles = (int)((nrows + eval.tile_m - 1) / eval.tile_m);
  }
  if (!otf && !pb->C) { set_error("C is NULL"); return MDOT_EINVAL; }
  if (!pb->r || !pb->c) { set_error("r or c is NULL"); return MDOT_EINVAL; }
  // marginals: validate on a host copy (2-D: the full marginals, n_glob long;
  // this rank keeps its row and column slices)
  const int64_t ng = two_d() ? n_glob : n;
  std::vector<double> hr(ng), hc(ng);
  if (dev) {
    CK(cudaMemcpyAsync(hr.data(), pb->r, sizeof(double) * ng, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), pb->c, sizeof(double) * ng, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else {
    memcpy(hr.data(), pb->r, sizeof(double) * ng);
    memcpy(hc.data(), pb->c, sizeof(double) * ng);
  }
  CKS(validate_marginal(hr.data(), ng, "r"));
  CKS(validate_marginal(hc.data(), ng, "c"));
  CK(cudaMemcpyAsync(r, hr.data() + row0, sizeof(double) * nrows, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c, hc.data() + (two_d() ? col0 : 0), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  // cost
  if (otf) {
    if (dev) {
      Xdev = pb->X; Ydev = pb->Y;
    } else {
      CK(cudaMallocAsync((void**)&owned_X, sizeof(float) * nrows * d, st));
      CK(cudaMallocAsync((void**)&owned_Y, sizeof(float) * n * d, st));
      CK(cudaMemcpyAsync(owned_X, pb->X, sizeof(float) * nrows * d, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(owned_Y, pb->Y, sizeof(float) * n * d, cudaMemcpyHostToDevice, st));
      Xdev = owned_X; Ydev = owned_Y;
    }
  } else {
    const size_t esz = c_f64 ? 8 : 4;
    if (dev) {
      Cdev = pb->C;
    } else {
      CK(cudaMallocAsync(&owned_C, esz * nrows * n, st));
      CK(cudaMemcpyAsync(owned_C, pb->C, esz * nrows * n, cudaMemcpyHostToDevice, st));
      Cdev = owned_C;
    }
    // sampled check C in [0,1]: one gather launch into the
    // mapped scalar block (doubles 128..191, unused by the solver) or a host read
    const int S = 64;
    double* samp = scal_host + 128;
    if (dev) {
      CKL(launch_sample_c(pb->C, c_f64, nrows * n, S, scal_host_dev + 128, st));
      CK(cudaStreamSynchronize(st));
    } else {
      for (int q = 0; q < S; ++q) {
        const int64_t idx = (int64_t)(((uint64_t)q * 2654435761ull) % (uint64_t)(nrows * n));
        samp[q] = c_f64 ? ((const double*)pb->C)[idx] : (double)((const float*)pb->C)[idx];
      }
    }
    for (int q = 0; q < S; ++q) {
      const double v = ((volatile double*)samp)[q];
      if (!(v >= 0.0 && v <= 1.0)) { set_error("C entry %g outside [0,1] (PAPER.md:42)", v); return MDOT_EINVAL; }
    }
  }
  eval.C = (const float*)Cdev;
  eval.ldc = n;
  eval.X = Xdev; eval.Y = Ydev; eval.d = d; eval.scale = scale; eval.otf_dot = otf == 2;
  use_nrm = otf == 2;
  if (use_nrm) {   // Z22b: |x_i|^2, |y_j|^2 once per solve; prep carries them to K2 in rowp/colp .w
    CKL(launch_sqnorms(Xdev, nrows, (int)d, nrm, st));
    CKL(launch_sqnorms(Ydev, n, (int)d, nrm + nrows, st));
  }
  use_tma = false;
  if (!otf && !c_f64 && getenv("MDOT_DISABLE_TMA") == nullptr && tma_supported(eval)) {
    if (make_tma_map(eval, tmap) == cudaSuccess) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t tiles = (int64_t)eval.n_row_tiles * eval.n_col_tiles;
      tma_grid = (int)std::min<int64_t>(tiles, 2 * (int64_t)sms);
      use_tma = true;
      int l2 = 0;
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
      eval.keep_l2 = (4.0 * (double)nrows * (double)n <= 0.6 * (double)l2) ? 1 : 0;
      if (const char* kl = getenv("MDOT_K1_KEEP_L2")) eval.keep_l2 = atoi(kl) != 0;   // A/B only
      // C larger than L2: a quarter of L2 keeps the first tiles resident
      // across evaluations (evict_last), the rest streams (evict_first);
      // config 4: K1 171.8 -> 168.5 us, time-to-eps -1.5 %; 64 / 96 MB
      // crowd out the partials and parameters (profiles/README.md)
      double res_bytes = eval.keep_l2 ? 0.0 : 0.25 * (double)l2;
      if (const char* mb = getenv("MDOT_K1_L2RES_MB")) res_bytes = atof(mb) * 1048576.0;   // A/B
      eval.l2_res_tiles = (int64_t)(res_bytes / (4.0 * eval.tile_m * kTileN));
      // sharded: the persistent path needs the fused peer exchange
      // (mdot_comm_enable_peer); CTAs per rank from the transport
      if (getenv("MDOT_NO_PERSIST") || persist_ncta < 0 || two_d()) pers_grid = 0;
      else if (sharded()) pers_grid = comm_peer_ncta(comm, n, persist_grid());
      else pers_grid = comm ? 0 : persist_grid();
      if (persist_ncta > 0 && pers_grid > persist_ncta) pers_grid = persist_ncta;
      if (persist_ncta == 0 && getenv("MDOT_PERSIST_NCTA") && pers_grid > atoi(getenv("MDOT_PERSIST_NCTA")))
        pers_grid = atoi(getenv("MDOT_PERSIST_NCTA"));   // A/B only
      if (pers_grid > 0 && (nrows + n + pers_grid - 1) / pers_grid > persist_max_chunk()) pers_grid = 0;
    }
  }
  if (getenv("MDOT_DEBUG"))
    fprintf(stderr, "[mdot] n=%lld nrows=%lld tile_m=%d tiles=%dx%d use_tma=%d grid=%d persist_grid=%d\n", (long long)n,
            (long long)nrows, eval.tile_m, eval.n_row_tiles, eval.n_col_tiles, (int)use_tma, tma_grid, pers_grid);
  return MDOT_OK;
}

// Checked builds: every guard band must still hold its 0xA5 fill.
mdot_status Workspace::check_guards() {
#ifdef MDOT_CHECKED
  if (!base) return MDOT_OK;
  std::vector<unsigned char> h(kGuardDbl * sizeof(double));
  for (size_t k = 0; k < guards.size(); ++k) {
    CK(cudaMemcpyAsync(h.data(), reinterpret_cast<double*>(base) + guards[k], h.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (size_t b = 0; b < h.size(); ++b)
      if (h[b] != 0xA5) {
        set_error("MDOT_CHECKED: guard band %zu of %zu (workspace double %zu) overwritten at byte %zu", k,
                  guards.size(), guards[k], b);
        return MDOT_ECUDA;
      }
  }
#endif
  return MDOT_OK;
}

// K1 fetched the first tiles of C (all of C when it fits in L2) with an
// evict_last policy; give those lines normal priority before returning so
// later kernels of the caller -- or a solve on another C -- are not crowded
// out by lines nobody reads any more (the data stays cached, only its
// priority changes).
mdot_status Workspace::l2_reset() {
  if (!use_tma || !Cdev) return MDOT_OK;
  int64_t rows = 0;
  if (eval.keep_l2) rows = nrows;
  else if (eval.l2_res_tiles > 0)
    rows = std::min<int64_t>(nrows, (eval.l2_res_tiles + eval.n_col_tiles - 1) / eval.n_col_tiles * eval.tile_m);
  if (rows > 0) CKL(launch_l2_normal(Cdev, (size_t)rows * (size_t)n * sizeof(float), st));
  return MDOT_OK;
}

void Workspace::free_owned() {
  if (owned_C) cudaFreeAsync(owned_C, st);
  if (owned_X) cudaFreeAsync(owned_X, st);
  if (owned_Y) cudaFreeAsync(owned_Y, st);
  owned_C = nullptr; owned_X = owned_Y = nullptr;
}

void apply_fault_env() {
  static int last = 0;
  const char* e = getenv("MDOT_FAULT_NAN");
  const int mode = e ? atoi(e) : 0;
  if (mode == last && mode == 0) return;
  fault_set_kernels(mode);
  fault_set_persist(mode);
  fault_set_batch(mode);
  last = mode;
}

mdot_status Workspace::setup(const mdot_options& o) {
  set_smem_carveout();
  apply_fault_env();
  time_kernels = o.time_kernels;
  if (time_kernels) {
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
  }
  // fp32 entries resolve the marginals to ~1e-7 relative (DESIGN.md "K1
  // numerics"): AUTO evaluates in fp64 for fp64 costs and for targets below
  // that resolution (the same rule as the batched solver, mdot_solve_batch)
  exact_mode = (o.precision == MDOT_PREC_F64P) || (o.precision == MDOT_PREC_AUTO && (c_f64 || o.eps < 5e-8));
  jacobi = o.projector == MDOT_PROJ_PNCG_JACOBI;
  // NC2 scalar-only trials: sharded host loop, fp32 entries, opt-in
  // (a net loss at the BASELINE sizes on the fused path)
  {
    const char* e = getenv("MDOT_NC2");
    nc2 = e && atoi(e) == 1 && (sharded() || two_d()) && !exact_mode;
  }
  if (!exact_mode && c_f64) {
    set_error("fp32-entry precision requested for an fp64 cost; use MDOT_PREC_F64P or AUTO");
    return MDOT_EINVAL;
  }
  CKL(launch_setup(nrows, r, logr, rho_r, st));
  CKL(launch_setup(n, c, logc, sig_c, st));
  // K2s (screen.cu): graph-slot control on the on-the-fly cost, one rank
  const char* se = getenv("MDOT_SCREEN");
  const bool al16 = ((reinterpret_cast<uintptr_t>(Xdev) | reinterpret_cast<uintptr_t>(Ydev)) & 15) == 0;
  // row-sharded: only with the graph-capturable NCCL transport (device control), where
  // every rank runs the same slots; the screen's decisions are allreduced (project_device)
  screen_cap = otf && !two_d() && (!sharded() || comm->capturable()) && screen_supported(d) && al16 && !(se && atoi(se) == 0);
  if (const char* e = getenv("MDOT_SCREEN_T")) screen_T = (float)atof(e);
  if (const char* e = getenv("MDOT_SCREEN_FMAX")) screen_fmax = atof(e);
  if (screen_cap) {
    CKL(launch_norm_max(Ydev, n, d, sop_ymax, st));
    CKL(launch_sop_pad(sopA, nrows, sopB, n, st));
  }
  return MDOT_OK;
}

// gauge: (U - d, V + d) leaves P unchanged; d chosen so that
// <r,U> = <c,V> (Z19).  Same for the step potentials (u, v).
mdot_status Workspace::gauge_center(double* X_, double* Y_) {
  const double* xs[2] = {r, c};
  const double* ys[2] = {X_, Y_};
  // rows (possibly sharded) and columns (replicated) separately
  CKL(launch_dots(nrows, 1, &xs[0], &ys[0], blockpart, ticket, scal_dev, scal_host_dev, st));
  double a = 0.0;
  if (sharded() || two_d()) {
    CKS(comm_allreduce(comm, scal_dev, 1, COMM_SUM, st));
    CK(cudaMemcpyAsync(&a, scal_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else {
    CK(cudaStreamSynchronize(st));
    a = scal_host[0];
  }
  CKL(launch_dots(n, 1, &xs[1], &ys[1], blockpart, ticket, scal_dev, scal_host_dev, st));
  double b = 0.0;
  if (two_d()) {   // this rank's column block: sum over the row team
    CKS(comm_allreduce(comm_row, scal_dev, 1, COMM_SUM, st));
    CK(cudaMemcpyAsync(&b, scal_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else {
    CK(cudaStreamSynchronize(st));
    b = scal_host[0];
  }
  const double dd = 0.5 * (a - b);
  CKL(launch_add_scalar(nrows, -dd, X_, st));
  CKL(launch_add_scalar(n, dd, Y_, st));
  return MDOT_OK;
}

// Rounding + cost, fp64 kernels (round.cu):
// R0 rows -> x (from an exact fp64 r(F): with x_i r_i(F) <= r_i the row error
// err_r = r - r(F'') is >= 0 and G lies in U(r,c), Altschuler's precondition;
// the last evaluation's fp32-entry marginals resolve r(F) only to ~1e-7),
// R2 columns -> y, err_c, R3 rows -> err_r and the costs.  Sharded: column
// sums and the final scalars are allreduced.
mdot_status Workspace::round_and_cost(float* P_out_dev, double* cost_F, double* cost_G) {
  RoundArgs a{};
  a.C = Cdev; a.ldc = n; a.c_f64 = c_f64;
  a.X = Xdev; a.Y = Ydev; a.d = d; a.scale = scale; a.otf = otf;
  a.n = n; a.nrows = nrows; a.gbar = gbar;
  a.logr = logr; a.logc = logc;
  const int chr = round_chunks(a, true), chc = round_chunks(a, false);
  if (two_d() && P_out_dev) { set_error("2-D sharded solve: no dense plan output"); return MDOT_EINVAL; }
  const size_t dbl = (size_t)(4 + 3 * chr + (two_d() ? 3 : 0)) * nrows + (size_t)(3 + chc) * n;
  double* buf = nullptr;
#ifdef MDOT_CHECKED
  CK(cudaMallocAsync((void**)&buf, (dbl + kGuardDbl) * sizeof(double), st));
  CK(cudaMemsetAsync(buf + dbl, 0xA5, kGuardDbl * sizeof(double), st));
#else
  CK(cudaMallocAsync((void**)&buf, dbl * sizeof(double), st));
#endif
  double* logx = buf;
  double* Ap = logx + nrows;
  double* er = Ap + nrows;
  double* rowcostF = er + nrows;
  double* rowS = rowcostF + nrows;
  double* rowC = rowS + (size_t)chr * nrows;
  double* rowE = rowC + (size_t)chr * nrows;
  double* Bpp = rowE + (size_t)chr * nrows;
  double* ec = Bpp + n;
  double* cs = ec + n;
  double* colS = cs + n;
  // 2-D: row sums of this rank's column block, summed over the row team
  double* rowT = colS + (size_t)chc * n;   // [3][nrows] (S, C, E)
  auto row_team_sum = [&](int k) -> mdot_status {
    const double* src[3] = {rowS, rowC, rowE};
    for (int q = 0; q < k; ++q) {
      CKL(launch_sum_chunks(src[q], chr, nrows, rowT + (size_t)q * nrows, st));
    }
    CKS(comm_allreduce(comm_row, rowT, (size_t)k * nrows, COMM_SUM, st));
    return MDOT_OK;
  };
  mdot_status stt = MDOT_OK;
  auto run = [&]() -> mdot_status {
    // R0: r(F), <C, F> per row
    a.A = U; a.B = V; a.chunks = chr; a.rowS = rowS; a.rowC = rowC; a.rowE = rowE;
    CKL(launch_round_rows(a, 0, st));
    if (two_d()) {
      CKS(row_team_sum(2));
      CKL(launch_round_x(nrows, 1, rowT, rowT + nrows, r, U, logx, Ap, rowcostF, st));
    } else {
      CKL(launch_round_x(nrows, chr, rowS, rowC, r, U, logx, Ap, rowcostF, st));
    }
    // R2: c(F') per column (partial over this rank's rows)
    a.A = Ap; a.B = V; a.chunks = chc; a.colS = colS;
    CKL(launch_round_cols(a, st));
    const double* colsum = colS;
    int colchunks = chc;
    if (sharded() || two_d()) {
      CKL(launch_sum_chunks(colS, chc, n, cs, st));
      CKS(comm_allreduce(comm, cs, (size_t)n, COMM_SUM, st));
      colsum = cs;
      colchunks = 1;
    }
    CKL(launch_round_y(n, colchunks, colsum, c, V, Bpp, ec, st));
    // R3: r(F''), <C, F''>, C err_c per row
    a.A = Ap; a.B = Bpp; a.ec = ec; a.chunks = chr;
    CKL(launch_round_rows(a, 1, st));
    if (two_d()) {
      CKS(row_team_sum(3));
      CKL(launch_round_fin(nrows, 1, rowT, rowT + nrows, rowT + 2 * nrows, rowcostF, r, er, blockpart, ticket,
                           scal_dev, scal_host_dev, st));
    } else {
      CKL(launch_round_fin(nrows, chr, rowS, rowC, rowE, rowcostF, r, er, blockpart, ticket, scal_dev, scal_host_dev,
                           st));
    }
    double ner, cF2, corr, cF;
    if (sharded() || two_d()) {
      CKS(comm_allreduce(comm, scal_dev, 4, COMM_SUM, st));
      double h4[4];
      CK(cudaMemcpyAsync(h4, scal_dev, sizeof(h4), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ner = h4[0]; cF2 = h4[1]; corr = h4[2]; cF = h4[3];
    } else {
      CK(cudaStreamSynchronize(st));
      ner = scal_host[0]; cF2 = scal_host[1]; corr = scal_host[2]; cF = scal_host[3];
    }
    if (cost_F) *cost_F = cF;
    if (cost_G) *cost_G = cF2 + (ner >= 1e-300 ? corr / ner : 0.0);   // Z18
    if (P_out_dev) {
      a.A = Ap; a.B = Bpp; a.er = er; a.ec = ec;
      a.plan = P_out_dev;
      a.inv_ner = ner >= 1e-300 ? 1.0 / ner : 0.0;
      CKL(launch_round_plan(a, st));
    }
    return MDOT_OK;
  };
  stt = run();
#ifdef MDOT_CHECKED
  if (stt == MDOT_OK) {
    std::vector<unsigned char> h(kGuardDbl * sizeof(double));
    CK(cudaMemcpyAsync(h.data(), buf + dbl, h.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (unsigned char b : h)
      if (b != 0xA5) { set_error("MDOT_CHECKED: rounding buffer overrun"); stt = MDOT_ECUDA; break; }
  }
#endif
  cudaFreeAsync(buf, st);
  return stt;
}

}  // namespace mdot

// ===========================================================================
// C ABI
// ===========================================================================
using namespace mdot;

extern "C" {

static thread_local double g_screen_stats[5] = {0, 0, 0, 0, 0};
mdot_status mdot_last_screen_stats(double* out) {
  if (!out) return MDOT_EINVAL;
  for (int q = 0; q < 5; ++q) out[q] = g_screen_stats[q];
  return MDOT_OK;
}

const char* mdot_last_error(void) { return g_last_error.c_str(); }
int32_t mdot_abi_version(void) { return MDOT_ABI_VERSION; }

void mdot_options_default(mdot_options* o) {
  memset(o, 0, sizeof(*o));
  o->eps = 1e-6;
  o->stop = 0;
  o->projector = MDOT_PROJ_PNCG;
  o->beta = MDOT_BETA_PPR;
  o->c1 = 0.1;
  o->c2 = 0.4;
  o->warm = MDOT_WARM_SCALED;
  o->precision = MDOT_PREC_AUTO;
  o->ls_max_trials = 100;
  o->max_evals = 10000000;
  o->device_control = 1;
}

void mdot_schedule_default(mdot_schedule* s) {
  memset(s, 0, sizeof(*s));
  s->kind = MDOT_SCHED_FIXED;
  s->gamma_bar = 4096.0;
  s->step_max = 256.0;
  s->gamma0 = 1.0;
}

static mdot_status solve_impl(const mdot_problem* pb, const mdot_schedule* sched, const mdot_options* opt_in,
                              double* u_out, double* v_out, float* P_out, mdot_result* res, int force_sinkhorn,
                              Comm* comm = nullptr, int64_t row0 = 0, int64_t nrows_in = -1,
                              int persist_ncta = 0, Comm* comm_row = nullptr, int64_t col0 = 0,
                              int64_t ncols_in = -1) {
  g_last_error.clear();
  if (!res) { set_error("result pointer is NULL"); return MDOT_EINVAL; }
  memset(res, 0, sizeof(*res));
  const double t0 = now_s();
  mdot_options o;
  if (opt_in) o = *opt_in; else mdot_options_default(&o);
  if (force_sinkhorn) o.projector = MDOT_PROJ_SINKHORN;
  if (o.ls_max_trials <= 0) o.ls_max_trials = 100;
  if (o.max_evals <= 0) o.max_evals = 10000000;
  if (!(o.eps > 0)) { set_error("eps must be > 0"); res->status = MDOT_EINVAL; return MDOT_EINVAL; }
  if (!pb || pb->n < 1) { set_error("problem is NULL or n < 1"); res->status = MDOT_EINVAL; return MDOT_EINVAL; }
  std::vector<double> gam;
  mdot_status st = build_schedule(sched, gam);
  if (st != MDOT_OK) { res->status = st; return st; }
  const bool adaptive = sched->kind == MDOT_SCHED_ADAPTIVE;
  cudaStream_t stream = (cudaStream_t)o.stream;
  const int64_t n = pb->n;
  const int64_t nr = nrows_in < 0 ? n : nrows_in;
  if (row0 < 0 || nr < 1 || row0 + nr > n) { set_error("bad row range"); res->status = MDOT_EINVAL; return MDOT_EINVAL; }
  // columns held by this rank: all n, or (2-D) the block [col0, col0 + nc)
  const int64_t nc = comm_row ? ncols_in : n;
  if (comm_row && (col0 < 0 || nc < 1 || col0 + nc > n)) {
    set_error("bad column range"); res->status = MDOT_EINVAL; return MDOT_EINVAL;
  }
  // 2-D: device control (graph slots with both teams' NCCL allreduces
  // captured) when both transports are capturable, else the host loop
  if (comm_row && !(comm && comm->capturable() && comm_row->capturable())) o.device_control = 0;
  // sharded: device control (CUDA-graph slots with the NCCL allreduce captured
  // inside) needs a capturable transport; the in-process transport syncs on
  // the host in every allreduce, so it runs the host loop
  // (with the fused peer exchange the persistent projection runs device-side
  // on any transport; when it cannot, such a solve takes the host loop)
  if (comm && (comm->nranks > 1 || comm->nccl) && !comm->capturable() && !comm->peer) o.device_control = 0;
  Workspace w;
  w.comm = comm;
  w.row0 = row0;
  w.comm_row = comm_row;
  w.col0 = comm_row ? col0 : 0;
  w.n_glob = n;
  w.persist_ncta = persist_ncta;
  // MDOT_TRACE: host timestamps per stage (synchronizes between stages)
  const bool trace = getenv("MDOT_TRACE") != nullptr;
  double tr_last = t0;
  NvtxRange solve_range("mdot solve");
  auto trace_mark = [&](const char* what, long long a0, long long a1) {
    if (!trace) return;
    cudaStreamSynchronize(stream);
    const double now = now_s();
    fprintf(stderr, "[mdot-trace] %-10s %9.3f ms  (%lld, %lld)\n", what, (now - tr_last) * 1e3, a0, a1);
    tr_last = now;
  };
  st = w.alloc(stream, nc, nr);
  if (st == MDOT_OK && o.trace && o.trace_cap > 0) {
    w.trace_cap = o.trace_cap;
    const size_t recs = (size_t)std::min<int64_t>(o.trace_cap, kTraceDevCap);
    if (cudaMallocAsync((void**)&w.trace_dev, recs * sizeof(mdot_trace_rec) + 64, stream) != cudaSuccess) {
      set_error("trace buffer allocation failed");
      st = MDOT_ENOMEM;
    } else {
      w.trace_len_dev = reinterpret_cast<long long*>(reinterpret_cast<char*>(w.trace_dev) + recs * sizeof(mdot_trace_rec));
    }
  }
  trace_mark("alloc", 0, 0);
  if (st == MDOT_OK) st = w.load_problem(pb, row0);
  trace_mark("load", 0, 0);
  if (st == MDOT_OK) st = w.setup(o);
  trace_mark("setup", 0, 0);
  mdot_status solve_st = MDOT_OK;
  if (st == MDOT_OK) {
    // P0 = r c^T -> U = log r, V = log c ; u = v = 0 (Alg. 1 line 2)
    if (o.p0_ones) {
      ++w.launches; launch_fill(nr, 0.0, w.U, stream);
      ++w.launches; launch_fill(nc, 0.0, w.V, stream);
    } else {
      cudaMemcpyAsync(w.U, w.logr, sizeof(double) * nr, cudaMemcpyDeviceToDevice, stream);
      cudaMemcpyAsync(w.V, w.logc, sizeof(double) * nc, cudaMemcpyDeviceToDevice, stream);
    }
    ++w.launches; launch_fill(nr, 0.0, w.u, stream);
    ++w.launches; launch_fill(nc, 0.0, w.v, stream);
    double gb = 0.0, gprev = 0.0;
    // ADAPTIVE (Z29): steps chosen after each projection from its cost
    double next = adaptive ? gam[0] : 0.0, eta_prev = 0.0;
    int final_next = adaptive && gam[0] >= sched->gamma_bar;
    for (size_t t = 1; adaptive || t <= gam.size(); ++t) {
      const double gt = adaptive ? next : gam[t - 1];
      const bool last = adaptive ? final_next != 0 : t == gam.size();
      gb = (adaptive && last) ? sched->gamma_bar : gb + gt;   // the last adaptive step lands on gamma_bar exactly
      if (t <= 64) res->gammas[t - 1] = gt;
      const int64_t evals_before = w.evals;
      w.set_gamma(gb);
      if (o.warm == MDOT_WARM_ZERO) {
        ++w.launches; launch_fill(nr, 0.0, w.u, stream);
        ++w.launches; launch_fill(nc, 0.0, w.v, stream);
      } else if (o.warm == MDOT_WARM_SCALED && t > 1 && gt != gprev) {
        ++w.launches; launch_axpby(nr, 0.0, w.u, gt / gprev, w.u, stream);   // Z4: scale by gamma_t / gamma_{t-1}
        ++w.launches; launch_axpby(nc, 0.0, w.v, gt / gprev, w.v, stream);
      }
      // intermediate MD steps may stop at the looser eps_md (Lemma 2; mdot.h)
      mdot_options ot = o;
      if (!last && o.eps_md > o.eps) ot.eps = o.eps_md;
      w.md_last = last;
      NvtxRange md_range("md step %d gbar %g", (int)t, gb);
      if (o.device_control == 1 && w.pers_grid > 0 && !w.exact_mode) solve_st = project_persistent(w, ot, (int)t, res);
      else if (o.device_control && !(w.sharded() && (w.exact_mode || !comm->capturable())))
        solve_st = project_device(w, ot, (int)t, res);
      else if (o.projector == MDOT_PROJ_SINKHORN) solve_st = project_sinkhorn(w, ot, (int)t, res);
      else solve_st = project_pncg(w, ot, (int)t, res);
      res->md_steps = (int64_t)t;
      trace_mark("project", (long long)t, (long long)w.evals);
      ++w.launches; launch_axpby(nr, 1.0, w.u, 1.0, w.U, stream);   // U += u
      ++w.launches; launch_axpby(nc, 1.0, w.v, 1.0, w.V, stream);   // V += v
      if (solve_st != MDOT_OK && solve_st != MDOT_ENOCONV) break;
      st = w.gauge_center(w.U, w.V);
      if (st == MDOT_OK) st = w.gauge_center(w.u, w.v);
      if (st != MDOT_OK) break;
      gprev = gt;
      trace_mark("step-end", (long long)t, 0);
      if (solve_st != MDOT_OK || (adaptive && last)) break;
      if (adaptive)
        next = adaptive_next_gamma((int)t, gt, (double)(w.evals - evals_before), gb, sched->gamma_bar, &eta_prev,
                                   &final_next);
    }
    res->gamma_bar = gb;
    if (st == MDOT_OK && (solve_st == MDOT_OK || solve_st == MDOT_ENOCONV)) {
      float* Pdev = nullptr;
      float* Pown = nullptr;
      if (P_out) {
        if (pb->mem == MDOT_MEM_DEVICE) Pdev = P_out;
        else if (cudaMallocAsync((void**)&Pown, sizeof(float) * nr * nc, stream) == cudaSuccess) Pdev = Pown;
      }
      {
        NvtxRange rr("rounding (Altschuler) + cost");
        st = w.round_and_cost(Pdev, &res->cost_unrounded, &res->cost_rounded);
      }
      if (st == MDOT_OK && Pown) {
        if (cudaMemcpyAsync(P_out, Pown, sizeof(float) * nr * nc, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
          st = MDOT_ECUDA;
      }
      if (Pown) cudaFreeAsync(Pown, stream);
      trace_mark("round", 0, 0);
    }
    const cudaMemcpyKind k = pb->mem == MDOT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (u_out) cudaMemcpyAsync(u_out, w.U, sizeof(double) * nr, k, stream);
    if (v_out) cudaMemcpyAsync(v_out, w.V, sizeof(double) * nc, k, stream);
  }
  if (st == MDOT_OK) st = w.l2_reset();
  if (st == MDOT_OK) st = w.check_guards();
  if (o.trace && o.trace_cap > 0) {
    const int64_t len = std::min<int64_t>((int64_t)w.trace_host.size(), o.trace_cap);
    if (len > 0) memcpy(o.trace, w.trace_host.data(), sizeof(mdot_trace_rec) * (size_t)len);
    if (o.trace_len) *o.trace_len = len;
  }
  res->evaluations = w.evals;
  res->fallbacks = w.fallbacks;
  g_screen_stats[0] = (double)w.screen_kept; g_screen_stats[1] = (double)w.screen_total;
  g_screen_stats[2] = (double)w.screen_slots; g_screen_stats[3] = w.screen_ms; g_screen_stats[4] = (double)w.screen_timed;
  res->kernel_ms = w.kernel_ms;
  res->kernel_launches = w.kernel_launches;
  res->all_launches = w.launches;
  for (int q = 0; q < 4; ++q) res->stage_ms[q] = w.stage_ms[q];
  res->stage_samples = w.stage_samples;
  w.free_owned();
  w.release();
  cudaError_t ce = cudaStreamSynchronize(stream);
  trace_mark("release", 0, 0);
  if (st == MDOT_OK && ce != cudaSuccess) {
    set_error("CUDA error at exit: %s", cudaGetErrorString(ce));
    st = MDOT_ECUDA;
  }
  if (st == MDOT_OK) st = solve_st;
  res->status = st;
  res->seconds = now_s() - t0;
  return st;
}

// Small dense problems run the whole solve in one CTA on-chip (the K8
// kernel with one instance): below a few hundred points an evaluation is a
// few thousand entries and the grid-wide paths pay ~20 us of launch /
// barrier / control latency per evaluation instead.  Threshold: MDOT_SMALL_N
// (default 512: crossover between n = 512 and 784 once K8 runs on thread-block clusters with the
// narrow-tile mapping; it was 320 before, profiles/r01_small_n_route.txt); the host control
// loop (device_control = 0) and dense plan outputs keep the general path.
static bool small_route(const mdot_problem* pb, const mdot_options* opt, const float* P_out) {
  if (!pb || P_out || pb->n < 1) return false;
  if (pb->kind != MDOT_COST_DENSE_F32 && pb->kind != MDOT_COST_DENSE_F64) return false;
  if (opt && opt->device_control == 0) return false;
  if (getenv("MDOT_NO_BATCH_KERNEL")) return false;
  int64_t lim = 512;
  if (const char* e = getenv("MDOT_SMALL_N")) lim = atoll(e);
  return pb->n <= lim;
}

// The one-CTA solver exponentiates anchored fp64 entries without a max
// shift and has no exact-evaluator fallback for its line search: plans
// beyond the fp64 range (|exponent| > ~690 from the anchor) report
// MDOT_EINSTABLE there, degenerate cases can fail the fp32-noise line search
// (n = 1 at gbar 4096); both are re-solved on the general path, whose exact
// evaluator is a max-shifted log-sum-exp.
mdot_status mdot_solve(const mdot_problem* pb, const mdot_schedule* sched, const mdot_options* opt,
                       double* u_out, double* v_out, float* P_out, mdot_result* res) {
  if (small_route(pb, opt, P_out)) {
    const mdot_status st = mdot_solve_batch(pb, 1, pb->r, pb->c, sched, opt, u_out, v_out, res);
    if (st != MDOT_EINSTABLE && st != MDOT_ELINESEARCH) return st;
  }
  return solve_impl(pb, sched, opt, u_out, v_out, P_out, res, 0);
}

mdot_status mdot_sinkhorn(const mdot_problem* pb, const mdot_schedule* sched, const mdot_options* opt,
                          double* u_out, double* v_out, float* P_out, mdot_result* res) {
  if (small_route(pb, opt, P_out)) {
    mdot_options o;
    if (opt) o = *opt; else mdot_options_default(&o);
    o.projector = MDOT_PROJ_SINKHORN;
    const mdot_status st = mdot_solve_batch(pb, 1, pb->r, pb->c, sched, &o, u_out, v_out, res);
    if (st != MDOT_EINSTABLE && st != MDOT_ELINESEARCH) return st;
  }
  return solve_impl(pb, sched, opt, u_out, v_out, P_out, res, 1);
}

mdot_status mdot_solve_sharded(mdot_comm* c, const mdot_problem* local_rows, int64_t row0, int64_t n_local,
                               const mdot_schedule* sched, const mdot_options* opt, double* u_local_out,
                               double* v_out, mdot_result* res) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm || !local_rows) { set_error("bad arguments"); return MDOT_EINVAL; }
  if (cudaSetDevice(cm->device) != cudaSuccess) { set_error("cudaSetDevice failed"); return MDOT_ECUDA; }
  return solve_impl(local_rows, sched, opt, u_local_out, v_out, nullptr, res, 0, cm, row0, n_local);
}

// 2-D (row x column) sharding: the block
// evaluation's row sums travel over the row team, its column sums over the
// column team; the host loop runs the Appx. C line search on the summed
// scalars (identical on every rank of the grid).
mdot_status mdot_solve_sharded_2d(mdot_comm* row_comm, mdot_comm* col_comm, const mdot_problem* block,
                                  int64_t row0, int64_t n_rows, int64_t col0, int64_t n_cols,
                                  const mdot_schedule* sched, const mdot_options* opt, double* u_local_out,
                                  double* v_local_out, mdot_result* res) {
  Comm* cr = reinterpret_cast<Comm*>(row_comm);
  Comm* cc = reinterpret_cast<Comm*>(col_comm);
  auto fail = [&](mdot_status e, const char* msg) {
    set_error("%s", msg);
    if (res) { memset(res, 0, sizeof(*res)); res->status = e; }
    return e;
  };
  if (!cr || !cc || !block) return fail(MDOT_EINVAL, "bad arguments");
  if (cr->device != cc->device) return fail(MDOT_EINVAL, "row and column communicators on different devices");
  if (cudaSetDevice(cc->device) != cudaSuccess) return fail(MDOT_ECUDA, "cudaSetDevice failed");
  return solve_impl(block, sched, opt, u_local_out, v_local_out, nullptr, res, 0, cc, row0, n_rows, 0, cr, col0,
                    n_cols);
}

// Throughput mode, lockstep ("including as
// a batch process"): B instances sharing one dense fp32 C advance together,
// one evaluation slot for all of them at a time, with ONE launch per phase for
// the whole batch -- k_ctrl_multi (every controller), k_prep_multi,
// k_eval_tma_multi (one persistent TMA pass over the virtual tile list
// (active instance, tile): a CTA streams several tiles, so the ring reaches
// steady state even where one instance has fewer tiles than the grid has
// CTAs) and k_finalize_multi -- captured in CUDA graphs of K slots.
// Instances whose projection has converged drop out of K1 and finalize; the
// MD step ends when every instance's has.  Each instance keeps its own
// workspace, controller and results, so it takes exactly the decisions of a
// device-control solve of its own (up to summation-order bits).  Returns
// MDOT_EGEN when the batch cannot run this way (the caller then uses the
// worker-stream path).  Opt-in (MDOT_BATCH_LOCKSTEP=1): without sharing the
// C reads between instances the batched K1 is bound by the same ~4.6 TB/s
// stream as one instance's (n = 4096, C "L2-resident" at 64 MB), so it does
// not beat the concurrent worker streams (16 x n = 4096, eps_md 1e-3: 264 vs
// 163 ms; profiles/r02_throughput_lockstep.txt).  A K1 that evaluates every
// instance on one read of each C stage is the lever; DESIGN.md section 10.
static mdot_status solve_batch_lockstep(const mdot_problem* shared, int32_t Bn, const double* r, const double* c,
                                        const mdot_schedule* sched, const mdot_options* opt_in, double* u_out,
                                        double* v_out, mdot_result* res) {
  mdot_options o;
  if (opt_in) o = *opt_in; else mdot_options_default(&o);
  if (o.ls_max_trials <= 0) o.ls_max_trials = 100;
  if (o.max_evals <= 0) o.max_evals = 10000000;
  if (Bn < 2 || Bn > kMaxBatchLockstep || shared->kind != MDOT_COST_DENSE_F32 || shared->mem != MDOT_MEM_DEVICE ||
      !sched || sched->kind == MDOT_SCHED_ADAPTIVE || o.device_control == 0 || o.trace ||
      !(getenv("MDOT_BATCH_LOCKSTEP") && atoi(getenv("MDOT_BATCH_LOCKSTEP")) == 1))
    return MDOT_EGEN;
  std::vector<double> gam;
  mdot_status st = build_schedule(sched, gam);
  if (st != MDOT_OK) return st;
  const double t0 = now_s();
  cudaStream_t stream = (cudaStream_t)o.stream;
  const int64_t n = shared->n;
  std::vector<std::unique_ptr<Workspace>> W;
  for (int32_t b = 0; b < Bn; ++b) {
    memset(&res[b], 0, sizeof(mdot_result));
    W.emplace_back(new Workspace());
    Workspace& w = *W.back();
    w.persist_ncta = -1;   // no persistent projection: the batch has its own slots
    CKS(w.alloc(stream, n, n));
    mdot_problem p = *shared;
    p.r = r + (int64_t)b * n;
    p.c = c + (int64_t)b * n;
    CKS(w.load_problem(&p, 0));
    CKS(w.setup(o));
    if (!w.use_tma || w.exact_mode || w.otf) return MDOT_EGEN;
    // P0 = r c^T: U = log r, V = log c; u = v = 0 (Alg. 1
    // line 2) -- as in the single solve; the workspace comes from the memory
    // pool and holds whatever the last user left there
    if (o.p0_ones) {
      launch_fill(n, 0.0, w.U, stream);
      launch_fill(n, 0.0, w.V, stream);
    } else {
      CK(cudaMemcpyAsync(w.U, w.logr, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(w.V, w.logc, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
    }
    launch_fill(n, 0.0, w.u, stream);
    launch_fill(n, 0.0, w.v, stream);
  }
  // argument arrays (pointers fixed for the whole solve: device control
  // accepts by element-wise copies, never by swapping buffers)
  std::vector<PrepArgs> hp(Bn);
  std::vector<EvalArgs> he(Bn);
  std::vector<FinalizeArgs> hf(Bn);
  std::vector<CtrlState*> hc(Bn);
  for (int32_t b = 0; b < Bn; ++b) {
    Workspace& w = *W[b];
    PrepArgs& a = hp[b];
    a = PrepArgs{};
    a.n = n; a.nrows = n; a.mode = 0;
    a.U = w.U; a.V = w.V; a.u = w.u; a.v = w.v; a.tu = w.tu; a.tv = w.tv;
    a.p = w.p; a.s = w.cur->s; a.pprev = w.pprev; a.lm = w.cur->lm;
    a.logr = w.logr; a.logc = w.logc; a.rho_r = w.rho_r; a.sig_c = w.sig_c;
    a.Aout = w.A; a.Bout = w.B;
    a.rowp = w.rowp; a.colp = w.colp; a.flag = w.flag;
    a.ctrl = w.ctrl;
    a.cur_lm = w.cur->lm; a.cur_m = w.cur->m; a.cur_s = w.cur->s; a.cur_g = w.cur->g;
    a.tr_lm = w.trial->lm; a.tr_m = w.trial->m; a.tr_s = w.trial->s; a.tr_g = w.trial->g;
    EvalArgs& e = he[b];
    e = w.eval;
    e.gpair = w.ctrl->gpair;
    e.done = &w.ctrl->done;
    FinalizeArgs& f = hf[b];
    f = FinalizeArgs{};
    f.n = n; f.nrows = n;
    f.rho_r = w.rho_r; f.sig_c = w.sig_c;
    f.r = w.r; f.c = w.c; f.logr = w.logr; f.logc = w.logc;
    f.gcur = w.cur->g; f.pcur = w.p;
    f.lm = w.trial->lm; f.m = w.trial->m; f.s = w.trial->s; f.g = w.trial->g;
    f.blockpart = w.blockpart; f.ticket = w.ticket;
    f.scalars_dev = w.ctrl->sc; f.scalars_host = nullptr;
    f.prep_flag = w.flag;
    f.jacobi = w.jacobi;
    f.done = &w.ctrl->done;
    f.from_partials = 1;
    f.rowpart = w.rowpart; f.n_col_tiles = w.eval.n_col_tiles;
    f.colpart = w.colpart; f.n_row_tiles = w.eval.n_row_tiles;
    hc[b] = w.ctrl;
  }
  const size_t bytes = sizeof(PrepArgs) * Bn + sizeof(EvalArgs) * Bn + sizeof(FinalizeArgs) * Bn +
                       sizeof(CtrlState*) * Bn + 4 * 256;
  char* dargs = nullptr;
  CK(cudaMallocAsync((void**)&dargs, bytes, stream));
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  PrepArgs* dp = reinterpret_cast<PrepArgs*>(dargs);
  EvalArgs* de = reinterpret_cast<EvalArgs*>(dargs + al(sizeof(PrepArgs) * Bn));
  FinalizeArgs* df = reinterpret_cast<FinalizeArgs*>(dargs + al(sizeof(PrepArgs) * Bn) + al(sizeof(EvalArgs) * Bn));
  CtrlState** dc = reinterpret_cast<CtrlState**>(dargs + al(sizeof(PrepArgs) * Bn) + al(sizeof(EvalArgs) * Bn) +
                                                 al(sizeof(FinalizeArgs) * Bn));
  CK(cudaMemcpyAsync(dp, hp.data(), sizeof(PrepArgs) * Bn, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(de, he.data(), sizeof(EvalArgs) * Bn, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(df, hf.data(), sizeof(FinalizeArgs) * Bn, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(dc, hc.data(), sizeof(CtrlState*) * Bn, cudaMemcpyHostToDevice, stream));
  // done flags: mapped pinned (the host polls them after each graph)
  int* done_h = nullptr;
  int* done_d = nullptr;
  CK(cudaHostAlloc((void**)&done_h, sizeof(int) * kMaxBatchLockstep, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&done_d, done_h, 0));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = 2 * sms;
  Workspace& w0 = *W[0];
  // K1 with shared C reads (MDOT_BATCH_SHARED_C=0: one pass per instance, A/B)
  const bool shared_c = !(getenv("MDOT_BATCH_SHARED_C") && atoi(getenv("MDOT_BATCH_SHARED_C")) == 0);
  // one graph of K slots [ctrl, prep, K1, finalize] for the whole batch (~2 ms of work)
  cudaStream_t cap = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const double est = (4.0 * (double)n * n / 5.0e12) * Bn + 20e-6;
  const int K = (int)std::max(2.0, std::min(64.0, ceil(2e-3 / est)));
  auto slot = [&](cudaStream_t s2, bool with_ctrl) -> mdot_status {
    if (with_ctrl) CK(launch_ctrl_multi(dc, Bn, done_d, s2));
    CK(launch_prep_multi(dp, hp[0], Bn, s2));
    if (shared_c) CK(launch_eval_tma_shared(w0.tmap, de, Bn, grid, s2));
    else CK(launch_eval_tma_multi(w0.tmap, de, Bn, grid, s2));
    CK(launch_finalize_multi(df, hf[0], Bn, s2));
    return MDOT_OK;
  };
  mdot_status stt = MDOT_OK;
  {
    CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < K && stt == MDOT_OK; ++k) stt = slot(cap, true);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cap, &g);
    if (stt != MDOT_OK || ce != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      set_error("lockstep graph capture failed");
      return stt != MDOT_OK ? stt : MDOT_ECUDA;
    }
    const cudaError_t ie = cudaGraphInstantiate(&gexec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) { set_error("lockstep graph instantiate failed"); return MDOT_ECUDA; }
  }
  int64_t launches = 0;
  double gb = 0.0, gprev = 0.0;
  std::vector<mdot_status> sts((size_t)Bn, MDOT_OK);
  // Decoupled MD steps (default): an instance whose projection has converged
  // starts its next MD step at once (own gamma, warm start, controller reset
  // and its initial evaluation on its own slot body) instead of waiting for
  // the slowest instance of the batch, so the shared-C slots stay full; each
  // instance still takes exactly the decisions of its own device-control solve.
  // MDOT_BATCH_SYNC_MD=1: every instance changes step together (A/B).
  const bool sync_md = getenv("MDOT_BATCH_SYNC_MD") && atoi(getenv("MDOT_BATCH_SYNC_MD")) == 1;
  if (!sync_md) {
    std::vector<size_t> tb((size_t)Bn, 0);
    std::vector<double> gbb((size_t)Bn, 0.0);
    std::vector<char> fin((size_t)Bn, 0);
    auto begin_step = [&](int32_t b) -> mdot_status {
      Workspace& w = *W[b];
      const size_t t = ++tb[b];
      const double gt = gam[t - 1];
      const double gp = t > 1 ? gam[t - 2] : 0.0;
      gbb[b] += gt;
      const bool last = t == gam.size();
      w.set_gamma(gbb[b]);
      if (o.warm == MDOT_WARM_ZERO) {
        launch_fill(n, 0.0, w.u, stream);
        launch_fill(n, 0.0, w.v, stream);
      } else if (o.warm == MDOT_WARM_SCALED && t > 1 && gt != gp) {
        launch_axpby(n, 0.0, w.u, gt / gp, w.u, stream);
        launch_axpby(n, 0.0, w.v, gt / gp, w.v, stream);
      }
      CtrlState h{};
      h.eps = (!last && o.eps_md > o.eps) ? o.eps_md : o.eps;
      h.c1 = o.c1; h.c2 = o.c2;
      h.noise = ls_noise(false, gbb[b]);
      h.stop_rho = o.stop; h.ncg = o.projector == MDOT_PROJ_NCG; h.sinkhorn = o.projector == MDOT_PROJ_SINKHORN;
      h.beta_kind = o.beta; h.ls_max_trials = o.ls_max_trials;
      h.max_evals = o.max_evals - w.evals;
      h.gpair[0] = w.eval.gh; h.gpair[1] = w.eval.gl;
      h.mode = PREP_CUR; h.phase = 0; h.alpha_prev = 1.0;
      h.md_t = (int)t;
      CK(cudaMemcpyAsync(w.ctrl, &h, sizeof(h), cudaMemcpyHostToDevice, stream));
      done_h[b] = 0;
      CKS(w.launch_slot_body(stream, 0, false));   // this instance's initial evaluation
      launches += 3;
      return MDOT_OK;
    };
    auto end_step = [&](int32_t b) -> mdot_status {
      Workspace& w = *W[b];
      const size_t t = tb[b];
      const double gt = gam[t - 1];
      const bool last = t == gam.size();
      CtrlState h{};
      CK(cudaMemcpyAsync(&h, w.ctrl, sizeof(h), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      mdot_result* R = &res[b];
      w.evals += h.evals;
      R->iterations += h.iterations;
      R->ls_evaluations += h.ls_evals;
      R->resets += h.resets;
      R->ls_restarts += h.restarts;
      if (t <= 64) {
        R->rho0[t - 1] = h.rho_0;
        R->l10[t - 1] = h.l1_0;
        R->iters_step[t - 1] += h.iterations;
        R->gammas[t - 1] = gt;
      }
      R->l1_final = h.l1;
      R->rho_final = h.rho;
      R->md_steps = (int64_t)t;
      R->control_path = 4;
      mdot_options ot = o;
      if (!last && o.eps_md > o.eps) ot.eps = o.eps_md;
      w.md_last = last;
      mdot_status ps = MDOT_OK;
      if (h.status == CTRL_NOCONV) ps = MDOT_ENOCONV;
      else if (h.status == CTRL_LS_FAIL) {
        set_error("instance %d: line search failed twice at MD step %d (lockstep batch)", (int)b, (int)t);
        ps = MDOT_ELINESEARCH;
      } else if (h.status == CTRL_NEED_HOST) {
        w.fallbacks++;
        ps = (o.projector == MDOT_PROJ_SINKHORN) ? project_sinkhorn(w, ot, (int)t, R) : project_pncg(w, ot, (int)t, R);
      }
      launch_axpby(n, 1.0, w.u, 1.0, w.U, stream);   // U += u
      launch_axpby(n, 1.0, w.v, 1.0, w.V, stream);
      if (ps != MDOT_OK && ps != MDOT_ENOCONV) { sts[b] = ps; return MDOT_OK; }
      mdot_status gs = w.gauge_center(w.U, w.V);
      if (gs == MDOT_OK) gs = w.gauge_center(w.u, w.v);
      if (gs != MDOT_OK) return gs;
      if (ps == MDOT_ENOCONV) sts[b] = ps;
      return MDOT_OK;
    };
    for (int32_t b = 0; b < Bn && stt == MDOT_OK; ++b) stt = begin_step(b);
    while (stt == MDOT_OK) {
      bool any = false;
      for (int32_t b = 0; b < Bn; ++b) any = any || !fin[b];
      if (!any) break;
      CK(cudaGraphLaunch(gexec, stream));
      launches += 4 * (int64_t)K;
      CK(cudaStreamSynchronize(stream));
      for (int32_t b = 0; b < Bn && stt == MDOT_OK; ++b) {
        if (fin[b] || !((volatile int*)done_h)[b]) continue;
        stt = end_step(b);
        if (stt != MDOT_OK) break;
        if (sts[b] != MDOT_OK || tb[b] == gam.size()) {
          fin[b] = 1;
          const int one = 1;   // sits out the remaining graphs
          CK(cudaMemcpyAsync(&W[b]->ctrl->done, &one, sizeof(int), cudaMemcpyHostToDevice, stream));
          done_h[b] = 1;
        } else {
          stt = begin_step(b);
        }
      }
    }
    for (double g : gam) gb += g;
  }
  for (size_t t = 1; sync_md && t <= gam.size() && stt == MDOT_OK; ++t) {
    const double gt = gam[t - 1];
    gb += gt;
    const bool last = t == gam.size();
    for (int32_t b = 0; b < Bn; ++b) {
      Workspace& w = *W[b];
      if (sts[b] != MDOT_OK) continue;
      w.set_gamma(gb);
      if (o.warm == MDOT_WARM_ZERO) {
        launch_fill(n, 0.0, w.u, stream);
        launch_fill(n, 0.0, w.v, stream);
      } else if (o.warm == MDOT_WARM_SCALED && t > 1 && gt != gprev) {
        launch_axpby(n, 0.0, w.u, gt / gprev, w.u, stream);
        launch_axpby(n, 0.0, w.v, gt / gprev, w.v, stream);
      }
      CtrlState h{};
      h.eps = (!last && o.eps_md > o.eps) ? o.eps_md : o.eps;
      h.c1 = o.c1; h.c2 = o.c2;
      h.noise = ls_noise(false, gb);
      h.stop_rho = o.stop; h.ncg = o.projector == MDOT_PROJ_NCG; h.sinkhorn = o.projector == MDOT_PROJ_SINKHORN;
      h.beta_kind = o.beta; h.ls_max_trials = o.ls_max_trials;
      h.max_evals = o.max_evals - w.evals;
      h.gpair[0] = w.eval.gh; h.gpair[1] = w.eval.gl;
      h.mode = PREP_CUR; h.phase = 0; h.alpha_prev = 1.0;
      h.md_t = (int)t;
      CK(cudaMemcpyAsync(w.ctrl, &h, sizeof(h), cudaMemcpyHostToDevice, stream));
      done_h[b] = 0;
    }
    // instances that already failed sit out (their controller is marked done)
    for (int32_t b = 0; b < Bn; ++b)
      if (sts[b] != MDOT_OK) {
        const int one = 1;
        CK(cudaMemcpyAsync(&W[b]->ctrl->done, &one, sizeof(int), cudaMemcpyHostToDevice, stream));
        done_h[b] = 1;
      }
    // initial evaluation of every instance (no controller), then graphs
    stt = slot(stream, false);
    launches += 3;
    while (stt == MDOT_OK) {
      CK(cudaGraphLaunch(gexec, stream));
      launches += 4 * (int64_t)K;
      CK(cudaStreamSynchronize(stream));
      bool all = true;
      for (int32_t b = 0; b < Bn; ++b) all = all && ((volatile int*)done_h)[b] != 0;
      if (all) break;
    }
    for (int32_t b = 0; b < Bn && stt == MDOT_OK; ++b) {
      Workspace& w = *W[b];
      if (sts[b] != MDOT_OK) continue;
      CtrlState h{};
      CK(cudaMemcpyAsync(&h, w.ctrl, sizeof(h), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      mdot_result* R = &res[b];
      w.evals += h.evals;
      R->iterations += h.iterations;
      R->ls_evaluations += h.ls_evals;
      R->resets += h.resets;
      R->ls_restarts += h.restarts;
      if (t <= 64) {
        R->rho0[t - 1] = h.rho_0;
        R->l10[t - 1] = h.l1_0;
        R->iters_step[t - 1] += h.iterations;
        R->gammas[t - 1] = gt;
      }
      R->l1_final = h.l1;
      R->rho_final = h.rho;
      R->md_steps = (int64_t)t;
      R->control_path = 4;
      mdot_options ot = o;
      if (!last && o.eps_md > o.eps) ot.eps = o.eps_md;
      w.md_last = last;
      mdot_status ps = MDOT_OK;
      if (h.status == CTRL_NOCONV) ps = MDOT_ENOCONV;
      else if (h.status == CTRL_LS_FAIL) {
        set_error("instance %d: line search failed twice at MD step %d (lockstep batch)", (int)b, (int)t);
        ps = MDOT_ELINESEARCH;
      } else if (h.status == CTRL_NEED_HOST) {
        // range guard: this instance finishes the projection under host control
        w.fallbacks++;
        ps = (o.projector == MDOT_PROJ_SINKHORN) ? project_sinkhorn(w, ot, (int)t, R) : project_pncg(w, ot, (int)t, R);
      }
      launch_axpby(n, 1.0, w.u, 1.0, w.U, stream);   // U += u
      launch_axpby(n, 1.0, w.v, 1.0, w.V, stream);
      if (ps != MDOT_OK && ps != MDOT_ENOCONV) { sts[b] = ps; continue; }
      mdot_status gs = w.gauge_center(w.U, w.V);
      if (gs == MDOT_OK) gs = w.gauge_center(w.u, w.v);
      if (gs != MDOT_OK) { stt = gs; break; }
      if (ps == MDOT_ENOCONV) sts[b] = ps;
    }
    gprev = gt;
  }
  mdot_status first = stt;
  for (int32_t b = 0; b < Bn; ++b) {
    Workspace& w = *W[b];
    mdot_result* R = &res[b];
    R->gamma_bar = gb;
    if (stt == MDOT_OK && (sts[b] == MDOT_OK || sts[b] == MDOT_ENOCONV)) {
      const mdot_status rs = w.round_and_cost(nullptr, &R->cost_unrounded, &R->cost_rounded);
      if (rs != MDOT_OK && first == MDOT_OK) first = rs;
    }
    if (u_out) cudaMemcpyAsync(u_out + (int64_t)b * n, w.U, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream);
    if (v_out) cudaMemcpyAsync(v_out + (int64_t)b * n, w.V, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream);
    R->evaluations = w.evals;
    R->fallbacks = w.fallbacks;
    R->all_launches = w.launches + launches / Bn;
    R->status = (stt != MDOT_OK) ? stt : sts[b];
    if (first == MDOT_OK && sts[b] != MDOT_OK) first = sts[b];
  }
  if (stt == MDOT_OK) W[0]->l2_reset();
  cudaGraphExecDestroy(gexec);
  cudaStreamDestroy(cap);
  cudaFreeAsync(dargs, stream);
  for (auto& w : W) { w->free_owned(); w->release(); }
  cudaStreamSynchronize(stream);
  cudaFreeHost(done_h);
  const double secs = now_s() - t0;
  for (int32_t b = 0; b < Bn; ++b) res[b].seconds = secs;
  return first;
}

// mdot_solve_batch for costs the K8 kernel cannot hold (SURVEY 8(f) rank 4,
// throughput mode): device-resident instances are solved concurrently by up
// to MDOT_BATCH_WORKERS (default 8) host workers, each on its own stream
// (ordered after the caller's stream) with the CUDA-graph control path --
// the persistent kernel is a cooperative grid over every SM and would
// serialise them.  The evaluations of different instances then overlap on
// the GPU (a shared C stays L2-resident when it fits).  Host-memory inputs
// run one instance after the other.
static mdot_status solve_batch_loop(const mdot_problem* shared, int32_t Bn, const double* r, const double* c,
                                    const mdot_schedule* sched, const mdot_options* opt, double* u_out,
                                    double* v_out, mdot_result* res) {
  mdot_options o;
  if (opt) o = *opt; else mdot_options_default(&o);
  const int64_t n = shared->n;
  auto one = [&](int32_t b, const mdot_options* ob, int persist_ncta) {
    mdot_problem p = *shared;
    p.r = r + (int64_t)b * n;
    p.c = c + (int64_t)b * n;
    return solve_impl(&p, sched, ob, u_out ? u_out + (int64_t)b * n : nullptr,
                      v_out ? v_out + (int64_t)b * n : nullptr, nullptr, &res[b], 0, nullptr, 0, -1, persist_ncta);
  };
  int W = 8;
  if (const char* e = getenv("MDOT_BATCH_WORKERS")) W = atoi(e);
  W = std::max(1, std::min<int>(W, Bn));
  if (W == 1 || shared->mem != MDOT_MEM_DEVICE) {
    mdot_status first = MDOT_OK;
    for (int32_t b = 0; b < Bn; ++b) {
      const mdot_status s = one(b, &o, 0);
      if (s != MDOT_OK && first == MDOT_OK) first = s;
    }
    return first;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  // graph-path control in every worker: cooperative persistent launches from
  // several workers (each on a slice of the grid) measured slower than one
  // after the other (profiles/r01_throughput_mode_n4096.txt)
  const int slice = -1;
  cudaEvent_t ready = nullptr;
  CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CK(cudaEventRecord(ready, (cudaStream_t)o.stream));
  std::atomic<int32_t> next{0};
  std::vector<mdot_status> sts((size_t)Bn, MDOT_OK);
  std::vector<std::string> errs((size_t)Bn);
  auto worker = [&]() {
    cudaSetDevice(dev);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return;
    cudaStreamWaitEvent(s, ready, 0);
    mdot_options ow = o;
    ow.stream = s;
    for (int32_t b = next++; b < Bn; b = next++) {
      sts[(size_t)b] = one(b, &ow, slice);
      if (sts[(size_t)b] != MDOT_OK) errs[(size_t)b] = mdot_last_error();
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  };
  std::vector<std::thread> th;
  for (int k = 0; k < W; ++k) th.emplace_back(worker);
  for (auto& x : th) x.join();
  cudaEventDestroy(ready);
  for (int32_t b = 0; b < Bn; ++b)
    if (sts[(size_t)b] != MDOT_OK) {
      set_error("instance %d: %s", (int)b, errs[(size_t)b].c_str());
      return sts[(size_t)b];
    }
  return MDOT_OK;
}

mdot_status mdot_solve_batch(const mdot_problem* shared, int32_t Bn, const double* r, const double* c,
                             const mdot_schedule* sched, const mdot_options* opt_in,
                             double* u_out, double* v_out, mdot_result* res) {
  g_last_error.clear();
  if (!shared || Bn < 1 || !r || !c || !res) { set_error("bad batch arguments"); return MDOT_EINVAL; }
  mdot_options o;
  if (opt_in) o = *opt_in; else mdot_options_default(&o);
  if (o.ls_max_trials <= 0) o.ls_max_trials = 100;
  if (o.max_evals <= 0) o.max_evals = 10000000;
  const int64_t n = shared->n;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const bool c64 = shared->kind == MDOT_COST_DENSE_F64;
  const bool fits = (shared->kind == MDOT_COST_DENSE_F32 || c64) && n >= 1 &&
                    (int64_t)batch_smem_bytes((int)n) <= optin && getenv("MDOT_NO_BATCH_KERNEL") == nullptr &&
                    !(c64 && o.precision == MDOT_PREC_F32P);   // rejected by the per-instance path
  if (!fits) {
    const mdot_status ls = solve_batch_lockstep(shared, Bn, r, c, sched, opt_in, u_out, v_out, res);
    if (ls != MDOT_EGEN) return ls;
    return solve_batch_loop(shared, Bn, r, c, sched, opt_in, u_out, v_out, res);
  }
  const double t0 = now_s();
  for (int32_t b = 0; b < Bn; ++b) memset(&res[b], 0, sizeof(mdot_result));
  if (!(o.eps > 0)) { set_error("eps must be > 0"); return MDOT_EINVAL; }
  std::vector<double> gam;
  mdot_status st = build_schedule(sched, gam);
  if (st != MDOT_OK) return st;
  cudaStream_t stream = (cudaStream_t)o.stream;
  const bool dev_mem = shared->mem == MDOT_MEM_DEVICE;
  const size_t vb = sizeof(double) * (size_t)Bn * n;
  // validate every instance's marginals on a host copy
  std::vector<double> hr((size_t)Bn * n), hc((size_t)Bn * n);
  if (dev_mem) {
    CK(cudaMemcpyAsync(hr.data(), r, vb, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(hc.data(), c, vb, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  } else {
    memcpy(hr.data(), r, vb);
    memcpy(hc.data(), c, vb);
  }
  for (int32_t b = 0; b < Bn; ++b) {
    CKS(validate_marginal(hr.data() + (size_t)b * n, n, "r"));
    CKS(validate_marginal(hc.data() + (size_t)b * n, n, "c"));
  }
  {
    // C in [0,1]: every entry (n^2 <= ~0.6 M here)
    double mm[2] = {0.0, 0.0};
    if (dev_mem) {
      double* dmm = nullptr;
      CK(cudaMallocAsync((void**)&dmm, 2 * sizeof(double), stream));
      CK(launch_minmax(shared->C, c64 ? 1 : 0, n * n, dmm, stream));
      CK(cudaMemcpyAsync(mm, dmm, sizeof(mm), cudaMemcpyDeviceToHost, stream));
      CK(cudaFreeAsync(dmm, stream));
      CK(cudaStreamSynchronize(stream));
    } else {
      mm[0] = INFINITY;
      mm[1] = -INFINITY;
      for (int64_t k = 0; k < n * n; ++k) {
        const double v = c64 ? ((const double*)shared->C)[k] : (double)((const float*)shared->C)[k];
        if (v != v) { mm[0] = -INFINITY; break; }
        mm[0] = std::min(mm[0], v);
        mm[1] = std::max(mm[1], v);
      }
    }
    if (!(mm[0] >= 0.0 && mm[1] <= 1.0)) {
      set_error("C entries in [%g, %g], outside [0,1] (PAPER.md:42)", mm[0], mm[1]);
      return MDOT_EINVAL;
    }
  }
  // device buffers: [r | c | gammas | U | V | results | C (host input)]
  const size_t cbytes = (c64 ? sizeof(double) : sizeof(float)) * (size_t)n * n;
  auto r256 = [](size_t k) { return (k + 255) / 256 * 256; };   // every take() below is 256-byte aligned
  const size_t bytes = 4 * r256(vb) + r256(sizeof(double) * gam.size()) + r256(sizeof(BatchResult) * Bn) +
                       (dev_mem ? 0 : r256(cbytes));
  char* base = nullptr;
  CK(cudaMallocAsync((void**)&base, bytes, stream));
  char* q = base;
  auto take = [&](size_t k) { char* x = q; q += (k + 255) / 256 * 256; return x; };
  double* dr = (double*)take(vb);
  double* dc = (double*)take(vb);
  double* dU = (double*)take(vb);
  double* dV = (double*)take(vb);
  double* dg = (double*)take(sizeof(double) * gam.size());
  BatchResult* dres = (BatchResult*)take(sizeof(BatchResult) * Bn);
  const void* dC = shared->C;
  if (!dev_mem) {
    void* cc = take(cbytes);
    CK(cudaMemcpyAsync(cc, shared->C, cbytes, cudaMemcpyHostToDevice, stream));
    dC = cc;
  }
  CK(cudaMemcpyAsync(dr, hr.data(), vb, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(dc, hc.data(), vb, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(dg, gam.data(), sizeof(double) * gam.size(), cudaMemcpyHostToDevice, stream));
  BatchArgs a{};
  a.C = c64 ? nullptr : (const float*)dC;
  a.C64 = c64 ? (const double*)dC : nullptr;
  a.n = (int)n; a.r = dr; a.c = dc; a.gammas = dg; a.T = (int)gam.size();
  a.adaptive = sched->kind == MDOT_SCHED_ADAPTIVE;
  a.gamma_bar = sched->gamma_bar;
  a.gamma1 = gam[0];
  mdot_trace_rec* dtrace = nullptr;
  if (o.trace && o.trace_cap > 0) {
    const size_t recs = (size_t)std::min<int64_t>(o.trace_cap, kTraceDevCap);
    CK(cudaMallocAsync((void**)&dtrace, recs * sizeof(mdot_trace_rec) + 64, stream));
    a.trace = dtrace;
    a.trace_cap = (long long)recs;
    a.trace_len = reinterpret_cast<long long*>(reinterpret_cast<char*>(dtrace) + recs * sizeof(mdot_trace_rec));
    CK(cudaMemsetAsync(a.trace_len, 0, sizeof(long long), stream));
  }
  a.eps = o.eps; a.eps_md = o.eps_md > o.eps ? o.eps_md : o.eps; a.c1 = o.c1; a.c2 = o.c2;
  a.stop_rho = o.stop; a.projector = o.projector; a.beta_kind = o.beta; a.ls_max_trials = o.ls_max_trials;
  a.warm = o.warm; a.p0_ones = o.p0_ones;
  // fp32 entries resolve marginals to ~1e-7 (K1 numerics): tighter
  // targets run the fp64-entry evaluation
  a.f64 = c64 || (o.precision == MDOT_PREC_F64P) || (o.precision == MDOT_PREC_AUTO && o.eps < 5e-8);
  a.max_evals = o.max_evals;
  a.U_out = dU; a.V_out = dV; a.res = dres;
  unsigned long long* kdbg = nullptr;   // MDOT_DEBUG_K8 (MDOT_DIAG_K8 builds): per-phase clocks of instance 0
  if (getenv("MDOT_DEBUG_K8") && cudaMalloc((void**)&kdbg, 8 * sizeof(unsigned long long)) == cudaSuccess) {
    cudaMemsetAsync(kdbg, 0, 8 * sizeof(unsigned long long), stream);
    a.dbg = kdbg;
  }
  apply_fault_env();
  cudaError_t e = launch_batch(a, Bn, stream);
  if (e != cudaSuccess) {
    cudaFreeAsync(base, stream);
    set_error("batch kernel launch failed: %s", cudaGetErrorString(e));
    return MDOT_ECUDA;
  }
  if (getenv("MDOT_DEBUG")) {
    const cudaError_t es = cudaStreamSynchronize(stream);
    fprintf(stderr, "[mdot] batch kernel n=%lld B=%d smem=%zu f64=%d c64=%d: %s\n", (long long)n, (int)Bn,
            batch_smem_bytes((int)n), a.f64, (int)c64, cudaGetErrorString(es));
  }
  std::vector<BatchResult> hres(Bn);
  CK(cudaMemcpyAsync(hres.data(), dres, sizeof(BatchResult) * Bn, cudaMemcpyDeviceToHost, stream));
  if (dtrace) {
    long long len = 0;
    CK(cudaMemcpyAsync(&len, a.trace_len, sizeof(len), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    len = std::min<long long>(len, (long long)o.trace_cap);
    if (len > 0)
      CK(cudaMemcpyAsync(o.trace, dtrace, sizeof(mdot_trace_rec) * (size_t)len, cudaMemcpyDeviceToHost, stream));
    if (o.trace_len) *o.trace_len = len;
  }
  const cudaMemcpyKind k = dev_mem ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (u_out) CK(cudaMemcpyAsync(u_out, dU, vb, k, stream));
  if (v_out) CK(cudaMemcpyAsync(v_out, dV, vb, k, stream));
  CK(cudaStreamSynchronize(stream));
  if (kdbg) {
    unsigned long long h[8];
    cudaMemcpy(h, kdbg, sizeof(h), cudaMemcpyDeviceToHost);
    const double k = h[7] ? (double)h[7] : 1.0;
    fprintf(stderr, "[mdot] K8 cycles per evaluation (instance 0, CTA 0): ctrl %.0f prep %.0f eval %.0f "
            "(tile loops %.0f, tile epilogues + tail %.0f) cluster-combine %.0f finalize %.0f (%llu evaluations)\n",
            h[0] / k, h[1] / k, h[2] / k, h[5] / k, h[6] / k, h[3] / k, h[4] / k, h[7]);
    cudaFree(kdbg);
  }
  cudaFreeAsync(base, stream);
  if (dtrace) cudaFreeAsync(dtrace, stream);
  const double secs = now_s() - t0;
  mdot_status first = MDOT_OK;
  for (int32_t b = 0; b < Bn; ++b) {
    mdot_result& R = res[b];
    const BatchResult& h = hres[b];
    R.cost_rounded = h.cost_rounded;
    R.cost_unrounded = h.cost_unrounded;
    R.l1_final = h.l1_final;
    R.rho_final = h.rho_final;
    R.gamma_bar = h.gamma_bar;
    R.seconds = secs;
    R.md_steps = h.md_steps;
    R.iterations = h.iterations;
    R.evaluations = h.evaluations;
    R.ls_evaluations = h.ls_evaluations;
    R.resets = h.resets;
    R.ls_restarts = h.ls_restarts;
    R.status = h.status;
    R.control_path = 3;   // K8 batched kernel
    for (int q = 0; q < 64 && q < h.md_steps; ++q) {
      R.rho0[q] = h.rho0[q];
      R.l10[q] = h.l10[q];
      R.iters_step[q] = h.iters_step[q];
      R.gammas[q] = h.gammas[q];
    }
    R.all_launches = 1;
    if (h.status != MDOT_OK && first == MDOT_OK) {
      first = (mdot_status)h.status;
      set_error("batch instance %d finished with status %d", b, h.status);
    }
  }
  return first;
}

mdot_status mdot_marginals(const mdot_problem* pb, const double* Ain, const double* Bin, double gbar,
                           double* lr, double* lc, const mdot_options* opt_in, int32_t* fallback_out) {
  g_last_error.clear();
  mdot_options o;
  if (opt_in) o = *opt_in; else mdot_options_default(&o);
  if (!pb || pb->n < 1 || !Ain || !Bin || !lr || !lc) { set_error("bad arguments"); return MDOT_EINVAL; }
  cudaStream_t stream = (cudaStream_t)o.stream;
  const int64_t n = pb->n;
  Workspace w;
  mdot_status st = w.alloc(stream, n, n);
  if (st == MDOT_OK) st = w.load_problem(pb, 0);
  if (st == MDOT_OK) st = w.setup(o);
  if (st == MDOT_OK) {
    w.set_gamma(gbar);
    const double* dA = Ain;
    const double* dB = Bin;
    if (pb->mem != MDOT_MEM_DEVICE) {
      cudaMemcpyAsync(w.tu, Ain, sizeof(double) * n, cudaMemcpyHostToDevice, stream);
      cudaMemcpyAsync(w.tv, Bin, sizeof(double) * n, cudaMemcpyHostToDevice, stream);
      dA = w.tu;
      dB = w.tv;
    }
    double sc[kNumScalars];
    st = w.prep(PREP_AB, 0, 0, nullptr, dA, dB);
    if (st == MDOT_OK) st = w.evaluate(w.cur, nullptr, nullptr, sc);
    if (st == MDOT_OK) {
      const cudaMemcpyKind k = pb->mem == MDOT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      cudaMemcpyAsync(lr, w.cur->lm, sizeof(double) * n, k, stream);
      cudaMemcpyAsync(lc, w.cur->lm + n, sizeof(double) * n, k, stream);
    }
    if (fallback_out) *fallback_out = (int32_t)w.fallbacks;
    if (st == MDOT_OK) st = w.l2_reset();
    if (st == MDOT_OK) st = w.check_guards();
  }
  w.free_owned();
  w.release();
  cudaError_t ce = cudaStreamSynchronize(stream);
  if (st == MDOT_OK && ce != cudaSuccess) { set_error("%s", cudaGetErrorString(ce)); st = MDOT_ECUDA; }
  return st;
}

mdot_status mdot_round(const mdot_problem* pb, const double* U, const double* V, double gbar,
                       float* P_out, double* cost_F, double* cost_G, const mdot_options* opt_in) {
  g_last_error.clear();
  mdot_options o;
  if (opt_in) o = *opt_in; else mdot_options_default(&o);
  if (!pb || pb->n < 1 || !U || !V) { set_error("bad arguments"); return MDOT_EINVAL; }
  o.precision = MDOT_PREC_F64P;   // rounding runs on the fp64 kernels
  cudaStream_t stream = (cudaStream_t)o.stream;
  const int64_t n = pb->n;
  Workspace w;
  mdot_status st = w.alloc(stream, n, n);
  if (st == MDOT_OK) st = w.load_problem(pb, 0);
  if (st == MDOT_OK) st = w.setup(o);
  float* Pown = nullptr;
  if (st == MDOT_OK) {
    w.set_gamma(gbar);
    const cudaMemcpyKind kin = pb->mem == MDOT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    cudaMemcpyAsync(w.U, U, sizeof(double) * n, kin, stream);
    cudaMemcpyAsync(w.V, V, sizeof(double) * n, kin, stream);
    ++w.launches; launch_fill(n, 0.0, w.u, stream);
    ++w.launches; launch_fill(n, 0.0, w.v, stream);
    double sc[kNumScalars];
    st = w.prep(PREP_CUR, 0, 0, nullptr, nullptr, nullptr);
    if (st == MDOT_OK) st = w.evaluate(w.cur, nullptr, nullptr, sc);
    float* Pdev = nullptr;
    if (st == MDOT_OK && P_out) {
      if (pb->mem == MDOT_MEM_DEVICE) Pdev = P_out;
      else if (cudaMallocAsync((void**)&Pown, sizeof(float) * n * n, stream) == cudaSuccess) Pdev = Pown;
    }
    if (st == MDOT_OK) st = w.round_and_cost(Pdev, cost_F, cost_G);
    if (st == MDOT_OK && Pown) cudaMemcpyAsync(P_out, Pown, sizeof(float) * n * n, cudaMemcpyDeviceToHost, stream);
  }
  if (Pown) cudaFreeAsync(Pown, stream);
  w.free_owned();
  w.release();
  cudaError_t ce = cudaStreamSynchronize(stream);
  if (st == MDOT_OK && ce != cudaSuccess) { set_error("%s", cudaGetErrorString(ce)); st = MDOT_ECUDA; }
  return st;
}

}  // extern "C"

// paper_2307_08507_b200/csrc/persist.cu -- persistent cooperative slot
// kernel: one launch runs a whole Bregman projection (Alg. 2 PNCG with the
// Appx. C line search, or Alg. 3 Sinkhorn) on the GPU.
//
// Every CTA of the co-resident grid (2 per SM, 8 consumer warps + 1 TMA
// producer warp) repeats, per evaluation slot:
//   ctrl      each CTA runs the controller (ops.cuh ctrl_body) on its own
//             shared-memory copy of the state: every CTA holds the same
//             scalars, so every CTA takes the same decision (no barrier)
//   prep      grid-stride over the 2n row/column items (accept copy,
//             direction p = -s + beta p_prev, trial potentials, exponent split)
//   -- grid barrier --
//   K1        the TMA-fed fused marginal pass over this CTA's tiles
//   -- grid barrier --
//   finalize  grid-stride over items: partial sums, log marginals, s, grad,
//             the 16 scalars -> per-CTA partial
//   -- grid barrier --
//   every CTA combines the per-CTA partials in the same fixed order.
// Kernel launches, graph nodes and host round trips disappear from the loop;
// the host launches once per MD step and reads the state back.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"
#include "k1_tma.cuh"
#include "ops.cuh"

namespace mdot {

// TMA ring + the CTA's copy of the controller state.  The finalize scratch
// (per-warp scalar partials, the cross-CTA combine) reuses tma.sred, which is
// only live at K1 tile ends: 2 CTAs/SM fit (2 x 115.3 KB).
struct PersistSmem {
  TmaSmem tma;
  CtrlState st;
};
static_assert(sizeof(double) * ((kTmaThreads / 32) * kNumScalars + 512) <= sizeof(TmaSmem::sred),
              "finalize scratch must fit in tma.sred");
// finalize chunk totals live at fin + 256 in tma.sred: items per CTA must fit
constexpr int kPersistMaxChunk = (int)(sizeof(TmaSmem::sred) / sizeof(double)) - (kTmaThreads / 32) * kNumScalars - 256;

// Sense-reversal grid barrier over co-resident CTAs (cooperative launch):
// bar[0] = arrivals, bar[1] = generation.  One gpu-scope fence per CTA on each
// side; the CTA barriers make every thread's prior writes part of it.
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_release(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Count barrier: every CTA's thread 0 arrives with a release-add on a
// monotonic counter (zeroed before every launch) and polls it with acquire
// loads until it reaches gen x ncta -- no last-arriver release step, so one
// L2 round trip less than a sense-reversal barrier.  The CTA barrier orders
// every thread's writes before thread 0's release-add.  L1 is not relied
// upon across phases (phase data is read with coherent loads or after this
// acquire).  bench/gridbar.cu, 296 CTAs x 288 threads: 1.37 us per barrier
// vs 1.85 us for the sense-reversal one with a register generation
// (profiles/r02_gridbar.txt); MDOT_GRIDBAR_SENSE=1 restores that one (A/B).
#ifndef MDOT_GRIDBAR_SENSE
#define MDOT_GRIDBAR_SENSE 0
#endif
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int ncta, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
#if MDOT_GRIDBAR_SENSE
    if (atom_add_acqrel(&bar[0], 1u) == ncta - 1) {
      bar[0] = 0u;
      red_release(&bar[1], 1u);
    } else {
      while (ld_acquire(&bar[1]) == gen) __nanosleep(8);
    }
    ++gen;
#else
    ++gen;
    red_release(&bar[0], 1u);
    const unsigned int tgt = gen * ncta;
    while ((int)(ld_acquire(&bar[0]) - tgt) < 0) {
    }
#endif
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// a record wait longer than this means a peer is gone: record and fall
// through (garbage scalars, no hang; the host reports MDOT_ENCCL)
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
// Self-validating 16-byte records of the peer exchange: {lo32, ex, hi32, ex}.
// Each aligned 8-byte half {data, ex} is single-copy atomic, so a reader
// that sees `ex` in both halves holds this exchange's value (NVLink stores
// of one 16-byte vector may land as two 8-byte halves; each is checked).
__device__ __forceinline__ uint4 ll_pack(double x, unsigned int ex) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return make_uint4((unsigned int)b, ex, (unsigned int)(b >> 32), ex);
}
__device__ __forceinline__ void ll_store(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ double ll_poll(const uint4* p, unsigned int ex, int* err) {
  uint4 v;
  unsigned long long t0 = 0;
  for (;;) {
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    if (v.y == ex && v.w == ex) break;
    if (*(volatile int*)err) break;   // an earlier wait already timed out
    if (t0 == 0) t0 = global_ns();
    else if (global_ns() - t0 > kPeerTimeoutNs) {
      *err = 1;
      break;
    }
    __nanosleep(20);
  }
  return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x));
}

// Finalize partial totals of items [i_lo, i_lo + cnt): (item, sub) tasks over
// all threads (a warp always holds whole octets); every partial load of up
// to kMaxRounds rounds is issued before the first add.  tots[q] <- total.
__device__ __forceinline__ void fin_totals(const FinalizeArgs& f, int64_t i_lo, int cnt, double* tots) {
  const int tid = threadIdx.x;
  constexpr int kMaxRounds = 2;
  const int rounds = (cnt * kFinTPI + blockDim.x - 1) / blockDim.x;
  for (int r0 = 0; r0 < rounds; r0 += kMaxRounds) {
    double acc[kMaxRounds];
#pragma unroll
    for (int rr = 0; rr < kMaxRounds; ++rr) {
      acc[rr] = 0.0;
      const int task = (r0 + rr) * blockDim.x + tid;
      const int q = task / kFinTPI, sub = task % kFinTPI;
      if (r0 + rr < rounds && q < cnt) {
        const int64_t k = i_lo + q;
        const double* base;
        int64_t stride;
        int m;
        if (k < f.nrows) { base = f.rowpart + k; stride = f.nrows; m = f.n_col_tiles; }
        else { base = f.colpart + (k - f.nrows); stride = f.n; m = f.n_row_tiles; }
        double z = 0.0;
        for (int tt = sub; tt < m; tt += 4 * kFinTPI) {
          const double y0 = base[(int64_t)tt * stride];
          const double y1 = tt + kFinTPI < m ? base[(int64_t)(tt + kFinTPI) * stride] : 0.0;
          const double y2 = tt + 2 * kFinTPI < m ? base[(int64_t)(tt + 2 * kFinTPI) * stride] : 0.0;
          const double y3 = tt + 3 * kFinTPI < m ? base[(int64_t)(tt + 3 * kFinTPI) * stride] : 0.0;
          z += y0; z += y1; z += y2; z += y3;
        }
        acc[rr] = z;
      }
    }
#pragma unroll
    for (int rr = 0; rr < kMaxRounds; ++rr) {
      double x = acc[rr];
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      x += __shfl_xor_sync(0xffffffffu, x, 4);
      const int task = (r0 + rr) * blockDim.x + tid;
      const int q = task / kFinTPI, sub = task % kFinTPI;
      if (r0 + rr < rounds && q < cnt && sub == 0) tots[q] = x;
    }
  }
}

// CTA partial of the 16 scalars (fixed order: warp shuffle tree, then warps
// in order) -> out[0..15].  red: [warps][16] shared scratch.
__device__ __forceinline__ void cta_partial(const double (&v)[kNumScalars], double* red, double* out) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int q = 0; q < kNumScalars; ++q) {
    double y = v[q];
    for (int off = 16; off > 0; off >>= 1) y += __shfl_xor_sync(0xffffffffu, y, off);
    if (lane == 0) red[warp * kNumScalars + q] = y;
  }
  __syncthreads();
  if (tid < kNumScalars) {
    double y = 0.0;
    for (int w = 0; w < kTmaThreads / 32; ++w) y += red[w * kNumScalars + tid];
    out[tid] = y;
  }
}

// Sum of the ncta CTA partials in a fixed order (identical in every CTA).
// Result in fin[0..15] and, when sc != null, in sc[] (+ add_tail: rank-slot
// row scalars of the peer exchange, summed in rank order, added last).
__device__ __forceinline__ void combine_partials(const double* cta_part, int ncta, double* fin, double* sc,
                                                 const double* add_tail = nullptr, int nranks = 0, int64_t ld = 0) {
  const int tid = threadIdx.x;
  constexpr int G = 256 / kNumScalars;
  double y = 0.0;
  if (tid < 256) {
    const int q = tid % kNumScalars;
    for (unsigned b = tid / kNumScalars; b < (unsigned)ncta; b += G) y += __ldcg(&cta_part[(int64_t)b * kNumScalars + q]);
    fin[tid] = y;
  }
  __syncthreads();
  double z = 0.0;
  if (tid < kNumScalars) {
    for (int g = 0; g < G; ++g) z += fin[g * kNumScalars + tid];
    if (add_tail) {
      double t = 0.0;
      for (int p = 0; p < nranks; ++p) t += __ldcg(add_tail + (int64_t)p * ld + tid);
      z += t;
    }
  }
  __syncthreads();
  if (tid < kNumScalars) {
    fin[tid] = z;
    if (sc) sc[tid] = z;
  }
  __syncthreads();
}

// The projection loop of one instance, run by `ncta` CTAs (cta = index among
// them; the whole co-resident grid for k_persist).  Barriers, tile
// round-robin, finalize chunks and the scalar combine use (cta, ncta) only.
// A grouped variant (several instances sharing C, one slice of the grid
// each, MD steps in lockstep) measured slower than concurrent graph-path
// solves and was removed (profiles/README.md).
template <bool PEER>
__device__ __forceinline__ void persist_body(const CUtensorMap& tmap, const PersistArgs& a, const int cta,
                                             const int ncta, const PeerNet* net = nullptr,
                                             const PeerGroup* pg = nullptr) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
  PersistSmem& S = *reinterpret_cast<PersistSmem*>(smem_raw + pad);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* red = &S.tma.sred[0][0];                     // [9 warps][16]
  double* fin = red + (kTmaThreads / 32) * kNumScalars;  // [256]
  constexpr int kWords = (int)(sizeof(CtrlState) / sizeof(unsigned long long));
  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&S.tma.full[s], 1);
      mbar_init(&S.tma.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const unsigned long long* g = reinterpret_cast<const unsigned long long*>(a.ctrl);
    unsigned long long* sh = reinterpret_cast<unsigned long long*>(&S.st);
    for (int i = tid; i < kWords; i += blockDim.x) sh[i] = g[i];
  }
  __syncthreads();
  // one trace writer: CTA 0's controller copy (every CTA takes the same decisions)
  if (tid == 0 && cta != 0) S.st.trace = nullptr;
  if (warp == kConsumerWarps && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");

  const int64_t items = a.p.nrows + a.p.n;
  const int64_t gstride = (int64_t)ncta * blockDim.x;
  uint32_t it = 0;
  // producer: prefetch the first stages of the first pass right away
  const int cta_stages = tma_cta_stages(a.e, cta, ncta);
  const int pre = cta_stages < kTmaStages ? cta_stages : kTmaStages;
  TmaCursor cur{(int64_t)cta, 0};
  if (warp == kConsumerWarps && lane == 0 && cta_stages > 0) tma_produce_n(S.tma, &tmap, a.e, cur, it, pre, cta, ncta);
  // CTA 0 phase timers (%globaltimer), kept in global memory (thread 0 of CTA
  // 0 only; no registers or smem live across the loop): tm[0..3] = [ctrl+prep
  // +barrier, K1+barrier, finalize+barrier, combine], tm[4..6] finalize
  // sub-phases, tm[8] = K1 phase count, tm[9..11] = timestamps
  const bool timer = (cta == 0 && tid == 0);
  unsigned long long* tm = a.k1_ns + 2;
  if (timer) tm[9] = global_ns();
  bool first = a.initial != 0;
  unsigned int bar_gen = 0;   // grid-barrier generation (thread 0; a.gbar is zeroed before every launch)
  // peer exchange counter (every CTA of every rank counts the same exchanges)
  unsigned int epoch = 0;
  if constexpr (PEER) epoch = __ldcg(pg->epoch);
  for (long long slot = 0; slot < a.max_slots; ++slot) {
    // ---------------------------------------------------------------- ctrl
    if (!first) {
      if (tid == 0) ctrl_body(&S.st, 0, cta == 0 ? a.done_host : nullptr, nullptr);
      __syncthreads();
      if (S.st.done) {
        // the accept copy requested together with `done` still applies
        if (S.st.accept_marg || S.st.accept_pot)
          for (int64_t k = (int64_t)cta * blockDim.x + tid; k < items; k += gstride)
            prep_item(a.p, k, &S.st);
        // drain the stages the producer prefetched for a pass that will not
        // run (no TMA may still target shared memory when the CTA exits)
        if (warp < kConsumerWarps) {
          for (int q = 0; q < pre; ++q, ++it) mbar_wait(&S.tma.full[it % kTmaStages], (it / kTmaStages) & 1u);
        }
        break;
      }
    }
    first = false;
    // ---------------------------------------------------------------- prep
    for (int64_t k = (int64_t)cta * blockDim.x + tid; k < items; k += gstride) prep_item(a.p, k, &S.st);
    grid_barrier(a.gbar, ncta, bar_gen);
    if (timer) {
      const unsigned long long t0 = global_ns();
      tm[0] += t0 - tm[9];
      tm[10] = t0;
    }
    // ------------------------------------------------------------------ K1
    if (warp == kConsumerWarps) {
      // the rest of this pass, then the prefetch of the next pass's first stages
      if (lane == 0 && cta_stages > 0) {
        tma_produce_n(S.tma, &tmap, a.e, cur, it, cta_stages - pre, cta, ncta);
        tma_produce_n(S.tma, &tmap, a.e, cur, it, pre, cta, ncta);
      }
    } else {
      tma_consume_pass<true>(S.tma, a.e, it, S.st.gpair[0], S.st.gpair[1], cta, ncta);
    }
    if (a.dbg_fin && slot < 64) {
      __syncthreads();
      if (tid == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.dbg_fin[slot * ncta + cta] = (global_ns() << 8) | (smid & 255u);
      }
    }
    grid_barrier(a.gbar, ncta, bar_gen);
    if (timer) {
      const unsigned long long t1 = global_ns();
      tm[1] += t1 - tm[10];
      tm[8] += 1;
      tm[10] = t1;
    }
    // ------------------------------------------------------------ finalize
    double v[kNumScalars];
#pragma unroll
    for (int q = 0; q < kNumScalars; ++q) v[q] = 0.0;
    // this CTA's contiguous chunk of items; (item, sub) tasks over all 288
    // threads (a warp always holds whole octets), totals to smem
    const int64_t per = (items + ncta - 1) / ncta;
    const int64_t i_lo = (int64_t)cta * per;
    const int64_t i_hi = (i_lo + per < items) ? i_lo + per : items;
    const int cnt = i_hi > i_lo ? (int)(i_hi - i_lo) : 0;
    MDOT_DCHECK(cnt <= kPersistMaxChunk);
    double* tots = fin + 256;   // [cnt]
    fin_totals(a.f, i_lo, cnt, tots);
    __syncthreads();
    if (timer) tm[4] += global_ns() - tm[10];
    if constexpr (!PEER) {
      // one thread per item for the fp64 log / exp / scalar work
      for (int q = tid; q < cnt; q += blockDim.x) finalize_item(a.f, i_lo + q, tots[q], v);
      __syncthreads();
      if (timer) tm[5] += global_ns() - tm[10];
      cta_partial(v, red, a.cta_part + (int64_t)cta * kNumScalars);
      if (timer) tm[6] += global_ns() - tm[10];
      grid_barrier(a.gbar, ncta, bar_gen);
      if (timer) {
        const unsigned long long t2 = global_ns();
        tm[2] += t2 - tm[10];
        tm[11] = t2;
      }
      // every CTA combines all CTA partials in the same order -> identical scalars
      combine_partials(a.cta_part, ncta, fin, S.st.sc);
    } else {
      // F1: local rows finalize; this CTA's column totals and its row-scalar
      // partial go to slot `me` of every rank's receive block as
      // self-validating 16-byte records {lo32, ex, hi32, ex} (the exchange
      // index travels with every 8-byte half, as in NCCL's LL protocol): no
      // fence, no flag -- a fence.sc.sys costs ~6 us per CTA here
      const int me = pg->rank, R = net->nranks;
      const int64_t ld = net->ld;
      MDOT_DCHECK(me < R && R <= kMaxPeers && a.f.n + kNumScalars * (int64_t)ncta <= ld);
      const unsigned int ex = ++epoch;
      uint4* const* recv = reinterpret_cast<uint4* const*>(net->recv);
      const int64_t slot_off = ((int64_t)(ex & 1u) * R + me) * ld;
      for (int q = tid; q < cnt; q += blockDim.x) {
        const int64_t k = i_lo + q;
        if (k < a.f.nrows) {
          finalize_item(a.f, k, tots[q], v);
        } else {
          const uint4 rec = ll_pack(tots[q], ex);
          const int64_t j = k - a.f.nrows;
#pragma unroll 1
          for (int p = 0; p < R; ++p) ll_store(recv[p] + slot_off + j, rec);
        }
      }
      cta_partial(v, red, fin);   // fin[0..15] (tid < 16 wrote them)
      if (tid < kNumScalars) {
        const uint4 rec = ll_pack(fin[tid], ex);
#pragma unroll 1
        for (int p = 0; p < R; ++p) ll_store(recv[p] + slot_off + a.f.n + kNumScalars * cta + tid, rec);
      }
      if (timer) tm[5] += global_ns() - tm[10];
      // F2: replicated columns, chunked identically on every rank (the
      // scalars, and so every decision, are bitwise identical across ranks);
      // each record is polled until it carries this exchange's index
#pragma unroll
      for (int q = 0; q < kNumScalars; ++q) v[q] = 0.0;
      const uint4* rb = recv[me] + (int64_t)(ex & 1u) * R * ld;
      const int64_t per2 = (a.f.n + ncta - 1) / ncta;
      const int64_t j_lo = (int64_t)cta * per2;
      const int64_t j_hi = (j_lo + per2 < a.f.n) ? j_lo + per2 : a.f.n;
      for (int64_t j = j_lo + tid; j < j_hi; j += blockDim.x) {
        double t = 0.0;
#pragma unroll 1
        for (int p = 0; p < R; ++p) t += ll_poll(rb + (int64_t)p * ld + j, ex, pg->err);
        finalize_item(a.f, a.f.nrows + j, t, v);
      }
      cta_partial(v, red, fin);
      if (tid < kNumScalars) {
        // + the row-scalar partials of CTA slot `cta` of every rank (rank order)
        double t = 0.0;
#pragma unroll 1
        for (int p = 0; p < R; ++p) t += ll_poll(rb + (int64_t)p * ld + a.f.n + kNumScalars * cta + tid, ex, pg->err);
        a.cta_part[(int64_t)cta * kNumScalars + tid] = fin[tid] + t;
      }
      if (timer) tm[6] += global_ns() - tm[10];
      grid_barrier(a.gbar, ncta, bar_gen);
      if (timer) {
        const unsigned long long t2 = global_ns();
        tm[2] += t2 - tm[10];
        tm[11] = t2;
      }
      // identical on every rank: same partials, same order
      combine_partials(a.cta_part, ncta, fin, S.st.sc);
    }
    if (timer) {
      tm[9] = global_ns();
      tm[3] += tm[9] - tm[11];
    }
    // the per-CTA partial buffer is reused next slot: nobody may overwrite it
    // before every CTA has read it (the next write happens after two more
    // grid barriers, so no extra barrier is needed here)
  }
  // write the state back (CTA 0) and the K1 phase timing
  if (cta == 0) {
    const unsigned long long* sh = reinterpret_cast<const unsigned long long*>(&S.st);
    unsigned long long* g = reinterpret_cast<unsigned long long*>(a.ctrl);
    __syncthreads();
    for (int i = tid; i < kWords; i += blockDim.x) g[i] = sh[i];
    if (tid == 0) {
      a.k1_ns[0] = tm[1];
      a.k1_ns[1] = tm[8];
      if constexpr (PEER) *pg->epoch = epoch;
    }
  }
}

__global__ void __launch_bounds__(kTmaThreads, 2)
    k_persist(const __grid_constant__ CUtensorMap tmap, PersistArgs a) {
  persist_body<false>(tmap, a, blockIdx.x, gridDim.x);
}

// Row-sharded projection with the fused peer exchange: group = rank slot of
// this launch (one group per GPU; G groups when one GPU emulates G ranks).
__global__ void __launch_bounds__(kTmaThreads, 2) k_persist_peer(const __grid_constant__ PeerLaunch L) {
  const int grp = blockIdx.x / L.cta_per_group;
  if (grp >= L.groups) return;
  const PeerGroup& g = L.g[grp];
  persist_body<true>(*reinterpret_cast<const CUtensorMap*>(&L.tmap[grp][0]), g.a, blockIdx.x % L.cta_per_group,
                     L.cta_per_group, &L.net, &g);
}

static int g_persist_grid = -1;
static const void* persist_fn() { return (const void*)k_persist; }

int persist_grid() {
  if (g_persist_grid >= 0) return g_persist_grid;
  const int smem = (int)sizeof(PersistSmem) + 128;
  if (cudaFuncSetAttribute(persist_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
    g_persist_grid = 0;
    return 0;
  }
  cudaFuncSetAttribute(persist_fn(), cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
  int per_sm = 0, dev = 0, sms = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persist_fn(), kTmaThreads, smem) != cudaSuccess)
    per_sm = 0;
  if (getenv("MDOT_DEBUG")) {
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, persist_fn());
    fprintf(stderr, "[mdot] k_persist regs %d smem %d coop %d per_sm %d\n", at.numRegs, smem, coop, per_sm);
  }
  // the K1 pass needs 2 CTAs per SM (18 warps) to keep HBM busy; with one the
  // graph-driven path is faster, so the persistent path is used only at 2/SM
  g_persist_grid = per_sm >= 2 ? 2 * sms : 0;
  return g_persist_grid;
}

int persist_max_chunk() { return kPersistMaxChunk; }

cudaError_t launch_persist_peer(const PeerLaunch& L, cudaStream_t st) {
  const int smem = (int)sizeof(PersistSmem) + 128;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k_persist_peer, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute((const void*)k_persist_peer, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    attr = true;
  }
  void* args[] = {const_cast<PeerLaunch*>(&L)};
  return cudaLaunchCooperativeKernel((const void*)k_persist_peer, dim3(L.groups * L.cta_per_group), dim3(kTmaThreads),
                                     args, (size_t)smem, st);
}

cudaError_t launch_persist(const void* map, const PersistArgs& a, int grid, cudaStream_t st) {
  const int smem = (int)sizeof(PersistSmem) + 128;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(map);
  void* args[] = {const_cast<CUtensorMap*>(m), const_cast<PersistArgs*>(&a)};
  return cudaLaunchCooperativeKernel(persist_fn(), dim3(grid), dim3(kTmaThreads), args, (size_t)smem, st);
}

void fault_set_persist(int mode) { fault_set_tu(mode); }

}  // namespace mdot

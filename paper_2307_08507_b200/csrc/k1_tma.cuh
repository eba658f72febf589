// paper_2307_08507_b200/csrc/k1_tma.cuh -- the TMA-fed K1 pass (producer /
// consumer device functions), shared by the persistent K1 kernel
// (eval_tma.cu) and the persistent cooperative slot kernel (persist.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "entry.cuh"
#include "internal.cuh"

namespace mdot {

constexpr int kTmaRows = 32;
constexpr int kTmaStages = 3;
constexpr int kConsumerWarps = 8;
constexpr int kTmaThreads = (kConsumerWarps + 1) * 32;

struct TmaSmem {
  float stage[kTmaStages][kTmaRows][kTileN];   // 96 KiB
  double sred[kConsumerWarps][kTileN];          // 16 KiB
  unsigned long long full[kTmaStages];
  unsigned long long empty[kTmaStages];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// L2 policy for the C stream: evict_first when C is larger than L2 (keeps
// the partials and O(n) vectors resident), evict_last when C fits (C then
// stays L2-resident across evaluations).
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t pol;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                 unsigned long long* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ double shfl_xor_dd(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

__device__ __forceinline__ double warp_reduce4_t(double v0, double v1, double v2, double v3, int lane) {
  const bool up = lane & 16;
  double k0 = up ? v2 : v0, k1 = up ? v3 : v1;
  double s0 = up ? v0 : v2, s1 = up ? v1 : v3;
  k0 += shfl_xor_dd(s0, 16);
  k1 += shfl_xor_dd(s1, 16);
  const bool up2 = lane & 8;
  double kk = up2 ? k1 : k0, ss = up2 ? k0 : k1;
  kk += shfl_xor_dd(ss, 8);
  kk += shfl_xor_dd(kk, 4);
  kk += shfl_xor_dd(kk, 2);
  kk += shfl_xor_dd(kk, 1);
  return kk;
}

// Producer: one elected lane streams this CTA's tiles (round-robin over the
// persistent grid) as 32-row x 256-column TMA boxes into the stage ring.
// `it` is the running stage counter (kept across passes by the caller).
// One tile's stages (tile = tr * n_col_tiles + tc of `a`).
__device__ __forceinline__ void tma_produce_tile(TmaSmem& sm, const CUtensorMap* tmap, const EvalArgs& a,
                                                 uint32_t& it, int64_t tile, uint64_t pol_stream, uint64_t pol_keep) {
  const int nct = a.n_col_tiles;
  const int tr = (int)(tile / nct), tc = (int)(tile % nct);
  const int64_t i0 = (int64_t)tr * a.tile_m;
  int nst = a.tile_m / kTmaRows;
  if (i0 + (int64_t)nst * kTmaRows > a.nrows) nst = (int)((a.nrows - i0 + kTmaRows - 1) / kTmaRows);
  for (int k = 0; k < nst; ++k, ++it) {
    const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
    mbar_wait(&sm.empty[s], ph ^ 1u);
    mbar_expect_tx(&sm.full[s], (uint32_t)(kTmaRows * kTileN * sizeof(float)));
    tma_load_2d_hint(&sm.stage[s][0][0], tmap, tc * kTileN, (int)(i0 + k * kTmaRows), &sm.full[s],
                     tile < a.l2_res_tiles ? pol_keep : pol_stream);
  }
}

__device__ __forceinline__ void tma_produce_pass(TmaSmem& sm, const CUtensorMap* tmap, const EvalArgs& a,
                                                 uint32_t& it) {
  const uint64_t pol_stream = l2_policy(a.keep_l2 != 0), pol_keep = l2_policy(true);   // L2 residency as tma_produce_n
  const int64_t total = (int64_t)a.n_row_tiles * a.n_col_tiles;
  for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x)
    tma_produce_tile(sm, tmap, a, it, tile, pol_stream, pol_keep);
}

// Stages of C this CTA streams per pass (its tiles, round-robin over the
// ncta CTAs working on this evaluation; cta = this CTA's index among them).
__device__ __forceinline__ int tma_cta_stages(const EvalArgs& a, int cta, int ncta) {
  const int nct = a.n_col_tiles;
  const int64_t total = (int64_t)a.n_row_tiles * nct;
  const int spt = a.tile_m / kTmaRows;
  int cnt = 0;
  for (int64_t tile = cta; tile < total; tile += ncta) {
    const int64_t i0 = (int64_t)(tile / nct) * a.tile_m;
    int nst = spt;
    if (i0 + (int64_t)nst * kTmaRows > a.nrows) nst = (int)((a.nrows - i0 + kTmaRows - 1) / kTmaRows);
    cnt += nst;
  }
  return cnt;
}

// Producer over the endless sequence pass, pass, ... of this CTA's stages:
// issues `count` stages from the cursor (tile, k).  The persistent kernel
// uses it to prefetch the first stages of the next pass while the grid runs
// finalize / control / prep (C does not depend on the potentials).
struct TmaCursor {
  int64_t tile;
  int k;
};
__device__ __forceinline__ void tma_produce_n(TmaSmem& sm, const CUtensorMap* tmap, const EvalArgs& a,
                                              TmaCursor& cur, uint32_t& it, int count, int cta, int ncta) {
  // L2 residency: the first l2_res_tiles tiles are read with evict_last, so
  // they stay in L2 across evaluations when C is larger than L2
  const uint64_t pol_stream = l2_policy(a.keep_l2 != 0), pol_keep = l2_policy(true);
  const int nct = a.n_col_tiles;
  const int64_t total = (int64_t)a.n_row_tiles * nct;
  const int spt = a.tile_m / kTmaRows;
  for (int q = 0; q < count; ++q, ++it) {
    const int tr = (int)(cur.tile / nct), tc = (int)(cur.tile % nct);
    const int64_t i0 = (int64_t)tr * a.tile_m;
    int nst = spt;
    if (i0 + (int64_t)nst * kTmaRows > a.nrows) nst = (int)((a.nrows - i0 + kTmaRows - 1) / kTmaRows);
    const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
    mbar_wait(&sm.empty[s], ph ^ 1u);
    mbar_expect_tx(&sm.full[s], (uint32_t)(kTmaRows * kTileN * sizeof(float)));
    tma_load_2d_hint(&sm.stage[s][0][0], tmap, tc * kTileN, (int)(i0 + cur.k * kTmaRows), &sm.full[s],
                     cur.tile < a.l2_res_tiles ? pol_keep : pol_stream);
    if (++cur.k == nst) {
      cur.k = 0;
      cur.tile += ncta;
      if (cur.tile >= total) cur.tile = cta;   // next pass
    }
  }
}

// Consumers (warps 0..7): the fused exp-reduce over the stages of this CTA's
// tiles; row totals -> rowpart[tc][i], column totals per tile -> colpart[tr][j].
// COHERENT: the parameters were written earlier in the same (persistent)
// launch -> a plain (L1-allocating, coherent) load; the grid barrier's
// gpu-scope fence invalidates L1 between phases.  Otherwise the read-only path.
template <bool COHERENT = false>
__device__ __forceinline__ float4 ld_param(const float4* p) {
  if (COHERENT) return *p;
  return __ldg(p);
}

// Row parameters: all of a warp's rows in the tile (<= 16 stages x 4 rows)
// are loaded once at the tile start, two rows per lane, and broadcast per row
// with shuffles.  Per-stage global loads of them were the top stall of the
// pass (long scoreboard on the first use after the mbarrier wait, ~15 % of
// the warp samples; profiles/README.md) and measured 4 us slower in-solve.
//
// Tried and rejected (profiles/README.md): releasing the ring slot before the
// arithmetic (rows staged in registers; needs a proxy fence before the
// release and spills at the 96-register cap of 18 warps/SM: 190 vs 185 us
// in-solve), packed f32x2 arithmetic (186 vs 185 us).
template <bool COHERENT = false>
__device__ __forceinline__ void tma_consume_tile(TmaSmem& sm, const EvalArgs& a, uint32_t& it, float gh, float gl,
                                                 int64_t tile);

template <bool COHERENT = false>
__device__ __forceinline__ void tma_consume_pass(TmaSmem& sm, const EvalArgs& a, uint32_t& it, float gh,
                                                 float gl, int cta, int ncta) {
  const int64_t total = (int64_t)a.n_row_tiles * a.n_col_tiles;
  for (int64_t tile = cta; tile < total; tile += ncta) tma_consume_tile<COHERENT>(sm, a, it, gh, gl, tile);
}

// One tile of `a` (tile = tr * n_col_tiles + tc): the consumers' share of the pass.
template <bool COHERENT>
__device__ __forceinline__ void tma_consume_tile(TmaSmem& sm, const EvalArgs& a, uint32_t& it, float gh, float gl,
                                                 int64_t tile) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = a.n, nrows = a.nrows;
  const int nct = a.n_col_tiles;
  const int stages_per_tile = a.tile_m / kTmaRows;
  {
    const int tr = (int)(tile / nct), tc = (int)(tile % nct);
    const int64_t i0 = (int64_t)tr * a.tile_m;
    const int64_t j0 = (int64_t)tc * kTileN;
    int nst = stages_per_tile;
    if (i0 + (int64_t)nst * kTmaRows > nrows) nst = (int)((nrows - i0 + kTmaRows - 1) / kTmaRows);

    float bh[8], T[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
      if (j < n) {
        const float4 cp = ld_param<COHERENT>(&a.colp[j]);
        bh[q] = cp.x; T[q] = cp.z;
      } else {
        bh[q] = -1.0e30f; T[q] = 0.f;
      }
    }
    // column multiplier 2^bl of the column this thread writes at the tile end
    const int64_t jw = j0 + threadIdx.x;
    const float Mcol = (threadIdx.x < kTileN && jw < n) ? ld_param<COHERENT>(&a.colp[jw]).y : 0.f;
    // fp64 column accumulators live in this warp's row of sm.sred (warp-
    // private; no registers held across the tile), fp32 over 8 rows first
    float cacc32[8];
    double* csum = &sm.sred[warp][0];
#pragma unroll
    for (int q = 0; q < 8; ++q) { csum[4 * lane + (q & 3) + 128 * (q >> 2)] = 0.0; cacc32[q] = 0.f; }
#if MDOT_K1_PACKED
    // packed f32x2 entry arithmetic (entry.cuh): column pairs (2p, 2p+1)
    ColPairs cpp;
#pragma unroll
    for (int p = 0; p < 4; ++p) { cpp.bh[p] = pk2(bh[2 * p], bh[2 * p + 1]); cpp.T[p] = pk2(T[2 * p], T[2 * p + 1]); }
    u64 cacc2[4] = {0ull, 0ull, 0ull, 0ull};
    const u64 ngh2 = pk2(-gh, -gh), ngl2 = pk2(-gl, -gl);
#endif

    // lane l holds rows (stage l/2, u = 2 (l & 1) + {0, 1}) of this warp
    float4 rq0, rq1;
    {
      const int kk = lane >> 1;
      const int64_t ib = i0 + (int64_t)kk * kTmaRows + 4 * warp + 2 * (lane & 1);
      const float4 none = make_float4(-1.0e30f, 0.f, 0.f, 0.f);
      rq0 = (kk < nst && ib < nrows) ? ld_param<COHERENT>(&a.rowp[ib]) : none;
      rq1 = (kk < nst && ib + 1 < nrows) ? ld_param<COHERENT>(&a.rowp[ib + 1]) : none;
    }
    for (int k = 0; k < nst; ++k, ++it) {
      const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
      const int64_t ib = i0 + (int64_t)k * kTmaRows + 4 * warp;
      mbar_wait(&sm.full[s], ph);
      float rs[4];   // fp32 lane sums of the 4 rows
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4& q = (u & 1) ? rq1 : rq0;
        const int src = 2 * k + (u >> 1);
        const float ah = __shfl_sync(0xffffffffu, q.x, src);
        const float S = __shfl_sync(0xffffffffu, q.z, src);
        const float* row = &sm.stage[s][4 * warp + u][0];
        const float4 x0 = *reinterpret_cast<const float4*>(row + 4 * lane);
        const float4 x1 = *reinterpret_cast<const float4*>(row + 128 + 4 * lane);
#if MDOT_K1_PACKED
        const u64 c2[4] = {pk2(x0.x, x0.y), pk2(x0.z, x0.w), pk2(x1.x, x1.y), pk2(x1.z, x1.w)};
        rs[u] = entry_row8_f(c2, make_float4(ah, 0.f, S, 0.f), cpp, ngh2, ngl2, cacc2);
#else
        const float cv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        float rsum = 0.f;
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8) {
          const float cij = cv[q8];
          const float zh = fmaf(-gh, cij, ah + bh[q8]);
          const float e = ex2_fast(fmaf(-gl, cij, zh));
          rsum = fmaf(e, T[q8], rsum);
          cacc32[q8] = fmaf(e, S, cacc32[q8]);
        }
        rs[u] = rsum;
#endif
      }
      // release the slot.  The reads above are generic-proxy shared-memory
      // loads and the refill is an async-proxy (TMA) write: without this
      // proxy fence nothing stops the arrive (and the refill) from overtaking
      // loads whose data has not returned yet (ptxas may schedule their
      // consumers after the arrive).  Observed as one corrupted row at
      // n = 16384 under a different instruction schedule
      // (test_tma_kernel_bitwise_equals_generic_kernel_config4).
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
#if MDOT_K1_ROWRED_F32
      const double tot = (double)warp_reduce4_f(rs[0], rs[1], rs[2], rs[3], lane);
#else
      const double tot = warp_reduce4_t(rs[0], rs[1], rs[2], rs[3], lane);
#endif
      // row multiplier M_i = 2^al_i of the row this lane writes (u = 2 h + l)
      const int srcm = 2 * k + ((lane >> 4) & 1);
      const float m0 = __shfl_sync(0xffffffffu, rq0.y, srcm);
      const float m1 = __shfl_sync(0xffffffffu, rq1.y, srcm);
      const float Mrow = (lane & 8) ? m1 : m0;
      const int64_t i = ib + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
      if ((lane & 7) == 0 && i < nrows) a.rowpart[(int64_t)tc * nrows + i] = tot * (double)Mrow;
      if ((k % MDOT_K1_COLFLUSH) == MDOT_K1_COLFLUSH - 1) {
#if MDOT_K1_PACKED
#pragma unroll
        for (int p = 0; p < 4; ++p) { up2(cacc2[p], cacc32[2 * p], cacc32[2 * p + 1]); cacc2[p] = 0ull; }
#endif
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8) {
          csum[4 * lane + (q8 & 3) + 128 * (q8 >> 2)] += (double)cacc32[q8];
          cacc32[q8] = 0.f;
        }
      }
    }
#if MDOT_K1_PACKED
#pragma unroll
    for (int p = 0; p < 4; ++p) up2(cacc2[p], cacc32[2 * p], cacc32[2 * p + 1]);
#endif
#pragma unroll
    for (int q8 = 0; q8 < 8; ++q8) csum[4 * lane + (q8 & 3) + 128 * (q8 >> 2)] += (double)cacc32[q8];

    // column sums of this tile (8 warps, fixed order) -> partial of row tile tr
    consumer_bar();
    {
      const int tt = threadIdx.x;
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) acc += sm.sred[w][tt];
      const int64_t j = j0 + tt;
      if (j < n) a.colpart[(int64_t)tr * n + j] = acc * (double)Mcol;
    }
    consumer_bar();   // sred / last flags reused by the next tile
  }
}

// Shared-C multi-instance consumer (lockstep throughput batch,
// k_eval_tma_shared): consumer warp w evaluates instance `b` (< 0: idle) on
// ALL 32 rows of every stage of the tile, so one read of C serves up to eight
// instances per CTA.  The warp's columns belong to it alone: its column sums
// (fp32 over 16 rows, then fp64 in its private row of sm.sred) become the
// tile's column partial without a cross-warp reduction, and its row totals are
// complete per (row, column tile) after the 4-row butterfly, as in
// tma_consume_tile.  Lane l holds stage row l's parameters (one load per stage)
// and broadcasts them with shuffles.
#ifndef MDOT_SHARED_UNROLL
#define MDOT_SHARED_UNROLL 8
#endif
// 4-row group loop of the shared-C consumer, fully unrolled: lockstep batch
// 518.9 -> 507.8 ms (16 x n = 4096, paper protocol; identical evaluations;
// profiles/r02_shared_unroll_ab.txt); MDOT_SHARED_UNROLL=1: A/B
constexpr int kSharedUnroll = MDOT_SHARED_UNROLL;
__device__ __forceinline__ void tma_consume_tile_shared(TmaSmem& sm, const EvalArgs& a, int b, uint32_t& it,
                                                        int64_t tile) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = a.n, nrows = a.nrows;
  const int nct = a.n_col_tiles;
  const int tr = (int)(tile / nct), tc = (int)(tile % nct);
  const int64_t i0 = (int64_t)tr * a.tile_m;
  const int64_t j0 = (int64_t)tc * kTileN;
  int nst = a.tile_m / kTmaRows;
  if (i0 + (int64_t)nst * kTmaRows > nrows) nst = (int)((nrows - i0 + kTmaRows - 1) / kTmaRows);
  if (b < 0) {   // no instance for this warp: keep the ring protocol only
    for (int k = 0; k < nst; ++k, ++it) {
      const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
      mbar_wait(&sm.full[s], ph);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    return;
  }
  float bh[8], T[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
    if (j < n) {
      const float4 cp = __ldg(&a.colp[j]);
      bh[q] = cp.x; T[q] = cp.z;
    } else {
      bh[q] = -1.0e30f; T[q] = 0.f;
    }
  }
  ColPairs cpp;
#pragma unroll
  for (int p = 0; p < 4; ++p) { cpp.bh[p] = pk2(bh[2 * p], bh[2 * p + 1]); cpp.T[p] = pk2(T[2 * p], T[2 * p + 1]); }
  const float gh = a.gpair ? a.gpair[0] : a.gh;
  const float gl = a.gpair ? a.gpair[1] : a.gl;
  const u64 ngh2 = pk2(-gh, -gh), ngl2 = pk2(-gl, -gl);
  double* csum = &sm.sred[warp][0];
#pragma unroll
  for (int q = 0; q < 8; ++q) csum[4 * lane + (q & 3) + 128 * (q >> 2)] = 0.0;
  u64 cacc2[4] = {0ull, 0ull, 0ull, 0ull};
  int grp = 0;
  const float4 none = make_float4(-1.0e30f, 0.f, 0.f, 0.f);
  // row parameters one stage ahead (their L2 latency was the top stall:
  // long scoreboard 2.5 warps per issue, profiles/r02_shared_k1_ncu.md)
  float4 rq_next = (i0 + lane < nrows) ? __ldg(&a.rowp[i0 + lane]) : none;
  for (int k = 0; k < nst; ++k, ++it) {
    const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
    const float4 rq = rq_next;
    if (k + 1 < nst) {
      const int64_t irow = i0 + (int64_t)(k + 1) * kTmaRows + lane;
      rq_next = (irow < nrows) ? __ldg(&a.rowp[irow]) : none;
    }
    mbar_wait(&sm.full[s], ph);
#pragma unroll kSharedUnroll
    for (int g = 0; g < kTmaRows / 4; ++g) {
      float rs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rl = 4 * g + u;
        const float ah = __shfl_sync(0xffffffffu, rq.x, rl);
        const float S = __shfl_sync(0xffffffffu, rq.z, rl);
        const float* row = &sm.stage[s][rl][0];
        const float4 x0 = *reinterpret_cast<const float4*>(row + 4 * lane);
        const float4 x1 = *reinterpret_cast<const float4*>(row + 128 + 4 * lane);
        const u64 c2[4] = {pk2(x0.x, x0.y), pk2(x0.z, x0.w), pk2(x1.x, x1.y), pk2(x1.z, x1.w)};
        rs[u] = entry_row8_f(c2, make_float4(ah, 0.f, S, 0.f), cpp, ngh2, ngl2, cacc2);
      }
      const double tot = (double)warp_reduce4_f(rs[0], rs[1], rs[2], rs[3], lane);
      const int rw = 4 * g + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
      const float Mrow = __shfl_sync(0xffffffffu, rq.y, rw);
      const int64_t i = i0 + (int64_t)k * kTmaRows + rw;
      if ((lane & 7) == 0 && i < nrows) a.rowpart[(int64_t)tc * nrows + i] = tot * (double)Mrow;
      if (++grp == MDOT_K1_COLFLUSH) {
        grp = 0;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          float lo, hi;
          up2(cacc2[p], lo, hi);
          csum[4 * lane + ((2 * p) & 3) + 128 * ((2 * p) >> 2)] += (double)lo;
          csum[4 * lane + ((2 * p + 1) & 3) + 128 * ((2 * p + 1) >> 2)] += (double)hi;
          cacc2[p] = 0ull;
        }
      }
    }
    // every row of the stage has been read: release the slot (generic-proxy
    // reads before the async-proxy refill, as in tma_consume_tile)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float lo, hi;
    up2(cacc2[p], lo, hi);
    csum[4 * lane + ((2 * p) & 3) + 128 * ((2 * p) >> 2)] += (double)lo;
    csum[4 * lane + ((2 * p + 1) & 3) + 128 * ((2 * p + 1) >> 2)] += (double)hi;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
    if (j < n) a.colpart[(int64_t)tr * n + j] = csum[4 * lane + (q & 3) + 128 * (q >> 2)] * (double)__ldg(&a.colp[j]).y;
  }
}

}  // namespace mdot

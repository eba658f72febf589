// paper_2307_08507_b200/csrc/batch.cu -- K8: batched MDOT solver for many
// independent (r, c) pairs sharing one cost (BASELINE config 2, the MNIST-
// shaped batch; "including as a batch process").
//
// One CTA (8 warps) per instance runs the WHOLE solve on-chip: MD loop
// (Alg. 1), PNCG / Sinkhorn projections with the device controller
// (ops.cuh ctrl_body), the fused row+column evaluation, and the final
// rounding + cost.  Every O(n) vector of the instance lives in
// shared memory (14 x 2n doubles + exponent parameters); C (n x n fp32, shared
// by all instances) is streamed from L2.  Instances converge independently;
// no cross-CTA communication, no host involvement until the batch is done.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/mdot.h"
#include "entry.cuh"
#include "internal.cuh"
#include "ops.cuh"

namespace mdot {

namespace cg = cooperative_groups;

// MDOT_K8_TAIL_REGULAR=1 (A/B): keep the regular 256-column mapping for the
// narrow last tile
__constant__ int g_k8_tail_regular = 0;
__device__ __forceinline__ bool batch_tail_regular() { return g_k8_tail_regular != 0; }

// 16 warps: one CTA per instance has an SM to itself and its evaluation is
// latency-bound (8 warps: 2 per scheduler, 13 % issue utilisation); the
// column-partial scratch stays [8][256] (two-round reduction)
constexpr int kBatchThreads = 512;
constexpr int kBatchWarps = kBatchThreads / 32;
constexpr int kSredRows = 8;

__device__ __forceinline__ float bex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double bshx(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ double bred4(double v0, double v1, double v2, double v3, int lane) {
  const bool up = lane & 16;
  double k0 = up ? v2 : v0, k1 = up ? v3 : v1;
  double s0 = up ? v0 : v2, s1 = up ? v1 : v3;
  k0 += bshx(s0, 16);
  k1 += bshx(s1, 16);
  const bool up2 = lane & 8;
  double kk = up2 ? k1 : k0, ss = up2 ? k0 : k1;
  kk += bshx(ss, 8);
  kk += bshx(kk, 4);
  kk += bshx(kk, 2);
  kk += bshx(kk, 1);
  return kk;
}

// deterministic block reduction of NS doubles (all threads call; result in out)
template <int NS>
__device__ __forceinline__ void block_sum(double (&v)[NS], double* scratch /*[kBatchWarps][NS]*/, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (NS == 16) {
    // reduce-scatter butterfly: each stage halves the values a lane holds (the
    // half it keeps is chosen by its lane bit) and adds the partner's other
    // half -- 16 + 8 + 4 + 2 + 1 = 31 fp64 shuffles instead of 16 x 5 = 80;
    // after the stages lane l (l < 16 after the last) holds scalar q(l) summed
    // over the warp in a fixed order
    double a[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) a[q] = v[q];
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      const int half = 8 >> st;            // values kept after this stage
      const int off = 16 >> st;            // partner lane distance
      const bool up = lane & off;
#pragma unroll
      for (int q = 0; q < half; ++q) {
        const double send = up ? a[q] : a[q + half];
        const double keep = up ? a[q + half] : a[q];
        a[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    // one value per lane: scalar index from the lane bits 16, 8, 4, 2 (bit 1 pairs stay to be added)
    const double x = a[0] + __shfl_xor_sync(0xffffffffu, a[0], 1);
    const int q = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
    if ((lane & 1) == 0) scratch[warp * NS + q] = x;
  } else {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      double x = v[q];
      for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      if (lane == 0) scratch[warp * NS + q] = x;
    }
  }
  __syncthreads();
  if (threadIdx.x < NS) {
    double x = 0.0;
    for (int w = 0; w < kBatchWarps; ++w) x += scratch[w * NS + threadIdx.x];
    out[threadIdx.x] = x;
  }
  __syncthreads();
}

struct BatchSmem;
__host__ __device__ inline size_t batch_smem_bytes_d(int n);
struct BatchSmem {
  // arrays of 2n doubles (rows then columns) follow in dynamic smem
  CtrlState st;
  double out[kNumScalars];
  double sred[kSredRows][kTileN];   // column partials of batch_eval; block_sum scratch otherwise
};

__host__ __device__ inline size_t batch_smem_bytes_d(int n) {
  return sizeof(BatchSmem) + (size_t)15 * 2 * n * sizeof(double) + (size_t)2 * n * 16;
}

// Fused evaluation of one instance: rowtot[i] = sum_j 2^w T_j and
// coltot[j] = sum_i 2^w S_i (anchored units, internal.cuh "K1 numerics").
// F64: w assembled and exponentiated in fp64 (fp64-entry mode, eps < 1e-7,
// and the range-guard fallback).
// Narrow last column tile (w = n - j0 <= 64 columns, fp32 entries, packed
// arithmetic): the regular mapping gives every lane 8 columns of ONE row, so
// a 16-column tail (n = 784 = 3 x 256 + 16, config 2) would keep 28 of 32
// lanes idle for a full tile's worth of row steps.  Here Lp = pow2ceil(w/8)
// lanes share a row (8 columns each) and a warp step covers 32/Lp rows; rows
// follow the cluster split of batch_eval (64-row blocks, block b to CTA
// b % CL), so row totals stay with their owner.  Column sums: per lane over
// its rows, fp32 over 16 rows then fp64, then the lanes of one column group
// (shuffles) and the warps (shared memory) in a fixed order.
__device__ void batch_eval_tail_packed(const float* __restrict__ C, int n, int j0, const float4* prm, float gh,
                                       float gl, double* rowtot, double* coltot, double (*sred)[kTileN], int q_rank,
                                       int CL) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4* rowp = prm;
  const float4* colp = prm + n;
  const int w = n - j0;
  int Lp = 1;
  while (8 * Lp < w) Lp *= 2;                 // lanes per row (<= 8)
  const int R = 32 / Lp;                      // rows per warp step
  const int rr = lane / Lp, cl = lane % Lp;   // this lane's row slot and column group
  const int jc = j0 + 8 * cl;                 // first of this lane's 8 columns
  // column pairs of this lane (masked past n)
  ColPairs cpp;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float b2[2], t2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = jc + 2 * p + h;
      if (j < n) { const float4 c = colp[j]; b2[h] = c.x; t2[h] = c.z; }
      else { b2[h] = -1.0e30f; t2[h] = 0.f; }
    }
    cpp.bh[p] = pk2(b2[0], b2[1]);
    cpp.T[p] = pk2(t2[0], t2[1]);
  }
  const u64 ngh2 = pk2(-gh, -gh), ngl2 = pk2(-gl, -gl);
  u64 cacc2[4] = {0ull, 0ull, 0ull, 0ull};
  double c64[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) c64[k] = 0.0;
  // rows owned by this CTA: 64-row blocks b = q_rank + CL m
  const int nblk = (n + 63) / 64;
  const int own_blocks = (nblk - q_rank + CL - 1) / CL;
  const int own_rows = own_blocks * 64;        // row slots (some past n)
  int fl = 0;
  for (int base = warp * R; base < own_rows; base += R * kBatchWarps) {
    const int slot = base + rr;
    const int i = 64 * (q_rank + CL * (slot / 64)) + (slot % 64);
    const bool ok = slot < own_rows && i < n;
    float4 rp = make_float4(-1.0e30f, 0.f, 0.f, 0.f);
    u64 c2[4] = {0ull, 0ull, 0ull, 0ull};
    if (ok) {
      rp = rowp[i];
      const float* crow = C + (int64_t)i * n;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int j = jc + 2 * p;
        const float x0 = (j < n) ? __ldg(crow + j) : 0.f;
        const float x1 = (j + 1 < n) ? __ldg(crow + j + 1) : 0.f;
        c2[p] = pk2(x0, x1);
      }
    }
    float rsum = entry_row8_f(c2, rp, cpp, ngh2, ngl2, cacc2);
    // the Lp lanes of this row: xor 1 .. Lp/2 (fixed tree)
    for (int off = 1; off < Lp; off <<= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, off);
    if (ok && cl == 0) {
      const double v = (double)rsum * (double)rp.y;   // times M_i
      rowtot[i] = (j0 == 0) ? v : rowtot[i] + v;
    }
    if (++fl == 4) {   // 4 steps of fp32 column sums -> fp64
      fl = 0;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float lo, hi;
        up2(cacc2[p], lo, hi);
        c64[2 * p] += (double)lo;
        c64[2 * p + 1] += (double)hi;
        cacc2[p] = 0ull;
      }
    }
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float lo, hi;
    up2(cacc2[p], lo, hi);
    c64[2 * p] += (double)lo;
    c64[2 * p + 1] += (double)hi;
  }
  // lanes with the same column group: xor Lp, 2 Lp, .. 16 (fixed tree)
#pragma unroll
  for (int k = 0; k < 8; ++k)
    for (int off = Lp; off < 32; off <<= 1) c64[k] += __shfl_xor_sync(0xffffffffu, c64[k], off);
  // warps in a fixed order through the shared scratch (two rounds, as batch_eval)
  if (rr == 0 && warp >= kSredRows) {
#pragma unroll
    for (int k = 0; k < 8; ++k) sred[warp - kSredRows][8 * cl + k] = c64[k];
  }
  __syncthreads();
  if (rr == 0 && warp < kSredRows) {
#pragma unroll
    for (int k = 0; k < 8; ++k) sred[warp][8 * cl + k] = c64[k] + sred[warp][8 * cl + k];
  }
  __syncthreads();
  if (threadIdx.x < 8 * Lp) {
    const int t = threadIdx.x;
    MDOT_DCHECK(t < kTileN);
    double acc = 0.0;
#pragma unroll
    for (int ww = 0; ww < kSredRows; ++ww) acc += sred[ww][t];
    if (j0 + t < n) coltot[j0 + t] = acc * (double)colp[j0 + t].y;   // times M_j
  }
  __syncthreads();
}

// fp64-entry evaluation: exponents below this (relative to the entry's
// anchor 2^(rho_i + sig_j) ~ sqrt(r_i c_j)) contribute < 1e-26 of that scale
// and are not exponentiated.  The finalize range guard (f64_tot_min) redoes
// an evaluation exactly whenever a total is small enough that the skipped
// entries could exceed 1e-16 of it
#ifndef MDOT_F64_SKIP_Z
#define MDOT_F64_SKIP_Z -60.0
#endif
constexpr double kF64SkipZ = MDOT_F64_SKIP_Z;

// Narrow last tile (<= 64 columns), fp64 entries: the lane layout of
// batch_eval_tail_packed (Lp lanes per row, 8 columns each, 32 / Lp rows per
// warp step, the same 64-row cluster blocks) with the exact fp64 entry of
// batch_eval.  Config 1 (n = 64) is one such tile: the regular layout kept
// 16 of 32 lanes busy on 4 columns each.  Column sums fp64 per lane, then the
// lanes of one column group and the warps in a fixed order.
template <typename CT>
__device__ void batch_eval_tail_f64(const CT* __restrict__ C, int n, int j0, const float4* prm, double gbar,
                                    double* rowtot, double* coltot, double (*sred)[kTileN], int q_rank, int CL,
                                    double skip_z) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4* rowp = prm;
  const float4* colp = prm + n;
  const int w = n - j0;
  int Lp = 1;
  while (8 * Lp < w) Lp *= 2;                 // lanes per row (<= 8)
  const int R = 32 / Lp;                      // rows per warp step
  const int rr = lane / Lp, cl = lane % Lp;
  const int jc = j0 + 8 * cl;
  // anchors are small integers: (double)rho_i + (double)sig_j is exact and
  // equals batch_eval's (double)(rho_i + sig_j), without a conversion per entry
  double Bd[8], Td[8], Wd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = jc + q;
    if (j < n) {
      const float4 cp = colp[j];
      Bd[q] = *reinterpret_cast<const double*>(&cp.x); Td[q] = (double)cp.z; Wd[q] = (double)cp.w;
    } else {
      Bd[q] = 0.0; Td[q] = 0.0; Wd[q] = 0.0;
    }
  }
  double c64[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) c64[k] = 0.0;
  const int nblk = (n + 63) / 64;
  const int own_blocks = (nblk - q_rank + CL - 1) / CL;
  const int own_rows = own_blocks * 64;
  for (int base = warp * R; base < own_rows; base += R * kBatchWarps) {
    const int slot = base + rr;
    const int i = 64 * (q_rank + CL * (slot / 64)) + (slot % 64);
    const bool ok = slot < own_rows && i < n;
    double rsum = 0.0;
    if (ok) {
      const float4 rp = rowp[i];
      const double Ai = *reinterpret_cast<const double*>(&rp.x);
      const double rw = (double)rp.w, rz = (double)rp.z;
      const CT* crow = C + (int64_t)i * n;
      CT cv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) cv[q] = (jc + q < n) ? __ldg(crow + jc + q) : (CT)0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (jc + q < n) {
          const double z = (Ai + Bd[q]) - gbar * (double)cv[q] - (rw + Wd[q]) * LN2_D;
          if (z > skip_z) {
            const double e = exp(z);
            rsum += e * Td[q];
            c64[q] += e * rz;
          }
        }
      }
    }
    for (int off = 1; off < Lp; off <<= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, off);
    if (ok && cl == 0) rowtot[i] = (j0 == 0) ? rsum : rowtot[i] + rsum;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k)
    for (int off = Lp; off < 32; off <<= 1) c64[k] += __shfl_xor_sync(0xffffffffu, c64[k], off);
  if (rr == 0 && warp >= kSredRows) {
#pragma unroll
    for (int k = 0; k < 8; ++k) sred[warp - kSredRows][8 * cl + k] = c64[k];
  }
  __syncthreads();
  if (rr == 0 && warp < kSredRows) {
#pragma unroll
    for (int k = 0; k < 8; ++k) sred[warp][8 * cl + k] = c64[k] + sred[warp][8 * cl + k];
  }
  __syncthreads();
  if (threadIdx.x < 8 * Lp) {
    const int t = threadIdx.x;
    double acc = 0.0;
#pragma unroll
    for (int ww = 0; ww < kSredRows; ++ww) acc += sred[ww][t];
    if (j0 + t < n) coltot[j0 + t] = acc;
  }
  __syncthreads();
}

// Cluster split (CL CTAs per instance, q = this CTA's rank): the CTA takes
// the row groups ib = 4 (q W + w) + 4 W CL m; row totals are complete for
// its rows, column totals are partial over them (combined by the caller).
// R4: n % 4 == 0, so every row of a 4-row group exists (no per-row guards)
template <bool F64, bool PACKED, typename CT, bool R4 = false>
__device__ void batch_eval(const CT* __restrict__ C, int n, const float4* prm, float gh, float gl, double g2,
                           double gbar, double* rowtot, double* coltot, double (*sred)[kTileN], int q_rank,
                           int CL, double skip_z = -INFINITY, unsigned long long* dbgp = nullptr) {
#ifdef MDOT_DIAG_K8
  // sub-phase clocks of thread 0 (MDOT_DEBUG_K8): [5] tile main loops, [6] tile epilogues + tail tile
  unsigned long long dt0 = (dbgp && threadIdx.x == 0) ? clock64() : 0ull;
#define K8_SUB(slot)                                   \
  if (dbgp && threadIdx.x == 0) {                      \
    const unsigned long long dt1 = clock64();          \
    dbgp[slot] += dt1 - dt0;                           \
    dt0 = dt1;                                         \
  }
#else
#define K8_SUB(slot)
#endif
  static_assert(kBatchWarps == 2 * kSredRows, "two-round column reduction");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4* rowp = prm;
  const float4* colp = prm + n;
  const bool vec4 = (n % 4) == 0 && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  for (int j0 = 0; j0 < n; j0 += kTileN) {
    if (!F64 && PACKED && sizeof(CT) == 4 && n - j0 <= 64 && !batch_tail_regular()) {
      batch_eval_tail_packed(reinterpret_cast<const float*>(C), n, j0, prm, gh, gl, rowtot, coltot, sred, q_rank, CL);
      continue;
    }
    if (F64 && n - j0 <= 64 && !batch_tail_regular()) {
      batch_eval_tail_f64<CT>(C, n, j0, prm, gbar, rowtot, coltot, sred, q_rank, CL, skip_z);
      continue;
    }
    float bh[8], T[8];
    double Bd[F64 ? 8 : 1];
    double Wd[F64 ? 8 : 1];   // integer anchors sig_j (exact in fp64; see batch_eval_tail_f64)
    int jj[8];
    if (!F64) {
      // column parameters from shared memory: lane l's quad starts 64 B after
      // lane l-1's, so lanes l and l+2 hit the same banks (4-way conflict, 9 %
      // of the warp samples); each lane visits its quad rotated by (l/2) mod 4
      // and the values are put back in column order with static selects
      const int rot = (lane >> 1) & 3;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 t4[4];
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
          const int j = j0 + 4 * lane + ((s4 + rot) & 3) + 128 * h;
          t4[s4] = (j < n) ? colp[j] : make_float4(-1.0e30f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int src = (q - rot) & 3;
          const float4 v = src == 0 ? t4[0] : (src == 1 ? t4[1] : (src == 2 ? t4[2] : t4[3]));
          bh[4 * h + q] = v.x;
          T[4 * h + q] = v.z;
          jj[4 * h + q] = j0 + 4 * lane + q + 128 * h;
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
        jj[q] = j;
        if (j < n) {
          const float4 cp = colp[j];
          bh[q] = cp.x; T[q] = cp.z;
          Bd[q & (F64 ? 7 : 0)] = *reinterpret_cast<const double*>(&cp.x); Wd[q & (F64 ? 7 : 0)] = (double)cp.w;
        } else {
          bh[q] = -1.0e30f; T[q] = 0.f;
          Bd[q & (F64 ? 7 : 0)] = 0.0; Wd[q & (F64 ? 7 : 0)] = 0.0;
        }
      }
    }
    float c32[8];
    double c64[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { c32[q] = 0.f; c64[q] = 0.0; }
    // packed column parameters and fp32 column-pair accumulators (fp32 entries)
    ColPairs cpp;
    u64 cacc2[4] = {0ull, 0ull, 0ull, 0ull};
    const u64 ngh2 = pk2(-gh, -gh), ngl2 = pk2(-gl, -gl);
    if (!F64) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        cpp.bh[p] = pk2(bh[2 * p], bh[2 * p + 1]);
        cpp.T[p] = pk2(T[2 * p], T[2 * p + 1]);
      }
    }
    int step = 0;
    // the 4 rows' C values (L2) are loaded before any is used: with 8 warps
    // per SM the per-row loads were exposed (long-scoreboard stalls on their
    // first use: 32 % of the warp samples)
    // full 256-column tile, whole 4-row groups (n % 4 == 0), aligned fp32 C:
    // two float4 loads per row from one base pointer, no per-row bounds tests
    // (the general path below spent ~90 issue slots per 4-row step on them)
    const bool fast_tile = sizeof(CT) == 4 && vec4 && (n % 4) == 0 && j0 + kTileN <= n;
    auto load_group = [&](int ib, CT (&cvg)[4][8]) {
      if (fast_tile) {
        const float* base = reinterpret_cast<const float*>(C) + (int64_t)ib * n + j0 + 4 * lane;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 x0 = __ldg(reinterpret_cast<const float4*>(base + (int64_t)u * n));
          const float4 x1 = __ldg(reinterpret_cast<const float4*>(base + (int64_t)u * n + 128));
          cvg[u][0] = x0.x; cvg[u][1] = x0.y; cvg[u][2] = x0.z; cvg[u][3] = x0.w;
          cvg[u][4] = x1.x; cvg[u][5] = x1.y; cvg[u][6] = x1.z; cvg[u][7] = x1.w;
        }
        return;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ib + u;
        if (i < n) {
          const CT* crow = C + (int64_t)i * n;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const int j = jj[4 * g];
            if (sizeof(CT) == 4 && vec4 && j + 3 < n) {
              const float4 x = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(crow) + j));
              cvg[u][4 * g] = x.x; cvg[u][4 * g + 1] = x.y; cvg[u][4 * g + 2] = x.z; cvg[u][4 * g + 3] = x.w;
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) cvg[u][4 * g + q] = (j + q < n) ? __ldg(crow + j + q) : 0.f;
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) cvg[u][q] = 0.f;
        }
      }
    };
    for (int ib = 4 * (warp + q_rank * kBatchWarps); ib < n; ib += 4 * kBatchWarps * CL, ++step) {
      CT cvc[4][8];
      load_group(ib, cvc);
      double rs[4];    // fp64 entries
      float rsf[4];    // fp32 entries (no fp64 round trip before the fp32 row butterfly)
      float mrow[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ib + u;
        CT cv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cv[q] = cvc[u][q];
        const float4 rp = (R4 || i < n) ? rowp[i] : make_float4(-1.0e30f, 0.f, 0.f, 0.f);
        if (!F64 && !PACKED) {
          float rsum = 0.f;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float zh = fmaf(-gh, cv[q], rp.x + bh[q]);
            const float e = bex2(fmaf(-gl, cv[q], zh));
            rsum = fmaf(e, T[q], rsum);
            c32[q] = fmaf(e, rp.z, c32[q]);
          }
          rsf[u] = rsum;
          mrow[u] = rp.y;
        } else if (!F64) {
          // fp32 entries, parameter slots {ah, M, S'} / {bh, M, T'} (ops.cuh
          // split_param), on fp32 pairs (entry.cuh): the evaluation is
          // issue-bound once 16 warps hide the load latency (ncu: 54 % issue)
          u64 c2[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) c2[p] = pk2(cv[2 * p], cv[2 * p + 1]);
#if MDOT_K1_ROWRED_F32
          rsf[u] = entry_row8_f(c2, rp, cpp, ngh2, ngl2, cacc2);
#else
          rs[u] = entry_row8(c2, rp, cpp, ngh2, ngl2, cacc2);
#endif
          mrow[u] = rp.y;
        } else {
          // fp64 entries: exact z = A_i + B_j - gbar C_ij, anchored by the
          // integer (rho_i + sig_j) ln 2, fp64 exp
          double rsum = 0.0;
          const double Ai = *reinterpret_cast<const double*>(&rp.x);
          const double rw = (double)rp.w;
          const bool rowok = i < n;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (rowok && jj[q] < n) {
              const double z = (Ai + Bd[q]) - gbar * (double)cv[q] - (rw + Wd[q]) * LN2_D;
              // entries below e^kF64SkipZ of their anchor scale (P_ij < 1e-26
              // sqrt(r_i c_j)) are dropped without calling exp: at gbar ~ 4096
              // that is most of the matrix, and whole warps skip the exp
              if (z > skip_z) {
                const double e = exp(z);
                rsum += e * (double)T[q];
                c64[q] += e * (double)rp.z;
              }
            }
          }
          rs[u] = rsum;
        }
      }
      // fp32 entries: rs are fp32 values, reduced across the warp in fp32
      // (MDOT_K1_ROWRED_F32); fp64 entries keep the fp64 butterfly
      double tot;
      if (F64) {
        tot = bred4(rs[0], rs[1], rs[2], rs[3], lane);
      } else if (MDOT_K1_ROWRED_F32) {
        tot = (double)warp_reduce4_f(rsf[0], rsf[1], rsf[2], rsf[3], lane);
      } else if (PACKED) {
        tot = bred4(rs[0], rs[1], rs[2], rs[3], lane);
      } else {
        tot = bred4((double)rsf[0], (double)rsf[1], (double)rsf[2], (double)rsf[3], lane);
      }
      const int i = ib + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
      MDOT_DCHECK(i >= 0 && (i < n || i >= ib));
      if (!F64) tot *= (double)((lane & 16) ? ((lane & 8) ? mrow[3] : mrow[2]) : ((lane & 8) ? mrow[1] : mrow[0]));
      if ((lane & 7) == 0 && i < n) rowtot[i] = (j0 == 0) ? tot : rowtot[i] + tot;
      if (!F64 && (step % MDOT_K1_COLFLUSH) == MDOT_K1_COLFLUSH - 1) {
        if (PACKED) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            float lo, hi;
            up2(cacc2[p], lo, hi);
            c64[2 * p] += (double)lo;
            c64[2 * p + 1] += (double)hi;
            cacc2[p] = 0ull;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) { c64[q] += (double)c32[q]; c32[q] = 0.f; }
        }
      }
    }
    K8_SUB(5)
    if (!F64 && PACKED) {
#pragma unroll
      for (int p = 0; p < 4; ++p) up2(cacc2[p], c32[2 * p], c32[2 * p + 1]);
    }
    // column totals, fixed order: warp w + 8 parks its sums, warp w adds its
    // own, then 256 threads add the 8 rows
    if (warp >= kSredRows) {
#pragma unroll
      for (int q = 0; q < 8; ++q) sred[warp - kSredRows][4 * lane + (q & 3) + 128 * (q >> 2)] = c64[q] + (double)c32[q];
    }
    __syncthreads();
    if (warp < kSredRows) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double& x = sred[warp][4 * lane + (q & 3) + 128 * (q >> 2)];
        x = (c64[q] + (double)c32[q]) + x;
      }
    }
    __syncthreads();
    if (threadIdx.x < kTileN) {
      const int t = threadIdx.x;
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < kSredRows; ++w) acc += sred[w][t];
      if (j0 + t < n) coltot[j0 + t] = F64 ? acc : acc * (double)colp[j0 + t].y;   // fp32: times M_j = 2^bl_j
    }
    __syncthreads();
    K8_SUB(6)
  }
#undef K8_SUB
}

// C read as fp32 (DENSE_F32) or fp64 (DENSE_F64: fp64 entries only)
__device__ __forceinline__ double batch_cost(const BatchArgs& a, int64_t idx) {
  return a.C64 ? __ldg(a.C64 + idx) : (double)__ldg(a.C + idx);
}

// Cluster exchange after a split evaluation: every CTA of the instance ends
// with the full [rowtot | coltot]: row totals copied from the owning CTA,
// column totals summed over the CTAs in rank order 0..CL-1 (the same bits in
// every CTA, so every CTA's controller takes the same decisions).  Peers'
// partials are read through DSMEM between two cluster barriers, then written.
constexpr int kBatchMaxItemsPerThread = 4;   // 2n <= 4 x 512
__device__ __forceinline__ void cluster_combine(cg::cluster_group& cl, double* tot, int n, int q_rank, int CL) {
  const int n2 = 2 * n;
  double vals[kBatchMaxItemsPerThread];
  cl.sync();   // every CTA's partials are complete
#pragma unroll
  for (int m = 0; m < kBatchMaxItemsPerThread; ++m) {
    const int k = threadIdx.x + m * blockDim.x;
    vals[m] = 0.0;
    if (k < n2) {
      if (k < n) {
        const int owner = (k / (4 * kBatchWarps)) % CL;
        vals[m] = owner == q_rank ? tot[k] : *cl.map_shared_rank(tot + k, owner);
      } else {
        double y = 0.0;
        for (int q = 0; q < CL; ++q) y += (q == q_rank) ? tot[k] : *cl.map_shared_rank(tot + k, q);
        vals[m] = y;
      }
    }
  }
  cl.sync();   // every peer read is done before anyone overwrites its partials
#pragma unroll
  for (int m = 0; m < kBatchMaxItemsPerThread; ++m) {
    const int k = threadIdx.x + m * blockDim.x;
    if (k < n2) tot[k] = vals[m];
  }
  __syncthreads();
}

template <bool PACKED, typename CT>
__global__ void __launch_bounds__(kBatchThreads, 1) k_batch_solve(BatchArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BatchSmem& S = *reinterpret_cast<BatchSmem*>(smem_raw);
  const int n = a.n, n2 = 2 * a.n, tid = threadIdx.x;
#ifdef MDOT_CHECKED
  {  // the dynamic allocation must cover every vector of the instance
    unsigned int dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    MDOT_DCHECK((size_t)dyn >= batch_smem_bytes_d(n));
  }
#endif
  // CL CTAs (a thread-block cluster) per instance; CL = 1 without a cluster launch
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int q_rank = (int)cluster.block_rank();
  const int b = blockIdx.x / CL;
  double* D = reinterpret_cast<double*>(smem_raw + sizeof(BatchSmem));
  double* logt = D;            // log r | log c
  double* tgt = D + 1 * n2;    // r | c
  double* anc = D + 2 * n2;    // anchors rho | sig
  double* UV = D + 3 * n2;     // cumulative potentials U | V
  double* uv = D + 4 * n2;     // step potentials u | v
  double* tuv = D + 5 * n2;    // trial potentials
  double* p = D + 6 * n2;
  double* pprev = D + 7 * n2;
  double* cl = D + 8 * n2;     // current log marginals, s, grad
  double* cs = D + 9 * n2;
  double* cg = D + 10 * n2;
  double* tl = D + 11 * n2;    // trial log marginals, s, grad
  double* ts = D + 12 * n2;
  double* tg = D + 13 * n2;
  double* tot = D + 14 * n2;   // [2n] rowtot | coltot
  float4* prm = reinterpret_cast<float4*>(D + 15 * n2);   // [2n]

  // ---- setup (a1): targets, logs, anchors; U = log r, V = log c; u = v = 0
  for (int k = tid; k < n2; k += blockDim.x) {
    const double x = (k < n) ? a.r[(int64_t)b * n + k] : a.c[(int64_t)b * n + (k - n)];
    tgt[k] = x;
    const double lx = log(x);
    logt[k] = lx;
    double an = rint(0.5 * lx * L2E_D);
    anc[k] = an < -60.0 ? -60.0 : (an > 0.0 ? 0.0 : an);
    UV[k] = a.p0_ones ? 0.0 : lx;
    uv[k] = 0.0;
  }
  __syncthreads();

  PrepArgs pa{};
  pa.n = n; pa.nrows = n;
  pa.U = UV; pa.V = UV + n; pa.u = uv; pa.v = uv + n; pa.tu = tuv; pa.tv = tuv + n;
  pa.p = p; pa.pprev = pprev; pa.lm = cl;
  pa.logr = logt; pa.logc = logt + n; pa.rho_r = anc; pa.sig_c = anc + n;
  pa.rowp = prm; pa.colp = prm + n; pa.flag = nullptr;
  pa.f64_params = a.f64;
  pa.cur_lm = cl; pa.cur_m = nullptr; pa.cur_s = cs; pa.cur_g = cg;
  pa.tr_lm = tl; pa.tr_m = nullptr; pa.tr_s = ts; pa.tr_g = tg;
  FinalizeArgs fa{};
  fa.n = n; fa.nrows = n; fa.from_partials = 1;
  fa.rho_r = anc; fa.sig_c = anc + n;
  fa.r = tgt; fa.c = tgt + n; fa.logr = logt; fa.logc = logt + n;
  fa.gcur = cg; fa.pcur = p;
  fa.lm = tl; fa.m = nullptr; fa.s = ts; fa.g = tg;
  fa.jacobi = a.projector == MDOT_PROJ_PNCG_JACOBI;
  fa.fault_repl = CL;   // every CTA of the cluster finalizes every item (identical decisions)

  long long evals_total = 0, iters = 0, ls_evals = 0, resets = 0, restarts = 0;
  int status = 0;
  double gbar = 0.0, gprev = 0.0, l1 = 0.0, rho = 0.0;
  int t_done = 0;
  // ADAPTIVE schedule (Z29): the next step from this step's evaluation count
  double next = a.adaptive ? a.gamma1 : 0.0, eta_prev = 0.0;
  int final_next = a.adaptive && a.gamma1 >= a.gamma_bar;
  for (int t = 1; a.adaptive || t <= a.T; ++t) {
    const double gt = a.adaptive ? next : a.gammas[t - 1];
    const bool last = a.adaptive ? final_next != 0 : t == a.T;
    gbar = (a.adaptive && last) ? a.gamma_bar : gbar + gt;
    if (tid == 0 && q_rank == 0 && t <= 64) a.res[b].gammas[t - 1] = gt;
    const double g2 = gbar * L2E_D;
    const float gh = (float)g2, gl = (float)(g2 - (double)(float)g2);
    // warm start (Z4)
    if (a.warm == MDOT_WARM_ZERO) {
      for (int k = tid; k < n2; k += blockDim.x) uv[k] = 0.0;
    } else if (a.warm == MDOT_WARM_SCALED && t > 1 && gt != gprev) {
      const double w = gt / gprev;
      for (int k = tid; k < n2; k += blockDim.x) uv[k] *= w;
    }
    // controller state for this projection
    if (tid == 0) {
      CtrlState& h = S.st;
      memset(&h, 0, sizeof(CtrlState));
      h.eps = last ? a.eps : a.eps_md; h.c1 = a.c1; h.c2 = a.c2; h.noise = ls_noise(a.f64 != 0, gbar);
      h.stop_rho = a.stop_rho; h.ncg = a.projector == MDOT_PROJ_NCG; h.sinkhorn = a.projector == MDOT_PROJ_SINKHORN;
      h.beta_kind = a.beta_kind; h.ls_max_trials = a.ls_max_trials;
      h.max_evals = a.max_evals - evals_total;
      h.mode = PREP_CUR; h.phase = 0; h.alpha_prev = 1.0;
      h.md_t = t;
      if (a.trace && b == 0 && q_rank == 0) {   // one writer: instance 0, cluster rank 0
        h.trace = a.trace; h.trace_len = a.trace_len; h.trace_cap = a.trace_cap;
      }
    }
    __syncthreads();
    bool first = true;
    for (;;) {
#ifdef MDOT_DIAG_K8
      const bool dg = a.dbg && b == 0 && q_rank == 0 && tid == 0;
      unsigned long long d0 = dg ? clock64() : 0ull;
#define K8_MARK(slot)                                     \
  if (dg) {                                               \
    const unsigned long long d1 = clock64();              \
    a.dbg[slot] += d1 - d0;                               \
    d0 = d1;                                              \
  }
#else
#define K8_MARK(slot)
#endif
      if (!first) {
        if (tid == 0) ctrl_body(&S.st, 0, nullptr, nullptr);
        __syncthreads();
        K8_MARK(0)
        if (S.st.done) {
          if (S.st.accept_marg || S.st.accept_pot)
            for (int k = tid; k < n2; k += blockDim.x) prep_item(pa, k, &S.st);
          __syncthreads();
          break;
        }
      }
      first = false;
      for (int k = tid; k < n2; k += blockDim.x) prep_item(pa, k, &S.st);
      __syncthreads();
      K8_MARK(1)
      bool use64 = a.f64 != 0;
      double skip_z = kF64SkipZ;   // fp64 entries: tiny entries skipped, exact retry if that leaves a zero total
      for (int attempt = 0; attempt < 3; ++attempt) {
        if (use64) {
          // fp64-entry parameters for this evaluation: redo the exponent split
          if (attempt > 0 || !a.f64) {
            // range-guard retry: rebuild the parameter slots from the fp64 bases
            // without repeating the prep side effects (mode PREP_CUR/AB-like)
            for (int k = tid; k < n2; k += blockDim.x) {
              const bool row = k < n;
              const double base = row ? ((S.st.mode & PREP_TRIAL) ? UV[k] + tuv[k] : UV[k] + uv[k])
                                      : ((S.st.mode & PREP_TRIAL) ? UV[k] + tuv[k] : UV[k] + uv[k]);
              prm[k] = f64_param(base, anc[k]);
            }
            __syncthreads();
          }
          batch_eval<true, false, CT>(reinterpret_cast<const CT*>(a.C64 ? (const void*)a.C64 : (const void*)a.C), n, prm, gh, gl, g2, gbar, tot, tot + n, S.sred, q_rank, CL, skip_z);
        } else {
          const CT* Cb = reinterpret_cast<const CT*>(a.C64 ? (const void*)a.C64 : (const void*)a.C);
          unsigned long long* dbg = (a.dbg && b == 0 && q_rank == 0) ? a.dbg : nullptr;
          if ((n & 3) == 0)
            batch_eval<false, PACKED, CT, true>(Cb, n, prm, gh, gl, g2, gbar, tot, tot + n, S.sred, q_rank, CL, -INFINITY, dbg);
          else
            batch_eval<false, PACKED, CT, false>(Cb, n, prm, gh, gl, g2, gbar, tot, tot + n, S.sred, q_rank, CL, -INFINITY, dbg);
        }
        __syncthreads();
        K8_MARK(2)
        if (CL > 1) cluster_combine(cluster, tot, n, q_rank, CL);
        K8_MARK(3)
        double v[kNumScalars];
#pragma unroll
        for (int q = 0; q < kNumScalars; ++q) v[q] = 0.0;
        fa.f64_entries = use64 ? 1 : 0;
        // skipped entries (z <= skip_z) each carry < e^skip_z T_j (row) or
        // e^skip_z S_i (column) in anchored units, with T, S <= 1 (anchors
        // <= 0): a total below n e^skip_z / 1e-16 may have lost more than
        // 1e-16 of itself to the skip -- redo that evaluation exactly (far-off
        // trial points, or targets below the anchor clamp 2^-120)
        fa.f64_tot_min = (use64 && skip_z > -INFINITY) ? (double)n * exp(skip_z) * 1e16 : 0.0;
        for (int k = tid; k < n2; k += blockDim.x) finalize_item(fa, k, tot[k], v);
        block_sum<kNumScalars>(v, &S.sred[0][0], S.out);
        K8_MARK(4)
#ifdef MDOT_DIAG_K8
        if (dg) a.dbg[7] += 1;
#endif
        if (S.out[SC_BAD] == 0.0) break;
        if (!use64) { use64 = true; continue; }     // range guard fired: redo with fp64 entries
        if (skip_z > -INFINITY) { skip_z = -INFINITY; continue; }   // a total lost to the skip: redo exactly
        break;
      }
      if (tid < kNumScalars) S.st.sc[tid] = S.out[tid];
      __syncthreads();
    }
    // projection result
    const CtrlState& h = S.st;
    if (tid == 0 && q_rank == 0 && t <= 64) {
      a.res[b].rho0[t - 1] = h.rho_0;
      a.res[b].l10[t - 1] = h.l1_0;
      a.res[b].iters_step[t - 1] = h.iterations;
    }
    evals_total += h.evals;
    iters += h.iterations;
    ls_evals += h.ls_evals;
    resets += h.resets;
    restarts += h.restarts;
    l1 = h.l1;
    rho = h.rho;
    if (h.status == CTRL_NOCONV) status = MDOT_ENOCONV;
    else if (h.status == CTRL_LS_FAIL) status = MDOT_ELINESEARCH;
    else if (h.status == CTRL_NEED_HOST) status = MDOT_EINSTABLE;
    __syncthreads();
    // a9: U += u, V += v; gauge (U - d, V + d) with <r,U> = <c,V>, same for (u, v)
    for (int k = tid; k < n2; k += blockDim.x) UV[k] += uv[k];
    __syncthreads();
    {
      double v4[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = tid; k < n2; k += blockDim.x) {
        const int q = (k < n) ? 0 : 1;
        v4[q] += tgt[k] * UV[k];
        v4[2 + q] += tgt[k] * uv[k];
      }
      block_sum<4>(v4, &S.sred[0][0], S.out);
      const double d1 = 0.5 * (S.out[0] - S.out[1]), d2 = 0.5 * (S.out[2] - S.out[3]);
      for (int k = tid; k < n2; k += blockDim.x) {
        UV[k] += (k < n) ? -d1 : d1;
        uv[k] += (k < n) ? -d2 : d2;
      }
      __syncthreads();
    }
    gprev = gt;
    t_done = t;
    if (status != 0 && status != MDOT_ENOCONV) break;
    if (status == MDOT_ENOCONV) break;
    if (a.adaptive) {
      if (last) break;
      // every CTA of the cluster holds the same h.evals: same decision everywhere
      next = adaptive_next_gamma(t, gt, (double)h.evals, gbar, a.gamma_bar, &eta_prev, &final_next);
    }
  }

  // ---- rounding + cost (a10), fp64: F = exp(U + V - gbar C), x = min(r/r(F), 1)
  // (rank 0 of the cluster alone: once per solve, no DSMEM access after the
  // last evaluation, so the other CTAs may exit)
  if (q_rank != 0) return;
  double cost_F = 0.0, cost_G = 0.0;
  if (status == 0 || status == MDOT_ENOCONV) {
    double* logx = tuv;        // [n] log x
    double* Ap = tuv + n;      // [n] U + log x
    double* cF1 = p;           // [n] c(F')
    double* Bpp = p + n;       // [n] V + log y
    double* ec = pprev;        // [n] err_c
    double* er = pprev + n;    // [n] err_r (first holds 1/x)
    double* invx = er;
    const int lane = tid & 31, warp = tid >> 5;
    // x = min(r / r(F), 1) from an exact fp64 row pass over F: the last
    // evaluation's fp32-entry marginals resolve r(F) only to ~1e-7 relative,
    // and x_i r_i(F) <= r_i is what keeps err_r >= 0 and G in U(r,c)
    // (solver.cu round_and_cost)
    for (int i = warp; i < n; i += kBatchWarps) {
      double s = 0.0;
      for (int j = lane; j < n; j += 32) s += exp((UV[i] + UV[n + j]) - gbar * batch_cost(a, (int64_t)i * n + j));
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) logx[i] = fmin(logt[i] - log(s), 0.0);
    }
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      const double lx = logx[i];
      Ap[i] = UV[i] + lx;
      invx[i] = exp(-lx);
    }
    __syncthreads();
    // columns: c(F')_j and sum_i C_ij F_ij (cost of F)
    double vF[1] = {0.0};
    for (int j = tid; j < n; j += blockDim.x) {
      double s1 = 0.0, s2 = 0.0;
      const double Bj = UV[n + j];
      for (int i = 0; i < n; ++i) {
        const double cij = batch_cost(a, (int64_t)i * n + j);
        const double f1 = exp((Ap[i] + Bj) - gbar * cij);
        s1 += f1;
        s2 += cij * f1 * invx[i];
      }
      cF1[j] = s1;
      vF[0] += s2;
    }
    block_sum<1>(vF, &S.sred[0][0], S.out);
    cost_F = S.out[0];
    for (int j = tid; j < n; j += blockDim.x) {
      const double y = fmin(tgt[n + j] / cF1[j], 1.0);
      Bpp[j] = UV[n + j] + log(y);
      ec[j] = fmax(tgt[n + j] - y * cF1[j], 0.0);   // >= 0 in exact arithmetic (kernels.cu)
    }
    __syncthreads();
    // rows: r(F''), <C, F''>, (C err_c)_i ; warp per row
    double v3[3] = {0.0, 0.0, 0.0};   // |err_r|_1, <C,F''>, err_r . C err_c (lane 0 of each warp)
    for (int i = warp; i < n; i += kBatchWarps) {
      double s = 0.0, cs2 = 0.0, cr = 0.0;
      for (int j = lane; j < n; j += 32) {
        const double cij = batch_cost(a, (int64_t)i * n + j);
        const double f2 = exp((Ap[i] + Bpp[j]) - gbar * cij);
        s += f2;
        cs2 += cij * f2;
        cr += cij * ec[j];
      }
      for (int off = 16; off > 0; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        cs2 += __shfl_xor_sync(0xffffffffu, cs2, off);
        cr += __shfl_xor_sync(0xffffffffu, cr, off);
      }
      if (lane == 0) {
        const double e = fmax(tgt[i] - s, 0.0);
        er[i] = e;
        v3[0] += fabs(e);
        v3[1] += cs2;
        v3[2] += e * cr;
      }
    }
    block_sum<3>(v3, &S.sred[0][0], S.out);
    cost_G = S.out[1] + (S.out[0] >= 1e-300 ? S.out[2] / S.out[0] : 0.0);
  }
  // ---- outputs
  if (a.U_out) for (int i = tid; i < n; i += blockDim.x) a.U_out[(int64_t)b * n + i] = UV[i];
  if (a.V_out) for (int j = tid; j < n; j += blockDim.x) a.V_out[(int64_t)b * n + j] = UV[n + j];
  if (tid == 0) {
    BatchResult& R = a.res[b];
    R.cost_rounded = cost_G;
    R.cost_unrounded = cost_F;
    R.l1_final = l1;
    R.rho_final = rho;
    R.gamma_bar = gbar;
    R.evaluations = evals_total;
    R.iterations = iters;
    R.ls_evaluations = ls_evals;
    R.resets = resets;
    R.ls_restarts = restarts;
    R.md_steps = t_done;
    R.status = status;
  }
}

size_t batch_smem_bytes(int n) { return batch_smem_bytes_d(n); }

// CTAs per instance: split the rows of each instance over a thread-block
// cluster while the batch leaves SMs idle (config 2: 64 instances on 148
// SMs -> 2 per instance), keeping >= 128 rows per CTA; power of two <= 8.
// MDOT_K8_CLUSTER overrides (A/B).
int batch_cluster(int n, int B) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int cl = 1;
  while (cl < 8 && (int64_t)B * cl * 2 <= sms && n / (cl * 2) >= 128) cl *= 2;
  if (const char* e = getenv("MDOT_K8_CLUSTER")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) cl = v;
  }
  return cl;
}

cudaError_t launch_batch(const BatchArgs& a, int B, cudaStream_t st) {
  const size_t smem = batch_smem_bytes(a.n);
  if (2 * a.n > kBatchMaxItemsPerThread * kBatchThreads) return cudaErrorInvalidValue;
  // MDOT_K8_SCALAR: A/B switch, scalar fp32 entry arithmetic
  static const bool scalar = getenv("MDOT_K8_SCALAR") != nullptr;
  const void* fn = a.C64 ? (const void*)k_batch_solve<false, double>
                         : (scalar ? (const void*)k_batch_solve<false, float> : (const void*)k_batch_solve<true, float>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int CL = batch_cluster(a.n, B);
  {
    static int set = -1;
    const int v = getenv("MDOT_K8_TAIL_REGULAR") ? 1 : 0;
    if (set != v) {
      cudaMemcpyToSymbol(g_k8_tail_regular, &v, sizeof(int));
      set = v;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * CL));
  cfg.blockDim = dim3(kBatchThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.C64) return cudaLaunchKernelEx(&cfg, k_batch_solve<false, double>, a);
  if (scalar) return cudaLaunchKernelEx(&cfg, k_batch_solve<false, float>, a);
  return cudaLaunchKernelEx(&cfg, k_batch_solve<true, float>, a);
}

void fault_set_batch(int mode) { fault_set_tu(mode); }

}  // namespace mdot

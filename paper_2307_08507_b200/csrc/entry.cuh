// paper_2307_08507_b200/csrc/entry.cuh -- the per-entry arithmetic of the
// fused marginal evaluation in packed form, for the on-the-fly-cost kernel
// (K2, kernels.cu k_eval_otf).
//
// Entries are handled as fp32 PAIRS (two adjacent columns of one row) with
// sm_100a's packed FADD2 / FFMA2 / FMUL2 (PTX add/fma/mul.rn.f32x2): each
// lane of a pair is rounded exactly like the scalar IEEE op, so the value of
// every entry is that of the scalar recipe:
//   zh = fmaf(-gh, C, ah + bh)    (ah + bh exact: both on a 2^-8 grid)
//   e  = ex2(fmaf(-gl, C, zh))
//   row += e * T'_j  (fp32, even / odd columns in two chains)
//   col_j += e * S'_i
// (the 2^al / 2^bl multipliers are applied to the row / column totals by the
// kernel) and the FP32 issue count per entry halves.  Used by the FP32-bound
// on-the-fly kernel; the K1 kernels keep the scalar form.
#pragma once
#include <stdint.h>

namespace mdot {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk2(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(u64 v, float& lo, float& hi) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Column parameters of a lane's 8 columns as 4 pairs: columns
// j0 + 4*lane + {0,1 | 2,3} and j0 + 128 + 4*lane + {0,1 | 2,3}.
struct ColPairs {
  u64 bh[4], T[4];
};

// colp(j) -> float4 {bh, M, T', .}; columns >= n are masked (bh = -1e30).
template <typename Load>
__device__ __forceinline__ void load_col_pairs(ColPairs& cp, int64_t j0, int lane, int64_t n, Load ld) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float v[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = 2 * p + h;
      const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
      if (j < n) {
        const float4 c = ld(j);
        v[0][h] = c.x; v[1][h] = c.z;
      } else {
        v[0][h] = -1.0e30f; v[1][h] = 0.f;
      }
    }
    cp.bh[p] = pk2(v[0][0], v[0][1]);
    cp.T[p] = pk2(v[1][0], v[1][1]);
  }
}

// One row of a lane's 8 entries.  c2[p] = (C_j, C_j+1) pairs in column-pair
// order, rp = {ah, M, S', .} of the row, ng = (-gh,-gh) / (-gl,-gl).  Adds
// e * S' into the column pair accumulators and returns the row's
// sum_j e * T'_j as an fp64 value (even and odd chains added in fp64).
__device__ __forceinline__ double entry_row8(const u64 (&c2)[4], float4 rp, const ColPairs& cp, u64 ngh2, u64 ngl2,
                                             u64 (&cacc)[4]) {
  const u64 ah2 = pk2(rp.x, rp.x), S2 = pk2(rp.z, rp.z);
  u64 rsum = 0ull;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const u64 zh = fma2(ngh2, c2[p], add2(ah2, cp.bh[p]));
    float zl, zu;
    up2(fma2(ngl2, c2[p], zh), zl, zu);
    const u64 e = pk2(ex2_ftz(zl), ex2_ftz(zu));
    rsum = fma2(e, cp.T[p], rsum);
    cacc[p] = fma2(e, S2, cacc[p]);
  }
  float lo, hi;
  up2(rsum, lo, hi);
  return (double)lo + (double)hi;
}

// Same, row sum left in fp32 (lo + hi): the warp then reduces rows in fp32
// (MDOT_K1_ROWRED_F32).
__device__ __forceinline__ float entry_row8_f(const u64 (&c2)[4], float4 rp, const ColPairs& cp, u64 ngh2, u64 ngl2,
                                              u64 (&cacc)[4]) {
  const u64 ah2 = pk2(rp.x, rp.x), S2 = pk2(rp.z, rp.z);
  u64 rsum = 0ull;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const u64 zh = fma2(ngh2, c2[p], add2(ah2, cp.bh[p]));
    float zl, zu;
    up2(fma2(ngl2, c2[p], zh), zl, zu);
    const u64 e = pk2(ex2_ftz(zl), ex2_ftz(zu));
    rsum = fma2(e, cp.T[p], rsum);
    cacc[p] = fma2(e, S2, cacc[p]);
  }
  float lo, hi;
  up2(rsum, lo, hi);
  return lo + hi;
}

// The 8 fp32 cost values of a lane's columns from two float4 loads.
__device__ __forceinline__ void cost_pairs(const float4& x0, const float4& x1, u64 (&c2)[4]) {
  c2[0] = pk2(x0.x, x0.y);
  c2[1] = pk2(x0.z, x0.w);
  c2[2] = pk2(x1.x, x1.y);
  c2[3] = pk2(x1.z, x1.w);
}

}  // namespace mdot

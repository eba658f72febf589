// paper_2307_08507_b200/csrc/otf_cost.cuh -- the on-the-fly cost recipes of
// BASELINE config 5 (C_ij = ||x_i - y_j||^2 * scale from fp32 coordinates),
// each a FIXED fp32 op sequence that the oracle replicates bit for bit
// (Z22 / Z22b), for the scalar paths (exact evaluator, rounding,
// generic K2 fallback, dense plan output).  The packed K2 kernel performs the
// same operations on column pairs (kernels.cu k_eval_otf).
//   diff (MDOT_COST_SQEUCLID_F32):     acc = fmaf(x_k - y_k, x_k - y_k, acc), k = 0..d-1;  C = acc * scale
//   dot  (MDOT_COST_SQEUCLID_DOT_F32): nx = fmaf chain of x_k^2, ny likewise, s = fmaf chain of x_k y_k;
//                                      C = max(fmaf(-2, s, nx + ny), 0) * scale
#pragma once
#include <cuda_runtime.h>

namespace mdot {

__device__ __forceinline__ float sqnorm_recipe(const float* x, int d) {
  float a = 0.f;
  for (int k = 0; k < d; ++k) a = __fmaf_rn(x[k], x[k], a);
  return a;
}

// unscaled cost of one pair; otf = 1 (diff) or 2 (dot)
__device__ __forceinline__ float otf_cost_raw(const float* x, const float* y, int d, int otf) {
  if (otf == 2) {
    float s = 0.f;
    for (int k = 0; k < d; ++k) s = __fmaf_rn(x[k], y[k], s);
    return fmaxf(__fmaf_rn(-2.0f, s, __fadd_rn(sqnorm_recipe(x, d), sqnorm_recipe(y, d))), 0.0f);
  }
  float acc = 0.f;
  for (int k = 0; k < d; ++k) {
    const float dk = __fsub_rn(x[k], y[k]);
    acc = __fmaf_rn(dk, dk, acc);
  }
  return acc;
}

__device__ __forceinline__ double otf_cost(const float* x, const float* y, int d, float scale, int otf) {
  return (double)__fmul_rn(otf_cost_raw(x, y, d, otf), scale);
}

}  // namespace mdot

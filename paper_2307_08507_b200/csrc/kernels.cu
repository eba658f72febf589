// paper_2307_08507_b200/csrc/kernels.cu -- sm_100a kernels of the MDOT-PNCG
// hot path (arxiv 2307.08507).  No tensor cores: the path is an exp-reduce
// over the n x n cost, bound by HBM for a materialised C.
//
//   k_eval_fast   fused row+column marginal evaluation:
//                 r(P)_i = sum_j P_ij, c(P)_j = sum_i P_ij for
//                 P_ij = exp(A_i + B_j - gbar C_ij)
//   k_exact_*     fp64 two-pass online log-sum-exp evaluator (fallback /
//                 fp64-P mode)
//   k_finalize    partial reduction + O(n) update: log marginals, Sinkhorn
//                 direction s, gradient,
//                 L1, rho, the CG inner products
//                 and phi'(alpha), deterministic reductions.
//   k_prep        direction update p = -s + beta p_prev,
//                 trial potentials u + alpha p, Sinkhorn
//                 half-steps, exponent split.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "entry.cuh"
#include "internal.cuh"
#include "ops.cuh"
#include "otf_cost.cuh"

namespace mdot {


__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float ld_stream1(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ float f4get(const float4& v, int q) {
  return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Reduce 4 per-lane values (one per row) across the warp with a transposing
// butterfly: 3 fp64 shuffles per row instead of 10.  On return, lanes with
// (lane & 7) == 0 hold the total of row ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1).
__device__ __forceinline__ double warp_reduce4(double v0, double v1, double v2, double v3, int lane) {
  const bool up = lane & 16;
  double k0 = up ? v2 : v0, k1 = up ? v3 : v1;
  double s0 = up ? v0 : v2, s1 = up ? v1 : v3;
  k0 += shfl_xor_d(s0, 16);
  k1 += shfl_xor_d(s1, 16);
  const bool up2 = lane & 8;
  double kk = up2 ? k1 : k0, ss = up2 ? k0 : k1;
  kk += shfl_xor_d(ss, 8);
  kk += shfl_xor_d(kk, 4);
  kk += shfl_xor_d(kk, 2);
  kk += shfl_xor_d(kk, 1);
  return kk;
}

// ---------------------------------------------------------------------------
// Fused evaluation.  CTA = (col tile tc of 256 columns) x (row tile tr of
// tile_m rows); 8 warps; lane owns columns j0 + 4*lane + {0..3} and
// j0 + 128 + 4*lane + {0..3}; warp w walks rows i0 + 32*k + 4*w + {0..3}.
// Per entry (5 FP32 + 1 MUFU; parameter slots: ops.cuh split_param):
//   s = ah_i + bh_j                      (exact: both on a 2^-8 grid)
//   zh = fmaf(-gh, C_ij, s)              (one rounding of the cancellation)
//   e  = ex2(fmaf(-gl, C_ij, zh))        (= P_ij 2^-(rho_i + sig_j + al_i + bl_j))
//   row_i += e * T'_j ;  col_j += e * S'_i
// Row sums are reduced across lanes per 4 rows (fp64 butterfly) and scaled
// by M_i = 2^al_i; column sums are fp32 over 8 rows, then fp64, then fp64
// across warps in smem, scaled by M_j = 2^bl_j.
// ---------------------------------------------------------------------------
template <int KIND, bool VEC4>
__global__ void __launch_bounds__(kThreads, 2) k_eval_fast(EvalArgs a) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (a.done && *a.done) return;
  const int64_t j0 = (int64_t)blockIdx.x * kTileN;
  const int64_t i0 = (int64_t)blockIdx.y * a.tile_m;
  const int64_t n = a.n, nrows = a.nrows;
  const bool full_cols = (j0 + kTileN <= n);

  __shared__ double sred[kWarps][kTileN];
  // on-the-fly cost: Y tile transposed [d][256]
  extern __shared__ float sdyn[];

  float bh[8], T[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
    if (j < n) {
      const float4 cp = a.colp[j];
      bh[q] = cp.x; T[q] = cp.z;
    } else {
      bh[q] = -1.0e30f; T[q] = 0.f;
    }
  }

  if (KIND == 1) {
    // stage Y[j0:j0+256, :] transposed into smem: sY[k*256 + t]
    float* sY = sdyn;
    for (int idx = threadIdx.x; idx < kTileN * a.d; idx += kThreads) {
      const int t = idx / a.d, k = idx % a.d;
      const int64_t j = j0 + t;
      sY[k * kTileN + t] = (j < n) ? a.Y[j * a.d + k] : 0.f;
    }
    __syncthreads();
  }

  const float gh = a.gpair ? a.gpair[0] : a.gh;
  const float gl = a.gpair ? a.gpair[1] : a.gl;
  double cacc64[8];
  float cacc32[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { cacc64[q] = 0.0; cacc32[q] = 0.f; }
#if MDOT_K1_PACKED
  ColPairs cpp;
#pragma unroll
  for (int p = 0; p < 4; ++p) { cpp.bh[p] = pk2(bh[2 * p], bh[2 * p + 1]); cpp.T[p] = pk2(T[2 * p], T[2 * p + 1]); }
  u64 cacc2[4] = {0ull, 0ull, 0ull, 0ull};
  const u64 ngh2 = pk2(-gh, -gh), ngl2 = pk2(-gl, -gl);
#endif

  const int64_t tile_end = (i0 + a.tile_m < nrows) ? i0 + a.tile_m : nrows;
  int flush = 0;
  for (int64_t ib = i0 + 4 * warp; ib < tile_end; ib += kWarps * kUnroll) {
    float cv[kUnroll][8];
    float4 rp[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = ib + u;
      if (i < tile_end) {
        rp[u] = a.rowp[i];
        if (KIND == 0) {
          const float* crow = a.C + i * a.ldc + j0 + 4 * lane;
          if (VEC4 && full_cols) {
            const float4 x0 = ld_stream4(crow);
            const float4 x1 = ld_stream4(crow + 128);
            cv[u][0] = x0.x; cv[u][1] = x0.y; cv[u][2] = x0.z; cv[u][3] = x0.w;
            cv[u][4] = x1.x; cv[u][5] = x1.y; cv[u][6] = x1.z; cv[u][7] = x1.w;
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
              cv[u][q] = (j < n) ? ld_stream1(a.C + i * a.ldc + j) : 0.f;
            }
          }
        } else if (a.otf_dot) {
          // Z22b: C_ij = max(fmaf(-2, s, fl(nx_i + ny_j)), 0) * scale (otf_cost.cuh)
          const float* xr = a.X + i * a.d;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
            cv[u][q] = (j < n) ? (float)otf_cost(xr, a.Y + j * a.d, a.d, a.scale, 2) : 0.f;
          }
        } else {
          // C_ij = fl32(fmaf chain over k of (x_ik - y_jk)^2) * scale  (Z22)
          float acc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = 0.f;
          const float* xr = a.X + i * a.d;
          for (int k = 0; k < a.d; ++k) {
            const float xk = __ldg(xr + k);
            const float4 y0 = *reinterpret_cast<const float4*>(sdyn + k * kTileN + 4 * lane);
            const float4 y1 = *reinterpret_cast<const float4*>(sdyn + k * kTileN + 128 + 4 * lane);
            float dk;
            dk = __fsub_rn(xk, y0.x); acc[0] = __fmaf_rn(dk, dk, acc[0]);
            dk = __fsub_rn(xk, y0.y); acc[1] = __fmaf_rn(dk, dk, acc[1]);
            dk = __fsub_rn(xk, y0.z); acc[2] = __fmaf_rn(dk, dk, acc[2]);
            dk = __fsub_rn(xk, y0.w); acc[3] = __fmaf_rn(dk, dk, acc[3]);
            dk = __fsub_rn(xk, y1.x); acc[4] = __fmaf_rn(dk, dk, acc[4]);
            dk = __fsub_rn(xk, y1.y); acc[5] = __fmaf_rn(dk, dk, acc[5]);
            dk = __fsub_rn(xk, y1.z); acc[6] = __fmaf_rn(dk, dk, acc[6]);
            dk = __fsub_rn(xk, y1.w); acc[7] = __fmaf_rn(dk, dk, acc[7]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) cv[u][q] = __fmul_rn(acc[q], a.scale);
        }
      } else {
        rp[u] = make_float4(-1.0e30f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q) cv[u][q] = 0.f;
      }
    }

    #if MDOT_K1_ROWRED_F32
    float rs[kUnroll];
#else
    double rs[kUnroll];
#endif
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#if MDOT_K1_PACKED
      const u64 c2[4] = {pk2(cv[u][0], cv[u][1]), pk2(cv[u][2], cv[u][3]), pk2(cv[u][4], cv[u][5]),
                         pk2(cv[u][6], cv[u][7])};
      rs[u] = entry_row8_f(c2, rp[u], cpp, ngh2, ngl2, cacc2);
#else
      float rsum = 0.f;
      const float ah = rp[u].x, S = rp[u].z;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float cij = cv[u][q];
        const float s = ah + bh[q];
        const float zh = fmaf(-gh, cij, s);
        const float e = ex2_approx(fmaf(-gl, cij, zh));
        rsum = fmaf(e, T[q], rsum);
        cacc32[q] = fmaf(e, S, cacc32[q]);
      }
      rs[u] = rsum;
#endif
    }
    // row totals (butterfly over the warp, MDOT_K1_ROWRED_F32), times M_i = 2^al_i
    {
#if MDOT_K1_ROWRED_F32
      const double tot = (double)warp_reduce4_f(rs[0], rs[1], rs[2], rs[3], lane);
#else
      const double tot = warp_reduce4(rs[0], rs[1], rs[2], rs[3], lane);
#endif
      const int64_t i = ib + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
      const float Mrow = (lane & 16) ? ((lane & 8) ? rp[3].y : rp[2].y) : ((lane & 8) ? rp[1].y : rp[0].y);
      if ((lane & 7) == 0 && i < tile_end) a.rowpart[(int64_t)blockIdx.x * nrows + i] = tot * (double)Mrow;
    }
    if (++flush == MDOT_K1_COLFLUSH) {   // 4 x MDOT_K1_COLFLUSH rows of fp32 column sums -> fp64
      flush = 0;
#if MDOT_K1_PACKED
#pragma unroll
      for (int p = 0; p < 4; ++p) { up2(cacc2[p], cacc32[2 * p], cacc32[2 * p + 1]); cacc2[p] = 0ull; }
#endif
#pragma unroll
      for (int q = 0; q < 8; ++q) { cacc64[q] += (double)cacc32[q]; cacc32[q] = 0.f; }
    }
  }
#if MDOT_K1_PACKED
#pragma unroll
  for (int p = 0; p < 4; ++p) up2(cacc2[p], cacc32[2 * p], cacc32[2 * p + 1]);
#endif
#pragma unroll
  for (int q = 0; q < 8; ++q) cacc64[q] += (double)cacc32[q];

  // column totals of this tile: sum over the 8 warps (fixed order)
#pragma unroll
  for (int q = 0; q < 8; ++q) sred[warp][4 * lane + (q & 3) + 128 * (q >> 2)] = cacc64[q];
  __syncthreads();
  {
    const int t = threadIdx.x;
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += sred[w][t];
    const int64_t j = j0 + t;
    if (j < n) a.colpart[(int64_t)blockIdx.y * n + j] = tot * (double)a.colp[j].y;   // times M_j = 2^bl_j
  }
}

// ---------------------------------------------------------------------------
// On-the-fly squared-Euclidean cost with packed fp32
// pairs.  This kernel is bound by the FP32 pipe, not HBM: per pair of points
// the Z22 recipe costs d FADD + d FFMA for the distance and 7 more ops for the
// entry.  sm_100a executes FADD2/FFMA2/FMUL2 (PTX add/fma/mul.rn.f32x2) on
// two lanes of a 64-bit register pair with per-lane IEEE rounding, so every
// op below handles two columns at once and the per-element result is
// bit-identical to the scalar recipe.  Layout as
// k_eval_fast: lane owns columns j0 + 4*lane + {0..3} and
// j0 + 128 + 4*lane + {0..3} (pairs {0,1},{2,3} of each quad); X rows are
// staged in chunks of OtfChunk<D> rows as duplicated pairs (x, x) so each
// FADD2 reads its broadcast operand straight from shared memory.
// ---------------------------------------------------------------------------
// rows per staged X chunk: 256 for d <= 16 (half the CTA barriers per row;
// 2 x 72 KB of shared memory per SM at d = 16), 128 above (d = 32: 2 x 112 KB)
template <int D>
struct OtfChunk {
  static constexpr int value = D <= 16 ? 256 : 128;
};
// Row sums: each lane stores its 4 fp32 row partials (8 entries each) to
// shared memory and one thread per row adds the 32 partials in fp64 after the
// chunk (fixed order).  The per-iteration fp64 shuffle butterfly this replaces
// (MDOT_K2_ROWSMEM=0) was ~15 % of the loop's instructions and its most
// latency-bound part (profiles/r02_k2_dot_ncu.md).
#ifndef MDOT_K2_ROWSMEM
#define MDOT_K2_ROWSMEM 1
#endif

// POW2: scale is a power of two, so C = acc * scale is exact and -g * C ==
// (-g * scale) * acc exactly: the scale folds into (gh, gl) and the FMUL2 per
// pair of entries disappears, with the Z22 recipe's bits unchanged.
template <int D, bool POW2, bool DOT>
__global__ void __launch_bounds__(kThreads, 2) k_eval_otf(EvalArgs a) {
  constexpr int kOtfChunk = OtfChunk<D>::value;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (a.done && *a.done) return;
  const int64_t j0 = (int64_t)blockIdx.x * kTileN;
  const int64_t i0 = (int64_t)blockIdx.y * a.tile_m;
  const int64_t n = a.n, nrows = a.nrows;

  __shared__ double sred[kWarps][kTileN];
  __shared__ float4 sRP[2][kOtfChunk];   // row parameters, double-buffered by chunk
  extern __shared__ __align__(16) unsigned char sraw[];
  float* sY = reinterpret_cast<float*>(sraw);                          // [D][256]
  float* sX = reinterpret_cast<float*>(sraw + sizeof(float) * D * kTileN);   // [2][chunk][D]
#if MDOT_K2_ROWSMEM
  // [32 lanes][chunk + 4] fp32 row partials (the +4 pad spreads the lanes'
  // float4 stores over all banks)
  constexpr int kPartStride = kOtfChunk + 4;
  float* sPart = sX + 2 * kOtfChunk * D;
#endif
  // X chunks (and their row parameters) stream through a 2-deep cp.async
  // ring: the next chunk's copy overlaps this chunk's arithmetic.  Vector
  // copies need D % 4 == 0 and 16-byte aligned X, Y (else synchronous
  // staging).  The per-element load -> store staging of the first version was
  // the kernel's top stall (one L2 round trip per element; profiles/).
  const bool vec = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Y)) & 15) == 0;
  const int64_t tile_end = (i0 + a.tile_m < nrows) ? i0 + a.tile_m : nrows;
  auto rows_of = [&](int64_t c0) { return (int)((tile_end - c0 < kOtfChunk) ? tile_end - c0 : kOtfChunk); };
  auto issue_chunk = [&](int64_t c0, int buf) {   // cp.async (zero-fill past the tile end)
    const int rows_c = rows_of(c0);
    constexpr int kQ = (kOtfChunk * D / 4 + kThreads - 1) / kThreads;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int f = 4 * (q * kThreads + threadIdx.x);
      if (f < kOtfChunk * D) {
        const bool ok = f / D < rows_c;
        const float* src = ok ? a.X + c0 * D + f : a.X;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sX + buf * kOtfChunk * D + f))),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
    }
    if (threadIdx.x < kOtfChunk) {
      const bool ok = (int)threadIdx.x < rows_c;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&sRP[buf][threadIdx.x]))),
                   "l"(ok ? a.rowp + c0 + threadIdx.x : a.rowp), "r"(ok ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (vec && i0 < tile_end) issue_chunk(i0, 0);

  // Y[j0:j0+256, :] transposed (thread t = column j0 + t); columns past n are
  // zero points (masked by bh)
  {
    static_assert(kThreads == kTileN, "one thread per tile column");
    const int64_t j = j0 + threadIdx.x;
    float yv[D];
    if (j < n) {
      if (vec) {
#pragma unroll
        for (int q = 0; q < (D + 3) / 4; ++q) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(a.Y + j * D) + q);
          yv[4 * q] = v.x;
          if (4 * q + 1 < D) yv[4 * q + 1] = v.y;
          if (4 * q + 2 < D) yv[4 * q + 2] = v.z;
          if (4 * q + 3 < D) yv[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k) yv[k] = __ldg(a.Y + j * D + k);
      }
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) yv[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) sY[k * kTileN + threadIdx.x] = yv[k];
  }
  // Z22b: the lane's column pairs' squared norms |y_j|^2 (colp .w, written by
  // prep from the once-per-solve norms; the row norms come with sRP .w)
  u64 ny2[DOT ? 4 : 1];
  if (DOT) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = 2 * p + h;
        const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
        v[h] = j < n ? a.colp[j].w : 0.f;
      }
      ny2[p & (DOT ? 3 : 0)] = pk2(v[0], v[1]);
    }
  }

  ColPairs cpp;
  load_col_pairs(cpp, j0, lane, n, [&](int64_t j) { return a.colp[j]; });
  const float gh = a.gpair ? a.gpair[0] : a.gh;
  const float gl = a.gpair ? a.gpair[1] : a.gl;
  const float sg = POW2 ? a.scale : 1.f;
  const u64 ngh2 = pk2(-gh * sg, -gh * sg), ngl2 = pk2(-gl * sg, -gl * sg), scale2 = pk2(a.scale, a.scale);

  double cacc64[8];
  u64 cacc2[4];
#pragma unroll
  for (int q = 0; q < 8; ++q) cacc64[q] = 0.0;
#pragma unroll
  for (int p = 0; p < 4; ++p) cacc2[p] = 0ull;

  int flush = 0, cidx = 0;
  for (int64_t c0 = i0; c0 < tile_end; c0 += kOtfChunk, ++cidx) {
    const int rows_c = rows_of(c0);
    const int buf = vec ? (cidx & 1) : 0;
    if (vec) {
      if (c0 + kOtfChunk < tile_end) issue_chunk(c0 + kOtfChunk, buf ^ 1);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");   // this chunk's group has landed
      __syncthreads();   // ... for every thread (and sY is written)
    } else {
      __syncthreads();   // previous chunk consumed (and sY written on entry)
      float4 rpv = make_float4(-1.0e30f, 0.f, 0.f, 0.f);
      if (threadIdx.x < kOtfChunk && (int)threadIdx.x < rows_c) rpv = a.rowp[c0 + threadIdx.x];
      constexpr int kE = (kOtfChunk * D + kThreads - 1) / kThreads;
      float xv[kE];
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        const int idx = q * kThreads + threadIdx.x;
        xv[q] = (idx < kOtfChunk * D && idx / D < rows_c) ? __ldg(a.X + c0 * D + idx) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        const int idx = q * kThreads + threadIdx.x;
        if (idx < kOtfChunk * D) sX[idx] = xv[q];
      }
      if (threadIdx.x < kOtfChunk) sRP[0][threadIdx.x] = rpv;
      __syncthreads();
    }
    const float* xs = sX + buf * kOtfChunk * D;
    for (int rb = 4 * warp; rb < rows_c; rb += kWarps * kUnroll) {
      u64 acc[kUnroll][4];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[u][p] = 0ull;
      // C_ij = fl32(fmaf chain over k of (x_ik - y_jk)^2) * scale  (Z22)
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const ulonglong2 ya = *reinterpret_cast<const ulonglong2*>(sY + k * kTileN + 4 * lane);
        const ulonglong2 yb = *reinterpret_cast<const ulonglong2*>(sY + k * kTileN + 128 + 4 * lane);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const float x = xs[(rb + u) * D + k];
          const u64 xx = pk2(x, x);   // ptxas: a broadcast (.F32) operand of the packed ops
          if (DOT) {   // s = fmaf chain of x_k y_k (Z22b)
            acc[u][0] = fma2(xx, ya.x, acc[u][0]);
            acc[u][1] = fma2(xx, ya.y, acc[u][1]);
            acc[u][2] = fma2(xx, yb.x, acc[u][2]);
            acc[u][3] = fma2(xx, yb.y, acc[u][3]);
          } else {
            u64 dk;
            dk = sub2(xx, ya.x); acc[u][0] = fma2(dk, dk, acc[u][0]);
            dk = sub2(xx, ya.y); acc[u][1] = fma2(dk, dk, acc[u][1]);
            dk = sub2(xx, yb.x); acc[u][2] = fma2(dk, dk, acc[u][2]);
            dk = sub2(xx, yb.y); acc[u][3] = fma2(dk, dk, acc[u][3]);
          }
        }
      }
      if (DOT) {   // C / scale = max(fmaf(-2, s, fl(nx_i + ny_j)), 0), pairwise
        const u64 m2 = pk2(-2.0f, -2.0f);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const float nx = sRP[buf][rb + u].w;   // |x_i|^2 (0 on zero-filled rows past the tile)
          const u64 nx2 = pk2(nx, nx);
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            float lo, hi;
            up2(fma2(m2, acc[u][p], add2(nx2, ny2[p & (DOT ? 3 : 0)])), lo, hi);
            acc[u][p] = pk2(fmaxf(lo, 0.f), fmaxf(hi, 0.f));
          }
        }
      }
#if MDOT_K2_ROWSMEM
      float rs[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        float4 rp = sRP[buf][rb + u];   // broadcast
        if (rb + u >= rows_c) rp = make_float4(-1.0e30f, 0.f, 0.f, 0.f);   // zero-filled rows past the tile
        u64 c2[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) c2[p] = POW2 ? acc[u][p] : mul2(acc[u][p], scale2);
        rs[u] = entry_row8_f(c2, rp, cpp, ngh2, ngl2, cacc2);
      }
      // the lane's 4 row partials (8 entries each) -> sPart, reduced per row after the chunk
      *reinterpret_cast<float4*>(sPart + lane * kPartStride + rb) = make_float4(rs[0], rs[1], rs[2], rs[3]);
#else
      double rs[kUnroll];
      float mrow[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        float4 rp = sRP[buf][rb + u];   // broadcast
        if (rb + u >= rows_c) rp = make_float4(-1.0e30f, 0.f, 0.f, 0.f);   // zero-filled rows past the tile
        mrow[u] = rp.y;
        u64 c2[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) c2[p] = POW2 ? acc[u][p] : mul2(acc[u][p], scale2);
        rs[u] = entry_row8(c2, rp, cpp, ngh2, ngl2, cacc2);
      }
      {
        const double tot = warp_reduce4(rs[0], rs[1], rs[2], rs[3], lane);
        const int r = rb + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
        const float Mrow = (lane & 16) ? ((lane & 8) ? mrow[3] : mrow[2]) : ((lane & 8) ? mrow[1] : mrow[0]);
        if ((lane & 7) == 0 && r < rows_c) a.rowpart[(int64_t)blockIdx.x * nrows + c0 + r] = tot * (double)Mrow;
      }
#endif
      if (++flush == MDOT_K1_COLFLUSH) {   // 4 x MDOT_K1_COLFLUSH rows of fp32 column sums -> fp64
        flush = 0;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          float lo, hi;
          up2(cacc2[p], lo, hi);
          cacc64[2 * p] += (double)lo;
          cacc64[2 * p + 1] += (double)hi;
          cacc2[p] = 0ull;
        }
      }
    }
#if MDOT_K2_ROWSMEM
    __syncthreads();   // every lane's partials of this chunk are in sPart
    for (int r = threadIdx.x; r < rows_c; r += kThreads) {   // one row per thread: 32 partials in fp64, fixed order
      double tot = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) tot += (double)sPart[l * kPartStride + r];
      a.rowpart[(int64_t)blockIdx.x * nrows + c0 + r] = tot * (double)sRP[buf][r].y;   // times M_i = 2^al_i
    }
    __syncthreads();   // sPart and the chunk buffer free for the next chunk
#else
    if (vec) __syncthreads();   // chunk buffer free before the next iteration's copy into it
#endif
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float lo, hi;
    up2(cacc2[p], lo, hi);
    cacc64[2 * p] += (double)lo;
    cacc64[2 * p + 1] += (double)hi;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) sred[warp][4 * lane + (q & 3) + 128 * (q >> 2)] = cacc64[q];
  __syncthreads();
  {
    const int t = threadIdx.x;
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += sred[w][t];
    const int64_t j = j0 + t;
    if (j < n) a.colpart[(int64_t)blockIdx.y * n + j] = tot * (double)a.colp[j].y;   // times M_j = 2^bl_j
  }
}

template <int D, bool POW2, bool DOT>
static cudaError_t launch_otf_pt(const EvalArgs& a, cudaStream_t st) {
  dim3 grid(a.n_col_tiles, a.n_row_tiles);
  const size_t smem = sizeof(float) * D * kTileN + sizeof(float) * 2 * OtfChunk<D>::value * D +
                      (MDOT_K2_ROWSMEM ? sizeof(float) * 32 * (OtfChunk<D>::value + 4) : 0);
  static bool attr_set = false;
  if (!attr_set) {   // static (column sums, row parameters) + dynamic exceeds the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(k_eval_otf<D, POW2, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  k_eval_otf<D, POW2, DOT><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}
template <int D>
static cudaError_t launch_otf_t(const EvalArgs& a, cudaStream_t st) {
  int e2 = 0;
  const bool pow2 = a.scale > 0.f && frexpf(a.scale, &e2) == 0.5f && e2 > -100 && e2 < 100;
  if (a.otf_dot) return pow2 ? launch_otf_pt<D, true, true>(a, st) : launch_otf_pt<D, false, true>(a, st);
  return pow2 ? launch_otf_pt<D, true, false>(a, st) : launch_otf_pt<D, false, false>(a, st);
}

template <int KIND, bool VEC4>
static cudaError_t launch_fast_t(const EvalArgs& a, cudaStream_t st) {
  dim3 grid(a.n_col_tiles, a.n_row_tiles);
  size_t smem = (KIND == 1) ? (size_t)kTileN * a.d * sizeof(float) : 0;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_eval_fast<KIND, VEC4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  k_eval_fast<KIND, VEC4><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_eval_fast(const EvalArgs& a, int kind, cudaStream_t st) {
  if (kind == 0) {
    const bool vec4 = (a.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0);
    return vec4 ? launch_fast_t<0, true>(a, st) : launch_fast_t<0, false>(a, st);
  }
  const bool generic = getenv("MDOT_OTF_GENERIC") != nullptr;   // A/B switch
  if (!generic) {
    switch (a.d) {
      case 2: return launch_otf_t<2>(a, st);
      case 3: return launch_otf_t<3>(a, st);
      case 4: return launch_otf_t<4>(a, st);
      case 8: return launch_otf_t<8>(a, st);
      case 16: return launch_otf_t<16>(a, st);
      case 32: return launch_otf_t<32>(a, st);
      default: break;
    }
  }
  return launch_fast_t<1, false>(a, st);
}

// ---------------------------------------------------------------------------
// Exact fp64 evaluator: z = (A_i + B_j) - gbar * C_ij in fp64, online
// log-sum-exp with fp64 exp.  Rows: one warp per row.  Columns: one thread per
// column over a chunk of rows, (max, sum) partials per chunk.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double exact_cost(const ExactArgs& a, int64_t i, int64_t j) {
  if (a.otf) return otf_cost(a.X + i * a.d, a.Y + j * a.d, a.d, a.scale, a.otf);
  if (a.c_f64) return reinterpret_cast<const double*>(a.C)[i * a.ldc + j];
  return (double)reinterpret_cast<const float*>(a.C)[i * a.ldc + j];
}

__global__ void k_exact_rows(ExactArgs a) {
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= a.nrows) return;
  const double Ai = a.A[i];
  double m = -INFINITY, s = 0.0;
  for (int64_t j = lane; j < a.n; j += 32) {
    const double z = (Ai + a.B[j]) - a.gbar * exact_cost(a, i, j);
    lse_push(m, s, z);
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const double s2 = __shfl_xor_sync(0xffffffffu, s, off);
    lse_merge(m, s, m2, s2);
  }
  if (lane == 0) a.lr[i] = m + log(s);
}

__global__ void k_exact_cols(ExactArgs a) {
  if (a.done && *a.done) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  const int64_t rows_per = (a.nrows + a.chunks - 1) / a.chunks;
  const int64_t ib = chunk * rows_per;
  const int64_t ie = (ib + rows_per < a.nrows) ? ib + rows_per : a.nrows;
  if (j >= a.n) return;
  const double Bj = a.B[j];
  double m = -INFINITY, s = 0.0;
  for (int64_t i = ib; i < ie; ++i) {
    const double z = (a.A[i] + Bj) - a.gbar * exact_cost(a, i, j);
    lse_push(m, s, z);
  }
  a.colm[(int64_t)chunk * a.n + j] = m;
  a.cols[(int64_t)chunk * a.n + j] = s;
}

cudaError_t launch_exact_rows(const ExactArgs& a, cudaStream_t st) {
  const int wpb = 8;
  k_exact_rows<<<(unsigned)((a.nrows + wpb - 1) / wpb), wpb * 32, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_eval_exact(const ExactArgs& a, cudaStream_t st) {
  cudaError_t e = launch_exact_rows(a, st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.n + 255) / 256), a.chunks);
  k_exact_cols<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Block reduction of kNumScalars doubles + deterministic last-block combine.
// ---------------------------------------------------------------------------
template <int NS>
__device__ void block_reduce_and_publish(double (&v)[NS], double* blockpart, unsigned int* ticket,
                                         double* out_dev, double* out_host, const double* add_in = nullptr) {
  // fixed-order reduction: warp shuffle tree -> per-warp smem -> per-block
  // partial; the last block (ticket) combines all block partials with every
  // thread loading a fixed strided subset and a fixed smem tree (no serial
  // chain of loads, deterministic for a given grid).
  __shared__ double sm[32][NS];
  __shared__ double sfin[256];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    double x = v[k];
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    if (lane == 0) sm[warp][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < NS) {
    double x = 0.0;
    for (int w = 0; w < nw; ++w) x += sm[w][threadIdx.x];
    blockpart[(int64_t)blockIdx.x * NS + threadIdx.x] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // thread t: scalar k = t % NS, blocks b = t / NS, t / NS + G, ... (G = 256 / NS groups)
  constexpr int G = 256 / NS;
  const int t = threadIdx.x;
  double x = 0.0;
  if (t < G * NS) {
    const int k = t % NS;
    unsigned b = t / NS;
    for (; b + 3 * G < gridDim.x; b += 4 * G) {
      const double y0 = __ldcg(&blockpart[(int64_t)b * NS + k]);
      const double y1 = __ldcg(&blockpart[(int64_t)(b + G) * NS + k]);
      const double y2 = __ldcg(&blockpart[(int64_t)(b + 2 * G) * NS + k]);
      const double y3 = __ldcg(&blockpart[(int64_t)(b + 3 * G) * NS + k]);
      x += y0; x += y1; x += y2; x += y3;
    }
    for (; b < gridDim.x; b += G) x += __ldcg(&blockpart[(int64_t)b * NS + k]);
  }
  if (t < 256) sfin[t] = x;
  __syncthreads();
  if (t < NS) {
    double y = 0.0;
    for (int g = 0; g < G; ++g) y += sfin[g * NS + t];
    if (add_in) y += add_in[t];
    out_dev[t] = y;
    if (out_host) out_host[t] = y;
  }
  if (t == 0) *ticket = 0u;
}

// sum_{t < cnt} x[t * stride] in index order; loads issued 8 at a time
__device__ __forceinline__ double sum_strided(const double* x, int64_t stride, int cnt) {
  double acc = 0.0;
  int t = 0;
  for (; t + 8 <= cnt; t += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = x[(int64_t)(t + u) * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; t < cnt; ++t) acc += x[(int64_t)t * stride];
  return acc;
}

// ---------------------------------------------------------------------------
// finalize: marginals, s, grad, scalars
// ---------------------------------------------------------------------------
__device__ __forceinline__ void finalize_body(const FinalizeArgs& a);

__global__ void __launch_bounds__(256) k_finalize(FinalizeArgs a) { finalize_body(a); }

// Lockstep batch (throughput mode): blockIdx.y = instance, its own args,
// tickets and block partials (an instance whose controller is done exits).
__global__ void __launch_bounds__(256) k_finalize_multi(const FinalizeArgs* args) {
  const FinalizeArgs a = args[blockIdx.y];
  finalize_body(a);
}

__device__ __forceinline__ void finalize_body(const FinalizeArgs& a) {
  if (a.smin_reset && blockIdx.x == 0 && threadIdx.x < 2) a.smin_reset[threadIdx.x] = kKeyPosInf;   // K2s: next prep
  if (a.done && *a.done) return;
  const int sub = threadIdx.x & (kFinTPI - 1);
  const int64_t tot_items = a.item_end > 0 ? a.item_end : a.nrows + a.n;
  const int64_t groups = (tot_items - a.item_begin + (256 / kFinTPI) - 1) / (256 / kFinTPI);
  double v[kNumScalars];
#pragma unroll
  for (int q = 0; q < kNumScalars; ++q) v[q] = 0.0;
  // grid-stride over groups of 32 items (one octet per item); the grid is
  // capped at 2 x #SMs so the last-block combine stays short
  for (int64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
  const int64_t k = a.item_begin + grp * (256 / kFinTPI) + threadIdx.x / kFinTPI;
  const bool in_range = k < tot_items;
  const bool is_row = k < a.nrows;
  double tot = 0.0;
  if (a.from_partials == 1) {   // octet-parallel partial sums; the shuffles run on the whole warp
    double x = 0.0;
    if (in_range) {
      if (is_row) x = a.rowtot ? ((sub == 0) ? a.rowtot[k] : 0.0)   // already reduced (2-D sharded)
                               : octet_partial(a.rowpart + k, a.nrows, a.n_col_tiles, sub);
      else if (a.coltot) x = (sub == 0) ? a.coltot[k - a.nrows] : 0.0;   // already reduced (sharded)
      else x = octet_partial(a.colpart + (k - a.nrows), a.n, a.n_row_tiles, sub);
    }
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    tot = x;
  }
  if (in_range && sub == 0) finalize_item(a, k, tot, v);
  }
  block_reduce_and_publish<kNumScalars>(v, a.blockpart, a.ticket, a.scalars_dev, a.scalars_host, a.add_in);
}

cudaError_t launch_finalize_multi(const FinalizeArgs* args_dev, const FinalizeArgs& a0, int B, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = a0.nrows + a0.n;
  const int64_t groups = (items * kFinTPI + 255) / 256;
  // at least ~2 blocks per SM over the whole batch, at most 2 x #SMs per instance
  const int64_t cap = std::max<int64_t>(8, std::min<int64_t>(2 * sms, (4 * (int64_t)sms + B - 1) / B));
  const unsigned blocks = (unsigned)(groups < cap ? groups : cap);
  k_finalize_multi<<<dim3(blocks, (unsigned)B), 256, 0, st>>>(args_dev);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st) {
  static int cap = 0;
  if (!cap) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = 2 * sms;
  }
  const int64_t items = (a.item_end > 0 ? a.item_end : a.nrows + a.n) - a.item_begin;
  const int64_t groups = (items * kFinTPI + 255) / 256;
  const unsigned blocks = (unsigned)(groups < cap ? groups : cap);
  k_finalize<<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// prep: direction, trial potentials, Sinkhorn half-steps, exponent split
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Device-resident controller (single thread), mirrors project_pncg /
// project_sinkhorn in solver.cu step by step.
// ---------------------------------------------------------------------------

// One warp copies the ~0.7 KB state to shared memory (coalesced), lane 0 runs
// the control logic on the shared copy, the warp writes it back: two L2 round
// trips instead of one per field.
__global__ void k_ctrl(CtrlState* gst, int slot, int* done_host, int* ran_host) {
  __shared__ CtrlState sst;
  constexpr int kWords = (int)(sizeof(CtrlState) / sizeof(unsigned long long));
  static_assert(sizeof(CtrlState) % sizeof(unsigned long long) == 0, "CtrlState size");
  unsigned long long* g = reinterpret_cast<unsigned long long*>(gst);
  unsigned long long* sh = reinterpret_cast<unsigned long long*>(&sst);
  for (int i = threadIdx.x; i < kWords; i += 32) sh[i] = g[i];
  __syncwarp();
  if (threadIdx.x == 0) ctrl_body(&sst, slot, done_host, ran_host);
  __syncwarp();
  for (int i = threadIdx.x; i < kWords; i += 32) g[i] = sh[i];
}

__global__ void k_prep(PrepArgs a);
void set_smem_carveout_tma();
void set_smem_carveout() {
  static bool done = false;
  if (done) return;
  done = true;
  const int c = cudaSharedmemCarveoutMaxShared;
  cudaFuncSetAttribute(k_ctrl, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_prep, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_finalize, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_eval_fast<0, true>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_eval_fast<0, false>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  cudaFuncSetAttribute(k_eval_fast<1, false>, cudaFuncAttributePreferredSharedMemoryCarveout, c);
  set_smem_carveout_tma();
}

// Lockstep batch: block b runs instance b's controller; done_flags[b] (mapped
// host memory) mirrors its `done` so the host knows when every instance's
// projection has finished.
__global__ void k_ctrl_multi(CtrlState* const* gsts, int* done_flags) {
  __shared__ CtrlState sst;
  constexpr int kWords = (int)(sizeof(CtrlState) / sizeof(unsigned long long));
  unsigned long long* g = reinterpret_cast<unsigned long long*>(gsts[blockIdx.x]);
  unsigned long long* sh = reinterpret_cast<unsigned long long*>(&sst);
  for (int i = threadIdx.x; i < kWords; i += 32) sh[i] = g[i];
  __syncwarp();
  if (threadIdx.x == 0) {
    ctrl_body(&sst, 0, nullptr, nullptr);
    *((volatile int*)&done_flags[blockIdx.x]) = sst.done;
  }
  __syncwarp();
  for (int i = threadIdx.x; i < kWords; i += 32) g[i] = sh[i];
}

cudaError_t launch_ctrl_multi(CtrlState* const* sts_dev, int B, int* done_flags, cudaStream_t s) {
  k_ctrl_multi<<<B, 32, 0, s>>>(sts_dev, done_flags);
  return cudaGetLastError();
}

cudaError_t launch_ctrl(CtrlState* st, int slot, int* done_host, int* ran_host, cudaStream_t s) {
  k_ctrl<<<1, 32, 0, s>>>(st, slot, done_host, ran_host);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_prep(PrepArgs a) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = k < a.nrows + a.n;
  const double dlt = in ? prep_item(a, k, a.ctrl) : INFINITY;
  if (!a.sopA) return;
  // K2s screen bounds: per-side minimum shift, block-reduced, one atomic per side and block
  double mr = (in && k < a.nrows) ? dlt : INFINITY;
  double mc = (in && k >= a.nrows) ? dlt : INFINITY;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mr = fmin(mr, __shfl_xor_sync(0xffffffffu, mr, off));
    mc = fmin(mc, __shfl_xor_sync(0xffffffffu, mc, off));
  }
  __shared__ double sm[2][8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sm[0][w] = mr; sm[1][w] = mc; }
  __syncthreads();
  if (threadIdx.x < 2) {
    double m = INFINITY;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) m = fmin(m, sm[threadIdx.x][q]);
    if (m < INFINITY) atomicMin(&a.smin[threadIdx.x], double_key(m));
  }
}

__global__ void k_prep_multi(const PrepArgs* args) {
  const PrepArgs& a = args[blockIdx.y];
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.nrows + a.n) return;
  prep_item(a, k, a.ctrl);
}

cudaError_t launch_prep_multi(const PrepArgs* args_dev, const PrepArgs& a0, int B, cudaStream_t st) {
  const int64_t items = a0.nrows + a0.n;
  k_prep_multi<<<dim3((unsigned)((items + 255) / 256), (unsigned)B), 256, 0, st>>>(args_dev);
  return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st) {
  const int64_t items = a.nrows + a.n;
  k_prep<<<(unsigned)((items + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// K2s (screen.cu): max_j |y_j| over the points (the tf32 error bound), once
// per solve; one CTA, fixed-order reduction
__global__ void __launch_bounds__(1024) k_norm_max(const float* __restrict__ P, int64_t m, int d, double* out) {
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) s = __fma_rn((double)P[i * d + t], (double)P[i * d + t], s);
    mx = fmax(mx, sqrt(s));
  }
  __shared__ double sm[32];
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sm[w]);
    *out = __dmul_rn(mx, 1.0 + 1e-6);
  }
}
cudaError_t launch_norm_max(const float* P, int64_t m, int d, double* out, cudaStream_t st) {
  k_norm_max<<<1, 1024, 0, st>>>(P, m, d, out);
  return cudaGetLastError();
}
// K2s padding rows (past nrows / n up to the chunk / tile multiple): never kept
__global__ void k_sop_pad(float* sopA, int64_t nrows, int64_t nrows_p, float* sopB, int64_t n, int64_t n_p) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ka = nrows_p - nrows, kb = n_p - n;
  if (t >= ka + kb) return;
  const bool isA = t < ka;
  const int64_t r = isA ? nrows + t : n + (t - ka);
  float v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = 0.f;
  if (isA) { v[16] = -1.0e32f; v[20] = 1.f; v[21] = 1.f; }
  else { v[18] = -1.0e32f; }
  sop_store((isA ? sopA : sopB) + r * 32, r, v);
}
cudaError_t launch_sop_pad(float* sopA, int64_t nrows, float* sopB, int64_t n, cudaStream_t st) {
  const int64_t nrows_p = (nrows + 127) / 128 * 128 + 128, n_p = (n + 255) / 256 * 256;
  const int64_t tot = nrows_p - nrows + n_p - n;
  if (tot > 0) k_sop_pad<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(sopA, nrows, nrows_p, sopB, n, n_p);
  return cudaGetLastError();
}

// Z22b squared norms, once per solve (O(m d)): one thread per point.
__global__ void k_sqnorms(const float* __restrict__ P, int64_t m, int d, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = sqnorm_recipe(P + i * d, d);
}

cudaError_t launch_sqnorms(const float* P, int64_t m, int d, float* out, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_sqnorms<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(P, m, d, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
__global__ void k_setup(int64_t n, const double* r, double* logr, double* rho) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lr = log(r[i]);
  logr[i] = lr;
  double a = rint(0.5 * lr * L2E_D);
  if (a < -60.0) a = -60.0;
  if (a > 0.0) a = 0.0;
  rho[i] = a;
}
cudaError_t launch_setup(int64_t n, const double* r, double* logr, double* rho, cudaStream_t st) {
  k_setup<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, r, logr, rho);
  return cudaGetLastError();
}

// min / max of all entries of a cost (input validation of the small-problem
// paths): one CTA, grid-stride, NaN reported as -inf / +inf
__global__ void __launch_bounds__(1024) k_minmax(const void* C, int c64, int64_t count, double* out) {
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t k = threadIdx.x; k < count; k += blockDim.x) {
    const double v = c64 ? reinterpret_cast<const double*>(C)[k] : (double)reinterpret_cast<const float*>(C)[k];
    if (v != v) { lo = -INFINITY; hi = INFINITY; }
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  __shared__ double slo[32], shi[32];
  for (int off = 16; off > 0; off >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fmin(lo, slo[w]); hi = fmax(hi, shi[w]); }
    out[0] = fmin(lo, slo[0]);
    out[1] = fmax(hi, shi[0]);
  }
}
cudaError_t launch_minmax(const void* C, int c64, int64_t count, double* out, cudaStream_t st) {
  k_minmax<<<1, 1024, 0, st>>>(C, c64, count, out);
  return cudaGetLastError();
}

__global__ void k_axpby(int64_t n, double a, const double* x, double b, double* y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i] + b * y[i];
}
cudaError_t launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_axpby<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, a, x, b, y);
  return cudaGetLastError();
}

__global__ void k_add_scalar(int64_t n, double d, double* y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += d;
}
__global__ void k_sum_scalars(const double* a, const double* b, double* out, const int* done) {
  if (done && *done) return;
  const int q = threadIdx.x;
  if (q < kNumScalars) out[q] = a[q] + b[q];
}
cudaError_t launch_sum_scalars(const double* a, const double* b, double* out, const int* done, cudaStream_t st) {
  k_sum_scalars<<<1, 32, 0, st>>>(a, b, out, done);
  return cudaGetLastError();
}
__global__ void k_lse_finish(int64_t n, const double* M, const double* S, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = M[i] + log(S[i]);
}
cudaError_t launch_lse_finish(int64_t n, const double* M, const double* S, double* out, cudaStream_t st) {
  k_lse_finish<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, M, S, out);
  return cudaGetLastError();
}
cudaError_t launch_add_scalar(int64_t n, double d, double* y, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_add_scalar<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d, y);
  return cudaGetLastError();
}

__global__ void k_fill(int64_t n, double v, double* y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = v;
}
cudaError_t launch_fill(int64_t n, double v, double* y, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_fill<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, v, y);
  return cudaGetLastError();
}

struct DotPtrs { const double* x[4]; const double* y[4]; };
__global__ void k_dots(int64_t n, int npairs, DotPtrs P, double* blockpart, unsigned int* ticket,
                       double* out_dev, double* out_host) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < n) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < npairs) v[k] = P.x[k][i] * P.y[k][i];
  }
  block_reduce_and_publish<4>(v, blockpart, ticket, out_dev, out_host);
}
// NC2: the line-search scalars of a trial from this rank's
// partials alone, no vector exchange -- phi'(alpha) and the mass are linear in
// the marginals, so each rank sums its own partials' contributions
// (PAPER.md:694-696): out[0] = sum_i p_i R_i 2^rho_i, out[1] = sum_i R_i 2^rho_i,
// out[2] = sum_j p_j C_j 2^sig_j (R, C: this rank's anchored row / column
// partial totals), out[3] = non-finite count + the prep range flag.
__global__ void __launch_bounds__(256) k_nc2_trial(const double* rowpart, int nct, const double* colpart, int nrt,
                                                   int64_t nrows, int64_t n, const double* rho_r,
                                                   const double* sig_c, const double* p, const int* flag,
                                                   double* blockpart, unsigned int* ticket, double* out_dev) {
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nrows + n; k += (int64_t)gridDim.x * blockDim.x) {
    if (k < nrows) {
      const double R = sum_strided(rowpart + k, nrows, nct) * exp2(rho_r[k]);
      v[0] += p[k] * R;
      v[1] += R;
      if (!isfinite(R)) v[3] += 1.0;
    } else {
      const int64_t j = k - nrows;
      const double Cj = sum_strided(colpart + j, n, nrt) * exp2(sig_c[j]);
      v[2] += p[k] * Cj;
      if (!isfinite(Cj)) v[3] += 1.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && flag) v[3] += (double)(*flag);
  block_reduce_and_publish<4>(v, blockpart, ticket, out_dev, nullptr);
}
cudaError_t launch_nc2_trial(const double* rowpart, int nct, const double* colpart, int nrt, int64_t nrows, int64_t n,
                             const double* rho_r, const double* sig_c, const double* p, const int* flag,
                             double* blockpart, unsigned int* ticket, double* out_dev, cudaStream_t st) {
  const int64_t items = nrows + n;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 296));
  k_nc2_trial<<<blocks, 256, 0, st>>>(rowpart, nct, colpart, nrt, nrows, n, rho_r, sig_c, p, flag, blockpart, ticket,
                                      out_dev);
  return cudaGetLastError();
}

cudaError_t launch_dots(int64_t n, int npairs, const double* const* xs, const double* const* ys,
                        double* blockpart, unsigned int* ticket, double* out_dev, double* out_host,
                        cudaStream_t st) {
  DotPtrs P;
  for (int k = 0; k < 4; ++k) {
    P.x[k] = k < npairs ? xs[k] : nullptr;
    P.y[k] = k < npairs ? ys[k] : nullptr;
  }
  const unsigned blocks = (unsigned)((n + 255) / 256);
  k_dots<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(n, npairs, P, blockpart, ticket, out_dev, out_host);
  return cudaGetLastError();
}

// Sampled input check (C in [0, 1]): 64 entries at a fixed
// hash of the index gathered by one launch into a mapped host buffer (one
// synchronisation instead of one device-to-host copy per sample).
__global__ void k_sample_c(const void* C, int c64, int64_t count, int S, double* out) {
  const int q = threadIdx.x;
  if (q >= S) return;
  const int64_t idx = (int64_t)(((uint64_t)q * 2654435761ull) % (uint64_t)count);
  out[q] = c64 ? reinterpret_cast<const double*>(C)[idx] : (double)reinterpret_cast<const float*>(C)[idx];
}
cudaError_t launch_sample_c(const void* C, int c64, int64_t count, int S, double* out, cudaStream_t st) {
  k_sample_c<<<1, 64, 0, st>>>(C, c64, count, S, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// sharded helpers
// ---------------------------------------------------------------------------
__global__ void k_reduce_colpart(const double* colpart, int nt, int64_t n, double* coltot, const int* done) {
  if (done && *done) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  coltot[j] = sum_strided(colpart + j, n, nt);
}
cudaError_t launch_reduce_colpart(const double* colpart, int nt, int64_t n, double* coltot, cudaStream_t st,
                                  const int* done) {
  k_reduce_colpart<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(colpart, nt, n, coltot, done);
  return cudaGetLastError();
}
__global__ void k_exact_colcombine(const double* colm, const double* cols, int chunks, int64_t n, double* M,
                                   double* S) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double m = -INFINITY, s = 0.0;
  for (int c = 0; c < chunks; ++c) lse_merge(m, s, colm[(int64_t)c * n + j], cols[(int64_t)c * n + j]);
  M[j] = m;
  S[j] = s;
}
cudaError_t launch_exact_colcombine(const double* colm, const double* cols, int chunks, int64_t n, double* M,
                                    double* S, cudaStream_t st) {
  k_exact_colcombine<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(colm, cols, chunks, n, M, S);
  return cudaGetLastError();
}
__global__ void k_rescale_to_max(int64_t n, const double* Mloc, const double* Mglob, double* S) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  S[j] = (S[j] == 0.0) ? 0.0 : S[j] * exp(Mloc[j] - Mglob[j]);
}
cudaError_t launch_rescale_to_max(int64_t n, const double* Mloc, const double* Mglob, double* S, cudaStream_t st) {
  k_rescale_to_max<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, Mloc, Mglob, S);
  return cudaGetLastError();
}
__global__ void k_sum_chunks(const double* x, int chunks, int64_t n, double* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int c = 0; c < chunks; ++c) acc += x[(int64_t)c * n + j];
  out[j] = acc;
}
cudaError_t launch_sum_chunks(const double* x, int chunks, int64_t n, double* out, cudaStream_t st) {
  k_sum_chunks<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, chunks, n, out);
  return cudaGetLastError();
}

__global__ void k_l2_normal(const char* p, size_t lines) {
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < lines; q += (size_t)gridDim.x * blockDim.x)
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(p + 128 * q) : "memory");
}
cudaError_t launch_l2_normal(const void* p, size_t bytes, cudaStream_t st) {
  const uintptr_t b = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(127);
  const size_t lines = (reinterpret_cast<uintptr_t>(p) + bytes - b + 127) / 128;
  if (lines == 0) return cudaSuccess;
  k_l2_normal<<<296, 256, 0, st>>>(reinterpret_cast<const char*>(b), lines);
  return cudaGetLastError();
}


void fault_set_kernels(int mode) { fault_set_tu(mode); }

}  // namespace mdot

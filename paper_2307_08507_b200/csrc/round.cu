// paper_2307_08507_b200/csrc/round.cu -- a10: rounding onto U(r,c) and the
// cost <C, G> ("rounded onto U(r,c) via Alg. 2 of Altschuler et
// al."; the procedure as restated in SPEC.md:331):
//   x = min(r / r(F), 1); F' = D(x) F; y = min(c / c(F'), 1); F'' = F' D(y)
//   err_r = r - r(F''); err_c = c - c(F''); G = F'' + err_r err_c^T / |err_r|_1
//   <C, G> = <C, F''> + err_r^T C err_c / |err_r|_1
// with F = exp(U + V - gbar C), in fp64 (once per solve), as three passes:
//   R0 rows (r(F), <C, F>), R2 columns (c(F')), R3 rows (r(F''), <C, F''>,
//   C err_c).
// Two cost kinds:
//   dense C    row passes: one warp per row (coalesced float4 rows of C);
//              column pass: one thread per column over a chunk of rows
//   on the fly row passes: one thread per row, 128-column tiles of Y staged
//              in shared memory and read as broadcasts; column pass: one
//              thread per column, 128-row tiles of X staged.  The distance is
//              the Z22 fp32 recipe (acc = fmaf(x_k - y_k, x_k - y_k, acc),
//              times scale) op for op, so every pass sees the same C_ij bits
//              as the solve.
// Entries whose exponent lies more than 50 below the log target of their
// pass's marginal (log r_i for row passes, log c_j for the column pass) are
// not exponentiated: each is < e^-50 = 2e-22 of that target, so a pass drops
// < n x 2e-22 of the total mass (1.3e-17 at n = 65536) -- below the fp64
// resolution of every quantity the rounding produces.  At gbar = 4096 that is
// almost every entry (effective support ~2 per row), so a pass costs the
// cost read (dense: HBM) or the distance (on the fly: FP32 pipe), not fp64 exp.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "internal.cuh"
#include "otf_cost.cuh"

namespace mdot {

constexpr double kRoundSkip = 50.0;
constexpr int kRT = 128;   // rows / columns per on-the-fly tile and per CTA

// unscaled pair cost with the thread's own point in registers (x, its squared
// norm nx for the dot form) and the other point y (norm ny) from shared memory;
// the dot form is symmetric bit for bit (fl(nx + ny) and the exact products)
template <int D, bool DOT>
__device__ __forceinline__ float pair_cost_t(const float (&x)[D], float nx, const float* y, float ny) {
  if (DOT) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) s = __fmaf_rn(x[k], y[k], s);
    return fmaxf(__fmaf_rn(-2.0f, s, __fadd_rn(nx, ny)), 0.0f);
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float dk = __fsub_rn(x[k], y[k]);
    acc = __fmaf_rn(dk, dk, acc);
  }
  return acc;
}
template <int D>
__device__ __forceinline__ float sqnorm_t(const float (&x)[D]) {
  float a = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) a = __fmaf_rn(x[k], x[k], a);
  return a;
}

// ---------------------------------------------------------------- dense rows
// warp per row; lane j-stride 32 (float4 groups of 4 columns when n % 4 == 0)
template <bool CORR>
__global__ void __launch_bounds__(256) k_round_rows_dense(RoundArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= a.nrows) return;
  const double Ai = a.A[i], thr = a.logr[i] - kRoundSkip, g = a.gbar;
  double s = 0.0, cs = 0.0, cr = 0.0;
  auto one = [&](double cij, int64_t j) {
    const double z = (Ai + a.B[j]) - g * cij;
    if (z > thr) {
      const double f = exp(z);
      s += f;
      cs += cij * f;
    }
    if (CORR) cr += cij * a.ec[j];
  };
  if (!a.c_f64 && (a.n & 3) == 0 && (a.ldc & 3) == 0) {
    const float4* row = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.C) + i * a.ldc);
#pragma unroll 4
    for (int64_t q = lane; q < a.n / 4; q += 32) {
      const float4 c4 = __ldg(row + q);
      one((double)c4.x, 4 * q);
      one((double)c4.y, 4 * q + 1);
      one((double)c4.z, 4 * q + 2);
      one((double)c4.w, 4 * q + 3);
    }
  } else {
    for (int64_t j = lane; j < a.n; j += 32) {
      const double cij = a.c_f64 ? reinterpret_cast<const double*>(a.C)[i * a.ldc + j]
                                 : (double)reinterpret_cast<const float*>(a.C)[i * a.ldc + j];
      one(cij, j);
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, off);
    cs += __shfl_xor_sync(0xffffffffu, cs, off);
    if (CORR) cr += __shfl_xor_sync(0xffffffffu, cr, off);
  }
  if (lane == 0) {
    a.rowS[i] = s;
    a.rowC[i] = cs;
    if (CORR) a.rowE[i] = cr;
  }
}

// ------------------------------------------------------------- dense columns
// thread per column, rows of chunk blockIdx.y
__global__ void __launch_bounds__(256) k_round_cols_dense(RoundArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  const int64_t rows_per = (a.nrows + a.chunks - 1) / a.chunks;
  const int64_t ib = chunk * rows_per;
  const int64_t ie = (ib + rows_per < a.nrows) ? ib + rows_per : a.nrows;
  if (j >= a.n) return;
  const double Bj = a.B[j], thr = a.logc[j] - kRoundSkip, g = a.gbar;
  double s = 0.0;
  // 8 rows' loads in flight per thread (the loop is otherwise one dependent
  // L2/HBM round trip per row: 0.9 TB/s on config 4)
#pragma unroll 8
  for (int64_t i = ib; i < ie; ++i) {
    const double cij = a.c_f64 ? __ldg(reinterpret_cast<const double*>(a.C) + i * a.ldc + j)
                               : (double)__ldg(reinterpret_cast<const float*>(a.C) + i * a.ldc + j);
    const double z = (__ldg(a.A + i) + Bj) - g * cij;
    if (z > thr) s += exp(z);
  }
  a.colS[(int64_t)chunk * a.n + j] = s;
}

// ---------------------------------------------------------- on-the-fly rows
// thread per row (128 rows per CTA), columns of chunk blockIdx.y in tiles of
// 128: Y tile, B and err_c staged in shared memory, read as broadcasts
template <int D, bool CORR, bool DOT>
__global__ void __launch_bounds__(kRT) k_round_rows_otf(RoundArgs a) {
  __shared__ __align__(16) float sY[kRT * D];
  __shared__ double sB[kRT], sE[kRT];
  __shared__ float sN[kRT];
  const int t = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * kRT + t;
  const bool ok = i < a.nrows;
  float x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = ok ? a.X[i * D + k] : 0.f;
  const float nx = DOT ? sqnorm_t<D>(x) : 0.f;
  const double Ai = ok ? a.A[i] : 0.0, thr = ok ? a.logr[i] - kRoundSkip : INFINITY, g = a.gbar;
  const int64_t cols_per = ((a.n + a.chunks - 1) / a.chunks + kRT - 1) / kRT * kRT;
  const int64_t jb = (int64_t)blockIdx.y * cols_per;
  const int64_t je = (jb + cols_per < a.n) ? jb + cols_per : a.n;
  double s = 0.0, cs = 0.0, cr = 0.0;
  for (int64_t j0 = jb; j0 < je; j0 += kRT) {
    const int w = (int)((je - j0) < kRT ? (je - j0) : kRT);
    __syncthreads();
    for (int q = t; q < kRT * D; q += kRT) sY[q] = (q / D < w) ? a.Y[j0 * D + q] : 0.f;
    if (t < w) {
      sB[t] = a.B[j0 + t];
      if (CORR) sE[t] = a.ec[j0 + t];
    }
    __syncthreads();
    if (DOT) {   // column squared norms of the tile (Z22b), one per thread
      if (t < w) sN[t] = sqnorm_recipe(sY + t * D, D);
      __syncthreads();
    }
    for (int jj = 0; jj < w; ++jj) {
      const double cij = (double)__fmul_rn(pair_cost_t<D, DOT>(x, nx, sY + jj * D, DOT ? sN[jj] : 0.f), a.scale);
      const double z = (Ai + sB[jj]) - g * cij;
      if (z > thr) {
        const double f = exp(z);
        s += f;
        cs += cij * f;
      }
      if (CORR) cr += cij * sE[jj];
    }
  }
  if (ok) {
    MDOT_DCHECK((int)blockIdx.y < a.chunks && a.chunks <= kRoundMaxChunks);
    const int64_t o = (int64_t)blockIdx.y * a.nrows + i;
    a.rowS[o] = s;
    a.rowC[o] = cs;
    if (CORR) a.rowE[o] = cr;
  }
}

// ------------------------------------------------------- on-the-fly columns
// thread per column (128 columns per CTA), rows of chunk blockIdx.y in tiles
// of 128: X tile and A staged in shared memory
template <int D, bool DOT>
__global__ void __launch_bounds__(kRT) k_round_cols_otf(RoundArgs a) {
  __shared__ __align__(16) float sX[kRT * D];
  __shared__ double sA[kRT];
  __shared__ float sN[kRT];
  const int t = threadIdx.x;
  const int64_t j = (int64_t)blockIdx.x * kRT + t;
  const bool ok = j < a.n;
  float y[D];
#pragma unroll
  for (int k = 0; k < D; ++k) y[k] = ok ? a.Y[j * D + k] : 0.f;
  const float ny = DOT ? sqnorm_t<D>(y) : 0.f;
  const double Bj = ok ? a.B[j] : 0.0, thr = ok ? a.logc[j] - kRoundSkip : INFINITY, g = a.gbar;
  const int64_t rows_per = ((a.nrows + a.chunks - 1) / a.chunks + kRT - 1) / kRT * kRT;
  const int64_t ib = (int64_t)blockIdx.y * rows_per;
  const int64_t ie = (ib + rows_per < a.nrows) ? ib + rows_per : a.nrows;
  double s = 0.0;
  for (int64_t i0 = ib; i0 < ie; i0 += kRT) {
    const int w = (int)((ie - i0) < kRT ? (ie - i0) : kRT);
    __syncthreads();
    for (int q = t; q < kRT * D; q += kRT) sX[q] = (q / D < w) ? a.X[i0 * D + q] : 0.f;
    if (t < w) sA[t] = a.A[i0 + t];
    __syncthreads();
    if (DOT) {
      if (t < w) sN[t] = sqnorm_recipe(sX + t * D, D);
      __syncthreads();
    }
    for (int ii = 0; ii < w; ++ii) {
      // the diff recipe is symmetric in the operand order only up to the sign
      // of x - y, whose square is exact: (x_k - y_k)^2 == (y_k - x_k)^2 bitwise
      const double cij = (double)__fmul_rn(pair_cost_t<D, DOT>(y, ny, sX + ii * D, DOT ? sN[ii] : 0.f), a.scale);
      const double z = (sA[ii] + Bj) - g * cij;
      if (z > thr) s += exp(z);
    }
  }
  if (ok) a.colS[(int64_t)blockIdx.y * a.n + j] = s;
}

// ------------------------------------------- on-the-fly, any d (generic path)
template <bool CORR>
__global__ void __launch_bounds__(256) k_round_rows_otf_any(RoundArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= a.nrows) return;
  const double Ai = a.A[i], thr = a.logr[i] - kRoundSkip, g = a.gbar;
  double s = 0.0, cs = 0.0, cr = 0.0;
  for (int64_t j = lane; j < a.n; j += 32) {
    const double cij = otf_cost(a.X + i * a.d, a.Y + j * a.d, a.d, a.scale, a.otf);
    const double z = (Ai + a.B[j]) - g * cij;
    if (z > thr) {
      const double f = exp(z);
      s += f;
      cs += cij * f;
    }
    if (CORR) cr += cij * a.ec[j];
  }
  for (int off = 16; off > 0; off >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, off);
    cs += __shfl_xor_sync(0xffffffffu, cs, off);
    if (CORR) cr += __shfl_xor_sync(0xffffffffu, cr, off);
  }
  if (lane == 0) {
    a.rowS[i] = s;
    a.rowC[i] = cs;
    if (CORR) a.rowE[i] = cr;
  }
}

__global__ void __launch_bounds__(256) k_round_cols_otf_any(RoundArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  const int64_t rows_per = (a.nrows + a.chunks - 1) / a.chunks;
  const int64_t ib = chunk * rows_per;
  const int64_t ie = (ib + rows_per < a.nrows) ? ib + rows_per : a.nrows;
  if (j >= a.n) return;
  const double Bj = a.B[j], thr = a.logc[j] - kRoundSkip, g = a.gbar;
  double s = 0.0;
  for (int64_t i = ib; i < ie; ++i) {
    const double cij = otf_cost(a.X + i * a.d, a.Y + j * a.d, a.d, a.scale, a.otf);
    const double z = (a.A[i] + Bj) - g * cij;
    if (z > thr) s += exp(z);
  }
  a.colS[(int64_t)chunk * a.n + j] = s;
}

// ------------------------------------------------------------------- plan
__global__ void k_round_plan(RoundArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= a.n || i >= a.nrows) return;
  double cij;
  if (a.otf) cij = otf_cost(a.X + i * a.d, a.Y + j * a.d, a.d, a.scale, a.otf);
  else if (a.c_f64) cij = reinterpret_cast<const double*>(a.C)[i * a.ldc + j];
  else cij = (double)reinterpret_cast<const float*>(a.C)[i * a.ldc + j];
  double gij = exp((a.A[i] + a.B[j]) - a.gbar * cij);
  if (a.inv_ner > 0.0) gij += a.er[i] * a.ec[j] * a.inv_ner;
  a.plan[i * a.n + j] = (float)gij;
}

// ------------------------------------------------------------ combines
__global__ void k_round_x(int64_t nrows, int chunks, const double* rowS, const double* rowC, const double* r,
                          const double* U, double* logx, double* Aout, double* rowcostF) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0, cs = 0.0;
  for (int q = 0; q < chunks; ++q) {
    s += rowS[(int64_t)q * nrows + i];
    cs += rowC[(int64_t)q * nrows + i];
  }
  // log x = min(log r - log r(F), 0); r(F) = 0 (every entry skipped: r(F) <
  // n e^-50 r_i) leaves x = 1
  const double lx = (s > 0.0) ? fmin(log(r[i]) - log(s), 0.0) : 0.0;
  logx[i] = lx;
  Aout[i] = U[i] + lx;
  rowcostF[i] = cs;
}

__global__ void k_round_y(int64_t n, int chunks, const double* colS, const double* c, const double* V,
                          double* Bout, double* ec) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double cf = 0.0;
  for (int q = 0; q < chunks; ++q) cf += colS[(int64_t)q * n + j];
  const double y = (cf > 0.0) ? fmin(c[j] / cf, 1.0) : 1.0;
  Bout[j] = V[j] + log(y);
  // c(F'') = y c(F') <= c in exact arithmetic; the clamp removes the
  // last-bit sign flips of the fp64 product
  ec[j] = fmax(c[j] - y * cf, 0.0);
}

// one CTA, fixed order: thread t sums items t, t + 1024, ...; then a fixed tree
__global__ void __launch_bounds__(1024) k_round_fin(int64_t nrows, int chunks, const double* rowS,
                                                    const double* rowC, const double* rowE, const double* rowcostF,
                                                    const double* r, double* er, double* out_dev, double* out_host) {
  __shared__ double red[4][1024];
  const int t = threadIdx.x;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  for (int64_t i = t; i < nrows; i += 1024) {
    double s = 0.0, cs = 0.0, cr = 0.0;
    for (int q = 0; q < chunks; ++q) {
      s += rowS[(int64_t)q * nrows + i];
      cs += rowC[(int64_t)q * nrows + i];
      cr += rowE[(int64_t)q * nrows + i];
    }
    // r(F'') <= x r(F) <= r in exact arithmetic (x from the fp64 r(F)); the
    // clamp keeps G >= 0 against fp64 rounding of the row sums
    const double e = fmax(r[i] - s, 0.0);
    er[i] = e;
    v0 += e;
    v1 += cs;
    v2 += e * cr;
    v3 += rowcostF[i];
  }
  red[0][t] = v0; red[1][t] = v1; red[2][t] = v2; red[3][t] = v3;
  __syncthreads();
  for (int h = 512; h > 0; h >>= 1) {
    if (t < h)
      for (int q = 0; q < 4; ++q) red[q][t] += red[q][t + h];
    __syncthreads();
  }
  if (t < 4) {
    out_dev[t] = red[t][0];
    if (out_host) out_host[t] = red[t][0];
  }
}

// ------------------------------------------------------------ launchers
static bool otf_tiled(int d) { return d == 2 || d == 3 || d == 4 || d == 8 || d == 16 || d == 32; }

int round_chunks(const RoundArgs& a, bool rows) {
  // enough CTAs for ~2 waves of 148 SMs; at most kRoundMaxChunks partials
  if (!a.otf) return rows ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(kRoundMaxChunks, (8 * 148) / ((a.n + 255) / 256)));
  if (!otf_tiled(a.d)) return rows ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(kRoundMaxChunks, (8 * 148) / ((a.n + 255) / 256)));
  const int64_t blocks = rows ? (a.nrows + kRT - 1) / kRT : (a.n + kRT - 1) / kRT;
  int ch = 1;
  while (ch < kRoundMaxChunks && blocks * ch < 16 * 148) ch *= 2;
  return ch;
}

template <int D>
static cudaError_t rows_otf_t(const RoundArgs& a, int corr, cudaStream_t st) {
  dim3 grid((unsigned)((a.nrows + kRT - 1) / kRT), (unsigned)a.chunks);
  const bool dot = a.otf == 2;
  if (corr) {
    if (dot) k_round_rows_otf<D, true, true><<<grid, kRT, 0, st>>>(a);
    else k_round_rows_otf<D, true, false><<<grid, kRT, 0, st>>>(a);
  } else {
    if (dot) k_round_rows_otf<D, false, true><<<grid, kRT, 0, st>>>(a);
    else k_round_rows_otf<D, false, false><<<grid, kRT, 0, st>>>(a);
  }
  return cudaGetLastError();
}
template <int D>
static cudaError_t cols_otf_t(const RoundArgs& a, cudaStream_t st) {
  dim3 grid((unsigned)((a.n + kRT - 1) / kRT), (unsigned)a.chunks);
  if (a.otf == 2) k_round_cols_otf<D, true><<<grid, kRT, 0, st>>>(a);
  else k_round_cols_otf<D, false><<<grid, kRT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_round_rows(const RoundArgs& a, int with_corr, cudaStream_t st) {
  if (a.otf) {
    switch (a.d) {
      case 2: return rows_otf_t<2>(a, with_corr, st);
      case 3: return rows_otf_t<3>(a, with_corr, st);
      case 4: return rows_otf_t<4>(a, with_corr, st);
      case 8: return rows_otf_t<8>(a, with_corr, st);
      case 16: return rows_otf_t<16>(a, with_corr, st);
      case 32: return rows_otf_t<32>(a, with_corr, st);
      default: break;
    }
    // any other d: one warp per row, chunks must be 1
    const unsigned blocks = (unsigned)((a.nrows + 7) / 8);
    if (with_corr) k_round_rows_otf_any<true><<<blocks, 256, 0, st>>>(a);
    else k_round_rows_otf_any<false><<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  const unsigned blocks = (unsigned)((a.nrows + 7) / 8);
  if (with_corr) k_round_rows_dense<true><<<blocks, 256, 0, st>>>(a);
  else k_round_rows_dense<false><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_round_cols(const RoundArgs& a, cudaStream_t st) {
  if (a.otf) {
    switch (a.d) {
      case 2: return cols_otf_t<2>(a, st);
      case 3: return cols_otf_t<3>(a, st);
      case 4: return cols_otf_t<4>(a, st);
      case 8: return cols_otf_t<8>(a, st);
      case 16: return cols_otf_t<16>(a, st);
      case 32: return cols_otf_t<32>(a, st);
      default: break;
    }
    dim3 grid((unsigned)((a.n + 255) / 256), (unsigned)a.chunks);
    k_round_cols_otf_any<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((a.n + 255) / 256), (unsigned)a.chunks);
  k_round_cols_dense<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_round_plan(const RoundArgs& a, cudaStream_t st) {
  dim3 grid((unsigned)((a.n + 255) / 256), (unsigned)a.nrows);
  k_round_plan<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_round_x(int64_t nrows, int chunks, const double* rowS, const double* rowC, const double* r,
                           const double* U, double* logx, double* Aout, double* rowcostF, cudaStream_t st) {
  k_round_x<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(nrows, chunks, rowS, rowC, r, U, logx, Aout, rowcostF);
  return cudaGetLastError();
}

cudaError_t launch_round_y(int64_t n, int chunks, const double* colS, const double* c, const double* V,
                           double* Bout, double* ec, cudaStream_t st) {
  k_round_y<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, chunks, colS, c, V, Bout, ec);
  return cudaGetLastError();
}

cudaError_t launch_round_fin(int64_t nrows, int chunks, const double* rowS, const double* rowC, const double* rowE,
                             const double* rowcostF, const double* r, double* er, double* /*blockpart*/,
                             unsigned int* /*ticket*/, double* out_dev, double* out_host, cudaStream_t st) {
  k_round_fin<<<1, 1024, 0, st>>>(nrows, chunks, rowS, rowC, rowE, rowcostF, r, er, out_dev, out_host);
  return cudaGetLastError();
}

}  // namespace mdot

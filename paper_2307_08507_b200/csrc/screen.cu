// paper_2307_08507_b200/csrc/screen.cu -- K2s: the on-the-fly-cost marginal
// evaluation with a tensor-core screen.
//
// The fused evaluation sums P_ij = exp(A_i + B_j - gbar C_ij) over every
// (i, j) (Alg. 2).  At the gbar of the later
// MD steps almost all of those n^2 entries are far below both their row's and
// their column's total (config 5, gbar 4096: ~0.05 % of them are within e^-40
// of either, profiles/r02_screen_fraction.txt), yet the dense kernel (K2,
// kernels.cu k_eval_otf) pays d + 7 FP32 ops and one MUFU op for each.
//
// K2s evaluates the SAME entries with the SAME fp32 recipe (Z22 / Z22b, bit
// for bit: e = ex2(fma(-gl, C, fma(-gh, C, ah + bh)))), but only where a
// rigorous bound says the entry can matter.  Per 128-row chunk x 256-column
// tile the 5th-generation tensor core computes (kind::tf32, K = 24, one
// elected thread, accumulator in TMEM)
//     t_ij = <2g x~_i, y~_j> + alpha_i + beta_j
// with g = gbar log2(e) scale, x~, y~ the coordinates rounded to tf32, and
//     alpha_i = log2(row factor_i) - g |x_i|^2 - theta_i + m + T + delta_i,
//     beta_j  = log2(col factor_j) - g |y_j|^2 - phi_j
// carried as tf32 hi/lo pairs in four extra K columns, so that
//     t_ij = log2 P_ij - (theta_i + phi_j - m - T) + (delta_i - tf32 error).
// theta_i = min(lr_i, m), phi_j = min(lc_j, m), m = -log2 n, where lr_i, lc_j
// are LOWER bounds (log2) of the row / column totals at the new potentials
// (prep: the accepted iterate's log marginals + this row's potential shift +
// the smallest shift on the other side; a total can only shrink by that
// much).  For every m, theta_i + phi_j - m <= min(lr_i, lc_j), so an entry
// with t_ij < 0 is below 2^-T of its row total AND of its column total;
// dropping all of them changes any marginal by < n 2^-T relative (T = 56:
// < 1e-12 at n = 65536, far below the fp32 entries' 1e-7).  delta_i bounds
// the tf32 error of the dot product: |<2g x~, y~> - <2g x, y>| <=
// 2g |x_i| max_j |y_j| 2^-10 (both operands rounded to nearest tf32, 2^-11
// relative each; Cauchy-Schwarz), plus 2 for the recipe's own rounding, the
// hi/lo splits and the fp32 accumulation in the tensor core.
//
// Entries with t_ij >= 0 ("survivors") are recomputed exactly from the fp32
// coordinates in registers / shared memory with the recipe's op order, so
// every kept entry has the dense kernel's bits; row sums stay with the lane
// that owns the row (TMEM lane = row), column sums are reduced over the
// warp's lanes in a fixed butterfly and accumulated in fp64 per row quarter
// -- deterministic, like every other evaluation kernel.  Outputs are the
// dense kernel's [col tile][nrows] row partials and [row tile][n] column
// partials, so k_finalize is unchanged.
//
// CTA: 256 threads, 2 per SM (TMEM: 256 of the SM's 512 columns each).
// Warp w reads TMEM lanes 32 (w & 3) .. +31 (its rows) and columns
// 128 (w >> 2) .. +127 of the accumulator.  One CTA per (256-column tile,
// row tile); the B operand (Y tile) is built once per CTA, the A operand
// (X chunk) per 128-row chunk.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "entry.cuh"
#include "internal.cuh"
#include "umma.cuh"

namespace mdot {

constexpr int kScrM = 128;          // rows per chunk = MMA M = TMEM lanes
constexpr int kScrN = 256;          // columns per CTA = MMA N = TMEM columns
constexpr int kScrKSteps = 3;       // K = 24 tf32: 16 coordinates (zero-padded) + alpha hi/lo + beta hi/lo
constexpr int kScrThreads = 256;
constexpr int kScrWarps = kScrThreads / 32;
constexpr int kScrMaxD = 16;
constexpr int kScrLCap = 64;        // survivor list entries per warp

struct ScrSmem {
  unsigned char B[kScrN * 128];     // operand B, K-major SW128 (1024-aligned: offset 0)
  unsigned char A[kScrM * 128];     // operand A (offset 32768, 1024-aligned)
  float Y[kScrN][kScrMaxD];         // raw y of the tile's columns (exact path; row stride D)
  float X[2][kScrM][kScrMaxD];      // raw x of the chunk's rows, double-buffered (row stride D)
  float4 colp[kScrN];               // {bh, M_j, T'_j, |y_j|^2 (dot recipe)}
  float4 rowp[2][kScrM];            // {ah, M_i, S'_i, |x_i|^2} of the chunk's rows
  double col[4][kScrN];             // column partials per row quarter (fp64)
  double row[2][2][kScrM];          // row partials of the two column halves, double-buffered by chunk
  uint32_t lidx[kScrWarps][kScrLCap];   // survivor list: (group << 10) | (row << 5) | column
  float lrow[kScrWarps][kScrLCap];      // e * T'_j
  float lcol[kScrWarps][kScrLCap];      // e * S'_i
  unsigned long long mbar_ld[2];    // bulk copies of a chunk (and the tile) landed, one barrier per buffer:
                                    // the prefetch of chunk c + 1 must not complete a second phase of the
                                    // barrier a slow warp still waits on for chunk c
  unsigned long long mbar_mma;      // the chunk's MMAs completed
  uint32_t tbase;
};

__device__ __forceinline__ double key_to_double(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void scr_mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "SCR_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra SCR_DONE;\n"
      "bra SCR_WAIT;\n"
      "SCR_DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void scr_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, 16-byte aligned), completion on the mbarrier
__device__ __forceinline__ void scr_bulk(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}

// 16-byte chunk c (4 floats) of operand row r
__device__ __forceinline__ void put_chunk(unsigned char* op, int r, int c, float4 v) {
  *reinterpret_cast<float4*>(op + umma::sw128_offset((uint32_t)r, (uint32_t)(4 * c))) = v;
}

// The recipe's entry (bit-identical to k_eval_otf's packed lanes):
// C~ (Z22 / Z22b, unscaled when the scale is a power of two and folded into
// ngh / ngl), e = ex2(fma(ngl, C~, fma(ngh, C~, ah + bh))).
template <int D, bool POW2, bool DOT>
__device__ __forceinline__ float exact_entry(const float* xr, const float* yj, float4 rp, float4 cp, float ngh,
                                             float ngl, float scale) {
  float cst;
  if (DOT) {   // Z22b: max(fmaf(-2, s, nx + ny), 0), s = fmaf chain (k ascending)
    float s = 0.f;
#pragma unroll
    for (int kk = 0; kk < D; ++kk) s = __fmaf_rn(xr[kk], yj[kk], s);
    cst = fmaxf(__fmaf_rn(-2.0f, s, __fadd_rn(rp.w, cp.w)), 0.f);
  } else {     // Z22: fmaf chain of (x - y)^2
    float acc = 0.f;
#pragma unroll
    for (int kk = 0; kk < D; ++kk) {
      const float dk = __fsub_rn(xr[kk], yj[kk]);
      acc = __fmaf_rn(dk, dk, acc);
    }
    cst = acc;
  }
  if (!POW2) cst = __fmul_rn(cst, scale);
  const float zh = __fmaf_rn(ngh, cst, __fadd_rn(rp.x, cp.x));
  return ex2_ftz(__fmaf_rn(ngl, cst, zh));
}

template <int D, bool POW2, bool DOT>
__global__ void __launch_bounds__(kScrThreads, 2) k_eval_screen(EvalArgs a) {
  static_assert(D <= kScrMaxD && D % 4 == 0, "screened kernel: d in {4, 8, 16}");
  if (a.done && *a.done) return;
  extern __shared__ unsigned char scr_raw[];
  const uint32_t pad = (1024u - (su32(scr_raw) & 1023u)) & 1023u;
  ScrSmem& S = *reinterpret_cast<ScrSmem*>(scr_raw + pad);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;
  const int64_t n = a.n, nrows = a.nrows;
  const int64_t j0 = (int64_t)blockIdx.x * kScrN;
  const int64_t i0 = (int64_t)blockIdx.y * a.tile_m;
  const int64_t tile_end = (i0 + a.tile_m < nrows) ? i0 + a.tile_m : nrows;
  const int ncols = (int)((n - j0 < kScrN) ? n - j0 : kScrN);

  const float gh = a.gpair ? a.gpair[0] : a.gh;
  const float gl = a.gpair ? a.gpair[1] : a.gl;
  // the grid-wide shift term G = min(D_r, D_c) of the separable bound (screen.cu header),
  // D_r = min column shift (row totals), D_c = min row shift (column totals), log2, -1 slack
  double G;
  {
    const double L2E = 1.4426950408889634;
    const double dr = __dsub_rn(__dmul_rn(key_to_double(a.smin[1]), L2E), 1.0);
    // the smallest row shift: over every rank's rows when the rows are sharded
    const double drow = a.smin_rows_neg ? -a.smin_rows_neg[0] : key_to_double(a.smin[0]);
    const double dc = __dsub_rn(__dmul_rn(drow, L2E), 1.0);
    G = fmin(dr, dc);
    if (!(G == G)) G = -INFINITY;
  }
  double mg = -G;
  if (!(mg < 1.0e30)) mg = 1.0e30;
  const float mgh = umma::to_tf32((float)mg), mgl = umma::to_tf32((float)__dsub_rn(mg, (double)mgh));

  if (warp == 0) umma::tmem_alloc(&S.tbase, kScrN);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&S.mbar_ld[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&S.mbar_ld[1])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&S.mbar_mma)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  S.col[0][tid] = 0.0; S.col[1][tid] = 0.0; S.col[2][tid] = 0.0; S.col[3][tid] = 0.0;
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  auto issue_chunk = [&](int64_t c0, int buf, bool with_tile) {   // thread 0
    const int rows_c = (int)((tile_end - c0 < kScrM) ? tile_end - c0 : kScrM);
    uint32_t bytes = kScrM * 128u + (uint32_t)rows_c * (uint32_t)(D * 4 + 16);
    if (with_tile) bytes += kScrN * 128u + (uint32_t)ncols * (uint32_t)(D * 4 + 16);
    unsigned long long* mb = &S.mbar_ld[buf];
    scr_expect_tx(mb, bytes);
    if (with_tile) {
      scr_bulk(S.B, a.sopB + j0 * 32, kScrN * 128u, mb);
      scr_bulk(&S.Y[0][0], a.Y + j0 * D, (uint32_t)ncols * D * 4u, mb);
      scr_bulk(S.colp, a.colp + j0, (uint32_t)ncols * 16u, mb);
    }
    scr_bulk(S.A, a.sopA + c0 * 32, kScrM * 128u, mb);
    scr_bulk(&S.X[buf][0][0], a.X + c0 * D, (uint32_t)rows_c * D * 4u, mb);
    scr_bulk(&S.rowp[buf][0], a.rowp + c0, (uint32_t)rows_c * 16u, mb);
  };
  if (tid == 0 && i0 < tile_end) issue_chunk(i0, 0, true);

  const uint32_t tmem = S.tbase;
  const uint32_t idesc = umma::idesc_tf32(kScrM, kScrN);
  const uint32_t a_addr = su32(S.A);
  const uint32_t b_addr = su32(S.B);
  const float sg = POW2 ? a.scale : 1.f;
  const float ngh = -gh * sg, ngl = -gl * sg;
  uint32_t* const lidx = S.lidx[warp];
  float* const lrow = S.lrow[warp];
  float* const lcol = S.lcol[warp];
  // raw rows are stored with stride D floats: view the buffers that way
  const float* const Yr = &S.Y[0][0];

  unsigned int kept = 0;
  uint32_t ph_ld[2] = {0u, 0u}, ph_mma = 0;
  int buf = 0;
  for (int64_t c0 = i0; c0 < tile_end; c0 += kScrM, buf ^= 1) {
    const int rows_c = (int)((tile_end - c0 < kScrM) ? tile_end - c0 : kScrM);
    scr_mbar_wait(&S.mbar_ld[buf], buf ? ph_ld[1] : ph_ld[0]);
    if (buf) ph_ld[1] ^= 1u;
    else ph_ld[0] ^= 1u;
    if (c0 == i0) {
      // the grid-wide shift into chunk 5 of every B row ({-G_hi, -G_lo, 0, 0} x A's {1, 1, 0, 0})
      put_chunk(S.B, tid, 5, make_float4(mgh, mgl, 0.f, 0.f));
      umma::fence_proxy_async();
      __syncthreads();
    }
    if (tid == 0) {
      umma::fence_after();
#pragma unroll
      for (int ks = 0; ks < kScrKSteps; ++ks)
        umma::mma_tf32(tmem, umma::smem_desc_sw128(a_addr + 32u * ks), umma::smem_desc_sw128(b_addr + 32u * ks),
                       idesc, ks > 0 ? 1u : 0u);
      umma::mma_commit(&S.mbar_mma);
    }
    scr_mbar_wait(&S.mbar_mma, ph_mma);
    ph_mma ^= 1u;
    umma::fence_after();
    // the operand A buffer is free: prefetch the next chunk (its x / row
    // parameters into the other buffer, last read by chunk c - 1)
    if (tid == 0 && c0 + kScrM < tile_end) issue_chunk(c0 + kScrM, buf ^ 1, false);
    const float* const Xr = &S.X[buf][0][0];
    const float4* const RPr = S.rowp[buf];

    // ---- screen: each warp's 32 rows x 128 columns, four 32-column groups.
    // Survivors go to the warp's list (lane order within a group, columns
    // ascending per lane); the list is evaluated 32 entries per warp step,
    // then every lane adds its own row's entries (list order) and lane k the
    // entries of column k of each group (list order = row order).
    double rsum = 0.0;   // fp64: a lane's row may collect many survivors
    double csum[4] = {0.0, 0.0, 0.0, 0.0};
    int L = 0;                 // list length (warp-uniform)
    int seg_off[4], seg_cnt[4];
#pragma unroll
    for (int gq = 0; gq < 4; ++gq) { seg_off[gq] = 0; seg_cnt[gq] = 0; }
    auto flush = [&]() {
      __syncwarp();
      for (int p = lane; p < L; p += 32) {
        const uint32_t idx = lidx[p];
        const int gq = (int)(idx >> 10), rl = 32 * q + (int)((idx >> 5) & 31u), jc = 128 * h + 32 * gq + (int)(idx & 31u);
        const float4 rpv = RPr[rl];
        const float4 cpv = S.colp[jc];
        float xr[kScrMaxD], yv[kScrMaxD];
#pragma unroll
        for (int c = 0; c < D / 4; ++c) {
          const float4 xx = *reinterpret_cast<const float4*>(Xr + rl * D + 4 * c);
          const float4 yy = *reinterpret_cast<const float4*>(Yr + jc * D + 4 * c);
          xr[4 * c] = xx.x; xr[4 * c + 1] = xx.y; xr[4 * c + 2] = xx.z; xr[4 * c + 3] = xx.w;
          yv[4 * c] = yy.x; yv[4 * c + 1] = yy.y; yv[4 * c + 2] = yy.z; yv[4 * c + 3] = yy.w;
        }
        const float e = exact_entry<D, POW2, DOT>(xr, yv, rpv, cpv, ngh, ngl, a.scale);
        lrow[p] = __fmul_rn(e, cpv.z);
        lcol[p] = __fmul_rn(e, rpv.z);
      }
      __syncwarp();
#pragma unroll
      for (int gq = 0; gq < 4; ++gq)
        for (int t = 0; t < seg_cnt[gq]; ++t) rsum += (double)lrow[seg_off[gq] + t];
      // column k of group gq: entries in list order (ascending rows); four at a time
      int p = 0;
      for (; p + 4 <= L; p += 4) {
        const uint4 i4 = *reinterpret_cast<const uint4*>(lidx + p);
        const float4 c4 = *reinterpret_cast<const float4*>(lcol + p);
        const uint32_t ii[4] = {i4.x, i4.y, i4.z, i4.w};
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((int)(ii[u] & 31u) == lane) {
            const int gq = (int)(ii[u] >> 10);
#pragma unroll
            for (int g2 = 0; g2 < 4; ++g2)
              if (g2 == gq) csum[g2] += (double)cc[u];
          }
      }
      for (; p < L; ++p) {
        const uint32_t idx = lidx[p];
        if ((int)(idx & 31u) == lane) {
          const int gq = (int)(idx >> 10);
#pragma unroll
          for (int g2 = 0; g2 < 4; ++g2)
            if (g2 == gq) csum[g2] += (double)lcol[p];
        }
      }
      kept += (unsigned)L;
      L = 0;
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) seg_cnt[gq] = 0;
      __syncwarp();
    };
#pragma unroll 1
    for (int grp = 0; grp < 4; ++grp) {
      const int cb = 128 * h + 32 * grp;   // first column of this group (CTA-local)
      uint32_t v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)cb, v);
      umma::tmem_ld_wait(v);   // binds v: nothing may read it before the asynchronous load lands
      // some t >= 0 in this lane's 32 values <=> the AND of their bit patterns has a clear sign bit
      uint32_t a0 = v[0] & v[1] & v[2] & v[3], a1 = v[4] & v[5] & v[6] & v[7];
      uint32_t a2 = v[8] & v[9] & v[10] & v[11], a3 = v[12] & v[13] & v[14] & v[15];
      a0 &= v[16] & v[17] & v[18] & v[19];
      a1 &= v[20] & v[21] & v[22] & v[23];
      a2 &= v[24] & v[25] & v[26] & v[27];
      a3 &= v[28] & v[29] & v[30] & v[31];
      // lanes past the chunk's rows (tile heights below 128 rows: the MMA ran
      // over the next tile's rows) never survive
      const bool live = 32 * q + lane < rows_c;
      const uint32_t andv = live ? ((a0 & a1) & (a2 & a3)) : 0x80000000u;
      if (!__any_sync(0xffffffffu, (andv >> 31) == 0u)) continue;
      // the lane's sign bits, bit k <-> column k (funnel shifts, 4 independent chains)
      uint32_t n0 = 0u, n1 = 0u, n2 = 0u, n3 = 0u;
#pragma unroll
      for (int k = 7; k >= 0; --k) {
        n0 = __funnelshift_l(v[k], n0, 1);
        n1 = __funnelshift_l(v[8 + k], n1, 1);
        n2 = __funnelshift_l(v[16 + k], n2, 1);
        n3 = __funnelshift_l(v[24 + k], n3, 1);
      }
      const uint32_t sb = live ? ~(n0 | (n1 << 8) | (n2 << 16) | (n3 << 24)) : 0u;
      const int cnt = __popc(sb);
      int incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (L + tot > kScrLCap) flush();
      if (tot > kScrLCap) {
        // more survivors than the list holds (dense region): column by column
        float rs = 0.f;
#pragma unroll 1
        for (int k = 0; k < 32; ++k) {
          const unsigned mk = __ballot_sync(0xffffffffu, (sb >> k) & 1u);
          if (mk == 0u) continue;
          const int jc = cb + k, rl = 32 * q + lane;
          const float4 rpv = RPr[rl];
          const float4 cpv = S.colp[jc];
          float xr[kScrMaxD], yv[kScrMaxD];
#pragma unroll
          for (int c = 0; c < D; ++c) { xr[c] = Xr[rl * D + c]; yv[c] = Yr[jc * D + c]; }
          float e = exact_entry<D, POW2, DOT>(xr, yv, rpv, cpv, ngh, ngl, a.scale);
          if (!((mk >> lane) & 1u)) e = 0.f;
          rs += __fmul_rn(e, cpv.z);
          float ce = __fmul_rn(e, rpv.z);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) ce += __shfl_xor_sync(0xffffffffu, ce, off);
          if (lane == k) {
#pragma unroll
            for (int gq = 0; gq < 4; ++gq)
              if (gq == grp) csum[gq] += (double)ce;
          }
          kept += (lane == 0) ? (unsigned)__popc(mk) : 0u;
        }
        rsum += (double)rs;
        continue;
      }
      const int off0 = L + incl - cnt;
      {
        uint32_t m = sb;
        int t = off0;
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1u;
          lidx[t++] = ((uint32_t)grp << 10) | ((uint32_t)lane << 5) | (uint32_t)k;
        }
      }
#pragma unroll
      for (int gq = 0; gq < 4; ++gq)   // static indices: the arrays stay in registers
        if (gq == grp) { seg_off[gq] = off0; seg_cnt[gq] = cnt; }
      L += tot;
    }
    if (L > 0) flush();
    // column partials of this warp's rows: lane k holds column k of each group
#pragma unroll
    for (int gq = 0; gq < 4; ++gq)
      if (csum[gq] != 0.0) S.col[q][128 * h + 32 * gq + lane] += csum[gq];
    S.row[buf][h][32 * q + lane] = rsum;
    // M_i before the barrier: the next chunk's copy may overwrite this row-parameter buffer right after it
    const float Mi = tid < rows_c ? RPr[tid].y : 0.f;
    umma::fence_before();
    __syncthreads();
    if (tid < rows_c) a.rowpart[(int64_t)blockIdx.x * nrows + c0 + tid] = (S.row[buf][0][tid] + S.row[buf][1][tid]) * (double)Mi;
  }
  __syncthreads();
  if (tid < ncols)
    a.colpart[(int64_t)blockIdx.y * n + j0 + tid] =
        (((S.col[0][tid] + S.col[1][tid]) + S.col[2][tid]) + S.col[3][tid]) * (double)S.colp[tid].y;
  if (a.scount) {
    // kept: every lane adds L in the list path; lane 0 alone in the dense-region path
    unsigned int kw = (lane == 0) ? kept : 0u;
    kw = __shfl_sync(0xffffffffu, kw, 0);
    if (lane == 0 && kw) atomicAdd(&a.scount[0], (unsigned long long)kw);
    if (tid == 0) atomicAdd(&a.scount[1], (unsigned long long)((tile_end - i0) * ncols));
  }
  if (warp == 0) umma::tmem_dealloc(tmem, kScrN);
}

size_t screen_smem_bytes() { return sizeof(ScrSmem) + 1024; }

__global__ void k_smin_neg(const unsigned long long* smin, double* out) {
  const double v = key_to_double(smin[0]);
  out[0] = (v == v) ? -v : INFINITY;   // NaN (no prep yet) -> +inf: the allreduced bound keeps everything
}
cudaError_t launch_smin_neg(const unsigned long long* smin, double* out, cudaStream_t st) {
  k_smin_neg<<<1, 1, 0, st>>>(smin, out);
  return cudaGetLastError();
}

template <int D, bool POW2, bool DOT>
static cudaError_t launch_screen_t(const EvalArgs& a, cudaStream_t st) {
  const size_t smem = screen_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_eval_screen<D, POW2, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(a.n_col_tiles, a.n_row_tiles);
  k_eval_screen<D, POW2, DOT><<<grid, kScrThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_screen_d(const EvalArgs& a, cudaStream_t st) {
  int e2 = 0;
  const bool pow2 = a.scale > 0.f && frexpf(a.scale, &e2) == 0.5f && e2 > -100 && e2 < 100;
  if (a.otf_dot) return pow2 ? launch_screen_t<D, true, true>(a, st) : launch_screen_t<D, false, true>(a, st);
  return pow2 ? launch_screen_t<D, true, false>(a, st) : launch_screen_t<D, false, false>(a, st);
}

bool screen_supported(int d) { return d == 4 || d == 8 || d == 16; }

cudaError_t launch_eval_screen(const EvalArgs& a, cudaStream_t st) {
  switch (a.d) {
    case 4: return launch_screen_d<4>(a, st);
    case 8: return launch_screen_d<8>(a, st);
    case 16: return launch_screen_d<16>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mdot

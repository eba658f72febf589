// Microbenchmark: per-SM entry rate of the K1 consumer loop (entry_row8_f on
// shared-memory C stages, 4-row butterfly, 16-row fp64 column flush) and of
// variants that move part of the exp2 from the MUFU to the FMA pipe (packed
// Cody-Waite + polynomial), drop the butterfly or the shared loads -- to find
// the per-SM resource that holds K1 (L2-resident), K8 and the shared-C K1 at
// ~6 entries / clk / SM against the 16 / clk / SM MUFU rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_08507_b200/csrc -o /tmp/er bench/entry_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include "entry.cuh"

using namespace mdot;

__device__ __forceinline__ u64 pk2c(float a) { return pk2(a, a); }

// 2^x for a pair on the FMA pipe: x clamped to >= -125, j = rint(x) by the
// 1.5 * 2^23 magic, f = x - j in [-0.5, 0.5], degree-5 polynomial, exponent
// added as an integer (j << 23).
__device__ __forceinline__ u64 exp2_poly2(u64 x) {
  float x0, x1;
  up2(x, x0, x1);
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  x = pk2(x0, x1);
  const u64 M = pk2c(12582912.f);
  const u64 t = add2(x, M);
  const u64 f = sub2(x, sub2(t, M));
  // relative-minimax degree 5 on [-0.5, 0.5]: 2.3e-7 in fp32 Horner
  u64 p = fma2(f, pk2c(0.001327647129073739f), pk2c(0.009675541892647743f));
  p = fma2(p, f, pk2c(0.05550713092088699f));
  p = fma2(p, f, pk2c(0.24022120237350464f));
  p = fma2(p, f, pk2c(0.6931469440460205f));
  p = fma2(p, f, pk2c(1.0000001192092896f));
  float p0, p1, t0, t1;
  up2(p, p0, p1);
  up2(t, t0, t1);
  const float r0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  const float r1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
  return pk2(r0, r1);
}

// V: 0 baseline, 1 pair 0 on the FMA pipe, 2 pairs 0-1, 3 all pairs,
//    4 baseline without the butterfly, 5 baseline with C from registers (no LDS),
//    6 butterfly of stage k-1 at the top of stage k, 7 no proxy fence,
//    8 row params by broadcast LDS (1 CTA/SM at 256 threads: smem), 9 by LDG one stage ahead,
//    10 row totals via smem, 11 butterfly without the row store, 12 row store without the butterfly
template <int V>
__device__ __forceinline__ float row8(const u64 (&c2)[4], float ah, float S, const ColPairs& cp, u64 ngh2, u64 ngl2,
                                      u64 (&cacc)[4]) {
  const u64 ah2 = pk2(ah, ah), S2 = pk2(S, S);
  u64 rsum = 0ull;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const u64 zh = fma2(ngh2, c2[p], add2(ah2, cp.bh[p]));
    const u64 z = fma2(ngl2, c2[p], zh);
    u64 e;
    const bool poly = (V == 1 && p == 0) || (V == 2 && p < 2) || (V == 3);
    if (poly) {
      e = exp2_poly2(z);
    } else {
      float zl, zu;
      up2(z, zl, zu);
      e = pk2(ex2_ftz(zl), ex2_ftz(zu));
    }
    rsum = fma2(e, cp.T[p], rsum);
    cacc[p] = fma2(e, S2, cacc[p]);
  }
  float lo, hi;
  up2(rsum, lo, hi);
  return lo + hi;
}

__device__ __forceinline__ float red4(float v0, float v1, float v2, float v3, int lane) {
  const bool up = lane & 16;
  float k0 = up ? v2 : v0, k1 = up ? v3 : v1;
  const float s0 = up ? v0 : v2, s1 = up ? v1 : v3;
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  const bool up2_ = lane & 8;
  float kk = up2_ ? k1 : k0;
  const float ss = up2_ ? k0 : k1;
  kk += __shfl_xor_sync(0xffffffffu, ss, 8);
  kk += __shfl_xor_sync(0xffffffffu, kk, 4);
  kk += __shfl_xor_sync(0xffffffffu, kk, 2);
  kk += __shfl_xor_sync(0xffffffffu, kk, 1);
  return kk;
}

template <int V>
__global__ void __launch_bounds__(512) k_rate(const float* Cg, const float4* rowp, const float4* colp, double* rowpart,
                                              double* colout, int stages, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float (*st)[32][256] = reinterpret_cast<float (*)[32][256]>(smem_raw);
  double (*sred)[256] = reinterpret_cast<double (*)[256]>(smem_raw + 3 * 32 * 256 * 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  for (int q = tid; q < 3 * 32 * 256; q += blockDim.x) (&st[0][0][0])[q] = Cg[q];
  ColPairs cpp;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int j = 4 * lane + ((2 * p) & 3) + 128 * ((2 * p) >> 2);
    const float4 a = colp[j], b = colp[j + 1];
    cpp.bh[p] = pk2(a.x, b.x);
    cpp.T[p] = pk2(a.z, b.z);
  }
  const float gh = 4096.f * 1.4426950408889634f, gl = 1e-5f;
  const u64 ngh2 = pk2c(-gh), ngl2 = pk2c(-gl);
  u64 cacc2[4] = {0ull, 0ull, 0ull, 0ull};
  double* csum = &sred[warp][0];
  for (int q = 0; q < 8; ++q) csum[4 * lane + (q & 3) + 128 * (q >> 2)] = 0.0;
  const float4 rq0 = rowp[lane], rq1 = rowp[32 + lane];
  float racc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  const int rows_per_warp_stage = 32 / nw;   // 4 (8 warps) or 2 (16 warps)
  float rp4[4] = {0.f, 0.f, 0.f, 0.f};   // V6: previous stage's row partials
  float4 cur[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) cur[u] = rowp[u];
  float2* prm = reinterpret_cast<float2*>(smem_raw + 3 * 32 * 256 * 4 + (size_t)nw * 256 * 8);
  if (V == 8)
    for (int q = tid; q < 256; q += blockDim.x) prm[q] = make_float2(rowp[q & 63].x, rowp[q & 63].z);
  for (int k = 0; k < stages; ++k) {
    const int s = k % 3;
    if (V == 6 && k > 0) {
      // deferred butterfly of stage k-1, in the same basic block as stage k's rows
      const float tot = red4(rp4[0], rp4[1], rp4[2], rp4[3], lane);
      if ((lane & 7) == 0) rowpart[(int64_t)blockIdx.x * 4096 + (((k - 1) * 32 + warp * 4 + (lane >> 3)) & 4095)] = (double)tot;
    }
    float rs[4] = {0.f, 0.f, 0.f, 0.f};
    float4 nx[4];
    if (V == 9) {
#pragma unroll
      for (int u = 0; u < 4; ++u) nx[u] = cur[u];
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = __ldg(&rowp[((k + 1) * 4 + u) & 63]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= rows_per_warp_stage) break;
      const float4& q = (u & 1) ? rq1 : rq0;
      const int src = (2 * k + (u >> 1)) & 31;
      float ah, S;
      if (V == 8) {   // row parameters as broadcast LDS.64 from a shared copy
        const float2 pr = prm[(k * 32 + rows_per_warp_stage * warp + u) & 255];
        ah = pr.x; S = pr.y;
      } else if (V == 9) {   // broadcast LDG (L1) issued one stage ahead
        ah = nx[u].x; S = nx[u].z;
      } else {
        ah = __shfl_sync(0xffffffffu, q.x, src);
        S = __shfl_sync(0xffffffffu, q.z, src);
      }
      u64 c2[4];
      if (V == 5) {
        c2[0] = pk2(0.1f * ah, 0.2f); c2[1] = pk2(0.3f, 0.4f * S); c2[2] = pk2(0.5f, 0.6f); c2[3] = pk2(0.7f, 0.8f);
      } else {
        const float* row = &st[s][rows_per_warp_stage * warp + u][0];
        const float4 x0 = *reinterpret_cast<const float4*>(row + 4 * lane);
        const float4 x1 = *reinterpret_cast<const float4*>(row + 128 + 4 * lane);
        cost_pairs(x0, x1, c2);
      }
      rs[u] = row8<(V >= 5) ? 0 : V>(c2, ah, S, cpp, ngh2, ngl2, cacc2);
    }
    if (V != 7) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (V == 4) {
      racc += rs[0] + rs[1] + rs[2] + rs[3];
    } else if (V == 11) {   // butterfly, no global store
      racc += red4(rs[0], rs[1], rs[2], rs[3], lane);
    } else if (V == 12) {   // global store, no butterfly
      if ((lane & 7) == 0) rowpart[(int64_t)blockIdx.x * 4096 + ((k * 32 + warp * 4 + (lane >> 3)) & 4095)] = (double)(rs[0] + rs[1] + rs[2] + rs[3]);
    } else if (V == 10) {
      // row totals through this warp's consumed rows of the stage: lane l
      // stores its 4 partials, lane (u, q) sums lanes 4q..4q+3 of row u, then xor 1, 2, 4
      float4* scr = reinterpret_cast<float4*>(&st[s][rows_per_warp_stage * warp][0]);
      scr[lane] = make_float4(rs[0], rs[1], rs[2], rs[3]);
      __syncwarp();
      const int u = lane >> 3, q = lane & 7;
      const float* f = reinterpret_cast<const float*>(scr);
      float t = f[(4 * q) * 4 + u] + f[(4 * q + 1) * 4 + u] + f[(4 * q + 2) * 4 + u] + f[(4 * q + 3) * 4 + u];
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      if ((lane & 7) == 0) rowpart[(int64_t)blockIdx.x * 4096 + ((k * 32 + warp * 4 + (lane >> 3)) & 4095)] = (double)t;
      __syncwarp();
    } else if (V == 6) {
#pragma unroll
      for (int u = 0; u < 4; ++u) rp4[u] = rs[u];
    } else {
      const float tot = red4(rs[0], rs[1], rs[2], rs[3], lane);
      if ((lane & 7) == 0) rowpart[(int64_t)blockIdx.x * 4096 + ((k * 32 + warp * 4 + (lane >> 3)) & 4095)] = (double)tot;
    }
    if ((k & 15) == 15) {
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
  long long t1 = clock64();
  __syncthreads();
  if (tid < 256) {
    double a = racc;
    for (int w = 0; w < nw; ++w) a += sred[w][tid];
    colout[blockIdx.x * 256 + tid] = a;
  }
  if (tid == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int V>
void run(const char* name, int threads, int ctas_per_sm, int sms, const float* C, const float4* rp, const float4* cp,
         double* rowpart, double* colout, long long* cyc) {
  const int stages = 4096;
  const int grid = sms * ctas_per_sm;
  const size_t smem = 3 * 32 * 256 * 4 + (size_t)(threads / 32) * 256 * 8 + (V == 8 ? 2048 : 0);
  cudaFuncSetAttribute(k_rate<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_rate<V><<<grid, threads, smem>>>(C, rp, cp, rowpart, colout, 64, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<V><<<grid, threads, smem>>>(C, rp, cp, rowpart, colout, stages, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const int rows_per_stage = (threads / 32) * ((32 / (threads / 32)) < 4 ? (32 / (threads / 32)) : 4);
  const double entries_cta = (double)stages * rows_per_stage * 256;
  printf("%-34s %4d thr x %d CTA/SM  %.2f entries/clk/SM (CTA 0 clock)  %.3e entries/s chip\n", name, threads,
         ctas_per_sm, entries_cta * ctas_per_sm / (double)c, entries_cta * grid / (ms * 1e-3));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nC = 3 * 32 * 256;
  float* hC = (float*)malloc(nC * 4);
  for (int q = 0; q < nC; ++q) hC[q] = (float)((q * 2654435761u) % 10007) / 10007.f;
  float4 hr[64], hc[256];
  for (int q = 0; q < 64; ++q) hr[q] = make_float4(-2.f - 0.01f * q, 1.f, 1.f, 0.f);
  for (int q = 0; q < 256; ++q) hc[q] = make_float4(-1.f - 0.001f * q, 1.f, 1.f, 0.f);
  float* C; float4 *rp, *cp; double *rowpart, *colout; long long* cyc;
  cudaMalloc(&C, nC * 4); cudaMalloc(&rp, sizeof(hr)); cudaMalloc(&cp, sizeof(hc));
  cudaMalloc(&rowpart, (size_t)sms * 2 * 4096 * 8); cudaMalloc(&colout, (size_t)sms * 2 * 256 * 8); cudaMalloc(&cyc, 8);
  cudaMemcpy(C, hC, nC * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(rp, hr, sizeof(hr), cudaMemcpyHostToDevice);
  cudaMemcpy(cp, hc, sizeof(hc), cudaMemcpyHostToDevice);
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int th = cfg == 0 ? 256 : 512, cps = cfg == 0 ? 2 : 1;
    run<0>("V0 baseline (K1 loop)", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<1>("V1 1/4 exp2 on FMA pipe", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<2>("V2 1/2 exp2 on FMA pipe", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<3>("V3 all exp2 on FMA pipe", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<4>("V4 no row butterfly", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<5>("V5 C from registers (no LDS)", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<6>("V6 butterfly deferred one stage", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<7>("V7 no proxy fence", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<11>("V11 butterfly, no row store", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<12>("V12 row store, no butterfly", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<8>("V8 row params by broadcast LDS", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<9>("V9 row params by LDG, stage ahead", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
    run<10>("V10 row totals via smem transpose", th, cps, sms, C, rp, cp, rowpart, colout, cyc);
  }
  // accuracy of the polynomial against the MUFU over the entry range
  return 0;
}

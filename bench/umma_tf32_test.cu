// bench/umma_tf32_test.cu -- layout check of the tcgen05 kind::tf32 MMA
// primitives in csrc/umma.cuh: D[128 x 256] = A[128 x K] * B[256 x K]^T with
// K-major SW128 operands written by threads, the commit -> mbarrier wait and
// the 32x32b TMEM loads.  Inputs are small multiples of 1/8, exact in tf32,
// so every product and sum is exact and D must equal the host result
// bit for bit.  Measurement / validation harness only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_08507_b200/csrc -o build/umma_tf32_test bench/umma_tf32_test.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include "umma.cuh"

using namespace mdot;

constexpr int M = 128, N = 256, KP = 32;

__device__ __forceinline__ void mbar_init_(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(128) k_test(const float* A, const float* B, float* D, int ksteps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - ((uint32_t)__cvta_generic_to_shared(sm) & 1023u)) & 1023u);
  unsigned char* sA = base;              // 128 x 128 B
  unsigned char* sB = base + M * 128;    // 256 x 128 B
  __shared__ unsigned long long mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int e = t; e < M * KP; e += blockDim.x) {
    const int r = e / KP, k = e % KP;
    *reinterpret_cast<float*>(sA + umma::sw128_offset(r, k)) = umma::to_tf32(A[e]);
  }
  for (int e = t; e < N * KP; e += blockDim.x) {
    const int r = e / KP, k = e % KP;
    *reinterpret_cast<float*>(sB + umma::sw128_offset(r, k)) = umma::to_tf32(B[e]);
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 256);
  if (t == 0) {
    mbar_init_(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t aa = (uint32_t)__cvta_generic_to_shared(sA), bb = (uint32_t)__cvta_generic_to_shared(sB);
    for (int ks = 0; ks < ksteps; ++ks)
      umma::mma_tf32(tm, umma::smem_desc_sw128(aa + 32 * ks), umma::smem_desc_sw128(bb + 32 * ks),
                     umma::idesc_tf32(M, N), ks > 0);
    umma::mma_commit(&mbar);
  }
  mbar_wait_(&mbar, 0);
  umma::fence_after();
  for (int c = 0; c < N; c += 32) {
    uint32_t v[32];
    umma::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    umma::tmem_ld_wait();
    for (int q = 0; q < 32; ++q) D[(32 * warp + lane) * N + c + q] = __uint_as_float(v[q]);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 256);
}

__global__ void __launch_bounds__(128) k_test_raw(const float* A, const float* B, float* D, int ksteps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - ((uint32_t)__cvta_generic_to_shared(sm) & 1023u)) & 1023u);
  unsigned char* sA = base;              // 128 x 128 B
  unsigned char* sB = base + M * 128;    // 256 x 128 B
  __shared__ unsigned long long mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int e = t; e < M * KP; e += blockDim.x) {
    const int r = e / KP, k = e % KP;
    *reinterpret_cast<float*>(sA + umma::sw128_offset(r, k)) = A[e];
  }
  for (int e = t; e < N * KP; e += blockDim.x) {
    const int r = e / KP, k = e % KP;
    *reinterpret_cast<float*>(sB + umma::sw128_offset(r, k)) = B[e];
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 256);
  if (t == 0) {
    mbar_init_(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t aa = (uint32_t)__cvta_generic_to_shared(sA), bb = (uint32_t)__cvta_generic_to_shared(sB);
    for (int ks = 0; ks < ksteps; ++ks)
      umma::mma_tf32(tm, umma::smem_desc_sw128(aa + 32 * ks), umma::smem_desc_sw128(bb + 32 * ks),
                     umma::idesc_tf32(M, N), ks > 0);
    umma::mma_commit(&mbar);
  }
  mbar_wait_(&mbar, 0);
  umma::fence_after();
  for (int c = 0; c < N; c += 32) {
    uint32_t v[32];
    umma::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    umma::tmem_ld_wait();
    for (int q = 0; q < 32; ++q) D[(32 * warp + lane) * N + c + q] = __uint_as_float(v[q]);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 256);
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, sizeof(float) * M * KP);
  cudaMallocManaged(&B, sizeof(float) * N * KP);
  cudaMallocManaged(&D, sizeof(float) * M * N);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < KP; ++k) A[i * KP + k] = (float)(((i * 7 + k * 3) % 17) - 8) / 8.0f;
  for (int j = 0; j < N; ++j)
    for (int k = 0; k < KP; ++k) B[j * KP + k] = (float)(((j * 5 + k * 11) % 13) - 6) / 4.0f;
  const int smem = 1024 + (M + N) * 128;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad_total = 0;
  for (int ksteps = 1; ksteps <= 4; ++ksteps) {
    cudaMemset(D, 0, sizeof(float) * M * N);
    k_test<<<1, 128, smem>>>(A, B, D, ksteps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 1;
    }
    int bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int k = 0; k < 8 * ksteps; ++k) s += (double)A[i * KP + k] * B[j * KP + k];
        if ((float)s != D[i * N + j]) {
          if (bad < 5) printf("  ksteps %d mismatch D[%d][%d] = %g, want %g\n", ksteps, i, j, D[i * N + j], s);
          ++bad;
        }
      }
    printf("ksteps %d (K = %d): %d mismatches of %d\n", ksteps, 8 * ksteps, bad, M * N);
    bad_total += bad;
  }
  printf(bad_total ? "FAIL\n" : "PASS\n");
  // raw fp32 operands (not tf32 images): how does the tensor core read them?
  {
    unsigned st = 12345u;
    auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (float)((st >> 8) & 0xFFFFFF) / 16777216.0f; };
    for (int e = 0; e < M * KP; ++e) A[e] = rnd();
    for (int e = 0; e < N * KP; ++e) B[e] = rnd();
    cudaFuncSetAttribute(k_test_raw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_test_raw<<<1, 128, smem>>>(A, B, D, 2);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("raw launch failed\n"); return 1; }
    double e_tr = 0, e_rn = 0, e_ex = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ex = 0, tr = 0, rn = 0;
        for (int k = 0; k < 16; ++k) {
          ex += (double)A[i * KP + k] * B[j * KP + k];
          unsigned ua, ub;
          memcpy(&ua, &A[i * KP + k], 4); memcpy(&ub, &B[j * KP + k], 4);
          unsigned ta = ua & 0xFFFFE000u, tb = ub & 0xFFFFE000u;
          unsigned ra = (ua + 0x1000u) & 0xFFFFE000u, rb = (ub + 0x1000u) & 0xFFFFE000u;
          float fta, ftb, fra, frb;
          memcpy(&fta, &ta, 4); memcpy(&ftb, &tb, 4); memcpy(&fra, &ra, 4); memcpy(&frb, &rb, 4);
          tr += (double)fta * ftb;
          rn += (double)fra * frb;
        }
        const double d = D[i * N + j];
        e_tr = fmax(e_tr, fabs(d - tr)); e_rn = fmax(e_rn, fabs(d - rn)); e_ex = fmax(e_ex, fabs(d - ex));
      }
    printf("raw fp32 operands, K = 16: max |D - truncated-tf32 dot| %.3g, |D - rounded-tf32 dot| %.3g, |D - exact| %.3g\n",
           e_tr, e_rn, e_ex);
  }
  return bad_total ? 1 : 0;
}

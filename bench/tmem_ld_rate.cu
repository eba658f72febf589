// bench/tmem_ld_rate.cu -- TMEM -> register load throughput on one SM
// (tcgen05.ld.32x32b.x32, 128 B per thread per load): W warps per CTA, one
// CTA per SM, every SM busy; reports bytes per cycle per SM.  Measurement
// harness for the K2s design: K2s reads 4 B of
// accumulator per screened entry.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_08507_b200/csrc -o build/tmem_ld_rate bench/tmem_ld_rate.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "umma.cuh"

using namespace mdot;

__global__ void k_rate(int iters, unsigned long long* cycles, unsigned* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) umma::tmem_alloc(&tbase, 512);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t t = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * ((warp >> 2) & 15));
  uint32_t acc = 0;
  const unsigned long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    umma::tmem_ld32(t, v);
    umma::tmem_ld_wait();
    uint32_t a = v[0];
#pragma unroll
    for (int k = 1; k < 32; ++k) a &= v[k];
    acc ^= a;
  }
  const unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
  if (acc == 0x12345678u) sink[0] = acc;
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tbase, 512);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  unsigned* sink;
  cudaMallocManaged(&cyc, sizeof(unsigned long long) * sms);
  cudaMallocManaged(&sink, 4);
  const int iters = 20000;
  for (int W : {1, 2, 4, 8, 12, 16}) {
    k_rate<<<sms, 32 * W>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    double mx = 0;
    for (int b = 0; b < sms; ++b) mx = mx > (double)cyc[b] ? mx : (double)cyc[b];
    const double bytes = (double)W * 32 * 128 * iters;
    printf("warps %2d: %.1f B/cycle/SM (%.1f cycles per warp-load)\n", W, bytes / mx, mx / iters);
  }
  return 0;
}

// Microbenchmark: MUFU.EX2 (ex2.approx.ftz.f32) and FFMA2 throughput per SM per clock on
// this GPU -- the denominators of the MUFU / FP32 floors quoted for K2 and K8.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu bench/mufu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ex2(float* out, int iters, float seed) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed * (threadIdx.x + k) * 1e-9f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[gridDim.x * blockDim.x] = (float)(t1 - t0);
}

__global__ void k_ffma2(float* out, int iters, float seed) {
  unsigned long long x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { float a = seed + k, b = seed - k; asm("mov.b64 %0, {%1,%2};" : "=l"(x[k]) : "f"(a), "f"(b)); }
  unsigned long long m; { float a = 0.999f; asm("mov.b64 %0, {%1,%1};" : "=l"(m) : "f"(a)); }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x[k]) : "l"(m));
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(x[k])); s += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[gridDim.x * blockDim.x] = (float)(t1 - t0);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, sizeof(float) * (sms * 1024 + 1));
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_ex2<<<sms, threads>>>(d, 16, 1.f);
    cudaEventRecord(e0);
    k_ex2<<<sms, threads>>>(d, iters, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float cyc; cudaMemcpy(&cyc, d + sms * threads, 4, cudaMemcpyDeviceToHost);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * threads * iters * 8;
    printf("ex2:   %4d thr/SM  %.3f ex2/clk/SM (clock64 of CTA 0)   %.3e ex2/s chip\n", threads,
           (double)threads * iters * 8 / cyc, ops / (ms * 1e-3));
    k_ffma2<<<sms, threads>>>(d, 16, 1.f);
    cudaEventRecord(e0);
    k_ffma2<<<sms, threads>>>(d, iters, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaMemcpy(&cyc, d + sms * threads, 4, cudaMemcpyDeviceToHost);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ffma2: %4d thr/SM  %.3f fp32 FMA lane-ops/clk/SM          %.3e flop/s chip\n", threads,
           (double)threads * iters * 8 * 2 / cyc, ops * 2 * 2 / (ms * 1e-3));
  }
  return 0;
}

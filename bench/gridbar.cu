// bench/gridbar.cu -- cost of one grid-wide barrier over a co-resident
// persistent grid (2 CTAs x 148 SMs, 288 threads): the flat sense-reversal
// barrier of persist.cu vs a two-level (grouped) variant.  Measurement
// harness only (profiles/README.md).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gridbar bench/gridbar.cu
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_acqrel(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ void bar_flat(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acq(&bar[1]);
    if (atom_acqrel(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      red_rel(&bar[1], 1u);
    } else {
      while (ld_acq(&bar[1]) == gen) __nanosleep(8);
    }
  }
  __syncthreads();
}
// flat, variants: spin without nanosleep; relaxed polling + one fence
template <int V>
__device__ void bar_flat_v(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acq(&bar[1]);
    if (atom_acqrel(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      red_rel(&bar[1], 1u);
    } else if (V == 0) {
      while (ld_acq(&bar[1]) == gen) {}
    } else {
      unsigned v;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&bar[1]) : "memory"); } while (v == gen);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}
// two levels: CTAs arrive on one of G group counters (separate 128-byte
// lines); the last of a group arrives on the top counter; waiters spin on the
// generation word
template <int G>
__device__ void bar_tree(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acq(&bar[1]);
    const unsigned grp = blockIdx.x % G;
    const unsigned gsize = (gridDim.x - grp + G - 1) / G;
    bool last = false;
    if (atom_acqrel(&bar[32 * (grp + 1)], 1u) == gsize - 1) {
      bar[32 * (grp + 1)] = 0u;
      last = atom_acqrel(&bar[0], 1u) == G - 1;
    }
    if (last) {
      bar[0] = 0u;
      red_rel(&bar[1], 1u);
    } else {
      while (ld_acq(&bar[1]) == gen) __nanosleep(8);
    }
  }
  __syncthreads();
}

// count barrier: every CTA arrives with a release-add on a monotonic counter
// and polls it until it reaches gen * ncta (no last-arriver release step)
__device__ void bar_count(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    red_rel(&bar[8], 1u);
    const unsigned tgt = gen * gridDim.x;
    while ((int)(ld_acq(&bar[8]) - tgt) < 0) {}
  }
  __syncthreads();
}
// count barrier variants: V=0 relaxed polls + one acquire fence; V=1 fence +
// relaxed red arrival, acquire polls; V=2 relaxed red after __threadfence,
// volatile polls, __threadfence (the classic cooperative-groups shape)
template <int V>
__device__ void bar_count_v(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    const unsigned tgt = gen * gridDim.x;
    if (V == 0) {
      red_rel(&bar[8], 1u);
      unsigned v;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&bar[8]) : "memory"); } while ((int)(v - tgt) < 0);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    } else if (V == 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&bar[8]), "r"(1u) : "memory");
      while ((int)(ld_acq(&bar[8]) - tgt) < 0) {}
    } else {
      __threadfence();
      atomicAdd(&bar[8], 1u);
      while ((int)(*((volatile unsigned*)&bar[8]) - tgt) < 0) {}
      __threadfence();
    }
  }
  __syncthreads();
}
// flat with the generation tracked in a register (persist.cu's grid_barrier)
__device__ void bar_flat_reg(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atom_acqrel(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      red_rel(&bar[1], 1u);
    } else {
      while (ld_acq(&bar[1]) == gen) __nanosleep(8);
    }
    ++gen;
  }
  __syncthreads();
}
template <int MODE>
__global__ void __launch_bounds__(288, 2) k(unsigned* bar, int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  unsigned gen = 0;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) bar_flat(bar);
    else if (MODE == 1) bar_tree<8>(bar);
    else if (MODE == 2) bar_tree<16>(bar);
    else if (MODE == 3) bar_flat_v<0>(bar);
    else if (MODE == 4) bar_flat_v<1>(bar);
    else if (MODE == 5) bar_count(bar, gen);
    else if (MODE == 6) bar_flat_reg(bar, gen);
    else if (MODE == 7) bar_count_v<0>(bar, gen);
    else if (MODE == 8) bar_count_v<1>(bar, gen);
    else bar_count_v<2>(bar, gen);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  unsigned long long* out;
  cudaMalloc(&bar, 4096 * 4);
  cudaMalloc(&out, 8);
  const int iters = 2000;
  const int grids[1] = {2 * sms};
  for (int gi = 0; gi < 1; ++gi)
  for (int mode = 5; mode < 10; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(bar, 0, 4096 * 4);
      int grid = grids[gi], iters_ = iters;
      void* args[] = {&bar, &iters_, &out};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const void* fns[10] = {(const void*)k<0>, (const void*)k<1>, (const void*)k<2>, (const void*)k<3>, (const void*)k<4>,
                             (const void*)k<5>, (const void*)k<6>, (const void*)k<7>, (const void*)k<8>, (const void*)k<9>};
      const void* fn = fns[mode];
      cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(288), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s) grid %d: %.3f us per barrier (%s)\n", mode, mode == 0 ? "flat" : mode == 1 ? "tree8" : mode == 2 ? "tree16" : mode == 3 ? "flat-spin" : mode == 4 ? "flat-relaxed" : mode == 5 ? "count" : mode == 6 ? "flat-reggen" : mode == 7 ? "count-relaxedpoll" : mode == 8 ? "count-fence-redrelaxed" : "count-cg",
             grid, 1000.0 * ms / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}

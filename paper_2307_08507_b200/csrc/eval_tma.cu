// paper_2307_08507_b200/csrc/eval_tma.cu -- K1 v2: persistent, TMA-fed fused
// marginal evaluation over a materialised fp32 C.
//
//   r(P)_i = sum_j P_ij,  c(P)_j = sum_i P_ij,  P_ij = exp(A_i + B_j - gbar C_ij)
//   (log form as in internal.cuh "K1 numerics").
//
// Structure (one or two CTAs per SM, grid <= 2 x #SMs, persistent):
//   * warp 8 = producer: one elected lane streams 32-row x 256-column boxes of C
//     into a 3-stage shared-memory ring with cp.async.bulk.tensor (TMA), each
//     stage guarded by a full/empty mbarrier pair;
//   * warps 0..7 = consumers: 4 rows x 8 columns per lane per stage, exponent
//     assembly + ex2 + row/column accumulation exactly as k_eval_fast;
//   * per tile, the column sums of the 8 warps are combined in smem and written
//     as a per-row-tile partial (rows: one partial per column tile); k_finalize
//     adds the partials in index order (deterministic, no float atomics, no
//     inter-CTA tickets on the streaming path).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"
#include "k1_tma.cuh"

namespace mdot {

__global__ void __launch_bounds__(kTmaThreads, 2)
    k_eval_tma(const __grid_constant__ CUtensorMap tmap, EvalArgs a) {
  if (a.done && *a.done) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
  TmaSmem& sm = *reinterpret_cast<TmaSmem*>(smem_raw + pad);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t it = 0;
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      tma_produce_pass(sm, &tmap, a, it);
    }
    return;
  }
  const float gh = a.gpair ? a.gpair[0] : a.gh;
  const float gl = a.gpair ? a.gpair[1] : a.gl;
  tma_consume_pass<false>(sm, a, it, gh, gl, blockIdx.x, gridDim.x);
}

// Lockstep batch (throughput mode): ONE persistent pass evaluates every
// active instance of a batch that shares C.  The virtual tile list is
// (active instance, tile) in instance-major order, round-robin over the grid
// as in k_eval_tma, so a CTA streams several tiles and the ring reaches steady
// state even when one instance has fewer tiles than CTAs (n = 4096: 256
// tiles).  Every instance keeps its own parameters and partials; instances
// whose controller is done are skipped (all CTAs read the same flags).
__global__ void __launch_bounds__(kTmaThreads, 2)
    k_eval_tma_multi(const __grid_constant__ CUtensorMap tmap, const EvalArgs* args, int B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
  TmaSmem& sm = *reinterpret_cast<TmaSmem*>(smem_raw + pad);
  __shared__ int act[kMaxBatchLockstep];
  __shared__ int nact;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    int k = 0;
    for (int b = 0; b < B; ++b)
      if (!(args[b].done && *args[b].done)) act[k++] = b;
    nact = k;
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t tpi = (int64_t)args[0].n_row_tiles * args[0].n_col_tiles;   // tiles per instance (same for all)
  const int64_t total = (int64_t)nact * tpi;
  uint32_t it = 0;
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      for (int64_t v = blockIdx.x; v < total; v += gridDim.x) {
        const EvalArgs& a = args[act[v / tpi]];
        tma_produce_tile(sm, &tmap, a, it, v % tpi, l2_policy(a.keep_l2 != 0), l2_policy(true));
      }
    }
    return;
  }
  for (int64_t v = blockIdx.x; v < total; v += gridDim.x) {
    const EvalArgs& a = args[act[v / tpi]];
    const float gh = a.gpair ? a.gpair[0] : a.gh;
    const float gl = a.gpair ? a.gpair[1] : a.gl;
    tma_consume_tile<false>(sm, a, it, gh, gl, v % tpi);
  }
}

// Shared-C variant: the virtual list is (tile, group of up to 8 active
// instances), tile-major, so one streamed copy of a C tile serves a whole
// group (consumer warp w = instance 8 g + w; tma_consume_tile_shared) and the
// groups of one tile run on neighbouring CTAs at about the same time (their
// second read of the tile hits L2).  C traffic per slot: ceil(active / 8)
// passes instead of one per instance.
__global__ void __launch_bounds__(kTmaThreads, 2)
    k_eval_tma_shared(const __grid_constant__ CUtensorMap tmap, const EvalArgs* args, int B) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
  TmaSmem& sm = *reinterpret_cast<TmaSmem*>(smem_raw + pad);
  __shared__ int act[kMaxBatchLockstep];
  __shared__ int nact;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    int k = 0;
    for (int b = 0; b < B; ++b)
      if (!(args[b].done && *args[b].done)) act[k++] = b;
    nact = k;
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const EvalArgs& a0 = args[0];   // geometry: identical for every instance of the batch
  const int64_t tpi = (int64_t)a0.n_row_tiles * a0.n_col_tiles;
  const int groups = (nact + kConsumerWarps - 1) / kConsumerWarps;
  const int64_t total = (int64_t)groups * tpi;
  uint32_t it = 0;
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      const uint64_t pol_stream = l2_policy(a0.keep_l2 != 0), pol_keep = l2_policy(true);
      for (int64_t v = blockIdx.x; v < total; v += gridDim.x)
        tma_produce_tile(sm, &tmap, a0, it, v / groups, pol_stream, pol_keep);
    }
    return;
  }
  for (int64_t v = blockIdx.x; v < total; v += gridDim.x) {
    const int g = (int)(v % groups);
    const int slot = g * kConsumerWarps + warp;
    const int b = slot < nact ? act[slot] : -1;
    tma_consume_tile_shared(sm, args[b >= 0 ? b : 0], b, it, v / groups);
  }
}

cudaError_t launch_eval_tma_shared(const void* map, const EvalArgs* args_dev, int B, int grid, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(TmaSmem) + 128;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_eval_tma_shared, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(k_eval_tma_shared, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    attr = true;
  }
  if (B > kMaxBatchLockstep) return cudaErrorInvalidValue;
  const CUtensorMap& m = *reinterpret_cast<const CUtensorMap*>(map);
  k_eval_tma_shared<<<grid, kTmaThreads, smem, st>>>(m, args_dev, B);
  return cudaGetLastError();
}

cudaError_t launch_eval_tma_multi(const void* map, const EvalArgs* args_dev, int B, int grid, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(TmaSmem) + 128;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_eval_tma_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(k_eval_tma_multi, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    attr = true;
  }
  if (B > kMaxBatchLockstep) return cudaErrorInvalidValue;
  const CUtensorMap& m = *reinterpret_cast<const CUtensorMap*>(map);
  k_eval_tma_multi<<<grid, kTmaThreads, smem, st>>>(m, args_dev, B);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    cudaError_t e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
    if (e == cudaSuccess && q == cudaDriverEntryPointSuccess && p) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    } else if (getenv("MDOT_DEBUG")) {
      fprintf(stderr, "[mdot] cuTensorMapEncodeTiled lookup failed: %s (query %d)\n", cudaGetErrorString(e), (int)q);
    }
  }
  return fn;
}

bool tma_supported(const EvalArgs& a) {
  return a.C != nullptr && (a.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 15) == 0) &&
         (a.tile_m % kTmaRows == 0) && get_encode() != nullptr;
}

cudaError_t make_tma_map(const EvalArgs& a, void* map_out /* CUtensorMap, 64 B aligned, 128 B */) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)a.n, (cuuint64_t)a.nrows};
  cuuint64_t strides[1] = {(cuuint64_t)a.ldc * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)kTileN, (cuuint32_t)kTmaRows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<float*>(a.C), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("MDOT_DEBUG")) fprintf(stderr, "[mdot] cuTensorMapEncodeTiled failed: %d\n", (int)r);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_eval_tma(const void* map, const EvalArgs& a, int grid, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(TmaSmem) + 128;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_eval_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const CUtensorMap& m = *reinterpret_cast<const CUtensorMap*>(map);
  k_eval_tma<<<grid, kTmaThreads, smem, st>>>(m, a);
  return cudaGetLastError();
}

void set_smem_carveout_tma() {
  cudaFuncSetAttribute(k_eval_tma, cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
}

int tma_smem_bytes() { return (int)sizeof(TmaSmem) + 128; }

}  // namespace mdot

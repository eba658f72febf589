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

namespace mdot {

constexpr int kTmaRows = 32;
constexpr int kTmaStages = 3;
constexpr int kConsumerWarps = 8;
constexpr int kTmaThreads = (kConsumerWarps + 1) * 32;

struct TmaSmem {
  float stage[kTmaStages][kTmaRows][kTileN];   // 96 KiB
  double sred[kConsumerWarps][kTileN];          // 16 KiB
  unsigned long long full[kTmaStages];
  unsigned long long empty[kTmaStages];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ double shfl_xor_dd(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

__device__ __forceinline__ double warp_reduce4_t(double v0, double v1, double v2, double v3, int lane) {
  const bool up = lane & 16;
  double k0 = up ? v2 : v0, k1 = up ? v3 : v1;
  double s0 = up ? v0 : v2, s1 = up ? v1 : v3;
  k0 += shfl_xor_dd(s0, 16);
  k1 += shfl_xor_dd(s1, 16);
  const bool up2 = lane & 8;
  double kk = up2 ? k1 : k0, ss = up2 ? k0 : k1;
  kk += shfl_xor_dd(ss, 8);
  kk += shfl_xor_dd(kk, 4);
  kk += shfl_xor_dd(kk, 2);
  kk += shfl_xor_dd(kk, 1);
  return kk;
}

__global__ void __launch_bounds__(kTmaThreads, 2)
    k_eval_tma(const __grid_constant__ CUtensorMap tmap, EvalArgs a) {
  if (a.done && *a.done) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
  TmaSmem& sm = *reinterpret_cast<TmaSmem*>(smem_raw + pad);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = a.n, nrows = a.nrows;
  const int nct = a.n_col_tiles;
  const int64_t total = (int64_t)a.n_row_tiles * nct;
  const int stages_per_tile = a.tile_m / kTmaRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int tr = (int)(tile / nct), tc = (int)(tile % nct);
        const int64_t i0 = (int64_t)tr * a.tile_m;
        int nst = stages_per_tile;
        if (i0 + (int64_t)nst * kTmaRows > nrows) nst = (int)((nrows - i0 + kTmaRows - 1) / kTmaRows);
        for (int k = 0; k < nst; ++k, ++it) {
          const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
          mbar_wait(&sm.empty[s], ph ^ 1u);
          mbar_expect_tx(&sm.full[s], (uint32_t)(kTmaRows * kTileN * sizeof(float)));
          tma_load_2d(&sm.stage[s][0][0], &tmap, tc * kTileN, (int)(i0 + k * kTmaRows), &sm.full[s]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const float gh = a.gpair ? a.gpair[0] : a.gh;
  const float gl = a.gpair ? a.gpair[1] : a.gl;
  uint32_t it = 0;
  for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const int tr = (int)(tile / nct), tc = (int)(tile % nct);
    const int64_t i0 = (int64_t)tr * a.tile_m;
    const int64_t j0 = (int64_t)tc * kTileN;
    int nst = stages_per_tile;
    if (i0 + (int64_t)nst * kTmaRows > nrows) nst = (int)((nrows - i0 + kTmaRows - 1) / kTmaRows);

    float bh[8], bl[8], T[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t j = j0 + 4 * lane + (q & 3) + 128 * (q >> 2);
      if (j < n) {
        const float4 cp = __ldg(&a.colp[j]);
        bh[q] = cp.x; bl[q] = cp.y; T[q] = cp.z;
      } else {
        bh[q] = -1.0e30f; bl[q] = 0.f; T[q] = 0.f;
      }
    }
    double cacc64[8];
    float cacc32[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { cacc64[q] = 0.0; cacc32[q] = 0.f; }

    for (int k = 0; k < nst; ++k, ++it) {
      const uint32_t s = it % kTmaStages, ph = (it / kTmaStages) & 1u;
      const int64_t ib = i0 + (int64_t)k * kTmaRows + 4 * warp;
      float4 rp[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        rp[u] = (ib + u < nrows) ? __ldg(&a.rowp[ib + u]) : make_float4(-1.0e30f, 0.f, 0.f, 0.f);
      mbar_wait(&sm.full[s], ph);
      double rs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float* row = &sm.stage[s][4 * warp + u][0];
        const float4 x0 = *reinterpret_cast<const float4*>(row + 4 * lane);
        const float4 x1 = *reinterpret_cast<const float4*>(row + 128 + 4 * lane);
        const float cv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const float ah = rp[u].x, al = rp[u].y, S = rp[u].z;
        float rsum = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float cij = cv[q];
          const float zh = fmaf(-gh, cij, ah + bh[q]);
          const float tt = fmaf(-gl, cij, al + bl[q]);
          const float e = ex2_fast(zh + tt);
          rsum = fmaf(e, T[q], rsum);
          cacc32[q] = fmaf(e, S, cacc32[q]);
        }
        rs[u] = rsum;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      const double tot = warp_reduce4_t(rs[0], rs[1], rs[2], rs[3], lane);
      const int64_t i = ib + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
      if ((lane & 7) == 0 && i < nrows) a.rowpart[(int64_t)tc * nrows + i] = tot;
      if (k & 1) {
#pragma unroll
        for (int q = 0; q < 8; ++q) { cacc64[q] += (double)cacc32[q]; cacc32[q] = 0.f; }
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) cacc64[q] += (double)cacc32[q];

    // column sums of this tile (8 warps, fixed order) -> partial of row tile tr
#pragma unroll
    for (int q = 0; q < 8; ++q) sm.sred[warp][4 * lane + (q & 3) + 128 * (q >> 2)] = cacc64[q];
    consumer_bar();
    {
      const int tt = threadIdx.x;
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) acc += sm.sred[w][tt];
      const int64_t j = j0 + tt;
      if (j < n) a.colpart[(int64_t)tr * n + j] = acc;
    }
    consumer_bar();   // sred / last flags reused by the next tile
  }
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

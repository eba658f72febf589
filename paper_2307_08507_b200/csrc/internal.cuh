// paper_2307_08507_b200/csrc/internal.cuh -- internal declarations of the
// MDOT-PNCG CUDA library (not part of the C ABI; see include/mdot.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/mdot.h"

namespace mdot {

// Checked builds (-DMDOT_CHECKED; tests/test_gpu_checked.py): device-side
// bounds / invariant checks that trap, and guard bands around every
// workspace sub-buffer verified when the call returns (solver.cu).  The
// sanitizer is not available on this pool; these are the replacement.
#ifdef MDOT_CHECKED
#define MDOT_DCHECK(c)                                                              \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("MDOT_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                   \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define MDOT_DCHECK(c) \
  do {                 \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// Fused marginal evaluation (rounding K6/K7).
//
// Entries are evaluated in an anchored base-2 form:
//   w_ij = a2_i + b2_j - g2 * C_ij,   a2_i = A_i log2(e) - rho_i,
//                                     b2_j = B_j log2(e) - sig_j,
//   P_ij = 2^w_ij * 2^rho_i * 2^sig_j,
// with integer anchors rho_i ~ log2(r_i)/2, sig_j ~ log2(c_j)/2 so that
// 2^w ~ 1 for the entries that carry the mass.  a2 = ah + al with ah on a
// 2^-8 grid (|ah| < 2^15), so ah + bh is exact in fp32 and fmaf(-gh, C, ah+bh)
// rounds the large cancellation once; g2 = gh + gl (fp32 pair).
// ---------------------------------------------------------------------------
constexpr int kTileN = 256;      // columns per tile (8 per lane)
constexpr int kWarps = 8;        // warps per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kUnroll = 4;       // rows per warp per inner step
constexpr int kNumScalars = 16;
constexpr long long kTraceDevCap = 1 << 20;   // device trace records per projection (mdot_options.trace)

// K1 reduction knobs, shared by the TMA kernels,
// k_eval_fast (bitwise-equal by test), K2 and the fp32-entry paths of K8: MDOT_K1_ROWRED_F32 = 1 reduces the 4
// rows' lane sums across the warp in fp32 (one conversion per row total
// instead of 4 conversions + 5 fp64 adds + 12 shuffles per lane and stage);
// MDOT_K1_COLFLUSH = 4-row steps of fp32 column sums per fp64 flush.
#ifndef MDOT_K1_ROWRED_F32
#define MDOT_K1_ROWRED_F32 1
#endif
#ifndef MDOT_K1_PACKED
#define MDOT_K1_PACKED 1
#endif
#ifndef MDOT_K1_COLFLUSH
#define MDOT_K1_COLFLUSH 4
#endif
__device__ __forceinline__ float warp_reduce4_f(float v0, float v1, float v2, float v3, int lane) {
  const bool up = lane & 16;
  float k0 = up ? v2 : v0, k1 = up ? v3 : v1;
  const float s0 = up ? v0 : v2, s1 = up ? v1 : v3;
  k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  const bool up2 = lane & 8;
  float kk = up2 ? k1 : k0;
  const float ss = up2 ? k0 : k1;
  kk += __shfl_xor_sync(0xffffffffu, ss, 8);
  kk += __shfl_xor_sync(0xffffffffu, kk, 4);
  kk += __shfl_xor_sync(0xffffffffu, kk, 2);
  kk += __shfl_xor_sync(0xffffffffu, kk, 1);
  return kk;
}

struct EvalArgs {
  // cost
  const float* C;          // dense fp32, row-major, rows of this shard (row stride ldc)
  int64_t ldc;             // row stride of C (== n)
  const float* X;          // on-the-fly: [nrows x d] (rows of this shard)
  const float* Y;          // on-the-fly: [n x d]
  int d;
  float scale;
  int otf_dot;             // on-the-fly cost recipe: 0 diff (Z22), 1 dot form (Z22b; otf_cost.cuh)
  int64_t n;               // number of columns (global n)
  int64_t nrows;           // number of rows evaluated (local rows)
  int tile_m;              // rows per tile (multiple of kWarps*kUnroll)
  int n_row_tiles, n_col_tiles;
  // per-row / per-column parameters
  const float4* rowp;      // [nrows] {ah, al, S=2^rho, w}  (w: |x_i|^2 for the dot recipe, else 0)
  const float4* colp;      // [n]     {bh, bl, T=2^sig, w}  (w: |y_j|^2 for the dot recipe, else 0)
  float gh, gl;            // g2 = gbar*log2(e) = gh + gl
  const float* gpair;      // device-resident {gh, gl} (device control), overrides gh/gl
  const int* done;         // device control: kernel returns at once when *done != 0
  int keep_l2;             // TMA path: C fits in L2 -> evict_last (stays resident), else evict_first
  int64_t l2_res_tiles;    // persistent TMA pass: tiles [0, l2_res_tiles) read with evict_last (MDOT_K1_L2RES_MB)
  // outputs
  double* rowpart;         // [n_col_tiles][nrows]  sum_j 2^w T_j
  double* colpart;         // [n_row_tiles][n]      sum_i 2^w S_i
  // screened on-the-fly evaluation (K2s, screen.cu): operand rows written by k_prep
  const float* sopA;                 // [nrows padded to 128][32] tf32 A rows (K-major SW128 image)
  const float* sopB;                 // [n padded to 256][32] tf32 B rows
  const unsigned long long* smin;    // [2] ordered keys: min potential shift over rows, over columns (nats)
  const double* smin_rows_neg;       // row-sharded: -(min row shift over ALL ranks) (allreduced), else null
  unsigned long long* scount;        // [2] += entries kept, entries screened (nullable)
};
// row-sharded K2s: out[0] = -(this rank's min row shift) for a MAX allreduce
cudaError_t launch_smin_neg(const unsigned long long* smin, double* out, cudaStream_t st);

bool tma_supported(const EvalArgs& a);
cudaError_t make_tma_map(const EvalArgs& a, void* map_out);
cudaError_t launch_eval_tma(const void* map, const EvalArgs& a, int grid, cudaStream_t st);
cudaError_t launch_eval_tma_multi(const void* map, const EvalArgs* args_dev, int B, int grid, cudaStream_t st);
// shared C reads: up to 8 instances per streamed tile (one per consumer warp)
cudaError_t launch_eval_tma_shared(const void* map, const EvalArgs* args_dev, int B, int grid, cudaStream_t st);
int tma_smem_bytes();

// Launch the fused evaluation over the (row tile x column tile) grid.
// kind: 0 dense fp32, 1 on-the-fly squared Euclidean.
cudaError_t launch_eval_fast(const EvalArgs& a, int kind, cudaStream_t st);
// K2s: on-the-fly cost with the tensor-core screen (screen.cu); d in {2, 4, 8, 16}
bool screen_supported(int d);
cudaError_t launch_eval_screen(const EvalArgs& a, cudaStream_t st);
size_t screen_smem_bytes();
// ordered 64-bit key of a double (unsigned order = numeric order; atomicMin)
__host__ __device__ inline unsigned long long double_key(double x) {
  unsigned long long b;
  memcpy(&b, &x, sizeof b);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
constexpr unsigned long long kKeyPosInf = 0xFFF0000000000000ull;   // double_key(+inf)

// Exact fp64 evaluator (two-pass online log-sum-exp, fp64 exp): fallback of
// the fp32 path and the fp64-P precision mode.  Writes lr (rows of this
// shard) and column (max, sum) partials.
struct ExactArgs {
  const void* C; int64_t ldc; int c_f64;  // dense (fp32 or fp64)
  const float* X; const float* Y; int d; float scale; int otf;   // otf: 0 dense, 1 diff recipe, 2 dot recipe
  int64_t n, nrows;
  const double* A;   // [nrows]
  const double* B;   // [n]
  double gbar;
  double* lr;        // [nrows]
  double* colm;      // [chunks][n]
  double* cols;      // [chunks][n]
  int chunks;        // row chunks for the column pass
  const int* done;   // device control early exit
};
cudaError_t launch_eval_exact(const ExactArgs& a, cudaStream_t st);
// rows only: lr = exact fp64 log row marginals (rounding)
cudaError_t launch_exact_rows(const ExactArgs& a, cudaStream_t st);

// ---------------------------------------------------------------------------
// O(n) kernels
// ---------------------------------------------------------------------------
// Scalars produced by finalize (fp64): indices
enum Scalar : int {
  SC_MASS = 0,     // sum r(P)
  SC_MASSC = 1,    // sum c(P)
  SC_L1 = 2,       // |r(P)-r|_1 + |c(P)-c|_1
  SC_RHO = 3,      // D_h(r(P)|r) + D_h(c(P)|c)
  SC_SG = 4,       // <s, g>
  SC_GCS = 5,      // <g_cur, s>
  SC_PCG = 6,      // <p_cur, g>      (= phi'(alpha) for a trial)
  SC_PRC = 7,      // <p_cur, (r,c)>
  SC_GG = 8,       // <g, g>
  SC_GCG = 9,      // <g_cur, g>
  SC_BAD = 10,     // count of invalid marginals (non-finite / out of range)
  SC_L1R = 11,     // |r(P)-r|_1
  SC_COST = 12,    // rounding: sum of cost partials
  SC_CORR = 13,    // rounding: correction term numerator
  SC_ERN = 14,     // rounding: |err_r|_1
  SC_AUX = 15
};

struct FinalizeArgs {
  int64_t n;             // global n (columns)
  int64_t nrows;         // local rows
  int from_partials;     // 2: totals rowtot/coltot; 1: reduce rowpart/colpart (rows) and colpart or coltot
                         // (cols, coltot when non-null); 0: exact (lr, col (m,s) partials)
  const double* rowtot; const double* coltot;
  const double* rowpart; int n_col_tiles;
  const double* colpart; int n_row_tiles;
  const double* rho_r;   // [nrows] anchors (fp64 integers)
  const double* sig_c;   // [n]
  const double* colm; const double* cols; int chunks;   // exact path column partials
  const double* lr_in;   // exact path rows
  const double* r; const double* c; const double* logr; const double* logc;   // r, logr: local rows
  const double* gcur;    // [nrows + n] current gradient (nullable)
  const double* pcur;    // [nrows + n] current direction (nullable)
  // outputs
  double* lm;            // [nrows + n] log marginals (rows then cols)
  double* m;             // [nrows + n] marginals
  double* s;             // [nrows + n] Sinkhorn direction
  double* g;             // [nrows + n] gradient
  double* blockpart;     // [gridDim][kNumScalars]
  unsigned int* ticket;
  double* scalars_dev;   // [kNumScalars]
  double* scalars_host;  // mapped host (nullable)
  int* prep_flag;        // nullable: added to SC_BAD, then reset to 0
  const int* done;       // device control: return at once when *done != 0
  int64_t item_begin, item_end;   // items processed: [begin, end) of [0, nrows + n) (end 0 = all)
  const double* add_in;  // nullable: kNumScalars values added before publishing (sharded rows)
  int cols_local_only;   // sharded: 1 -> column items produce raw partial sums (no log) ... (unused)
  int jacobi;            // 1: s = grad / diag(Hessian) (MDOT_PROJ_PNCG_JACOBI) instead of the Sinkhorn direction
  int f64_entries;       // partials from fp64 entries (K8): range guard at the fp64 limits, not fp32's
  int fault_repl;        // MDOT_FAULT_NAN=1 hook: copies of item 0 finalized per evaluation (K8 cluster: CL)
  double f64_tot_min;    // fp64 entries: totals below this (anchored units) are redone exactly -- the
                         // bound on the mass K8's entry skip may have dropped (batch.cu); 0 = 1e-300
  unsigned long long* smin_reset;   // nullable: [2] screen shift minima, reset to +inf (block 0) for the next prep
};
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st);
cudaError_t launch_finalize_multi(const FinalizeArgs* args_dev, const FinalizeArgs& a0, int B, cudaStream_t st);

// ---------------------------------------------------------------------------
// Device-resident PNCG / Sinkhorn control (one thread; k_ctrl).  The host
// enqueues CUDA graphs of [k_ctrl, k_prep, eval, k_finalize] slots; the
// controller reads the scalars of the previous slot's finalize, runs the
// line-search / direction logic of project_pncg (Alg. 2, Appx. C, Z5-Z10)
// and writes the next slot's mode, alpha, beta -- no host sync per trial.
// ---------------------------------------------------------------------------
enum CtrlStatus : int { CTRL_RUNNING = 0, CTRL_OK = 1, CTRL_NOCONV = 2, CTRL_LS_FAIL = 3, CTRL_NEED_HOST = 4 };
struct CtrlState {
  // configuration (host-written per projection)
  double eps, c1, c2, noise;
  int stop_rho, ncg, sinkhorn, beta_kind, ls_max_trials, pad0;
  long long max_evals;
  float gpair[2];
  // next slot
  int done, status, accept_marg, accept_pot, mode, phase;
  double alpha, beta;
  // iterate
  long long k, evals, ls_evals, resets, restarts, iterations;
  double mass, S_sg, S_gcs, S_pcg, S_gg, S_gcg, dphi0_prev, sg_prev, gg_prev, alpha_prev;
  double l1, rho, l1_0, rho_0;
  // line search
  double lo, dlo, hi, dhi, dphi0, dg;
  int have_hi, doublings, trials, attempt;
  // per-iteration trace (mdot_options.trace): device records written by the
  // ONE controller copy whose `trace` is non-null (CTA 0 of the persistent
  // grid, k_ctrl, instance 0 of K8); md_t = MD step of this projection
  mdot_trace_rec* trace;
  long long* trace_len;
  long long trace_cap;
  int md_t, reset_flag;
  // scalars published by k_finalize
  double sc[kNumScalars];
};
cudaError_t launch_ctrl(CtrlState* st, int slot, int* done_host, int* ran_host, cudaStream_t s);

// Lockstep batch (throughput mode, solver.cu solve_batch_lockstep): one launch
// per phase for every instance of a batch sharing a dense fp32 C; argument
// arrays in device memory, instance b = blockIdx.y (prep / finalize), block b
// (ctrl), or the b-th active instance of the virtual tile list (K1).
constexpr int kMaxBatchLockstep = 64;
cudaError_t launch_ctrl_multi(CtrlState* const* sts_dev, int B, int* done_flags, cudaStream_t s);
// Prefer the maximum shared-memory carveout for every kernel of the solve loop
// (one L1/smem configuration for the whole loop, no reconfiguration between
// the TMA kernel and the O(n) kernels).
void set_smem_carveout();

enum PrepMode : int {
  PREP_CUR = 0,         // A = U + u, B = V + v -> params
  PREP_AB = 16,         // A, B given (rows/cols) -> params
  PREP_TRIAL = 1,       // tu = u + alpha p_u, tv = v + alpha p_v ; A = U + tu, B = V + tv
  PREP_NEWDIR = 2,      // p = -s + beta*pprev  (or -s if beta==0 and reset)
  PREP_SK_ROW = 4,      // u += log r - lr  (Sinkhorn odd half-step)
  PREP_SK_COL = 8       // v += log c - lc
};
struct PrepArgs {
  int64_t n, nrows;
  int mode;
  double alpha, beta;
  const double* U; const double* V;   // cumulative (rows local, cols global)
  double* u; double* v;               // step potentials (in place for Sinkhorn)
  double* tu; double* tv;             // trial potentials
  double* p;                          // [nrows + n] direction (written in NEWDIR)
  const double* s;                    // [nrows + n]
  double* pprev;                      // [nrows + n]
  const double* lm;                   // [nrows + n] current log marginals (Sinkhorn)
  const double* logr; const double* logc;
  const double* rho_r; const double* sig_c;
  const double* Ain; const double* Bin;   // PREP_AB
  double* Aout; double* Bout;         // fp64 bases (for the exact path)
  float4* rowp; float4* colp;
  const float* nrm;                   // [nrows + n] squared norms (Z22b dot recipe) -> rowp/colp .w, or null
  int* flag;                          // set to 1 when |a2|,|b2| >= 2^15
  int f64_params;                     // 1: write {fp64 base, 2^anchor, anchor} (fp64-entry evaluation)
  // device control: mode/alpha/beta/accept come from ctrl; accept copies trial -> cur
  const CtrlState* ctrl;
  double *cur_lm, *cur_m, *cur_s, *cur_g;
  const double *tr_lm, *tr_m, *tr_s, *tr_g;
  // K2s screen operands (device control only; null = off): the accept copy
  // also carries the base potentials of the accepted evaluation (cur_bp),
  // prep writes this evaluation's bases to tr_bp, the item's 128-byte tf32
  // operand row (screen.cu) to sopA / sopB and the per-side minimum shift to
  // smin[2] (k_prep)
  double* cur_bp; double* tr_bp;
  float* sopA; float* sopB;
  unsigned long long* smin;
  const float* X; const float* Y; int d; float scale;   // on-the-fly coordinates
  const double* sop_ymax;            // max_j |y_j| (setup)
  float screen_T;                    // entries below 2^-T of their row and column totals are skipped
};
// one 128-byte operand row of K2s (screen.cu): 8 chunks of 16 bytes, chunk c
// stored at position c ^ (r & 7) -- the K-major SW128 image of row r
__device__ __forceinline__ void sop_store(float* rowbase, int64_t r, const float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(rowbase + 4 * (c ^ (int)(r & 7))) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
cudaError_t launch_norm_max(const float* P, int64_t m, int d, double* out, cudaStream_t st);
cudaError_t launch_sop_pad(float* sopA, int64_t nrows, float* sopB, int64_t n, cudaStream_t st);
cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st);
// out[i] = sqnorm_recipe(P + i d, d) for i < m (the Z22b recipe, otf_cost.cuh)
cudaError_t launch_sqnorms(const float* P, int64_t m, int d, float* out, cudaStream_t st);
cudaError_t launch_prep_multi(const PrepArgs* args_dev, const PrepArgs& a0, int B, cudaStream_t st);

// Persistent cooperative slot kernel (persist.cu): a whole projection in one
// launch (ctrl / prep / K1 / finalize phases separated by grid barriers).
struct PersistArgs {
  EvalArgs e;
  PrepArgs p;
  FinalizeArgs f;
  CtrlState* ctrl;             // global state (read at entry, written back by CTA 0 at exit)
  int* done_host;              // mapped flag (device alias), written by CTA 0's controller
  unsigned int* gbar;          // [2] grid barrier (zeroed before launch)
  double* cta_part;            // [grid][kNumScalars]
  unsigned long long* k1_ns;   // [2] += K1 phase ns (%globaltimer between grid barriers), count
  unsigned long long* dbg_fin; // MDOT_DEBUG_K1TAIL: [64 slots][grid] %globaltimer when each CTA's consumers end K1
  int initial;                 // 1: the first slot is the projection's initial evaluation
  long long max_slots;
};
int persist_grid();            // co-resident grid size (0 = unsupported)
int persist_max_chunk();       // max finalize items per CTA
cudaError_t launch_persist(const void* map, const PersistArgs& a, int grid, cudaStream_t st);

// Row-sharded persistent projection with the column exchange fused into the
// kernel over peer memory (SURVEY 8(e) NC1 without NCCL; DESIGN.md "Fused
// peer exchange").  Per evaluation every CTA of every rank stores its column
// totals and its row-scalar partial into slot `rank` of EVERY rank's receive
// block through peer-mapped pointers (NVLink) as self-validating 16-byte
// records {lo32, ex, hi32, ex}; each rank polls the records of its F2 column
// chunk until they carry the exchange index, sums the slots in rank order
// (identical on every rank) and finalizes the replicated columns.  Receive
// blocks are double-buffered by exchange parity: a rank writes parity p again
// only at exchange e + 2, after it has read every rank's exchange-(e + 1)
// records, which those ranks wrote after the grid barrier that ended their
// exchange-e reads.
constexpr int kMaxPeers = 8;
struct PeerNet {
  double* recv[kMaxPeers];         // rank q's receive block as seen from this GPU: [2][nranks][ld] 16-byte records
  unsigned int* flag[kMaxPeers];   // rank q's control words (after its records): [kMaxPeers] | epoch | err
  int nranks;
  int64_t ld;                      // slot stride (>= n + kNumScalars)
};
struct PeerGroup {                 // one rank's share of a launch
  PersistArgs a;
  int rank;                        // global rank
  unsigned int* epoch;             // this rank's exchange counter (own memory)
  int* err;                        // set to 1 when a flag wait timed out
};
// One cooperative launch runs `groups` ranks of cta_per_group CTAs each: 1 on
// a real multi-GPU rank (the peers run their own launches on their GPUs), G
// when one GPU emulates G ranks (the in-process transport; every "peer"
// pointer is then local and the ranks' CTAs are co-resident, so the flag
// waits cannot deadlock -- B200_PROFILING.md: emulate ranks as ONE kernel).
struct PeerLaunch {
  alignas(64) unsigned char tmap[kMaxPeers][128];
  PeerGroup g[kMaxPeers];
  PeerNet net;
  int groups, cta_per_group;
};
cudaError_t launch_persist_peer(const PeerLaunch& L, cudaStream_t st);

// misc vector kernels
cudaError_t launch_setup(int64_t n, const double* r, double* logr, double* rho, cudaStream_t st);
cudaError_t launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t st); // y = a x + b y
cudaError_t launch_add_scalar(int64_t n, double d, double* y, cudaStream_t st);
// 2-D sharded graph slots: out[q] = a[q] + b[q] for the kNumScalars control
// scalars (row side + column side), skipped once the controller is done
cudaError_t launch_sum_scalars(const double* a, const double* b, double* out, const int* done, cudaStream_t st);
// 2-D exact fallback: out[i] = M[i] + log(S[i]) (a log-sum-exp from its
// allreduced (max, scaled sum) form)
cudaError_t launch_lse_finish(int64_t n, const double* M, const double* S, double* out, cudaStream_t st);
// NC2 scalar-only line-search trial (kernels.cu k_nc2_trial): 4 doubles
cudaError_t launch_nc2_trial(const double* rowpart, int nct, const double* colpart, int nrt, int64_t nrows, int64_t n,
                             const double* rho_r, const double* sig_c, const double* p, const int* flag,
                             double* blockpart, unsigned int* ticket, double* out_dev, cudaStream_t st);
cudaError_t launch_fill(int64_t n, double v, double* y, cudaStream_t st);
// deterministic dot products: out[k] = sum_i x_k[i] * y_k[i] for up to 4 pairs
cudaError_t launch_dots(int64_t n, int npairs, const double* const* xs, const double* const* ys,
                        double* blockpart, unsigned int* ticket, double* out_dev, double* out_host,
                        cudaStream_t st);
// column partials -> local column totals (generic kernel, sharded mode)
cudaError_t launch_sample_c(const void* C, int c64, int64_t count, int S, double* out, cudaStream_t st);
cudaError_t launch_minmax(const void* C, int c64, int64_t count, double* out2, cudaStream_t st);
cudaError_t launch_reduce_colpart(const double* colpart, int n_row_tiles, int64_t n, double* coltot, cudaStream_t st,
                                  const int* done = nullptr);
// exact path, sharded: combine chunk (max, sum) pairs; rescale sums to a global max
cudaError_t launch_exact_colcombine(const double* colm, const double* cols, int chunks, int64_t n, double* M,
                                    double* S, cudaStream_t st);
cudaError_t launch_rescale_to_max(int64_t n, const double* Mloc, const double* Mglob, double* S, cudaStream_t st);
cudaError_t launch_sum_chunks(const double* x, int chunks, int64_t n, double* out, cudaStream_t st);

// rounding (fp64, once per solve; round.cu).  Altschuler et al. Alg. 2 as
// restated in SPEC.md:331 in three passes over the cost:
//   R0 rows:    r(F)_i, sum_j C_ij F_ij            F   = exp(U + V - gbar C)
//   R2 columns: c(F')_j                            F'  = D(x) F, x = min(r / r(F), 1)
//   R3 rows:    r(F'')_i, sum_j C F'', sum_j C_ij err_c_j   F'' = F' D(y)
// Entries below e^-50 of their pass's target marginal (r_i for row passes,
// c_j for the column pass) are not exponentiated: each is < 2e-22 of that
// target, so a pass drops < n * 2e-22 of total mass (1.3e-17 at n = 65536).
struct RoundArgs {
  const void* C; int64_t ldc; int c_f64;
  const float* X; const float* Y; int d; float scale; int otf;   // otf: 0 dense, 1 diff recipe, 2 dot recipe
  int64_t n, nrows;
  double gbar;
  const double* A;      // row exponent base of the pass (U or U + log x)
  const double* B;      // column exponent base of the pass (V or V + log y)
  const double* logr;   // [nrows] skip thresholds (log targets)
  const double* logc;   // [n]
  const double* ec;     // R3: err_c [n]
  int chunks;           // partial chunks: column chunks of a row pass / row chunks of the column pass
  double* rowS;         // [chunks][nrows] sum of entries
  double* rowC;         // [chunks][nrows] sum C * entry
  double* rowE;         // [chunks][nrows] sum_j C_ij err_c_j (R3)
  double* colS;         // [chunks][n] column sums (R2)
  // plan output
  const double* er; float* plan; double inv_ner;
};
constexpr int kRoundMaxChunks = 8;
int round_chunks(const RoundArgs& a, bool rows);           // chunks a pass launches with (<= kRoundMaxChunks)
cudaError_t launch_round_rows(const RoundArgs& a, int with_corr, cudaStream_t st);   // R0 / R3
cudaError_t launch_round_cols(const RoundArgs& a, cudaStream_t st);                  // R2
cudaError_t launch_round_plan(const RoundArgs& a, cudaStream_t st);
// x from R0's row sums: logx = min(log r - log r(F), 0), Aout = U + logx, rowcostF = sum of R0's C F chunks
cudaError_t launch_round_x(int64_t nrows, int chunks, const double* rowS, const double* rowC, const double* r,
                           const double* U, double* logx, double* Aout, double* rowcostF, cudaStream_t st);
// y from R2's column sums (chunks): Bout = V + log y, ec = max(c - y c(F'), 0)
cudaError_t launch_round_y(int64_t n, int chunks, const double* colS, const double* c, const double* V,
                           double* Bout, double* ec, cudaStream_t st);
// err_r = max(r - r(F''), 0); scalars [|err_r|_1, <C,F''>, err_r . (C err_c), <C,F>] published
cudaError_t launch_round_fin(int64_t nrows, int chunks, const double* rowS, const double* rowC, const double* rowE,
                             const double* rowcostF, const double* r, double* er, double* blockpart,
                             unsigned int* ticket, double* out_dev, double* out_host, cudaStream_t st);
// L2 lines of [p, p + bytes) back to evict_normal priority (K1 reads part or
// all of C with evict_last; the caller's later kernels must not inherit it)
cudaError_t launch_l2_normal(const void* p, size_t bytes, cudaStream_t st);
cudaError_t launch_round_cols(const RoundArgs& a, cudaStream_t st);
cudaError_t launch_round_rows3(const RoundArgs& a, cudaStream_t st);
cudaError_t launch_round_plan(const RoundArgs& a, cudaStream_t st);
cudaError_t launch_round_combine_cols(const RoundArgs& a, const double* c, const double* V, double* Bout,
                                      double* ec, double* blockpart, unsigned int* ticket,
                                      double* out_dev, double* out_host, cudaStream_t st);
cudaError_t launch_round_combine_rows(const RoundArgs& a, const double* r, double* blockpart,
                                      unsigned int* ticket, double* out_dev, double* out_host,
                                      cudaStream_t st);

// K8: batched solver, one CTA per instance (batch.cu)
// Decrease-safeguard tolerance of the line search (Z9), relative to
// max(1, sum P).  fp32 entries: the fp32-entry noise of sum P.  fp64 entries:
// the exponent z = A_i + B_j - gbar C_ij cancels terms of size ~gbar (the
// potentials grow with gbar), so a 4-ulp error of that size moves sum P by
// ~4u (gbar + 64) relative; a fixed 1e-14 rejected every trial near
// convergence at gbar = 4096 (config 2, eps 1e-8).
__host__ __device__ inline double ls_noise(bool f64, double gbar) {
  return f64 ? 4.4e-16 * (gbar + 64.0) : 6e-8;
}

struct BatchResult {
  double cost_rounded, cost_unrounded, l1_final, rho_final, gamma_bar;
  long long evaluations, iterations, ls_evaluations, resets, ls_restarts;
  int md_steps, status;
  double rho0[64], l10[64];      // per MD step (t <= 64): initial infeasibility / L1 of the projection
  long long iters_step[64];      // per MD step iterations
  double gammas[64];             // per MD step: realised gamma_t
};
// beta_k (Z6; FR PAPER.md:496-498; PR+) from the scalars of
// the current iterate; shared by the device controller and the host loop
__host__ __device__ inline double beta_k(bool ncg, int beta_kind, double S_sg, double S_gcs, double S_gg,
                                        double S_gcg, double dphi0_prev, double sg_prev, double gg_prev) {
  double num, den;
  if (ncg) { num = S_gg - S_gcg; den = gg_prev; }
  else if (beta_kind == MDOT_BETA_PPR || beta_kind == MDOT_BETA_PPR_PLUS) { num = S_sg - S_gcs; den = -dphi0_prev; }
  else if (beta_kind == MDOT_BETA_PPR_AF) { num = S_sg - S_gcs; den = sg_prev; }
  else { num = S_sg; den = sg_prev; }
  double b = (fabs(den) > 1e-300) ? num / den : 0.0;
  if (!ncg && beta_kind == MDOT_BETA_PPR_PLUS && b < 0.0) b = 0.0;   // PR+
  return b;
}

// ADAPTIVE schedule step rule (mdot.h MDOT_SCHED_ADAPTIVE, Z29),
// shared by the host loop (solver.cu) and K8: given the step just finished
// (gamma_t, its evaluation count E, the running gbar and the previous
// efficiency eta_prev), the next step; *final is set when it is the last.
__host__ __device__ inline double adaptive_next_gamma(int t, double gt, double evals, double gbar,
                                                      double gamma_bar, double* eta_prev, int* final) {
  const double eta = gt / (evals > 1.0 ? evals : 1.0);
  double g = (t == 1 || eta >= *eta_prev) ? 2.0 * gt : fmax(0.5 * gt, gamma_bar / 1024.0);
  *eta_prev = eta;
  const double rem = gamma_bar - gbar;
  *final = 0;
  if (g >= rem || rem - g < 0.25 * g || t + 1 >= 64) { g = rem; *final = 1; }
  return g;
}
struct BatchArgs {
  const float* C;          // shared n x n fp32 cost (device)
  const double* C64;       // or fp64 cost (DENSE_F64; fp64 entries), C unused
  int n;
  const double* r;         // [B][n] (device)
  const double* c;         // [B][n]
  const double* gammas;    // [T] schedule (device)
  int T;
  int adaptive;            // MDOT_SCHED_ADAPTIVE: steps chosen on the fly from gamma1, gamma_bar
  double gamma_bar, gamma1;
  mdot_trace_rec* trace;   // nullable device trace of instance 0
  long long* trace_len;
  long long trace_cap;
  double eps, eps_md, c1, c2;   // eps_md: intermediate MD steps (>= eps)
  int stop_rho, projector, beta_kind, ls_max_trials, warm, p0_ones, f64;
  long long max_evals;
  double* U_out;           // [B][n] nullable
  double* V_out;
  BatchResult* res;        // [B] (device)
  unsigned long long* dbg; // MDOT_DIAG_K8 builds: [8] phase clock sums of instance 0 (null otherwise)
};
size_t batch_smem_bytes(int n);
cudaError_t launch_batch(const BatchArgs& a, int B, cudaStream_t st);

// MDOT_FAULT_NAN test hook (ops.cuh): per translation unit setters; apply_fault_env()
// (solver.cu) reads the environment and sets all of them when it changes
void fault_set_kernels(int mode);
void fault_set_persist(int mode);
void fault_set_batch(int mode);
void apply_fault_env();

}  // namespace mdot

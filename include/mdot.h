/* include/mdot.h -- C ABI of the B200-native MDOT-PNCG hot path.
 *
 * Method: arxiv 2307.08507 ("MDOT-PNCG").  The library solves the discrete
 * OT problem  min_{P in U(r,c)} <P, C>  (Eq. opt:original-OT-
 * problem) by mirror descent (Alg. 1) whose Bregman
 * projections onto U(r,c) are computed by preconditioned nonlinear conjugate
 * gradients on the dual potentials (Alg. 2) or by Sinkhorn
 * scaling (Alg. 3), then rounds the plan onto U(r,c)
 * and returns <C, P>.
 *
 * All functions are synchronous on return, return an mdot_status, never throw
 * and never free caller memory.  The caller owns every input and output
 * buffer; the library owns only its internal workspaces (allocated per call on
 * the caller's stream and released before return).  The last error message
 * of the calling thread is available from mdot_last_error().
 *
 * Memory kinds: `mem` in mdot_problem says where C / X / Y / r / c live and
 * where the potential outputs are written (MDOT_MEM_HOST: pageable or pinned
 * host memory, copied in/out inside the call; MDOT_MEM_DEVICE: device
 * pointers of the current CUDA device, used in place).
 *
 * Layout: C is n*n row-major (C[i*n + j] = C_ij = cost of moving mass from
 * source i to sink j), entries in [0, 1].  X, Y are n*d
 * row-major fp32 point clouds; the on-the-fly cost is
 *   C_ij = fl32( fmaf-chain over k of (x_ik - y_jk)^2 ) * scale
 * with the exact fp32 op order of DESIGN.md "Z22".  r, c are fp64 [n],
 * strictly positive, summing to 1 within 1e-12 (checked with a
 * compensated sum).
 */
#ifndef MDOT_H
#define MDOT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDOT_ABI_VERSION 3

typedef enum {
  MDOT_OK = 0,
  MDOT_EINVAL = 1,       /* precondition violated (r,c <= 0, sums, n < 1, eps <= 0, C outside [0,1]) */
  MDOT_EGEN = 2,         /* reserved (input generation failure, SPEC exit 2) */
  MDOT_EINSTABLE = 3,    /* non-finite marginals even on the exact fp64 fallback evaluator */
  MDOT_ENOCONV = 4,      /* max_evals reached before the marginal error fell below eps */
  MDOT_ELINESEARCH = 5,  /* line search failed twice in a row (Z10) */
  MDOT_ECUDA = 6,        /* CUDA runtime error (message in mdot_last_error) */
  MDOT_ENCCL = 7,        /* NCCL error (sharded calls) */
  MDOT_ENOMEM = 8        /* device allocation failed */
} mdot_status;

typedef enum {
  MDOT_COST_DENSE_F32 = 0,     /* C: const float*  (n*n) */
  MDOT_COST_SQEUCLID_F32 = 1,  /* X, Y: const float* (n*d), scale; the difference recipe (Z22):
                                  acc = fmaf(x_k - y_k, x_k - y_k, acc) for k = 0..d-1, C = acc * scale */
  MDOT_COST_DENSE_F64 = 2,     /* C: const double* (n*n) */
  MDOT_COST_SQEUCLID_DOT_F32 = 3  /* the same squared distance in dot form (Z22b), 2d + 5 -> d + 7 FP32 ops per pair:
                                  nx = fmaf chain of x_k^2, ny likewise, s = fmaf chain of x_k y_k (k = 0..d-1),
                                  C = max(fmaf(-2, s, nx + ny), 0) * scale, every step one fp32 rounding */
} mdot_cost_kind;

typedef enum { MDOT_MEM_HOST = 0, MDOT_MEM_DEVICE = 1 } mdot_mem;

typedef struct {
  int64_t n;
  int32_t kind;            /* mdot_cost_kind */
  int32_t mem;             /* mdot_mem (inputs and potential outputs) */
  const void* C;           /* DENSE_*: n*n row-major */
  int32_t d;               /* SQEUCLID: coordinate dimension (1..64) */
  float scale;             /* SQEUCLID: C_ij = recipe(|x_i - y_j|^2) * scale */
  const float* X;          /* SQEUCLID: n*d */
  const float* Y;          /* SQEUCLID: n*d */
  const double* r;         /* [n] target row marginal */
  const double* c;         /* [n] target column marginal */
} mdot_problem;

typedef enum {
  MDOT_SCHED_FIXED = 0,     /* T equal steps gamma_t = gamma_bar/T; T = max(1, floor(gamma_bar/step_max))
                               when T == 0 */
  MDOT_SCHED_DOUBLING = 1,  /* cumulative gbar_t = gamma0 * 2^(t-1) up to gamma_bar (BASELINE config 1, Z13) */
  MDOT_SCHED_EXPLICIT = 2,  /* gammas[0..n_gammas-1] */
  MDOT_SCHED_ADAPTIVE = 3   /* variable step rule (PAPER.md:371 future work; Z29): gamma_1 =
                               min(step_max, gamma_bar); with E_t the O(n^2) evaluations step t took and
                               eta_t = gamma_t / E_t, gamma_2 = 2 gamma_1 and gamma_{t+1} = 2 gamma_t if
                               eta_t >= eta_{t-1}, else max(gamma_t / 2, gamma_bar / 1024); each step is
                               clipped to the remaining budget, a remainder below a quarter of the next step
                               is merged into it, step 64 takes the rest.  Lemma 2: the
                               final plan is the entropic plan at gamma_bar whatever the realised steps.
                               The realised schedule is returned in mdot_result.gammas. */
} mdot_sched_kind;

typedef struct {
  int32_t kind;            /* mdot_sched_kind */
  int32_t T;               /* FIXED: number of steps, 0 = paper rule */
  double gamma_bar;        /* total budget (sum of gamma_t) */
  double step_max;         /* FIXED paper rule cap, default 256 */
  double gamma0;           /* DOUBLING: first step, default 1 */
  const double* gammas;    /* EXPLICIT (host pointer) */
  int32_t n_gammas;
} mdot_schedule;

/* PNCG_JACOBI: Alg. 2 with the Jacobi preconditioner diag(Hessian)^-1 =
 * D(1/r(P), 1/c(P)) (Hessian block form), its diagonal
 * bounded below by the target marginals (max(r(P), r)), in place of the
 * Sinkhorn direction (SURVEY 8(f) rank 2 ablation of PAPER.md:257). */
typedef enum { MDOT_PROJ_PNCG = 0, MDOT_PROJ_SINKHORN = 1, MDOT_PROJ_NCG = 2, MDOT_PROJ_PNCG_JACOBI = 3 } mdot_projector;
/* PPR: Eq. beta_PPR_OT with the denominator sign of Z6;
 * PPR_AF: Al-Baali-Fletcher denominator <g_{k-1}, s_{k-1}> (equal under exact
 * line search); PFR: preconditioned Fletcher-Reeves <g_k, s_k> / <g_{k-1},
 * s_{k-1}>; PPR_PLUS: max(0, beta^PPR) (PR+, Gilbert &
 * Nocedal, cited at PAPER.md:499). */
typedef enum { MDOT_BETA_PPR = 0, MDOT_BETA_PPR_AF = 1, MDOT_BETA_PFR = 2, MDOT_BETA_PPR_PLUS = 3 } mdot_beta;
typedef enum { MDOT_WARM_SCALED = 0, MDOT_WARM_CARRY = 1, MDOT_WARM_ZERO = 2 } mdot_warm;
typedef enum { MDOT_PREC_AUTO = 0, MDOT_PREC_F32P = 1, MDOT_PREC_F64P = 2 } mdot_precision;

/* One record per PNCG iteration (accepted step) or Sinkhorn half-step, in
 * order ("SolveTrace"; the oracle's orc_trace_rec has the same
 * fields).  PNCG: l1, rho at the iterate BEFORE the update; alpha the accepted
 * step; dphi0 = phi'(0) = <p, grad g>; dphi_alpha = phi'(alpha);
 * dphi_value = phi(alpha) - phi(0); beta the beta_k used in p (0 after a reset);
 * gs = <grad g, s> at the iterate; trials = line-search evaluations; reset = 1
 * when p = -s was forced (Z5 / Z10).  Sinkhorn: alpha = 1, the rest 0. */
typedef struct {
  int32_t t, k;            /* MD step (1-based), iteration within the projection (1-based) */
  double l1, rho;
  double alpha, dphi0, dphi_alpha, dphi_value;
  int32_t trials, reset;
  double beta, gs;
} mdot_trace_rec;

typedef struct {
  double eps;              /* projection stop tolerance (> 0) */
  int32_t stop;            /* 0: L1 = |r(P)-r|_1 + |c(P)-c|_1 <= eps (Z2); 1: rho <= eps */
  int32_t projector;       /* mdot_projector */
  int32_t beta;            /* mdot_beta (Z6) */
  double c1, c2;           /* approximate Wolfe constants (Z7 defaults 0.1, 0.4) */
  int32_t warm;            /* mdot_warm (Z4) */
  int32_t precision;       /* mdot_precision: AUTO = fp32 entries for fp32 C and eps >= 5e-8, fp64 entries
                              (exact two-pass evaluation) for DENSE_F64 or eps < 5e-8 */
  int32_t p0_ones;         /* 1: P0 = 1 1^T (classic Sinkhorn special case) */
  int32_t ls_max_trials;   /* per line search, default 100 */
  int64_t max_evals;       /* cap on O(n^2) evaluations per solve, default 10^7 */
  int32_t time_kernels;    /* 1: time every evaluation kernel with CUDA events (result.kernel_ms) */
  int32_t device_control;  /* 1: device-resident line-search control (no host sync per trial) */
  void* stream;            /* cudaStream_t, NULL = legacy default stream */
  double eps_md;           /* tolerance of the intermediate MD steps t < T; 0 (default) = eps at every
                              step, as the paper ran it (Z11).  By Lemma 2
                              the final plan depends only on gamma_bar, and a Bregman projection onto
                              U(r,c) is invariant to diagonal scalings of its input, so an inexact
                              intermediate projection only moves the last step's starting point
                              (adaptive eps, the paper's stated future work). */
  mdot_trace_rec* trace;   /* nullable HOST buffer of trace_cap records; filled in iteration order
                              (mdot_solve_batch: instance 0 only; sharded: this rank's copy) */
  int64_t trace_cap;
  int64_t* trace_len;      /* nullable host pointer: number of records written (<= trace_cap) */
} mdot_options;

typedef struct {
  double cost_rounded;     /* <C, G>, G = rounded plan in U(r,c) */
  double cost_unrounded;   /* <C, P(U,V)> */
  double l1_final;         /* marginal L1 error of P(U,V) (device evaluation) */
  double rho_final;        /* D_h(r(P)|r) + D_h(c(P)|c) */
  double gamma_bar;
  double seconds;          /* host wall time of the call */
  double kernel_ms;        /* sum of evaluation-kernel durations (time_kernels = 1) */
  int64_t md_steps, iterations, evaluations, ls_evaluations, resets, ls_restarts;
  int64_t fallbacks;       /* evaluations redone on the exact fp64 evaluator */
  int64_t kernel_launches; /* evaluation kernels timed */
  int64_t all_launches;    /* every kernel this library launched during the call */
  double stage_ms[4];      /* time_kernels: per-slot durations, sums over stage_samples slots.
                              graph path (CUDA events, first slot of each graph): [ctrl, prep, K1, finalize];
                              persistent path (%globaltimer, every slot): [ctrl+prep, K1, finalize, combine],
                              each including its grid barrier */
  int64_t stage_samples;   /* number of sampled slots in stage_ms */
  int32_t status;
  int32_t control_path;    /* last projection's control: 0 host loop, 1 CUDA-graph slots, 2 persistent kernel,
                              3 one-CTA-per-instance kernel (mdot_solve_batch, small mdot_solve),
                              4 lockstep batch (mdot_solve_batch with MDOT_BATCH_LOCKSTEP=1) */
  double rho0[64];         /* per MD step: infeasibility at the warm start (Fig. 2 left) */
  double l10[64];          /* per MD step: L1 at the warm start */
  int64_t iters_step[64];  /* per MD step: projection iterations */
  double gammas[64];       /* per MD step: the realised gamma_t (ADAPTIVE chooses them on the fly) */
} mdot_result;

/* Fill defaults: eps 1e-6 on L1, PNCG, beta PPR (Z6), c1 0.1, c2 0.4,
 * warm scaled, precision auto, ls_max_trials 100, max_evals 1e7. */
void mdot_options_default(mdot_options* o);
/* FIXED, gamma_bar 4096, step_max 256, T 0 (paper rule -> 16 steps). */
void mdot_schedule_default(mdot_schedule* s);

/* MDOT-PNCG solve (Alg. 1 with Alg. 2 projections; projector option selects
 * Alg. 3 or vanilla NCG).
 *   u_out, v_out: [n] cumulative potentials (U, V) with P_ij = exp(U_i + V_j
 *                 - gamma_bar C_ij), gauge fixed so that <r,U> = <c,V> (Z19);
 *                 nullable.  Same memory kind as the problem.
 *   P_out:        nullable; n*n fp32 rounded plan G (dense write, same memory
 *                 kind as the problem).
 *   res:          required.
 * Errors: MDOT_EINVAL on precondition violations (checked on the host copy of
 * r, c; C in [0,1] is checked on a sample of entries), MDOT_ENOCONV,
 * MDOT_ELINESEARCH, MDOT_EINSTABLE, MDOT_ECUDA, MDOT_ENOMEM.  On error the
 * outputs hold the last iterate. */
mdot_status mdot_solve(const mdot_problem* pb, const mdot_schedule* sched, const mdot_options* opt,
                       double* u_out, double* v_out, float* P_out, mdot_result* res);

/* Same call with the projector forced to Sinkhorn (Alg. 3) on the same
 * evaluation kernels: the paper's baseline. */
mdot_status mdot_sinkhorn(const mdot_problem* pb, const mdot_schedule* sched, const mdot_options* opt,
                          double* u_out, double* v_out, float* P_out, mdot_result* res);

/* Batch of B independent instances sharing one cost (BASELINE config 2,
 * PAPER.md:699 "including as a batch process").  r, c: B*n row-major
 * (instance b at r + b*n); u_out, v_out: B*n, nullable; res: B results.
 * Dense fp32 costs whose per-instance state fits in one SM's shared memory
 * (n <= 784 on B200) run on the K8 kernel: one CTA per instance executes the
 * whole solve on-chip, C shared through L2.  precision AUTO uses fp64 entries
 * when eps < 5e-8.  Larger instances (throughput mode)
 * run concurrently on worker streams (MDOT_BATCH_WORKERS, default 8), or, with
 * environment MDOT_BATCH_LOCKSTEP=1 and a shared dense fp32 C on the device,
 * as a lockstep batch: one launch per phase for every instance, one streamed
 * copy of each C tile evaluated by every active instance (k_eval_tma_shared),
 * MD steps decoupled per instance (MDOT_BATCH_SYNC_MD=1: step-synchronous);
 * the two are measured at parity.  Returns the
 * first non-OK status (all instances run). */
mdot_status mdot_solve_batch(const mdot_problem* shared, int32_t B, const double* r, const double* c,
                             const mdot_schedule* sched, const mdot_options* opt,
                             double* u_out, double* v_out, mdot_result* res);

/* One fused marginal evaluation (the hot kernel):
 *   lr_i = log sum_j exp(A_i + B_j - gbar C_ij),  lc_j = log sum_i exp(...)
 * (PAPER.md:157-160 in log form).  A, B, lr, lc are [n] fp64 in the memory
 * kind of the problem (r, c are used only to anchor the fp32 exponent).
 * `fallback_out` (nullable) receives 1 if the exact fp64 evaluator was used. */
mdot_status mdot_marginals(const mdot_problem* pb, const double* A, const double* B, double gbar,
                           double* lr, double* lc, const mdot_options* opt, int32_t* fallback_out);

/* Rounding onto U(r,c) (Altschuler et al. Alg. 2 as restated in
 * SPEC.md:331) of F = exp(U + V - gbar C), without solving: writes <C,F>,
 * <C,G> and optionally the dense fp32 G (P_out, nullable). */
mdot_status mdot_round(const mdot_problem* pb, const double* U, const double* V, double gbar,
                       float* P_out, double* cost_F, double* cost_G, const mdot_options* opt);

/* ---- row-sharded multi-GPU (NCCL over NVLink; one process per GPU) ---- */
typedef struct mdot_comm mdot_comm;
/* nccl_unique_id: 128-byte ncclUniqueId from rank 0 (broadcast by the caller,
 * e.g. over a torch.distributed process group). */
mdot_status mdot_get_unique_id(void* nccl_unique_id_out);
mdot_status mdot_comm_create(const void* nccl_unique_id, int32_t nranks, int32_t rank, int32_t device,
                             mdot_comm** out);
/* In-process transport: `nranks` threads of ONE process (one stream each,
 * possibly on one GPU) form group `group`; every allreduce is a host-side
 * deterministic rank-ordered sum.  For tests of the sharded path on one GPU
 * (virtual ranks) and for single-process multi-GPU embedding. */
mdot_status mdot_comm_create_local(const char* group, int32_t nranks, int32_t rank, int32_t device,
                                   mdot_comm** out);
mdot_status mdot_comm_destroy(mdot_comm* comm);
/* Fused peer exchange (SURVEY 8(e) NC1 without a separate collective;
 * DESIGN.md "Fused peer exchange").  COLLECTIVE: every rank of `comm` calls
 * it with the same n_max.  Allocates this rank's exchange block
 * (2 x nranks x (n_max + 16) fp64, device memory, owned by the comm, freed by
 * mdot_comm_destroy) and maps every rank's block: NCCL transport -> CUDA IPC
 * handles gathered over the communicator, opened with peer access (NVLink);
 * in-process transport -> the group's blocks on the shared GPU.  Afterwards
 * mdot_solve_sharded with dense fp32 C (n <= n_max) runs each projection as
 * ONE persistent kernel per rank whose column-marginal exchange is plain
 * peer-memory stores + system-scope flags inside the kernel; the in-process
 * transport runs all of its ranks as groups of CTAs of ONE cooperative launch
 * (ranks that wait on each other must be co-resident on one GPU).
 * nranks <= 8.  Errors: MDOT_EINVAL (bad arguments, > 8 ranks, single-rank
 * in-process comm), MDOT_ECUDA (allocation / IPC / peer access failed on ANY
 * rank -- every rank returns it and keeps the NCCL / host path), MDOT_ENOMEM.
 * A solve whose in-kernel flag wait times out (a peer died) returns
 * MDOT_ENCCL.  MDOT_NO_PEER=1 in the environment disables the path;
 * n_max = 0 (collective) frees the exchange blocks and returns the comm to
 * the NCCL / host path. */
mdot_status mdot_comm_enable_peer(mdot_comm* comm, int64_t n_max);
/* local rows [row0, row0 + n_local) of C (local_rows->C points at row row0,
 * n_local*n entries) or of X (local_rows->X at row row0; Y, r, c full).
 * local_rows->n is the GLOBAL n.  u_local_out: [n_local], v_out: [n]. */
mdot_status mdot_solve_sharded(mdot_comm* comm, const mdot_problem* local_rows, int64_t row0, int64_t n_local,
                               const mdot_schedule* sched, const mdot_options* opt,
                               double* u_local_out, double* v_out, mdot_result* res);

/* 2-D (row x column) sharding (past the replicated
 * column vectors of mdot_solve_sharded).  The ranks form a Gr x Gc grid; this
 * rank owns the block rows [row0, row0 + n_rows) x columns
 * [col0, col0 + n_cols) of the n x n cost: block->C points at that block
 * (dense fp32, row-major, n_rows x n_cols, leading dimension n_cols), or, for
 * (dense fp64 for MDOT_COST_DENSE_F64), or, for
 * the on-the-fly costs (MDOT_COST_SQEUCLID_F32 / _DOT_F32), block->X at the
 * n_rows x d rows of X and block->Y at the n_cols x d rows of Y of the block;
 * block->n is the GLOBAL n; block->r, block->c are the FULL marginals,
 * validated as in mdot_solve.  An evaluation is K1 over the block, then
 * two allreduces: the block's row sums over `row_comm` (the Gc ranks of this
 * row block) and its column sums over `col_comm` (the Gr ranks of this column
 * block); rows and columns then finalize locally and the 16 control scalars
 * are summed over the other communicator (row items are replicated across
 * row_comm, column items across col_comm), so every rank holds identical
 * scalars and takes identical line-search decisions.
 * Rounding reduces its row sums over row_comm and its column
 * sums over col_comm the same way.  Either communicator may have one rank
 * (Gr = 1 or Gc = 1).  u_local_out: [n_rows], v_local_out: [n_cols] (the
 * rank's slices of the gauge-fixed potentials; identical across the
 * replicas).  Precision as mdot_solve: fp32 entries, with the exact fp64
 * evaluator distributed the same way ((max, sum) pairs: a max-allreduce, a
 * rescale and a sum-allreduce per side) for the range-guard fallback and for
 * fp64-entry solves (eps < 5e-8 with AUTO, F64P, fp64 C; host control).
 * Control: with both communicators on the NCCL
 * transport, options.device_control = 1 runs the line search on the device
 * (CUDA-graph slots with the four per-evaluation allreduces captured); the
 * in-process transport, or device_control = 0, runs the host control loop.
 * The screened on-the-fly evaluation (K2s), the persistent fused-exchange
 * kernel and the dense plan output are not part of the 2-D path.
 * Environment MDOT_NC2=1 (this call and mdot_solve_sharded, host control
 * loop, fp32 entries): scalar-only line-search trials --
 * a trial reduces 4 scalars, an accepted trial is completed with the vector
 * exchange (measured slower at the BASELINE sizes). */
mdot_status mdot_solve_sharded_2d(mdot_comm* row_comm, mdot_comm* col_comm, const mdot_problem* block,
                                  int64_t row0, int64_t n_rows, int64_t col0, int64_t n_cols,
                                  const mdot_schedule* sched, const mdot_options* opt, double* u_local_out,
                                  double* v_local_out, mdot_result* res);

/* Screened evaluation statistics of the calling thread's last mdot_solve /
 * mdot_sinkhorn (K2s): on-the-fly costs with
 * d in {2, 4, 8, 16} on one rank evaluate the graph-slot trials with a
 * tensor-core screen that skips the entries below 2^-T (T = 56 by default,
 * env MDOT_SCREEN_T) of both their row and column totals -- a rigorous bound,
 * < n 2^-T relative change of any marginal.  out[0] entries kept, out[1]
 * entries screened, out[2] screened evaluations, out[3] summed device time
 * of the timed screened evaluations (ms, options.time_kernels), out[4] their
 * count.  env MDOT_SCREEN=0 disables the screen.  out: 5 doubles (host). */
mdot_status mdot_last_screen_stats(double* out);

const char* mdot_last_error(void);
int32_t mdot_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MDOT_H */

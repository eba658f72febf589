/* oracle/mdot_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU oracle of the MDOT-PNCG hot path (arxiv 2307.08507).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  It shares no code, header, table or
 * constant with the CUDA library (paper_2307_08507_b200/, include/mdot.h).
 *
 * Readings of the paper that this oracle takes are the SURVEY.md section 8(c)
 * "Z" readings, restated in DESIGN.md; each function cites the passage it
 * follows as PAPER.md:<line> (section / equation / algorithm).
 */
#ifndef MDOT_ORACLE_H
#define MDOT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ORC_SQEUCLID_DOT_F32 (Z22b): the dot form of the same squared distance with
 * its own fixed fp32 op order, nx = fmaf chain of x_k^2, ny likewise, s = fmaf
 * chain of x_k y_k, C = max(fmaf(-2, s, nx + ny), 0) * scale. */
enum { ORC_DENSE_F32 = 0, ORC_SQEUCLID_F32 = 1, ORC_DENSE_F64 = 2, ORC_SQEUCLID_DOT_F32 = 3 };
/* ORC_PNCG_JACOBI: Alg. 2 with the Jacobi preconditioner diag(Hessian)^-1 in place
 * of the Sinkhorn direction (SURVEY 8(f) rank 2 ablation; Hessian PAPER.md:225). */
enum { ORC_PNCG = 0, ORC_SINKHORN = 1, ORC_NCG = 2, ORC_PNCG_JACOBI = 3 };
/* ORC_BETA_PPR_PLUS: max(0, beta^PPR), the PR+ safeguard of Gilbert & Nocedal
 * (cited at PAPER.md:499 for FR's unproductive directions). */
enum { ORC_BETA_PPR = 0, ORC_BETA_PPR_AF = 1, ORC_BETA_PFR = 2, ORC_BETA_PPR_PRINTED = 3, ORC_BETA_PPR_PLUS = 4 };
enum { ORC_WARM_SCALED = 0, ORC_WARM_CARRY = 1, ORC_WARM_ZERO = 2 };
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EINSTABLE = 3, ORC_ENOCONV = 4, ORC_ELINESEARCH = 5 };

typedef struct {
  int64_t n;
  int32_t kind;          /* ORC_DENSE_F32 / ORC_DENSE_F64 / ORC_SQEUCLID_F32 */
  int32_t d;             /* coordinate dimension (SQEUCLID) */
  const void* C;         /* n*n row-major, float or double */
  const float* X;        /* n*d (SQEUCLID) */
  const float* Y;        /* n*d */
  float scale;           /* C_ij = fp32 recipe(|x_i-y_j|^2) * scale */
  const double* r;       /* target row marginal, >0, sums to 1 */
  const double* c;       /* target column marginal */
} orc_problem;

typedef struct {
  double eps;            /* projection stop tolerance */
  int32_t stop_rho;      /* 0: L1 = |r(P)-r|_1+|c(P)-c|_1 <= eps (Z2); 1: rho <= eps */
  int32_t projector;     /* ORC_PNCG, ORC_SINKHORN, ORC_NCG */
  int32_t beta;          /* ORC_BETA_* (Z6) */
  double c1, c2;         /* approximate Wolfe constants (Z7: 0.1, 0.4) */
  int32_t warm;          /* ORC_WARM_* (Z4) */
  int32_t p0_ones;       /* 1: P0 = 1 1^T (classic Sinkhorn), 0: P0 = r c^T */
  int64_t max_evals;     /* cap on O(n^2) evaluations per solve (0 = 10^7) */
  int32_t ls_max_trials; /* per line search (0 = 100) */
  int32_t max_threads;   /* OpenMP threads (0 = default) */
  double eps_md;         /* tolerance of the intermediate MD steps t < T (0 = eps at every step, Z11).
                            Lemma 2 makes the final plan depend only on gbar, and the
                            projection is invariant to diagonal scalings of its input, so an inexact
                            intermediate projection changes only the final step's starting point
                            ("future work"). */
} orc_options;

typedef struct {         /* one PNCG / Sinkhorn iteration */
  int32_t t, k;
  double l1, rho;        /* at the iterate BEFORE this iteration's update */
  double alpha, dphi0, dphi_alpha, dphi_value; /* line search: phi'(0), phi'(alpha), phi(alpha)-phi(0) */
  int32_t trials, reset;
  double beta;
  double gs;             /* <grad g, s> at the iterate (the PPR_AF / PFR denominator of the next iteration) */
} orc_trace_rec;

typedef struct {
  double cost_unrounded, cost_rounded, l1_final, rho_final, gamma_bar, seconds;
  int64_t md_steps, iterations, evaluations, ls_evaluations, resets, ls_restarts;
  int32_t status;
  /* per-MD-step: initial infeasibility rho_0 and L1_0 (Fig. 2 left), iterations */
  double rho0[64], l10[64];
  int64_t iters_step[64];
} orc_result;

/* log r(P), log c(P) for P_ij = exp(A_i + B_j - gbar*C_ij) */
int orc_log_marginals(const orc_problem* pb, const double* A, const double* B, double gbar,
                      double* lr, double* lc);
int orc_log_marginal_rows(const orc_problem* pb, const double* A, const double* B, double gbar,
                          const int64_t* idx, int64_t k, double* out);
int orc_log_marginal_cols(const orc_problem* pb, const double* A, const double* B, double gbar,
                          const int64_t* idx, int64_t k, double* out);
/* C_ij as the oracle sees it (fp64 promotion of the input / Z22 recipe) */
double orc_cost(const orc_problem* pb, int64_t i, int64_t j);

/* One Bregman projection (Alg. 2 / Alg. 3) of P_hat = exp(U + V - gbar*C)
 * starting at potentials (u, v), which are updated in place. */
int orc_project(const orc_problem* pb, const double* U, const double* V, double gbar,
                double* u, double* v, const orc_options* opt, int32_t t,
                orc_result* res, orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len);

/* MDOT (Alg. 1) with schedule gammas[0..T-1]; outputs cumulative (U, V),
 * gauge fixed so that <r,U> = <c,V> (Z19), rounded cost and stats. */
int orc_mdot(const orc_problem* pb, const double* gammas, int32_t T, const orc_options* opt,
             double* U_out, double* V_out, orc_result* res,
             orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len);

/* phi'(alpha) and phi(alpha) - phi(0) of one line-search trial (PAPER.md:
 * 694-696); returns ORC_OK or an error status that aborts the search. */
typedef int (*orc_phi_fn)(void* ctx, double alpha, double* dphi, double* dval);
/* The hybrid secant / bisection line search of Appx. C
 * for the approximate Wolfe conditions with the decrease
 * safeguard phi(alpha) - phi(0) <= dec_tol (Z9) and bracket expansion by
 * doubling from alpha0 (Z8, cap 60).  Writes the accepted alpha, phi'(alpha),
 * phi(alpha) - phi(0), the trial count and *accepted (0: no alpha within
 * max_trials / 60 doublings).  Returns the callback's error status or ORC_OK. */
int orc_line_search(orc_phi_fn fn, void* ctx, double dphi0, double alpha0, double c1, double c2, double dec_tol,
                    int max_trials, double* alpha_out, double* dphi_out, double* dval_out, int* trials_out,
                    int* accepted_out);

/* sum_ij C_ij exp(A_i + B_j - gbar C_ij): <C, P(A,B)> in one pass (the
 * unrounded cost of north_star's parity gate, Z20). */
double orc_plan_cost(const orc_problem* pb, const double* A, const double* B, double gbar);

/* MDOT with the ADAPTIVE step rule (PAPER.md:371 future work, "variable
 * learning rate MD procedures that exploit the warm-starting of the dual
 * variables"; reading Z29): gamma_1 = min(gamma1, gamma_bar); after
 * step t with E_t evaluations, eta_t = gamma_t / E_t (progress in gbar per
 * O(n^2) pass); gamma_2 = 2 gamma_1; for t >= 2 gamma_{t+1} = 2 gamma_t if
 * eta_t >= eta_{t-1} else max(gamma_t / 2, gamma_bar / 1024); every step is
 * clipped to the remaining budget, a remainder below a quarter of the next
 * step is merged into it, and step 64 takes the whole remainder.  By Lemma 2
 * the final plan is the entropic plan at gamma_bar for
 * ANY such schedule.  gammas_out[0..md_steps-1] receives the schedule. */
int orc_mdot_adaptive(const orc_problem* pb, double gamma_bar, double gamma1, const orc_options* opt,
                      double* U_out, double* V_out, orc_result* res, double* gammas_out,
                      orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len);

/* Rounding onto U(r,c) (Altschuler et al. Alg. 2, as restated in SPEC.md:331)
 * of F = exp(U + V - gbar*C).  Writes cost <C,F>, cost <C,G>, and optionally
 * the dense G (n*n doubles) and its marginals. */
int orc_round(const orc_problem* pb, const double* U, const double* V, double gbar,
              double* cost_F, double* cost_G, double* G_out, double* rG, double* cG);

/* Schedules (BASELINE config 1 / Z13) */
int orc_schedule_fixed(double gamma_bar, double step_max, int32_t T, double* out, int32_t cap);
int orc_schedule_doubling(double gamma_bar, double gamma0, double* out, int32_t cap);
double orc_default_eps(double hmin, double gamma_bar);

#ifdef __cplusplus
}
#endif
#endif

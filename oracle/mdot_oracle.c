/* oracle/mdot_oracle.c -- TEST INFRASTRUCTURE ONLY (see mdot_oracle.h).
 *
 * A plain fp64 CPU implementation of MDOT (Alg. 1) with the PNCG (Alg. 2) and
 * Sinkhorn (Alg. 3) Bregman projections, the hybrid secant/bisection line
 * search of Appx. C, and the final rounding onto U(r,c).  Loops are written
 * as the definitions read; OpenMP only splits independent rows / columns
 * (each sum is still accumulated in index order, so results do not depend on
 * the thread count).  Built with -ffp-contract=off: no fused multiply-adds
 * unless written as fma().
 *
 * Parity status of each function:
 *   orc_log_marginals  pinned: direct fp64 sum on small n, shift invariance,
 *                      closed-form marginals of rank-1 P.
 *   orc_project        pinned: 2x2 closed form, Sinkhorn==PNCG fixed point,
 *                      descent identity, Wolfe post-hoc, alpha=1 along -s is
 *                      a Jacobi Sinkhorn step.
 *   orc_mdot           pinned: Lemma 2 (schedule invariance), Lemma 1,
 *                      Prop. 1 bound vs exact OT (enumeration / LP / 1-D
 *                      monotone coupling), delta marginal -> r c^T.
 *   orc_round          pinned: exact marginals, SPEC.md:337 worked example,
 *                      idempotence, L1 perturbation bound.
 * Absolute iteration counts are "parity unpinned" (no paper numbers).
 */
#include "mdot_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Cost access.  Dense: the input value promoted to double.  SQEUCLID: the
 * fixed fp32 recipe of DESIGN.md Z22:  acc = 0; for k: d = x_k - y_k;
 * acc = fmaf(d, d, acc);  C = acc * scale  (all fp32, round-to-nearest). */
double orc_cost(const orc_problem* pb, int64_t i, int64_t j) {
  const int64_t n = pb->n;
  if (pb->kind == ORC_DENSE_F32) return (double)((const float*)pb->C)[i * n + j];
  if (pb->kind == ORC_DENSE_F64) return ((const double*)pb->C)[i * n + j];
  if (pb->kind == ORC_SQEUCLID_DOT_F32) {
    /* Z22b: C = max(fl(nx + ny) - 2 s, 0) * scale, each fp32 step rounded once */
    const float* x = pb->X + i * pb->d;
    const float* y = pb->Y + j * pb->d;
    float nx = 0.0f, ny = 0.0f, sxy = 0.0f;
    for (int k = 0; k < pb->d; ++k) nx = fmaf(x[k], x[k], nx);
    for (int k = 0; k < pb->d; ++k) ny = fmaf(y[k], y[k], ny);
    for (int k = 0; k < pb->d; ++k) sxy = fmaf(x[k], y[k], sxy);
    const float t = nx + ny;
    const float cij = fmaxf(fmaf(-2.0f, sxy, t), 0.0f) * pb->scale;
    return (double)cij;
  }
  {
    const float* x = pb->X + i * pb->d;
    const float* y = pb->Y + j * pb->d;
    float acc = 0.0f;
    for (int k = 0; k < pb->d; ++k) {
      float dk = x[k] - y[k];
      acc = fmaf(dk, dk, acc);
    }
    float cij = acc * pb->scale;
    return (double)cij;
  }
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------ */
/* Log-marginals of P(A,B)_ij = exp(A_i + B_j - gbar C_ij), PAPER.md:54,
 * 157-160 (plan refinement with P^t = exp(U + V - gbar_prev C), PAPER.md:
 * 597-598).  Log domain (A34, mandated by north_star): each marginal is a
 * two-pass log-sum-exp, max first, then the sum of exp(z - max).            */
int orc_log_marginals(const orc_problem* pb, const double* A, const double* B, double gbar,
                      double* lr, double* lc) {
  const int64_t n = pb->n;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < n; ++i) {
    double m = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
      double z = (A[i] + B[j]) - gbar * orc_cost(pb, i, j);
      if (z > m) m = z;
    }
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double z = (A[i] + B[j]) - gbar * orc_cost(pb, i, j);
      s += exp(z - m);
    }
    lr[i] = m + log(s);
    if (!isfinite(lr[i])) bad = 1;
  }
  const int64_t JB = 64;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t j0 = 0; j0 < n; j0 += JB) {
    double m[64], s[64];
    int64_t j1 = j0 + JB < n ? j0 + JB : n;
    for (int64_t j = j0; j < j1; ++j) { m[j - j0] = -INFINITY; s[j - j0] = 0.0; }
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = j0; j < j1; ++j) {
        double z = (A[i] + B[j]) - gbar * orc_cost(pb, i, j);
        if (z > m[j - j0]) m[j - j0] = z;
      }
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = j0; j < j1; ++j) {
        double z = (A[i] + B[j]) - gbar * orc_cost(pb, i, j);
        s[j - j0] += exp(z - m[j - j0]);
      }
    for (int64_t j = j0; j < j1; ++j) {
      lc[j] = m[j - j0] + log(s[j - j0]);
      if (!isfinite(lc[j])) bad = 1;
    }
  }
  return bad ? ORC_EINSTABLE : ORC_OK;
}

/* The same log-sum-exp for selected rows / columns only (parity checks at
 * full size compute sampled outputs one by one). */
int orc_log_marginal_rows(const orc_problem* pb, const double* A, const double* B, double gbar,
                          const int64_t* idx, int64_t k, double* out) {
  const int64_t n = pb->n;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < k; ++q) {
    const int64_t i = idx[q];
    double m = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
      double z = (A[i] + B[j]) - gbar * orc_cost(pb, i, j);
      if (z > m) m = z;
    }
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s += exp((A[i] + B[j]) - gbar * orc_cost(pb, i, j) - m);
    out[q] = m + log(s);
  }
  return ORC_OK;
}

int orc_log_marginal_cols(const orc_problem* pb, const double* A, const double* B, double gbar,
                          const int64_t* idx, int64_t k, double* out) {
  const int64_t n = pb->n;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < k; ++q) {
    const int64_t j = idx[q];
    double m = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      double z = (A[i] + B[j]) - gbar * orc_cost(pb, i, j);
      if (z > m) m = z;
    }
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += exp((A[i] + B[j]) - gbar * orc_cost(pb, i, j) - m);
    out[q] = m + log(s);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Small vector helpers (plain loops). */
static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double sum(const double* a, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i];
  return s;
}

/* D_h(y|x) = sum_i x_i - y_i + y_i log(y_i/x_i).  rho uses
 * y = r(P), x = r (Alg. 2 line 3; Z1). */
static double gen_kl(const double* y, const double* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] - y[i] + y[i] * log(y[i] / x[i]);
  return s;
}

typedef struct {       /* marginals of the current plan */
  double *lr, *lc, *rP, *cP;
  double mass;         /* sum_ij P_ij */
} marg_t;

static int evaluate(const orc_problem* pb, const double* U, const double* V, const double* u,
                    const double* v, double gbar, double* A, double* B, marg_t* M) {
  const int64_t n = pb->n;
  for (int64_t i = 0; i < n; ++i) A[i] = U[i] + u[i];
  for (int64_t j = 0; j < n; ++j) B[j] = V[j] + v[j];
  int st = orc_log_marginals(pb, A, B, gbar, M->lr, M->lc);
  for (int64_t i = 0; i < n; ++i) M->rP[i] = exp(M->lr[i]);
  for (int64_t j = 0; j < n; ++j) M->cP[j] = exp(M->lc[j]);
  M->mass = sum(M->rP, n);
  return st;
}

static double l1_err(const marg_t* M, const double* r, const double* c, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += fabs(M->rP[i] - r[i]);
  for (int64_t j = 0; j < n; ++j) s += fabs(M->cP[j] - c[j]);
  return s;
}

static double rho_err(const marg_t* M, const double* r, const double* c, int64_t n) {
  return gen_kl(M->rP, r, n) + gen_kl(M->cP, c, n);
}

/* ------------------------------------------------------------------ */
/* Sinkhorn projection, Alg. 3 with the index typo of
 * line 430 read as dv_j = log(c_j / c_j(P)) (Z16).  Odd k updates u, even k
 * updates v; the stopping test uses both marginals of P^k (one evaluation
 * per half-step; Z26: an SA "iteration" is a half-step).                  */
static int sinkhorn_project(const orc_problem* pb, const double* U, const double* V, double gbar,
                            double* u, double* v, const orc_options* opt, int32_t t,
                            orc_result* res, orc_trace_rec* tr, int64_t cap, int64_t* tlen) {
  const int64_t n = pb->n;
  const double *r = pb->r, *c = pb->c;
  double* buf = (double*)malloc(sizeof(double) * 6 * n);
  double *A = buf, *B = buf + n;
  marg_t M = {buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, 0.0};
  int st = evaluate(pb, U, V, u, v, gbar, A, B, &M);
  res->evaluations++;
  double l1 = l1_err(&M, r, c, n), rho = rho_err(&M, r, c, n);
  if (t >= 1 && t <= 64) { res->rho0[t - 1] = rho; res->l10[t - 1] = l1; }
  int64_t k = 0;
  const int64_t cap_evals = opt->max_evals > 0 ? opt->max_evals : 10000000;
  while (st == ORC_OK && (opt->stop_rho ? rho : l1) > opt->eps) {
    if (res->evaluations >= cap_evals) { st = ORC_ENOCONV; break; }
    k++;
    if (tr && *tlen < cap) {
      orc_trace_rec* q = &tr[(*tlen)++];
      memset(q, 0, sizeof(*q));
      q->t = t; q->k = (int32_t)k; q->l1 = l1; q->rho = rho; q->alpha = 1.0;
    }
    if (k % 2 == 1) {
      for (int64_t i = 0; i < n; ++i) u[i] += log(r[i]) - M.lr[i];   /* log(r_i / r_i(P)) */
    } else {
      for (int64_t j = 0; j < n; ++j) v[j] += log(c[j]) - M.lc[j];   /* log(c_j / c_j(P)) */
    }
    st = evaluate(pb, U, V, u, v, gbar, A, B, &M);
    res->evaluations++;
    res->iterations++;
    if (t >= 1 && t <= 64) res->iters_step[t - 1]++;
    l1 = l1_err(&M, r, c, n);
    rho = rho_err(&M, r, c, n);
  }
  res->l1_final = l1;
  res->rho_final = rho;
  free(buf);
  return st;
}

/* ------------------------------------------------------------------ */
/* Line search, Appx. C: approximate Wolfe
 *   (2 c1 - 1) phi'(0) >= phi'(alpha) >= c2 phi'(0)
 * plus the decrease safeguard phi(alpha) - phi(0) <= dec_tol (Z9).  Bracket
 * [lo, hi] with phi'(lo) < 0 < phi'(hi): while there is no hi, alpha doubles
 * (Z8, at most 60 times); then alpha_sec = (lo phi'(hi) - hi phi'(lo)) /
 * (phi'(hi) - phi'(lo)) and alpha = alpha_sec / 2 + (lo + hi) / 4
 * ("alpha_hybrid"); bisection if phi'(hi) <= phi'(lo).          */
int orc_line_search(orc_phi_fn fn, void* ctx, double dphi0, double alpha0, double c1, double c2, double dec_tol,
                    int max_trials, double* alpha_out, double* dphi_out, double* dval_out, int* trials_out,
                    int* accepted_out) {
  double alpha = alpha0;
  double lo = 0.0, dlo = dphi0, hi = 0.0, dhi = 0.0;
  int have_hi = 0, doublings = 0, trials = 0, accepted = 0, st = ORC_OK;
  double dphi_a = 0.0, dval = 0.0;
  for (int tr_i = 0; tr_i < max_trials; ++tr_i) {
    st = fn(ctx, alpha, &dphi_a, &dval);
    trials++;
    if (st != ORC_OK) break;
    const int wolfe = ((2.0 * c1 - 1.0) * dphi0 >= dphi_a) && (dphi_a >= c2 * dphi0);
    const int decrease = dval <= dec_tol;
    if (wolfe && decrease) { accepted = 1; break; }
    if (dphi_a < 0.0 && decrease) {
      lo = alpha; dlo = dphi_a;
    } else {
      hi = alpha; dhi = dphi_a; have_hi = 1;
    }
    if (!have_hi) {
      if (++doublings > 60) break;
      alpha = 2.0 * alpha;
    } else if (dhi > dlo) {
      double a_sec = (lo * dhi - hi * dlo) / (dhi - dlo);
      alpha = 0.5 * a_sec + 0.5 * (hi + lo) / 2.0;
    } else {
      alpha = 0.5 * (lo + hi);
    }
  }
  *alpha_out = alpha;
  *dphi_out = dphi_a;
  *dval_out = dval;
  *trials_out = trials;
  *accepted_out = accepted;
  return st;
}

/* One trial of the PNCG line search: P(alpha) at (u + alpha p_u, v + alpha p_v). */
typedef struct {
  const orc_problem* pb;
  const double *U, *V, *u, *v, *p;
  double gbar, mass0, pr;
  double *A, *B, *trial_u, *trial_v;
  marg_t* T;
  orc_result* res;
} trial_ctx;

static int pncg_trial(void* vctx, double alpha, double* dphi, double* dval) {
  trial_ctx* c = (trial_ctx*)vctx;
  const int64_t n = c->pb->n;
  const double *r = c->pb->r, *cc = c->pb->c, *p = c->p;
  for (int64_t i = 0; i < n; ++i) c->trial_u[i] = c->u[i] + alpha * p[i];
  for (int64_t j = 0; j < n; ++j) c->trial_v[j] = c->v[j] + alpha * p[n + j];
  int st = evaluate(c->pb, c->U, c->V, c->trial_u, c->trial_v, c->gbar, c->A, c->B, c->T);
  c->res->evaluations++;
  c->res->ls_evaluations++;
  if (st != ORC_OK) return st;
  /* phi'(alpha) = <p_u, r(P(alpha)) - r> + <p_v, c(P(alpha)) - c> */
  double d = 0.0;
  for (int64_t i = 0; i < n; ++i) d += p[i] * (c->T->rP[i] - r[i]);
  for (int64_t j = 0; j < n; ++j) d += p[n + j] * (c->T->cP[j] - cc[j]);
  *dphi = d;
  /* phi(alpha) - phi(0) = sum P(alpha) - sum P(0) - alpha(<p_u,r> + <p_v,c>) */
  *dval = (c->T->mass - c->mass0) - alpha * c->pr;
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* PNCG projection, Alg. 2, with
 *   s   = (log r(P) - log r, log c(P) - log c)
 *   grad= (r(P) - r, c(P) - c)
 *   beta (Z6): <grad_k - grad_{k-1}, s_k> / (-<grad_{k-1}, p_{k-1}>), beta_1 = 0
 *        (PAPER.md:262 prints the denominator without the minus sign)
 *   p   = -s + beta p_prev; reset p = -s when <p, grad> >= 0 (Z5; PAPER.md:190
 *        prints "< 0")
 *   line search: approximate Wolfe with c1 = 0.1, c2 = 0.4
 *        (Z7), hybrid alpha = alpha_sec/2 + (alpha_lo+alpha_hi)/4
 *        (PAPER.md:692, 698), bracket expansion by doubling (Z8), decrease
 *        safeguard (Z9), reset-and-retry on failure (Z10).
 * NCG (projector ORC_NCG) uses grad in place of s and
 * beta^PR.                                                                 */
static int pncg_project(const orc_problem* pb, const double* U, const double* V, double gbar,
                        double* u, double* v, const orc_options* opt, int32_t t,
                        orc_result* res, orc_trace_rec* tr, int64_t cap, int64_t* tlen) {
  const int64_t n = pb->n, n2 = 2 * n;
  const double *r = pb->r, *c = pb->c;
  const int ncg = opt->projector == ORC_NCG;
  double* buf = (double*)malloc(sizeof(double) * (22 * n));
  double *A = buf, *B = buf + n;
  marg_t M = {buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, 0.0};
  marg_t T = {buf + 6 * n, buf + 7 * n, buf + 8 * n, buf + 9 * n, 0.0};
  double* s = buf + 10 * n;      /* [2n] (u part, v part) */
  double* g = buf + 12 * n;      /* [2n] */
  double* p = buf + 14 * n;      /* [2n] */
  double* gprev = buf + 16 * n;  /* [2n] */
  double* pprev = buf + 18 * n;  /* [2n] */
  double* trial_u = buf + 20 * n;
  double* trial_v = buf + 21 * n;
  double* sprev = (double*)malloc(sizeof(double) * n2);
  double rc_dot_prev = 0.0;

  int st = evaluate(pb, U, V, u, v, gbar, A, B, &M);
  res->evaluations++;
  double l1 = l1_err(&M, r, c, n), rho = rho_err(&M, r, c, n);
  if (t >= 1 && t <= 64) { res->rho0[t - 1] = rho; res->l10[t - 1] = l1; }
  int64_t k = 0;
  double alpha_prev = 1.0;
  const double c1 = opt->c1, c2 = opt->c2;
  const int max_trials = opt->ls_max_trials > 0 ? opt->ls_max_trials : 100;
  const int64_t cap_evals = opt->max_evals > 0 ? opt->max_evals : 10000000;

  while (st == ORC_OK && (opt->stop_rho ? rho : l1) > opt->eps) {
    if (res->evaluations >= cap_evals) { st = ORC_ENOCONV; break; }
    k++;
    /* Sinkhorn direction and gradient (Alg. 2 line 5). */
    for (int64_t i = 0; i < n; ++i) {
      s[i] = M.lr[i] - log(r[i]);
      g[i] = M.rP[i] - r[i];
    }
    for (int64_t j = 0; j < n; ++j) {
      s[n + j] = M.lc[j] - log(c[j]);
      g[n + j] = M.cP[j] - c[j];
    }
    /* Jacobi variant: s = D(diag Hessian)^-1 grad with diag = (r(P), c(P))
     * (Hessian block form), the diagonal bounded below by
     * the target, max(r(P), r): |s| < 1 far from feasibility (the plain
     * 1/r(P) overflows the first trial when r(P) << r); equal to D(1/r)
     * grad at the solution, where the Sinkhorn direction is too. */
    if (opt->projector == ORC_PNCG_JACOBI) {
      for (int64_t i = 0; i < n; ++i) s[i] = g[i] / fmax(M.rP[i], r[i]);
      for (int64_t j = 0; j < n; ++j) s[n + j] = g[n + j] / fmax(M.cP[j], c[j]);
    }
    const double* dir = ncg ? g : s;   /* preconditioned or vanilla */
    /* beta_k (Z6) */
    double beta = 0.0;
    if (k > 1) {
      double num = 0.0, den = 0.0;
      for (int64_t q = 0; q < n2; ++q) num += (g[q] - gprev[q]) * dir[q];
      if (ncg) {
        for (int64_t q = 0; q < n2; ++q) den += gprev[q] * gprev[q];  /* beta^PR */
      } else if (opt->beta == ORC_BETA_PPR) {
        den = -dot(gprev, pprev, n2);
      } else if (opt->beta == ORC_BETA_PPR_PRINTED) {
        den = dot(gprev, pprev, n2);
      } else if (opt->beta == ORC_BETA_PPR_AF) {
        den = rc_dot_prev;            /* <grad_{k-1}, s_{k-1}> */
      } else if (opt->beta == ORC_BETA_PPR_PLUS) {
        den = -dot(gprev, pprev, n2);
      } else { /* ORC_BETA_PFR: <grad_k, s_k> / <grad_{k-1}, s_{k-1}> (PAPER.md:497 preconditioned) */
        num = dot(g, s, n2);
        den = rc_dot_prev;
      }
      beta = (fabs(den) > 1e-300) ? num / den : 0.0;
      if (!ncg && opt->beta == ORC_BETA_PPR_PLUS && beta < 0.0) beta = 0.0;   /* PR+ */
    }
    /* direction and reset (Alg. 2 lines 6-9; Z5) */
    for (int64_t q = 0; q < n2; ++q) p[q] = -dir[q] + beta * pprev[q];
    double dphi0 = dot(p, g, n2);
    int reset = 0;
    if (!(dphi0 < 0.0)) {
      for (int64_t q = 0; q < n2; ++q) p[q] = -dir[q];
      dphi0 = dot(p, g, n2);
      reset = 1;
      res->resets++;
    }
    rc_dot_prev = dot(g, s, n2);

    /* line search (Alg. 2 line 10; Appx. C) */
    const double phi0 = M.mass - dot(u, r, n) - dot(v, c, n) - 1.0;  /* g(u,v) */
    const double dec_tol = 1e-14 * (fabs(phi0) > 1.0 ? fabs(phi0) : 1.0);
    double alpha = (k == 1) ? 1.0 : fmin(4.0, fmax(0.25, alpha_prev));   /* Z8 */
    int accepted = 0, trials = 0, attempt = 0;
    double dphi_a = 0.0, dval = 0.0;
    trial_ctx tc = {pb, U, V, u, v, p, gbar, M.mass, 0.0, A, B, trial_u, trial_v, &T, res};
    while (!accepted && attempt < 2) {
      tc.pr = dot(p, r, n) + dot(p + n, c, n);   /* <p_u,r> + <p_v,c> */
      int tr_n = 0;
      st = orc_line_search(pncg_trial, &tc, dphi0, alpha, c1, c2, dec_tol, max_trials, &alpha, &dphi_a, &dval,
                           &tr_n, &accepted);
      trials += tr_n;
      if (accepted || st != ORC_OK) break;
      /* Z10: restart along -s with a fresh bracket */
      attempt++;
      res->ls_restarts++;
      for (int64_t q = 0; q < n2; ++q) p[q] = -dir[q];
      dphi0 = dot(p, g, n2);
      alpha = 1.0;
      reset = 1;
    }
    if (st != ORC_OK) break;
    if (!accepted) { st = ORC_ELINESEARCH; break; }
    if (tr && *tlen < cap) {
      orc_trace_rec* q = &tr[(*tlen)++];
      q->t = t; q->k = (int32_t)k; q->l1 = l1; q->rho = rho; q->alpha = alpha;
      q->dphi0 = dphi0; q->dphi_alpha = dphi_a; q->dphi_value = dval;
      q->trials = trials; q->reset = reset; q->beta = reset ? 0.0 : beta;
      q->gs = rc_dot_prev;
    }
    /* accept: u += alpha p_u, v += alpha p_v (Alg. 2 line 11); the accepted
     * trial's marginals are those of the new iterate (lines 12-13). */
    for (int64_t i = 0; i < n; ++i) u[i] = trial_u[i];
    for (int64_t j = 0; j < n; ++j) v[j] = trial_v[j];
    { marg_t tmp = M; M = T; T = tmp; }
    memcpy(gprev, g, sizeof(double) * n2);
    memcpy(pprev, p, sizeof(double) * n2);
    memcpy(sprev, s, sizeof(double) * n2);
    alpha_prev = alpha;
    res->iterations++;
    if (t >= 1 && t <= 64) res->iters_step[t - 1]++;
    l1 = l1_err(&M, r, c, n);
    rho = rho_err(&M, r, c, n);
  }
  res->l1_final = l1;
  res->rho_final = rho;
  free(sprev);
  free(buf);
  return st;
}

int orc_project(const orc_problem* pb, const double* U, const double* V, double gbar,
                double* u, double* v, const orc_options* opt, int32_t t,
                orc_result* res, orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len) {
#ifdef _OPENMP
  if (opt->max_threads > 0) omp_set_num_threads(opt->max_threads);
#endif
  int64_t dummy = 0;
  if (!trace_len) trace_len = &dummy;
  if (opt->projector == ORC_SINKHORN)
    return sinkhorn_project(pb, U, V, gbar, u, v, opt, t, res, trace, trace_cap, trace_len);
  return pncg_project(pb, U, V, gbar, u, v, opt, t, res, trace, trace_cap, trace_len);
}

/* ------------------------------------------------------------------ */
/* Rounding ("rounded onto U(r,c) via Alg. 2 of Altschuler et
 * al."; procedure as restated in SPEC.md:331):
 *   x = min(r / r(F), 1); F' = D(x) F; y = min(c / c(F'), 1); F'' = F' D(y)
 *   err_r = r - r(F''); err_c = c - c(F''); G = F'' + err_r err_c^T / |err_r|_1
 * Entries of F are recomputed on the fly as exp(U_i + V_j - gbar C_ij). The
 * rank-1 term is skipped when |err_r|_1 < 1e-300 (Z18).                    */
int orc_round(const orc_problem* pb, const double* U, const double* V, double gbar,
              double* cost_F, double* cost_G, double* G_out, double* rG, double* cG) {
  const int64_t n = pb->n;
  const double *r = pb->r, *c = pb->c;
  double* buf = (double*)calloc(8 * n, sizeof(double));
  double *rF = buf, *x = buf + n, *cF1 = buf + 2 * n, *y = buf + 3 * n;
  double *rF2 = buf + 4 * n, *cF2 = buf + 5 * n, *er = buf + 6 * n, *ec = buf + 7 * n;
  double costF = 0.0;
  /* r(F) and <C,F> */
#pragma omp parallel for schedule(static) reduction(+ : costF)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0, cs = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double cij = orc_cost(pb, i, j);
      double f = exp((U[i] + V[j]) - gbar * cij);
      s += f;
      cs += cij * f;
    }
    rF[i] = s;
    costF += cs;
  }
  for (int64_t i = 0; i < n; ++i) x[i] = fmin(r[i] / rF[i], 1.0);
  /* c(F') with F' = D(x) F */
  const int64_t JB = 64;
#pragma omp parallel for schedule(static)
  for (int64_t j0 = 0; j0 < n; j0 += JB) {
    int64_t j1 = j0 + JB < n ? j0 + JB : n;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = j0; j < j1; ++j)
        cF1[j] += x[i] * exp((U[i] + V[j]) - gbar * orc_cost(pb, i, j));
  }
  for (int64_t j = 0; j < n; ++j) y[j] = fmin(c[j] / cF1[j], 1.0);
  /* r(F''), c(F''), <C,F''> */
  double costF2 = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : costF2)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0, cs = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double cij = orc_cost(pb, i, j);
      double f2 = x[i] * exp((U[i] + V[j]) - gbar * cij) * y[j];
      s += f2;
      cs += cij * f2;
    }
    rF2[i] = s;
    costF2 += cs;
  }
#pragma omp parallel for schedule(static)
  for (int64_t j0 = 0; j0 < n; j0 += JB) {
    int64_t j1 = j0 + JB < n ? j0 + JB : n;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = j0; j < j1; ++j)
        cF2[j] += x[i] * exp((U[i] + V[j]) - gbar * orc_cost(pb, i, j)) * y[j];
  }
  double ner = 0.0;
  for (int64_t i = 0; i < n; ++i) { er[i] = r[i] - rF2[i]; ner += fabs(er[i]); }
  for (int64_t j = 0; j < n; ++j) ec[j] = c[j] - cF2[j];
  /* <C, err_r err_c^T> / |err_r|_1 */
  double corr = 0.0;
  if (ner >= 1e-300) {
#pragma omp parallel for schedule(static) reduction(+ : corr)
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < n; ++j) s += orc_cost(pb, i, j) * ec[j];
      corr += er[i] * s;
    }
    corr /= ner;
  }
  if (cost_F) *cost_F = costF;
  if (cost_G) *cost_G = costF2 + corr;
  if (G_out || rG || cG) {
    if (rG) memset(rG, 0, sizeof(double) * n);
    if (cG) memset(cG, 0, sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        double gij = x[i] * exp((U[i] + V[j]) - gbar * orc_cost(pb, i, j)) * y[j];
        if (ner >= 1e-300) gij += er[i] * ec[j] / ner;
        if (G_out) G_out[i * n + j] = gij;
        if (rG) rG[i] += gij;
        if (cG) cG[j] += gij;
      }
  }
  free(buf);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Schedules.  Paper MNIST rule gamma_t = gbar / max(1, floor(gbar/256))
 * (PAPER.md:356, 362); fixed rate gamma_t = gbar/T;
 * doubling (BASELINE config 1, Z13): cumulative gbar_t = gamma0 * 2^(t-1).  */
int orc_schedule_fixed(double gamma_bar, double step_max, int32_t T, double* out, int32_t cap) {
  if (T <= 0) {
    double q = floor(gamma_bar / step_max);
    T = (int32_t)(q > 1.0 ? q : 1.0);
  }
  if (T > cap) return -1;
  for (int32_t t = 0; t < T; ++t) out[t] = gamma_bar / T;
  return T;
}

int orc_schedule_doubling(double gamma_bar, double gamma0, double* out, int32_t cap) {
  int32_t T = 0;
  double gb = 0.0;
  while (gb < gamma_bar * (1.0 - 1e-12)) {
    double next = (T == 0) ? gamma0 : gb;   /* gamma_1 = gamma0, gamma_t = gbar_{t-1} */
    if (gb + next > gamma_bar * (1.0 + 1e-12)) next = gamma_bar - gb;
    if (T >= cap) return -1;
    out[T++] = next;
    gb += next;
  }
  return T;
}

/* eps = min(1e-5, 1e-5 (H_min / gbar)^2), PAPER.md:356 (used on rho). */
double orc_default_eps(double hmin, double gamma_bar) {
  double e = 1e-5 * (hmin / gamma_bar) * (hmin / gamma_bar);
  return e < 1e-5 ? e : 1e-5;
}

/* ------------------------------------------------------------------ */
/* sum_ij C_ij exp(A_i + B_j - gbar C_ij) in index order per row. */
double orc_plan_cost(const orc_problem* pb, const double* A, const double* B, double gbar) {
  const int64_t n = pb->n;
  double* rowc = (double*)malloc(sizeof(double) * n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double cs = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double cij = orc_cost(pb, i, j);
      cs += cij * exp((A[i] + B[j]) - gbar * cij);
    }
    rowc[i] = cs;
  }
  const double tot = sum(rowc, n);
  free(rowc);
  return tot;
}

/* ------------------------------------------------------------------ */
/* MDOT, Alg. 1.
 *   P^0 = r c^T (PAPER.md:203 (i)) -> U = log r, V = log c;  u = v = 0.
 *   step t: gbar += gamma_t; P_hat^t = P^{t-1} exp(-gamma_t C), i.e. the plan
 *   exp(U + V - gbar C); warm start: the previous step's potentials are
 *   carried over (Z4), scaled by gamma_t/gamma_{t-1};
 *   project; U += u, V += v.  Gauge (u+d, v-d) is free: after
 *   each step U, V and u, v are re-centred so that <r,.> = <c,.> (Z19).
 * `adaptive` selects the step rule of orc_mdot_adaptive (Z29) instead of the
 * given schedule.                                                            */
static int mdot_run(const orc_problem* pb, const double* gammas, int32_t T, int adaptive, double gamma_bar,
                    double gamma1, const orc_options* opt, double* U, double* V, orc_result* res,
                    double* gammas_out, orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len) {
  const int64_t n = pb->n;
  const double *r = pb->r, *c = pb->c;
  memset(res, 0, sizeof(*res));
  if (n < 1 || (!adaptive && T < 1) || (adaptive && !(gamma_bar > 0 && gamma1 > 0)) || !(opt->eps > 0)) {
    res->status = ORC_EINVAL;
    return ORC_EINVAL;
  }
  double t0 = now_s();
  double* u = (double*)calloc(n, sizeof(double));
  double* v = (double*)calloc(n, sizeof(double));
  for (int64_t i = 0; i < n; ++i) U[i] = opt->p0_ones ? 0.0 : log(r[i]);
  for (int64_t j = 0; j < n; ++j) V[j] = opt->p0_ones ? 0.0 : log(c[j]);
  int64_t dummy = 0;
  if (!trace_len) trace_len = &dummy;
  *trace_len = 0;
  double gbar = 0.0, gprev = 0.0;
  double next = adaptive ? fmin(gamma1, gamma_bar) : 0.0, eta_prev = 0.0;
  int final_next = adaptive && gamma1 >= gamma_bar;
  int st = ORC_OK;
  for (int32_t t = 1; adaptive || t <= T; ++t) {
    double gt = adaptive ? next : gammas[t - 1];
    const int last = adaptive ? final_next : (t == T);
    gbar = (adaptive && last) ? gamma_bar : gbar + gt;   /* the last adaptive step lands on gamma_bar exactly */
    if (gammas_out && t <= 64) gammas_out[t - 1] = gt;
    if (opt->warm == ORC_WARM_ZERO) {
      memset(u, 0, sizeof(double) * n);
      memset(v, 0, sizeof(double) * n);
    } else if (opt->warm == ORC_WARM_SCALED && t > 1) {
      double w = gt / gprev;
      for (int64_t i = 0; i < n; ++i) u[i] *= w;
      for (int64_t j = 0; j < n; ++j) v[j] *= w;
    }
    orc_options ot = *opt;
    if (!last && opt->eps_md > opt->eps) ot.eps = opt->eps_md;
    const int64_t evals_before = res->evaluations;
    st = orc_project(pb, U, V, gbar, u, v, &ot, t, res, trace, trace_cap, trace_len);
    res->md_steps = t;
    for (int64_t i = 0; i < n; ++i) U[i] += u[i];
    for (int64_t j = 0; j < n; ++j) V[j] += v[j];
    double d1 = 0.5 * (dot(r, U, n) - dot(c, V, n));
    for (int64_t i = 0; i < n; ++i) U[i] -= d1;
    for (int64_t j = 0; j < n; ++j) V[j] += d1;
    double d2 = 0.5 * (dot(r, u, n) - dot(c, v, n));
    for (int64_t i = 0; i < n; ++i) u[i] -= d2;
    for (int64_t j = 0; j < n; ++j) v[j] += d2;
    gprev = gt;
    if (st != ORC_OK || (adaptive && last)) break;
    if (adaptive) {
      /* Z29: eta_t = gamma_t / E_t; double while eta does not fall, else halve */
      const double E = (double)(res->evaluations - evals_before);
      const double eta = gt / (E > 1.0 ? E : 1.0);
      double g = (t == 1 || eta >= eta_prev) ? 2.0 * gt : fmax(0.5 * gt, gamma_bar / 1024.0);
      eta_prev = eta;
      const double rem = gamma_bar - gbar;
      if (g >= rem || rem - g < 0.25 * g || t + 1 >= 64) { g = rem; final_next = 1; }
      next = g;
    }
  }
  res->gamma_bar = gbar;
  if (st == ORC_OK || st == ORC_ENOCONV)
    orc_round(pb, U, V, gbar, &res->cost_unrounded, &res->cost_rounded, NULL, NULL, NULL);
  res->seconds = now_s() - t0;
  res->status = st;
  free(u);
  free(v);
  return st;
}

int orc_mdot(const orc_problem* pb, const double* gammas, int32_t T, const orc_options* opt,
             double* U, double* V, orc_result* res,
             orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len) {
  return mdot_run(pb, gammas, T, 0, 0.0, 0.0, opt, U, V, res, NULL, trace, trace_cap, trace_len);
}

int orc_mdot_adaptive(const orc_problem* pb, double gamma_bar, double gamma1, const orc_options* opt,
                      double* U, double* V, orc_result* res, double* gammas_out,
                      orc_trace_rec* trace, int64_t trace_cap, int64_t* trace_len) {
  return mdot_run(pb, NULL, 0, 1, gamma_bar, gamma1, opt, U, V, res, gammas_out, trace, trace_cap, trace_len);
}

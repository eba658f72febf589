// paper_2307_08507_b200/csrc/ops.cuh -- device functions shared by the
// standalone loop kernels (kernels.cu) and the persistent cooperative slot
// kernel (persist.cu): log-sum-exp merge, exponent split, the per-item prep
// and finalize steps, and the PNCG / Sinkhorn controller.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.cuh"

namespace mdot {

#ifndef MDOT_L2E_LN2
#define MDOT_L2E_LN2
#define L2E_D 1.4426950408889634
#define LN2_D 0.6931471805599453
#endif

__device__ __forceinline__ void lse_push(double& m, double& s, double z) {
  if (z <= m) {
    s += exp(z - m);
  } else {
    s = s * exp(m - z) + 1.0;
    m = z;
  }
}

__device__ __forceinline__ void lse_merge(double& m, double& s, double m2, double s2) {
  if (s2 == 0.0) return;
  if (s == 0.0) { m = m2; s = s2; return; }
  if (m2 <= m) {
    s += s2 * exp(m2 - m);
  } else {
    s = s * exp(m - m2) + s2;
    m = m2;
  }
}

// fp32-entry parameter slot {ah, M = 2^al, S' = 2^anchor * M, 0} (DESIGN.md
// "K1 numerics"): a2 = base log2(e) - anchor = ah + al with ah on a 2^-8 grid
// (|ah| < 2^15, so ah_i + bh_j is exact in fp32) and |al| <= 2^-9.  The lo
// part leaves the exponent: the kernels exponentiate ah + bh - g2 C only and
// carry 2^al_i / 2^bl_j as the multipliers M (applied to the row / column
// totals) and S' / T' (the cross weights), so the entry costs 1 FADD + 2
// FFMA + 1 MUFU + 2 FFMA.  M is fp32-rounded once (<= 2^-24 relative);
// S' = 2^anchor * M is exact.
__device__ __forceinline__ float4 split_param(double base, double anchor, int* flag) {
  const double a2 = base * L2E_D - anchor;
  const double ah = rint(a2 * 256.0) * (1.0 / 256.0);
  if (!(fabs(ah) < 32768.0)) {
    if (flag) *flag = 1;
  }
  const double al = a2 - ah;
  const float M = (float)exp2(al);
  // integer anchors (k_setup rounds them): exp2(anchor) * M == ldexp(M, anchor) exactly
  const double S = (anchor == rint(anchor)) ? ldexp((double)M, (int)anchor) : exp2(anchor) * (double)M;
  return make_float4((float)ah, M, (float)S, 0.f);
}

__device__ __forceinline__ float screen_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// fp64-entry parameter slot: {base potential (fp64), 2^anchor (fp32), anchor (fp32)}
__device__ __forceinline__ float4 f64_param(double base, double anchor) {
  float4 r;
  *reinterpret_cast<double*>(&r.x) = base;
  r.z = (float)((anchor == rint(anchor)) ? ldexp(1.0, (int)anchor) : exp2(anchor));
  r.w = (float)anchor;
  return r;
}

// One row/column item of the prep step (k in [0, nrows + n)); the controller
// state `c` (device control) overrides mode / alpha / beta and requests the
// element-wise accept copy.
// Returns this item's potential shift against the accepted iterate (K2s
// screen operands, a.sopA set) or +inf.
__device__ __forceinline__ double prep_item(const PrepArgs& a, int64_t k, const CtrlState* c) {
  MDOT_DCHECK(k >= 0 && k < a.nrows + a.n);
  const bool is_row = k < a.nrows;
  const int64_t idx = is_row ? k : k - a.nrows;
  int mode = a.mode;
  double alpha = a.alpha, beta = a.beta;
  const double* sdir = a.s;
  if (c) {
    // accepted trial becomes the iterate (Alg. 2 lines 11-13): element-wise copy
    if (c->accept_marg) {
      a.cur_lm[k] = a.tr_lm[k];
      if (a.cur_m) a.cur_m[k] = a.tr_m[k];
      a.cur_s[k] = a.tr_s[k];
      a.cur_g[k] = a.tr_g[k];
      if (a.cur_bp) a.cur_bp[k] = a.tr_bp[k];
    }
    if (c->accept_pot) {
      a.pprev[k] = a.p[k];
      if (is_row) a.u[idx] = a.tu[idx];
      else a.v[idx] = a.tv[idx];
    }
    if (c->done) return INFINITY;
    mode = c->mode;
    alpha = c->alpha;
    beta = c->beta;
    sdir = c->ncg ? a.cur_g : a.cur_s;
  }
  double pk = 0.0;
  if (mode & PREP_NEWDIR) {
    pk = -sdir[k] + (beta != 0.0 ? beta * a.pprev[k] : 0.0);
    a.p[k] = pk;
  } else if (mode & PREP_TRIAL) {
    pk = a.p[k];
  }
  double base;
  if (is_row) {
    if (mode & PREP_TRIAL) {
      const double t = a.u[idx] + alpha * pk;
      a.tu[idx] = t;
      base = a.U[idx] + t;
    } else if (mode & PREP_SK_ROW) {
      const double t = a.u[idx] + (a.logr[idx] - a.lm[k]);
      a.u[idx] = t;
      base = a.U[idx] + t;
    } else if (mode & PREP_AB) {
      base = a.Ain[idx];
    } else {
      base = a.U[idx] + a.u[idx];
    }
    if (a.Aout) a.Aout[idx] = base;
    if (a.f64_params) {
      a.rowp[idx] = f64_param(base, a.rho_r[idx]);
    } else {
      float4 q = split_param(base, a.rho_r[idx], a.flag);
      if (a.nrm) q.w = a.nrm[idx];
      a.rowp[idx] = q;
    }
  } else {
    if (mode & PREP_TRIAL) {
      const double t = a.v[idx] + alpha * pk;
      a.tv[idx] = t;
      base = a.V[idx] + t;
    } else if (mode & PREP_SK_COL) {
      const double t = a.v[idx] + (a.logc[idx] - a.lm[k]);
      a.v[idx] = t;
      base = a.V[idx] + t;
    } else if (mode & PREP_AB) {
      base = a.Bin[idx];
    } else {
      base = a.V[idx] + a.v[idx];
    }
    if (a.Bout) a.Bout[idx] = base;
    if (a.f64_params) {
      a.colp[idx] = f64_param(base, a.sig_c[idx]);
    } else {
      float4 q = split_param(base, a.sig_c[idx], a.flag);
      if (a.nrm) q.w = a.nrm[a.nrows + idx];
      a.colp[idx] = q;
    }
  }
  if (!a.sopA) return INFINITY;
  // K2s (screen.cu): the marginal at the new potentials is at least the
  // accepted iterate's times e^(this shift + the other side's smallest
  // shift); the latter is a grid-wide minimum, folded in by the kernel
  // (every rounding explicit: the screen's decisions, and so the kept set,
  // must not depend on the compiler's contraction choices -- checked and
  // release builds give identical bits)
  double dlt = __dsub_rn(base, a.cur_bp[k]);
  if (!(dlt == dlt)) dlt = -INFINITY;
  a.tr_bp[k] = base;
  double sl = __dmul_rn(__dadd_rn(a.cur_lm[k], dlt), L2E_D);   // log2 of the predicted marginal, own shift only
  if (!(sl == sl)) sl = -INFINITY;
  const double mlog = -log2((double)a.n);
  const double g = __dmul_rn(__dadd_rn((double)c->gpair[0], (double)c->gpair[1]), (double)a.scale);
  const float4 q = is_row ? a.rowp[idx] : a.colp[idx];
  const float* P = (is_row ? a.X : a.Y) + idx * a.d;
  float v[32];
  double nrm2 = 0.0;
  const float tg = is_row ? (float)__dmul_rn(2.0, g) : 1.f;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const float x = t < a.d ? P[t] : 0.f;
    nrm2 = __fma_rn((double)x, (double)x, nrm2);
    v[t] = screen_tf32(__fmul_rn(tg, x));
  }
  double w = __dsub_rn(__dsub_rn(__dadd_rn((double)q.x, log2((double)q.z)), __dmul_rn(g, nrm2)), fmin(sl, mlog));
  if (is_row) {
    const double delta = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, g), sqrt(nrm2)), __dmul_rn(*a.sop_ymax, 1.001 / 1024.0)), 2.0);
    w = __dadd_rn(w, __dadd_rn(__dadd_rn(mlog, (double)a.screen_T), delta));
  }
  if (!(w < 1.0e30)) w = 1.0e30;   // +inf / NaN: keep the whole row / column
  const float wh = screen_tf32((float)w), wl = screen_tf32((float)__dsub_rn(w, (double)wh));
  if (is_row) {   // chunk 4 {alpha_hi, alpha_lo, 1, 1}, chunk 5 {1, 1, 0, 0}
    v[16] = wh; v[17] = wl; v[18] = 1.f; v[19] = 1.f; v[20] = 1.f; v[21] = 1.f;
  } else {        // chunk 4 {1, 1, beta_hi, beta_lo}, chunk 5 {-G_hi, -G_lo, 0, 0} (G: per CTA)
    v[16] = 1.f; v[17] = 1.f; v[18] = wh; v[19] = wl; v[20] = 0.f; v[21] = 0.f;
  }
#pragma unroll
  for (int t = 22; t < 32; ++t) v[t] = 0.f;
  sop_store((is_row ? a.sopA : a.sopB) + idx * 32, idx, v);
  return dlt;
}

// Fault injection for the error-path tests (MDOT_FAULT_NAN, solver.cu):
// 1 = the total of item 0 in the first fp32-entry evaluation becomes NaN
//     (the range guard must redo that evaluation exactly, the solve go on);
// 2 = item 0's log marginal is NaN in every evaluation, exact ones included
//     (the call must end with MDOT_EINSTABLE, not hang or return garbage).
// `static` in a header: every translation unit has its own copy, set by its
// own fault_set_* (no relocatable device code).
static __constant__ int c_fault_nan = 0;
static __device__ unsigned int g_fault_hits = 0;
static inline void fault_set_tu(int mode) {
  unsigned int z = 0;
  cudaMemcpyToSymbol(c_fault_nan, &mode, sizeof(int));
  cudaMemcpyToSymbol(g_fault_hits, &z, sizeof(z));
}

// 8 threads per item: the partial sums are split over the octet (t = lane%8,
// t+8, ...) in a fixed order and combined by a fixed shuffle tree, so every
// partial load of an item is in flight at once.
constexpr int kFinTPI = 8;
__device__ __forceinline__ double octet_partial(const double* x, int64_t stride, int cnt, int sub) {
  double acc = 0.0;
  int t = sub;
  for (; t + 3 * kFinTPI < cnt; t += 4 * kFinTPI) {
    const double v0 = x[(int64_t)t * stride], v1 = x[(int64_t)(t + kFinTPI) * stride];
    const double v2 = x[(int64_t)(t + 2 * kFinTPI) * stride], v3 = x[(int64_t)(t + 3 * kFinTPI) * stride];
    acc += v0; acc += v1; acc += v2; acc += v3;
  }
  for (; t < cnt; t += kFinTPI) acc += x[(int64_t)t * stride];
  return acc;
}

// Per-item finalize (row or column item k, marginal total `tot` in anchored
// units or, for the exact path, taken from lr_in / column (max, sum) chunks):
// log marginal, marginal, Sinkhorn direction s, gradient
// (PAPER.md:236-239), and this item's contributions to the 16 scalars.
__device__ __forceinline__ void finalize_item(const FinalizeArgs& a, int64_t k, double tot,
                                              double (&v)[kNumScalars]) {
  MDOT_DCHECK(k >= 0 && k < a.nrows + a.n);
  const bool is_row = k < a.nrows;
    double lm, bad = 0.0;
    if (c_fault_nan == 1 && k == 0 && a.from_partials == 1 &&
        atomicAdd(&g_fault_hits, 1u) < (unsigned)(a.fault_repl > 1 ? a.fault_repl : 1))
      tot = __longlong_as_double(0x7ff8000000000000ll);
    if (a.from_partials == 1) {
      const double anchor = is_row ? a.rho_r[k] : a.sig_c[k - a.nrows];
      lm = log(tot) + anchor * LN2_D;
      // fp32 entry range guard (K1 numerics): totals far from 1 in
      // anchored units mean under/overflowed entries -> exact re-evaluation
      if (a.f64_entries ? !(tot > fmax(a.f64_tot_min, 1e-300) && tot < 1e300)
                        : !(tot > 7.888609052210118e-31 && tot < 1.2676506002282294e30)) bad = 1.0;
    } else {
      if (is_row) {
        lm = a.lr_in[k];
      } else {
        const int64_t j = k - a.nrows;
        double m = -INFINITY, s = 0.0;
        for (int c = 0; c < a.chunks; ++c)
          lse_merge(m, s, a.colm[(int64_t)c * a.n + j], a.cols[(int64_t)c * a.n + j]);
        lm = m + log(s);
      }
      if (!isfinite(lm)) bad = 1.0;
    }
    if (c_fault_nan == 2 && k == 0) { lm = __longlong_as_double(0x7ff8000000000000ll); bad = 1.0; }
    const double tgt = is_row ? a.r[k] : a.c[k - a.nrows];
    const double ltg = is_row ? a.logr[k] : a.logc[k - a.nrows];
    const double mm = exp(lm);
    const double g = mm - tgt;
    const double lrat = lm - ltg;
    // preconditioned direction: the Sinkhorn direction log(m / target)
    // or, for the Jacobi ablation, g / diag(Hessian) with
    // the diagonal bounded below by the target: g / max(m, target)
    const double s = a.jacobi ? g / fmax(mm, tgt) : lrat;
    a.lm[k] = lm;
    if (a.m) a.m[k] = mm;
    a.s[k] = s;
    a.g[k] = g;
    const double gc = a.gcur ? a.gcur[k] : 0.0;
    const double pc = a.pcur ? a.pcur[k] : 0.0;
    if (is_row) v[SC_MASS] += mm;   // static indices only: v stays in registers
    else v[SC_MASSC] += mm;
    v[SC_L1] += fabs(g);
    v[SC_RHO] += tgt - mm + mm * lrat;         // D_h(y|x) term with y = m, x = tgt (Z1)
    v[SC_SG] += s * g;
    v[SC_GCS] += gc * s;
    v[SC_PCG] += pc * g;
    v[SC_PRC] += pc * tgt;
    v[SC_GG] += g * g;
    v[SC_GCG] += gc * g;
    v[SC_BAD] += bad;
    v[SC_L1R] += is_row ? fabs(g) : 0.0;
    if (a.prep_flag && k == a.item_begin) {
      v[SC_BAD] += (double)(*a.prep_flag);
      *a.prep_flag = 0;
    }
}

// ---------------------------------------------------------------------------
// Controller (single thread), mirrors project_pncg / project_sinkhorn in
// solver.cu step by step.
// ---------------------------------------------------------------------------
__device__ inline void ctrl_finish(CtrlState* st, int status, int* done_host) {
  st->done = 1;
  st->status = status;
  if (done_host) *((volatile int*)done_host) = 1;
}

__device__ inline void ctrl_trace(CtrlState* st, double alpha, double dphi_a, double dval) {
  if (!st->trace || *st->trace_len >= st->trace_cap) return;
  MDOT_DCHECK(*st->trace_len >= 0);
  mdot_trace_rec& q = st->trace[*st->trace_len];
  q.t = st->md_t; q.k = (int32_t)st->k;
  q.l1 = st->l1; q.rho = st->rho;
  q.alpha = alpha; q.dphi0 = st->sinkhorn ? 0.0 : st->dphi0; q.dphi_alpha = dphi_a; q.dphi_value = dval;
  q.trials = st->sinkhorn ? 0 : st->trials; q.reset = st->sinkhorn ? 0 : st->reset_flag;
  q.beta = st->sinkhorn ? 0.0 : st->beta; q.gs = st->sinkhorn ? 0.0 : st->S_sg;
  *st->trace_len += 1;
}

__device__ inline void ctrl_start_iteration(CtrlState* st) {
  st->k++;
  double beta = 0.0;
  if (st->k > 1)
    beta = beta_k(st->ncg, st->beta_kind, st->S_sg, st->S_gcs, st->S_gg, st->S_gcg, st->dphi0_prev, st->sg_prev,
                  st->gg_prev);
  const double dg = st->ncg ? st->S_gg : st->S_sg;
  double dphi0 = -dg + beta * st->S_pcg;
  st->reset_flag = 0;
  if (!(dphi0 < 0.0)) { beta = 0.0; dphi0 = -dg; st->resets++; st->reset_flag = 1; }   // Z5
  st->dg = dg;
  st->dphi0 = dphi0;
  st->beta = beta;
  st->alpha = (st->k == 1) ? 1.0 : fmin(4.0, fmax(0.25, st->alpha_prev));   // Z8
  st->lo = 0.0; st->dlo = dphi0; st->hi = 0.0; st->dhi = 0.0;
  st->have_hi = 0; st->doublings = 0; st->trials = 0; st->attempt = 0;
  st->mode = PREP_NEWDIR | PREP_TRIAL;
}

__device__ inline void ctrl_body(CtrlState* st, int slot, int* done_host, int* ran_host) {
  if (st->done) { if (ran_host) ran_host[slot] = 0; return; }
  st->accept_marg = 0;
  st->accept_pot = 0;
  const double* sc = st->sc;
  const bool bad = sc[SC_BAD] != 0.0;
  st->evals++;
  if (st->phase == 0) {   // initial evaluation of the projection
    if (bad) { ctrl_finish(st, CTRL_NEED_HOST, done_host); if (ran_host) ran_host[slot] = 0; return; }
    st->accept_marg = 1;
    st->l1 = sc[SC_L1]; st->rho = sc[SC_RHO]; st->l1_0 = st->l1; st->rho_0 = st->rho;
    st->mass = sc[SC_MASS];
    st->S_sg = sc[SC_SG]; st->S_gg = sc[SC_GG];
    st->S_gcs = 0.0; st->S_pcg = 0.0; st->S_gcg = 0.0;
    st->phase = 1;
    const double sv = st->stop_rho ? st->rho : st->l1;
    if (sv <= st->eps) { ctrl_finish(st, CTRL_OK, done_host); if (ran_host) ran_host[slot] = 0; return; }
    if (st->evals >= st->max_evals) { ctrl_finish(st, CTRL_NOCONV, done_host); if (ran_host) ran_host[slot] = 0; return; }
    if (st->sinkhorn) { st->k = 1; st->mode = PREP_SK_ROW; }
    else ctrl_start_iteration(st);
    if (ran_host) ran_host[slot] = 1;
    return;
  }
  if (st->sinkhorn) {   // Alg. 3 half-step result
    if (bad) { ctrl_finish(st, CTRL_NEED_HOST, done_host); if (ran_host) ran_host[slot] = 0; return; }
    ctrl_trace(st, 1.0, 0.0, 0.0);
    st->accept_marg = 1;
    st->iterations++;
    st->l1 = sc[SC_L1]; st->rho = sc[SC_RHO]; st->mass = sc[SC_MASS];
    const double sv = st->stop_rho ? st->rho : st->l1;
    if (sv <= st->eps) { ctrl_finish(st, CTRL_OK, done_host); if (ran_host) ran_host[slot] = 0; return; }
    if (st->evals >= st->max_evals) { ctrl_finish(st, CTRL_NOCONV, done_host); if (ran_host) ran_host[slot] = 0; return; }
    st->k++;
    st->mode = (st->k % 2 == 1) ? PREP_SK_ROW : PREP_SK_COL;
    if (ran_host) ran_host[slot] = 1;
    return;
  }
  // PNCG line-search trial result (Appx. C; Z7, Z9)
  st->ls_evals++;
  st->trials++;
  const double dphi_a = bad ? INFINITY : sc[SC_PCG];
  const double dval = bad ? INFINITY : (sc[SC_MASS] - st->mass) - st->alpha * sc[SC_PRC];
  const bool wolfe = ((2.0 * st->c1 - 1.0) * st->dphi0 >= dphi_a) && (dphi_a >= st->c2 * st->dphi0);
  const bool decrease = dval <= st->noise * fmax(1.0, st->mass);
  if (!bad && wolfe && decrease) {
    ctrl_trace(st, st->alpha, dphi_a, dval);
    st->accept_marg = 1;
    st->accept_pot = 1;
    st->iterations++;
    st->dphi0_prev = st->dphi0;
    st->sg_prev = st->S_sg;
    st->gg_prev = st->S_gg;
    st->S_sg = sc[SC_SG]; st->S_gcs = sc[SC_GCS]; st->S_pcg = sc[SC_PCG];
    st->S_gg = sc[SC_GG]; st->S_gcg = sc[SC_GCG];
    st->mass = sc[SC_MASS]; st->l1 = sc[SC_L1]; st->rho = sc[SC_RHO];
    st->alpha_prev = st->alpha;
    const double sv = st->stop_rho ? st->rho : st->l1;
    if (sv <= st->eps) { ctrl_finish(st, CTRL_OK, done_host); if (ran_host) ran_host[slot] = 0; return; }
    if (st->evals >= st->max_evals) { ctrl_finish(st, CTRL_NOCONV, done_host); if (ran_host) ran_host[slot] = 0; return; }
    ctrl_start_iteration(st);
    if (ran_host) ran_host[slot] = 1;
    return;
  }
  if (dphi_a < 0.0 && decrease) { st->lo = st->alpha; st->dlo = dphi_a; }
  else { st->hi = st->alpha; st->dhi = dphi_a; st->have_hi = 1; }
  bool fail = false;
  if (!st->have_hi) {
    if (++st->doublings > 60) fail = true;
    else st->alpha *= 2.0;
  } else if (st->dhi > st->dlo && isfinite(st->dhi)) {
    const double a_sec = (st->lo * st->dhi - st->hi * st->dlo) / (st->dhi - st->dlo);
    st->alpha = 0.5 * a_sec + 0.5 * (st->hi + st->lo) / 2.0;
  } else {
    st->alpha = 0.5 * (st->lo + st->hi);
  }
  if (st->trials >= st->ls_max_trials) fail = true;
  if (fail) {   // Z10
    st->attempt++;
    st->restarts++;
    if (st->attempt >= 2) { ctrl_finish(st, CTRL_LS_FAIL, done_host); if (ran_host) ran_host[slot] = 0; return; }
    st->dphi0 = -st->dg;
    st->alpha = 1.0;
    st->beta = 0.0;
    st->reset_flag = 1;
    st->lo = 0.0; st->dlo = st->dphi0; st->hi = 0.0; st->dhi = 0.0;
    st->have_hi = 0; st->doublings = 0; st->trials = 0;
    st->mode = PREP_NEWDIR | PREP_TRIAL;
  } else {
    st->mode = PREP_TRIAL;
  }
  if (ran_host) ran_host[slot] = 1;
}


}  // namespace mdot

"""fp64 CPU oracle of the MDOT-PNCG hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  The product package
(paper_2307_08507_b200) never imports it and shares no code with it.

ctypes wrapper around oracle/mdot_oracle.c (plain C, fp64, OpenMP over
independent rows/columns).  See the C header for the paper citations.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "mdot_oracle.c")

DENSE_F32, SQEUCLID_F32, DENSE_F64, SQEUCLID_DOT_F32 = 0, 1, 2, 3
PNCG, SINKHORN, NCG, PNCG_JACOBI = 0, 1, 2, 3
BETA_PPR, BETA_PPR_AF, BETA_PFR, BETA_PPR_PRINTED, BETA_PPR_PLUS = 0, 1, 2, 3, 4
WARM_SCALED, WARM_CARRY, WARM_ZERO = 0, 1, 2
STATUS = {0: "OK", 1: "EINVAL", 3: "EINSTABLE", 4: "ENOCONV", 5: "ELINESEARCH"}


def build(force=False):
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_POSIX_C_SOURCE=199309L", "-fopenmp",
               "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


class Problem(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("kind", ct.c_int32), ("d", ct.c_int32),
                ("C", ct.c_void_p), ("X", ct.c_void_p), ("Y", ct.c_void_p),
                ("scale", ct.c_float), ("r", ct.c_void_p), ("c", ct.c_void_p)]


class Options(ct.Structure):
    _fields_ = [("eps", ct.c_double), ("stop_rho", ct.c_int32), ("projector", ct.c_int32),
                ("beta", ct.c_int32), ("c1", ct.c_double), ("c2", ct.c_double),
                ("warm", ct.c_int32), ("p0_ones", ct.c_int32), ("max_evals", ct.c_int64),
                ("ls_max_trials", ct.c_int32), ("max_threads", ct.c_int32), ("eps_md", ct.c_double)]


class TraceRec(ct.Structure):
    _fields_ = [("t", ct.c_int32), ("k", ct.c_int32), ("l1", ct.c_double), ("rho", ct.c_double),
                ("alpha", ct.c_double), ("dphi0", ct.c_double), ("dphi_alpha", ct.c_double),
                ("dphi_value", ct.c_double), ("trials", ct.c_int32), ("reset", ct.c_int32),
                ("beta", ct.c_double), ("gs", ct.c_double)]


class Result(ct.Structure):
    _fields_ = [("cost_unrounded", ct.c_double), ("cost_rounded", ct.c_double),
                ("l1_final", ct.c_double), ("rho_final", ct.c_double),
                ("gamma_bar", ct.c_double), ("seconds", ct.c_double),
                ("md_steps", ct.c_int64), ("iterations", ct.c_int64),
                ("evaluations", ct.c_int64), ("ls_evaluations", ct.c_int64),
                ("resets", ct.c_int64), ("ls_restarts", ct.c_int64), ("status", ct.c_int32),
                ("rho0", ct.c_double * 64), ("l10", ct.c_double * 64),
                ("iters_step", ct.c_int64 * 64)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("rho0", "l10", "iters_step")}
        T = int(self.md_steps)
        d["rho0"] = list(self.rho0)[:T]
        d["l10"] = list(self.l10)[:T]
        d["iters_step"] = list(self.iters_step)[:T]
        d["status_name"] = STATUS.get(self.status, str(self.status))
        return d


_lib = None
PHI_FN = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_double, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double))


def lib():
    global _lib
    if _lib is None:
        build()
        L = ct.CDLL(_SO)
        P, D = ct.c_void_p, ct.c_double
        L.orc_log_marginals.argtypes = [ct.POINTER(Problem), P, P, D, P, P]
        L.orc_log_marginal_rows.argtypes = [ct.POINTER(Problem), P, P, D, P, ct.c_int64, P]
        L.orc_log_marginal_cols.argtypes = [ct.POINTER(Problem), P, P, D, P, ct.c_int64, P]
        L.orc_cost.argtypes = [ct.POINTER(Problem), ct.c_int64, ct.c_int64]
        L.orc_cost.restype = D
        L.orc_project.argtypes = [ct.POINTER(Problem), P, P, D, P, P, ct.POINTER(Options),
                                  ct.c_int32, ct.POINTER(Result), P, ct.c_int64,
                                  ct.POINTER(ct.c_int64)]
        L.orc_mdot.argtypes = [ct.POINTER(Problem), P, ct.c_int32, ct.POINTER(Options), P, P,
                               ct.POINTER(Result), P, ct.c_int64, ct.POINTER(ct.c_int64)]
        L.orc_round.argtypes = [ct.POINTER(Problem), P, P, D, ct.POINTER(D), ct.POINTER(D), P, P, P]
        L.orc_schedule_fixed.argtypes = [D, D, ct.c_int32, P, ct.c_int32]
        L.orc_schedule_doubling.argtypes = [D, D, P, ct.c_int32]
        L.orc_default_eps.argtypes = [D, D]
        L.orc_default_eps.restype = D
        L.orc_line_search.argtypes = [PHI_FN, P, D, D, D, D, D, ct.c_int, ct.POINTER(D), ct.POINTER(D),
                                      ct.POINTER(D), ct.POINTER(ct.c_int), ct.POINTER(ct.c_int)]
        L.orc_plan_cost.argtypes = [ct.POINTER(Problem), P, P, D]
        L.orc_plan_cost.restype = D
        L.orc_mdot_adaptive.argtypes = [ct.POINTER(Problem), D, D, ct.POINTER(Options), P, P,
                                        ct.POINTER(Result), P, P, ct.c_int64, ct.POINTER(ct.c_int64)]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


class OracleProblem:
    """Holds contiguous arrays alive for the C side."""

    def __init__(self, inst=None, *, C=None, r=None, c=None, X=None, Y=None, scale=0.0, recipe="diff"):
        if inst is not None:
            C, r, c, X, Y, scale = inst.C, inst.r, inst.c, inst.X, inst.Y, inst.scale
            if C is not None:
                X = Y = None
        self.r = np.ascontiguousarray(r, dtype=np.float64)
        self.c = np.ascontiguousarray(c, dtype=np.float64)
        self.n = len(self.r)
        self.C = self.X = self.Y = None
        if C is not None:
            C = np.ascontiguousarray(C)
            if C.dtype == np.float64:
                kind = DENSE_F64
            else:
                C = C.astype(np.float32, copy=False)
                kind = DENSE_F32
            self.C = C
            d = 0
        else:
            self.X = np.ascontiguousarray(X, dtype=np.float32)
            self.Y = np.ascontiguousarray(Y, dtype=np.float32)
            kind = SQEUCLID_DOT_F32 if recipe == "dot" else SQEUCLID_F32   # Z22 / Z22b
            d = self.X.shape[1]
        self.kind = kind
        self.s = Problem(self.n, kind, d, _ptr(self.C), _ptr(self.X), _ptr(self.Y),
                         float(scale), _ptr(self.r), _ptr(self.c))

    def cost(self, i, j):
        return lib().orc_cost(ct.byref(self.s), i, j)


def make_options(eps=1e-6, projector=PNCG, beta=BETA_PPR, c1=0.1, c2=0.4, warm=WARM_SCALED,
                 stop_rho=False, p0_ones=False, max_evals=0, ls_max_trials=0, threads=0, eps_md=0.0):
    return Options(eps, int(stop_rho), projector, beta, c1, c2, warm, int(p0_ones),
                   max_evals, ls_max_trials, threads, eps_md)


def log_marginals(prob: OracleProblem, A, B, gbar):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    lr = np.empty(prob.n)
    lc = np.empty(prob.n)
    st = lib().orc_log_marginals(ct.byref(prob.s), _ptr(A), _ptr(B), float(gbar), _ptr(lr), _ptr(lc))
    return lr, lc, st


def log_marginal_subset(prob: OracleProblem, A, B, gbar, rows=None, cols=None):
    """Oracle log-marginals of selected rows / columns only."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    out = {}
    for name, idx, fn in (("rows", rows, lib().orc_log_marginal_rows),
                          ("cols", cols, lib().orc_log_marginal_cols)):
        if idx is None:
            continue
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        o = np.empty(len(idx))
        fn(ct.byref(prob.s), _ptr(A), _ptr(B), float(gbar), _ptr(idx), len(idx), _ptr(o))
        out[name] = o
    return out


def schedule_fixed(gamma_bar, step_max=256.0, T=0):
    out = np.zeros(4096)
    T = lib().orc_schedule_fixed(float(gamma_bar), float(step_max), int(T), _ptr(out), 4096)
    return out[:T].copy()


def schedule_doubling(gamma_bar, gamma0=1.0):
    out = np.zeros(4096)
    T = lib().orc_schedule_doubling(float(gamma_bar), float(gamma0), _ptr(out), 4096)
    return out[:T].copy()


def default_eps(hmin, gamma_bar):
    return lib().orc_default_eps(float(hmin), float(gamma_bar))


def _trace_buf(cap):
    return (TraceRec * cap)() if cap else None


def _trace_list(buf, ln):
    out = []
    for k in range(ln):
        q = buf[k]
        out.append({f: getattr(q, f) for f, _ in TraceRec._fields_})
    return out


def project(prob: OracleProblem, U, V, gbar, u0=None, v0=None, opts=None, t=1, trace_cap=0):
    n = prob.n
    U = np.ascontiguousarray(U, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    u = np.zeros(n) if u0 is None else np.array(u0, dtype=np.float64)
    v = np.zeros(n) if v0 is None else np.array(v0, dtype=np.float64)
    opts = opts or make_options()
    res = Result()
    tb = _trace_buf(trace_cap)
    tl = ct.c_int64(0)
    st = lib().orc_project(ct.byref(prob.s), _ptr(U), _ptr(V), float(gbar), _ptr(u), _ptr(v),
                           ct.byref(opts), int(t), ct.byref(res),
                           ct.cast(tb, ct.c_void_p) if tb is not None else None,
                           trace_cap, ct.byref(tl))
    res.status = st
    res.md_steps = max(1, t)
    return u, v, res.as_dict(), _trace_list(tb, tl.value) if tb is not None else []


def mdot(prob: OracleProblem, gammas, opts=None, trace_cap=0):
    n = prob.n
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    U = np.empty(n)
    V = np.empty(n)
    opts = opts or make_options()
    res = Result()
    tb = _trace_buf(trace_cap)
    tl = ct.c_int64(0)
    lib().orc_mdot(ct.byref(prob.s), _ptr(g), len(g), ct.byref(opts), _ptr(U), _ptr(V),
                   ct.byref(res), ct.cast(tb, ct.c_void_p) if tb is not None else None,
                   trace_cap, ct.byref(tl))
    return U, V, res.as_dict(), _trace_list(tb, tl.value) if tb is not None else []


def round_plan(prob: OracleProblem, U, V, gbar, dense=False):
    n = prob.n
    U = np.ascontiguousarray(U, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    cF = ct.c_double(0)
    cG = ct.c_double(0)
    G = np.empty((n, n)) if dense else None
    rG = np.empty(n)
    cGm = np.empty(n)
    lib().orc_round(ct.byref(prob.s), _ptr(U), _ptr(V), float(gbar), ct.byref(cF), ct.byref(cG),
                    _ptr(G), _ptr(rG) if dense else None, _ptr(cGm) if dense else None)
    out = {"cost_F": cF.value, "cost_G": cG.value}
    if dense:
        out.update(G=G, rG=rG, cG=cGm)
    return out


def plan(prob: OracleProblem, U, V, gbar):
    """Dense P = exp(U_i + V_j - gbar C_ij) (small n only)."""
    n = prob.n
    C = np.array([[prob.cost(i, j) for j in range(n)] for i in range(n)]) if prob.C is None \
        else prob.C.astype(np.float64)
    return np.exp(U[:, None] + V[None, :] - gbar * C)


def line_search(phi, dphi0, alpha0=1.0, c1=0.1, c2=0.4, dec_tol=1e-14, max_trials=100):
    """Run the oracle's Appx. C line search on a Python phi: alpha -> (phi'(alpha),
    phi(alpha) - phi(0)).  Returns (alpha, phi'(alpha), dval, trials, accepted,
    [every trial alpha in order])."""
    seen = []

    def cb(_ctx, alpha, dphi, dval):
        seen.append(alpha)
        a, b = phi(alpha)
        dphi[0] = a
        dval[0] = b
        return 0

    f = PHI_FN(cb)
    al, dp, dv = ct.c_double(0), ct.c_double(0), ct.c_double(0)
    tr, acc = ct.c_int(0), ct.c_int(0)
    st = lib().orc_line_search(f, None, float(dphi0), float(alpha0), float(c1), float(c2), float(dec_tol),
                               int(max_trials), ct.byref(al), ct.byref(dp), ct.byref(dv), ct.byref(tr),
                               ct.byref(acc))
    assert st == 0
    return al.value, dp.value, dv.value, tr.value, bool(acc.value), seen


def plan_cost(prob: OracleProblem, A, B, gbar):
    """<C, P(A,B)> = sum_ij C_ij exp(A_i + B_j - gbar C_ij) (one pass)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    return lib().orc_plan_cost(ct.byref(prob.s), _ptr(A), _ptr(B), float(gbar))


def mdot_adaptive(prob: OracleProblem, gamma_bar, gamma1=256.0, opts=None, trace_cap=0):
    """MDOT with the ADAPTIVE step rule (Z29); returns (U, V, result, trace, gammas)."""
    n = prob.n
    U = np.empty(n)
    V = np.empty(n)
    g = np.zeros(64)
    opts = opts or make_options()
    res = Result()
    tb = _trace_buf(trace_cap)
    tl = ct.c_int64(0)
    lib().orc_mdot_adaptive(ct.byref(prob.s), float(gamma_bar), float(gamma1), ct.byref(opts), _ptr(U), _ptr(V),
                            ct.byref(res), _ptr(g), ct.cast(tb, ct.c_void_p) if tb is not None else None,
                            trace_cap, ct.byref(tl))
    T = int(res.md_steps)
    return U, V, res.as_dict(), _trace_list(tb, tl.value) if tb is not None else [], g[:T].copy()

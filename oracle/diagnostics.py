"""TEST INFRASTRUCTURE ONLY -- Fig. 3 diagnostics of arxiv 2307.08507 (SURVEY
8(f) rank 2): the dual Hessian, the two diagonal preconditioners and the
pseudo-condition number, in plain numpy (fp64, small n).

* Hessian of the dual objective g(u, v) (Eq. hessian):
      H = [[D(r(P)), P], [P^T, D(c(P))]]
  with the null vector (1_n, -1_n).
* Pseudo-condition number lambda_2n / lambda_2 of eigenvalues
  0 = lambda_1 <= ... <= lambda_2n.
* Sinkhorn-direction preconditioner M = D(s / grad), with
  s = log(m / target) and grad = m - target elementwise;
  M H is similar to the symmetric M^1/2 H M^1/2, whose spectrum is used.
* Jacobi preconditioner D(diag H)^-1 = D(1 / r(P), 1 / c(P)), its diagonal
  bounded below by the target as in the solver ablation
  (MDOT_PROJ_PNCG_JACOBI / oracle ORC_PNCG_JACOBI): D(1 / max(m, target)).

Only tests/ and scripts that produce profiles/ use this module; it shares no
code with the CUDA library.
"""
from __future__ import annotations

import numpy as np

from . import plan as _plan


def hessian(prob, U, V, gbar):
    """Dense 2n x 2n Hessian of g at the plan P = exp(U + V - gbar C)."""
    P = _plan(prob, np.asarray(U, dtype=np.float64), np.asarray(V, dtype=np.float64), gbar)
    n = P.shape[0]
    H = np.zeros((2 * n, 2 * n))
    H[:n, :n] = np.diag(P.sum(1))
    H[n:, n:] = np.diag(P.sum(0))
    H[:n, n:] = P
    H[n:, :n] = P.T
    return H, P


def _log_ratio_over_diff(m, t):
    """log(m / t) / (m - t) elementwise, -> 1 / t as m -> t (series for tiny |d|)."""
    d = m - t
    x = d / t
    out = np.empty_like(m)
    small = np.abs(x) < 1e-6
    out[~small] = np.log1p(x[~small]) / d[~small]
    xs = x[small]
    out[small] = (1.0 - xs / 2.0 + xs * xs / 3.0) / t[small]
    return out


def preconditioner(prob, U, V, gbar, kind="sinkhorn"):
    """Diagonal M (length 2n): 'sinkhorn' = s / grad,
    'jacobi' = 1 / diag(H)."""
    _, P = hessian(prob, U, V, gbar)
    m = np.concatenate([P.sum(1), P.sum(0)])
    t = np.concatenate([prob.r, prob.c])
    if kind == "jacobi":
        return 1.0 / np.maximum(m, t)
    return _log_ratio_over_diff(m, t)


def spectrum(H, M=None):
    """Ascending eigenvalues of H, or of M^1/2 H M^1/2 (similar to M H)."""
    if M is not None:
        sq = np.sqrt(M)
        H = sq[:, None] * H * sq[None, :]
    return np.linalg.eigvalsh(0.5 * (H + H.T))


def pseudo_condition(H, M=None):
    """lambda_2n / lambda_2."""
    w = spectrum(H, M)
    return w[-1] / w[1]

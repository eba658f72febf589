"""Exact OT values used as pins (test-only, independent of the oracle).

* permutation enumeration: for uniform marginals 1/n the vertices of U(r,c)
  are permutation matrices / n (Birkhoff), so OT = min_sigma sum_i C_{i,sigma(i)} / n.
* LP: scipy HiGHS on the transportation LP.
* 1-D monotone coupling: for C_ij = h(x_i - y_j) with h convex and sorted
  supports, the north-west-corner coupling is optimal for any marginals
  (textbook result on optimal transport on the line).
* 2x2 entropic closed form: with t = P_11 and
  kappa = exp(-gbar (C11 + C22 - C12 - C21)) the entropic plan in U(r,c)
  satisfies P11 P22 = kappa P12 P21, i.e.
  (1-kappa) t^2 + (1 - r1 - c1 + kappa (r1 + c1)) t - kappa r1 c1 = 0.
"""
import itertools

import numpy as np


def ot_enumerate_uniform(C):
    n = C.shape[0]
    best = np.inf
    for perm in itertools.permutations(range(n)):
        v = sum(C[i, perm[i]] for i in range(n))
        best = min(best, v)
    return best / n


def ot_lp(C, r, c):
    from scipy.optimize import linprog
    n, m = C.shape
    A_eq = np.zeros((n + m, n * m))
    for i in range(n):
        A_eq[i, i * m:(i + 1) * m] = 1.0
    for j in range(m):
        A_eq[n + j, j::m] = 1.0
    b_eq = np.concatenate([r, c])
    res = linprog(C.ravel(), A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs")
    assert res.status == 0, res.message
    return res.fun


def ot_line_nw(C, r, c):
    """North-west corner rule on sorted supports (C built from sorted x, y)."""
    i = j = 0
    ri, cj = float(r[0]), float(c[0])
    n, m = len(r), len(c)
    cost = 0.0
    while i < n and j < m:
        q = min(ri, cj)
        cost += q * C[i, j]
        ri -= q
        cj -= q
        if ri <= cj:
            i += 1
            if i < n:
                ri = float(r[i])
        else:
            j += 1
            if j < m:
                cj = float(c[j])
    return cost


def entropic_2x2(C, r, c, gbar):
    r1, c1 = r[0], c[0]
    kappa = np.exp(-gbar * (C[0, 0] + C[1, 1] - C[0, 1] - C[1, 0]))
    if kappa <= 1.0:
        a = 1.0 - kappa
        b = 1.0 - r1 - c1 + kappa * (r1 + c1)
        cc = -kappa * r1 * c1
    else:   # same equation divided by kappa (avoids overflow of b^2)
        a = 1.0 / kappa - 1.0
        b = (1.0 - r1 - c1) / kappa + (r1 + c1)
        cc = -r1 * c1
    lo = max(0.0, r1 + c1 - 1.0)
    hi = min(r1, c1)
    if abs(a) < 1e-300:
        t = -cc / b
    else:
        disc = np.sqrt(b * b - 4 * a * cc)
        q = -0.5 * (b + np.copysign(disc, b))       # stable quadratic roots
        roots = [q / a, cc / q]
        cand = [x for x in roots if lo - 1e-15 <= x <= hi + 1e-15]
        t = cand[0]
    return np.array([[t, r1 - t], [c1 - t, 1.0 - r1 - c1 + t]])

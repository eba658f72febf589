"""Seeded synthetic OT instances shaped like the paper's workloads.

This module is the ONLY code shared by the oracle side (tests, bench's
cpu_baseline) and the CUDA side (tests, bench).  It holds no arithmetic of the
method (no potentials, no marginals of P, no projections): it only draws the
inputs (C or point clouds X, Y, and target marginals r, c).

Recipes (BASELINE.json configs):
  RNG      numpy Generator(PCG64(seed)), seed = 1000*config + instance.
           Draw order: X, Y, then r, then c.
  config 1 n=64, the same 8x8 grid (coords 0..7) on both sides, C = |x-y|^2/98
           in fp64; r, c = softmax(N(0,1)).
  config 2 n=784, 28x28 grid both sides, C = |x-y|^2/1458 in fp32; marginals
           are synthetic "images": K~U{3..6} Gaussian blobs, centres
           ~U([0,27]^2), sigma~U(1,3) px, amplitude ~U(0.5,1.5), +1e-6 floor,
           normalised.  Stand-in for MNIST, which is not here.
  config 3 n=4096, X, Y ~ U[0,1]^2 independent, C = d^2/max(d^2) fp32;
           r, c proportional to exp(z/tau), z~N(0,1), tau bisected so that
           H(r)/log n hits {0.5, 0.9, 0.99}.
  config 4 n=16384, X, Y ~ U[0,1]^2, C = d^2/max fp32 (1 GiB); Dirichlet(1).
  config 5 n=65536, X, Y ~ U[0,1]^16 fp32; C is not materialised (on-the-fly
           C_ij = fixed fp32 recipe of |x_i-y_j|^2/16, Z22);
           Dirichlet(1).
The paper's own synthetic set (2n points on the unit sphere in
R^m, min-subtracted, max-normalised Euclidean distance, Dirichlet entropy
targeting) is provided as `paper_sphere_instance` for the paper-shaped pins.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def rng_for(config: int, instance: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(1000 * config + instance))


@dataclass
class Instance:
    n: int
    r: np.ndarray                 # fp64 [n], strictly positive, sums to 1
    c: np.ndarray                 # fp64 [n]
    C: np.ndarray | None = None   # [n, n] fp32 or fp64, row-major, in [0, 1]
    X: np.ndarray | None = None   # [n, d] fp32 (on-the-fly cost)
    Y: np.ndarray | None = None
    scale: float = 0.0            # on-the-fly: C_ij = scale * |x_i - y_j|^2
    name: str = ""
    meta: dict = field(default_factory=dict)


def _normalise(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x / x.sum()


def softmax_marginal(rng, n):
    z = rng.standard_normal(n)
    e = np.exp(z - z.max())
    return _normalise(e)


def dirichlet_marginal(rng, n, alpha=1.0):
    x = rng.dirichlet(np.full(n, alpha))
    x = np.maximum(x, np.finfo(np.float64).tiny)
    return _normalise(x)


def _entropy_frac(p):
    p = p[p > 0]
    return float(-(p * np.log(p)).sum() / math.log(len(p)) if len(p) > 1 else 0.0)


def entropy_targeted_marginal(rng, n, frac, tol=1e-3):
    """r proportional to exp(z/tau), tau bisected so that H(r)/log n = frac."""
    z = rng.standard_normal(n)

    def make(tau):
        e = np.exp((z - z.max()) / tau)
        return _normalise(e)

    lo, hi = 1e-3, 1e3   # H increases with tau
    for _ in range(200):
        mid = math.sqrt(lo * hi)
        h = _entropy_frac(make(mid))
        if abs(h - frac) < tol * 0.1:
            break
        if h < frac:
            lo = mid
        else:
            hi = mid
    return make(mid)


def sqdist_matrix(X, Y, dtype=np.float32, normalise="max", chunk=2048):
    """C_ij = |x_i - y_j|^2 / max_ij |x_i - y_j|^2 computed in fp64 with a fixed
    op order (acc += diff*diff over coordinates), then rounded to `dtype`."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    n, d = X.shape
    m = Y.shape[0]
    D = np.empty((n, m), dtype=np.float64 if dtype == np.float64 else np.float32)
    mx = 0.0
    # first pass: max (fp64)
    for i0 in range(0, n, chunk):
        acc = np.zeros((min(chunk, n - i0), m))
        for k in range(d):
            diff = X[i0:i0 + chunk, k][:, None] - Y[None, :, k]
            acc += diff * diff
        mx = max(mx, float(acc.max()))
    norm = mx if normalise == "max" else float(normalise)
    for i0 in range(0, n, chunk):
        acc = np.zeros((min(chunk, n - i0), m))
        for k in range(d):
            diff = X[i0:i0 + chunk, k][:, None] - Y[None, :, k]
            acc += diff * diff
        D[i0:i0 + chunk] = (acc / norm).astype(D.dtype)
    return D


def grid_points(side):
    g = np.arange(side, dtype=np.float64)
    yy, xx = np.meshgrid(g, g, indexing="ij")
    return np.stack([xx.ravel(), yy.ravel()], axis=1)


# --------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------

def config1(instance=0):
    """Tiny OT: n=64 on an 8x8 grid, C fp64 = |.|^2/98, softmax marginals."""
    rng = rng_for(1, instance)
    P = grid_points(8)
    C = sqdist_matrix(P, P, dtype=np.float64, normalise=98.0)
    r = softmax_marginal(rng, 64)
    c = softmax_marginal(rng, 64)
    return Instance(64, r, c, C=C, name=f"cfg1-tiny-n64-s{instance}")


def blob_image(rng, side=28):
    K = int(rng.integers(3, 7))
    P = grid_points(side)
    img = np.zeros(side * side)
    for _ in range(K):
        ctr = rng.uniform(0.0, side - 1.0, size=2)
        sig = rng.uniform(1.0, 3.0)
        amp = rng.uniform(0.5, 1.5)
        d2 = ((P - ctr) ** 2).sum(axis=1)
        img += amp * np.exp(-d2 / (2.0 * sig * sig))
    img += 1e-6
    return _normalise(img)


def config2(instance=0, pairs=64):
    """MNIST-shaped batch: n=784, C fp32 = |.|^2/1458, `pairs` blob pairs."""
    rng = rng_for(2, instance)
    P = grid_points(28)
    C = sqdist_matrix(P, P, dtype=np.float32, normalise=1458.0)
    R = np.stack([blob_image(rng) for _ in range(pairs)])
    Cc = np.stack([blob_image(rng) for _ in range(pairs)])
    return C, R, Cc


def config2_pair(instance=0, pair=0, pairs=64):
    C, R, Cc = config2(instance, pairs)
    return Instance(784, R[pair], Cc[pair], C=C, name=f"cfg2-mnistlike-n784-s{instance}-p{pair}")


def uniform_points_instance(config, n, d, instance, marg="dirichlet", frac=None,
                            dtype=np.float32, materialise=True):
    rng = rng_for(config, instance)
    X = rng.uniform(0.0, 1.0, size=(n, d))
    Y = rng.uniform(0.0, 1.0, size=(n, d))
    if marg == "dirichlet":
        r = dirichlet_marginal(rng, n)
        c = dirichlet_marginal(rng, n)
    elif marg == "entropy":
        r = entropy_targeted_marginal(rng, n, frac)
        c = entropy_targeted_marginal(rng, n, frac)
    elif marg == "softmax":
        r = softmax_marginal(rng, n)
        c = softmax_marginal(rng, n)
    else:
        raise ValueError(marg)
    inst = Instance(n, r, c, name=f"cfg{config}-n{n}-d{d}-s{instance}")
    if materialise:
        inst.C = sqdist_matrix(X, Y, dtype=dtype)
    inst.X = X.astype(np.float32)
    inst.Y = Y.astype(np.float32)
    return inst


def config3(instance=0, frac=0.9, n=4096):
    return uniform_points_instance(3, n, 2, instance, marg="entropy", frac=frac)


def config4(instance=0, n=16384):
    return uniform_points_instance(4, n, 2, instance, marg="dirichlet")


def config5(instance=0, n=65536, d=16):
    """On-the-fly cost: only X, Y (fp32) are produced; scale = 1/16."""
    rng = rng_for(5, instance)
    X = rng.uniform(0.0, 1.0, size=(n, d)).astype(np.float32)
    Y = rng.uniform(0.0, 1.0, size=(n, d)).astype(np.float32)
    r = dirichlet_marginal(rng, n)
    c = dirichlet_marginal(rng, n)
    return Instance(n, r, c, X=X, Y=Y, scale=1.0 / d, name=f"cfg5-otf-n{n}-d{d}-s{instance}")


def otf_instance(n, d, instance=0, config=5):
    """Smaller on-the-fly instances for parity tests (same recipe as config 5)."""
    return config5(instance, n=n, d=d) if config == 5 else None


# --------------------------------------------------------------------------
# Small instances for pins
# --------------------------------------------------------------------------

def random_small(n, seed, uniform_marginals=False, dtype=np.float64):
    rng = np.random.Generator(np.random.PCG64(seed))
    C = rng.uniform(0.0, 1.0, size=(n, n)).astype(dtype)
    if uniform_marginals:
        r = np.full(n, 1.0 / n)
        c = np.full(n, 1.0 / n)
    else:
        r = dirichlet_marginal(rng, n)
        c = dirichlet_marginal(rng, n)
    return Instance(n, r, c, C=C, name=f"small-n{n}-s{seed}")


def line_instance(n, seed, dtype=np.float64):
    """1-D point sets with C = (x_i - y_j)^2 (convex cost on a line), any
    marginals.  Exact OT is the monotone (north-west corner) coupling."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.sort(rng.uniform(0.0, 1.0, n))
    y = np.sort(rng.uniform(0.0, 1.0, n))
    C = ((x[:, None] - y[None, :]) ** 2).astype(dtype)
    r = dirichlet_marginal(rng, n)
    c = dirichlet_marginal(rng, n)
    inst = Instance(n, r, c, C=C, name=f"line-n{n}-s{seed}")
    inst.meta["x"] = x
    inst.meta["y"] = y
    return inst


def paper_sphere_instance(n, m, frac, seed):
    """PAPER.md:301 recipe: 2n points on the unit sphere of R^m (normalised
    Gaussians), Euclidean distances between first and second n
    points, min subtracted, divided by max; marginals with H/log n ~ frac
    (softmax-temperature targeting in place of the paper's Dirichlet search;
    both only aim at the entropy level)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    Z = rng.standard_normal((2 * n, m))
    Z /= np.linalg.norm(Z, axis=1, keepdims=True)
    X, Y = Z[:n], Z[n:]
    D = np.sqrt(((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1))
    D = D - D.min()
    D = D / D.max()
    r = entropy_targeted_marginal(rng, n, frac)
    c = entropy_targeted_marginal(rng, n, frac)
    r = r + 1e-8 if r.min() < 1e-8 else r
    c = c + 1e-8 if c.min() < 1e-8 else c
    return Instance(n, _normalise(r), _normalise(c), C=D, name=f"sphere-n{n}-m{m}-s{seed}")

"""A/B of the two on-the-fly cost recipes of K2 (Z22 difference form, Z22b
dot form) at BASELINE config 5 (n = 65536, d = 16): one fused marginal
evaluation timed with CUDA events (median of 20 after warm-up), and the full
config-5 solve (gbar 4096, T 16, L1 1e-5) timed once per recipe.  The
evaluation runs at potentials of a short gbar-256 solve (fast path, no
fallback).  argv: recipes to run (default diff dot diff dot).  Prints one
JSON line per recipe.  Product path only (no oracle)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

DEV = torch.device("cuda:0")


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def main():
    inst = S.config5(0)
    n, d = inst.n, inst.X.shape[1]
    X, Y, r, c = t(inst.X), t(inst.Y), t(inst.r), t(inst.c)
    # potentials on the fast (fp32-entry) path: a short gbar-256 solve
    A = torch.empty(n, dtype=torch.float64, device=DEV)
    B = torch.empty_like(A)
    gb = 256.0
    M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=1),
                 options=M.options(eps=1e-3), u_out=A, v_out=B)
    only = sys.argv[1:] or ["diff", "dot", "diff", "dot"]
    for recipe in only:
        for _ in range(3):
            _, _, fb = M.mdot_marginals(A, B, gb, X=X, Y=Y, scale=inst.scale, r=r, c=c, recipe=recipe)
        assert fb == 0
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            M.mdot_marginals(A, B, gb, X=X, Y=Y, scale=inst.scale, r=r, c=c, recipe=recipe)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        U = torch.empty(n, dtype=torch.float64, device=DEV)
        V = torch.empty_like(U)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0),
                           options=M.options(eps=1e-5), u_out=U, v_out=V, recipe=recipe)
        e1.record()
        e1.synchronize()
        ms = float(np.median(ts))
        ops = (d + 7) if recipe == "dot" else (2 * d + 5)
        peak = 148 * 128 * 1.965e9 / ops
        print(json.dumps({"recipe": recipe, "n": n, "d": d, "eval_call_ms_median": ms,
                          "pairs_per_s": n * n / (ms / 1e3), "fp32_floor_pairs_per_s": peak,
                          "frac": n * n / (ms / 1e3) / peak,
                          "solve_s": e0.elapsed_time(e1) / 1e3, "evaluations": res["evaluations"],
                          "status": res["status_name"], "cost_unrounded": res["cost_unrounded"],
                          "cost_rounded": res["cost_rounded"], "l1_final": res["l1_final"]}), flush=True)


if __name__ == "__main__":
    main()

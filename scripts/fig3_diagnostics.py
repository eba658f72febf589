"""Fig. 3 of the paper on synthetic sphere instances
(PAPER.md:301 recipe): left -- projection iterations vs entropy
level for Sinkhorn, PNCG, vanilla NCG and the Jacobi-preconditioned ablation,
on the GPU path (n = 8, m = 4, T = 1, gbar = 128, rho <= 1e-5); right -- the
ratio of pseudo-condition numbers kappa(H) / kappa(M H) along PNCG iterations
(n = 32, m = 4, gbar = 32), computed with the oracle's dense diagnostics
(numpy eigendecomposition; a CPU-side diagnostic, as in the paper)."""
import json
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402
from oracle import diagnostics as D  # noqa: E402


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def main():
    out = {"left": {}, "right": {}}
    names = {M.MDOT_PROJ_SINKHORN: "sinkhorn", M.MDOT_PROJ_PNCG: "pncg", M.MDOT_PROJ_NCG: "ncg",
             M.MDOT_PROJ_PNCG_JACOBI: "pncg_jacobi"}
    for frac in (0.2, 0.4, 0.6, 0.8):
        its = {v: [] for v in names.values()}
        for seed in range(32):
            inst = S.paper_sphere_instance(8, 4, frac, 200 + seed)
            C, r, c = t(inst.C), t(inst.r), t(inst.c)
            for p, nm in names.items():
                res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 128.0, T=1),
                                   options=M.options(eps=1e-5, stop=1, projector=p, max_evals=500000), check=False)
                its[nm].append(res["iterations"] if res["status"] == 0 else float("nan"))
        out["left"][frac] = {k: float(np.nanmean(v)) for k, v in its.items()}
        print("left", frac, out["left"][frac], flush=True)
    for frac in (0.2, 0.4, 0.6, 0.8):
        rows = {}
        for k in (5, 10, 20, 35, 50):
            rs, rj = [], []
            for seed in range(32):
                inst = S.paper_sphere_instance(32, 4, frac, 100 + seed)
                prob = O.OracleProblem(inst)
                U0, V0 = np.log(inst.r), np.log(inst.c)
                u, v, _, _ = O.project(prob, U0, V0, 32.0, opts=O.make_options(eps=1e-12, max_evals=k))
                U, V = U0 + u, V0 + v
                H, _ = D.hessian(prob, U, V, 32.0)
                kH = D.pseudo_condition(H)
                rs.append(kH / D.pseudo_condition(H, D.preconditioner(prob, U, V, 32.0)))
                rj.append(kH / D.pseudo_condition(H, D.preconditioner(prob, U, V, 32.0, "jacobi")))
            rows[k] = {"sinkhorn_precond": float(np.exp(np.mean(np.log(rs)))),
                       "jacobi_precond": float(np.exp(np.mean(np.log(rj))))}
        out["right"][frac] = rows
        print("right", frac, rows, flush=True)
    print("JSON " + json.dumps(out))


if __name__ == "__main__":
    main()

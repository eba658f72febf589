"""Adaptive eps per MD step on config 4 (n = 16384,
gamma_bar = 4096, final L1 <= 1e-6): time-to-eps and evaluations for
eps_md x T, device-timed with CUDA events around each synchronous solve.
Also config 3 (n = 4096) for both projectors.  Writes one JSON object."""
import json
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def timed(fn, reps=2):
    fn()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if best is None or ms < best[0]:
            best = (ms, r)
    return best


def main():
    which = sys.argv[1:] or ["4", "3"]
    out = {}
    if "4" in which:
        inst = S.config4(0)
        C, r, c = t(inst.C), t(inst.r), t(inst.c)
        del inst
        for T in (16, 4, 1):
            for em in ((0.0, 1e-4, 1e-3, 1e-2) if T > 1 else (0.0,)):
                ms, res = timed(lambda: M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=T),
                                                     options=M.options(eps=1e-6, eps_md=em), check=False))
                k = f"cfg4_T{T}_epsmd{em:g}"
                out[k] = {"ms": ms, "evals": res["evaluations"], "iterations": res["iterations"],
                          "cost_unrounded": res["cost_unrounded"], "l1": res["l1_final"],
                          "status": res["status_name"]}
                print(k, out[k], flush=True)
        del C
        torch.cuda.empty_cache()
    if "3" in which:
        for frac in (0.5, 0.9, 0.99):
            inst = S.config3(0, frac=frac)
            C, r, c = t(inst.C), t(inst.r), t(inst.c)
            for nm, proj in (("pncg", M.MDOT_PROJ_PNCG), ("sinkhorn", M.MDOT_PROJ_SINKHORN)):
                for em in (0.0, 1e-3):
                    ms, res = timed(lambda: M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                                                         options=M.options(eps=1e-6, eps_md=em, projector=proj,
                                                                           max_evals=300000), check=False), reps=1)
                    k = f"cfg3_H{frac}_{nm}_epsmd{em:g}"
                    out[k] = {"ms": ms, "evals": res["evaluations"], "iterations": res["iterations"],
                              "cost_unrounded": res["cost_unrounded"], "status": res["status_name"]}
                    print(k, out[k], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Secondary measurements over the BASELINE configs (not the driver's bench
line): time-to-eps and evaluations for configs 1, 3 (PNCG vs Sinkhorn on the
same kernels, three entropy levels) and 5 (on-the-fly cost), device-timed
with CUDA events around each synchronous solve.  Writes one JSON object."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def timed(fn, reps=2):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), r


def main():
    which = sys.argv[1:] or ["1", "3", "5"]
    out = {}
    if "1" in which:
        inst = S.config1(0)
        C, r, c = t(inst.C), t(inst.r), t(inst.c)
        for em in (0.0, 1e-3):
            ms, res = timed(lambda: M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_DOUBLING, 4096.0),
                                                 options=M.options(eps=1e-6, eps_md=em)))
            out[f"cfg1_n64_fp64_doubling_eps1e-6_epsmd{em:g}"] = {
                "ms": ms, "evals": res["evaluations"], "md_steps": res["md_steps"],
                "control_path": res["control_path"], "l1": res["l1_final"]}
        print(out, flush=True)
    if "3" in which:
        for frac in (0.5, 0.9, 0.99):
            inst = S.config3(0, frac=frac)
            C, r, c = t(inst.C), t(inst.r), t(inst.c)
            for gb, T in ((512.0, 1), (512.0, 4), (512.0, 16), (4096.0, 16)):
                row = {}
                for nm, proj in (("pncg", M.MDOT_PROJ_PNCG), ("sinkhorn", M.MDOT_PROJ_SINKHORN)):
                    ms, res = timed(lambda: M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=T),
                                                         options=M.options(eps=1e-6, projector=proj,
                                                                           max_evals=300000),
                                                         check=False), reps=1)
                    row[nm] = {"ms": ms, "evals": res["evaluations"], "iterations": res["iterations"],
                               "status": res["status_name"], "l1": res["l1_final"],
                               "control_path": res["control_path"]}
                row["speedup_time"] = row["sinkhorn"]["ms"] / row["pncg"]["ms"]
                row["speedup_iters"] = row["sinkhorn"]["iterations"] / max(1, row["pncg"]["iterations"])
                out[f"cfg3_n4096_H{frac}_gbar{int(gb)}_T{T}"] = row
                print(f"cfg3 H={frac} gbar={gb} T={T}", json.dumps(row), flush=True)
    if "5" in which:
        inst = S.config5(0)
        X, Y, r, c = t(inst.X), t(inst.Y), t(inst.r), t(inst.c)
        n = inst.n
        A = torch.from_numpy(np.log(inst.r)).cuda()
        B = torch.from_numpy(np.log(inst.c)).cuda()
        ms, _ = timed(lambda: M.mdot_marginals(A, B, 4096.0, X=X, Y=Y, scale=inst.scale, r=r, c=c), reps=3)
        pairs = float(n) * n
        out["cfg5_single_eval"] = {"ms_incl_setup": ms, "pairs_per_s": pairs / (ms / 1e3)}
        print(out["cfg5_single_eval"], flush=True)
        for em in (0.0, 1e-3):
            ms, res = timed(lambda: M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c,
                                                 schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0),
                                                 options=M.options(eps=1e-5, eps_md=em, time_kernels=1),
                                                 check=False), reps=1)
            k1 = res["kernel_ms"] / max(1, res["kernel_launches"])
            key = f"cfg5_n65536_d16_otf_gbar4096_eps1e-5_epsmd{em:g}"
            out[key] = {
                "ms": ms, "evals": res["evaluations"], "status": res["status_name"], "l1": res["l1_final"],
                "k1_ms": k1, "pairs_per_s_k1": pairs / (k1 / 1e3), "control_path": res["control_path"],
                "cost_unrounded": res["cost_unrounded"], "cost_rounded": res["cost_rounded"]}
            print(key, out[key], flush=True)
    print("JSON " + json.dumps(out))


if __name__ == "__main__":
    main()

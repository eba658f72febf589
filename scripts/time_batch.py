import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
Cd, Rd, Cmd = t(C), t(R), t(Cm)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
out = {}
for eps, em in ((1e-4, 0.0), (1e-6, 0.0), (1e-8, 0.0), (1e-4, 1e-3), (1e-6, 1e-3), (1e-8, 1e-3)):
    M.mdot_solve_batch(Cd, Rd[:2], Cmd[:2], schedule=sched, options=M.options(eps=eps, eps_md=em), check=False)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=eps, eps_md=em), check=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ev = sum(r["evaluations"] for r in res)
    st = sorted(set(r["status_name"] for r in res))
    out[f"{eps:g}/epsmd{em:g}"] = {"batch_s": dt, "evals_total": ev, "evals_per_s": ev / dt, "status": st,
                     "max_l1": max(r["l1_final"] for r in res), "mean_evals": ev / 64}
    print(eps, em, out[f"{eps:g}/epsmd{em:g}"], flush=True)
# per-instance loop for comparison (2 instances, eps 1e-6)
torch.cuda.synchronize(); t0 = time.perf_counter()
for b in range(2):
    M.mdot_solve(Cd, Rd[b], Cmd[b], schedule=sched, options=M.options(eps=1e-6))
torch.cuda.synchronize(); print("single-instance solves, 2 instances eps 1e-6:", time.perf_counter() - t0)

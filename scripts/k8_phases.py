"""K8 (config 2) phase clocks per evaluation (MDOT_DIAG_K8 build via MDOT_LIB) and batch times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
Cd, Rd, Cmd = t(C), t(R), t(Cm)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
for eps in [float(x) for x in (sys.argv[1:] or ["1e-6"])]:
    M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=eps), check=False)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=eps), check=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ev = [r["evaluations"] for r in res]
    print(f"eps {eps:g}: batch {dt*1e3:.1f} ms, evals mean {np.mean(ev):.0f} max {max(ev)}, "
          f"us/eval(max inst) {dt*1e6/max(ev):.1f}, status {sorted(set(r['status_name'] for r in res))}", flush=True)

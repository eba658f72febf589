#!/bin/bash
# K8 fp64-entry narrow-tail layout A/B: config 1 (n = 64, fp64 C) and config 2
# at eps 1e-8 (fp64 entries, 16-column tail), new layout vs MDOT_K8_TAIL_REGULAR.
for mode in new regular new regular; do
  if [ $mode = regular ]; then export MDOT_K8_TAIL_REGULAR=1; else unset MDOT_K8_TAIL_REGULAR; fi
  echo "== $mode"
  timeout 120 python scripts/cfg1_diag.py 2>&1 | tail -1
  timeout 300 python -c "
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
Cd, Rd, Cmd = t(C), t(R), t(Cm)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
for eps, em in ((1e-8, 0.0), (1e-8, 1e-3)):
    M.mdot_solve_batch(Cd, Rd[:2], Cmd[:2], schedule=sched, options=M.options(eps=eps, eps_md=em), check=False)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=eps, eps_md=em), check=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ev = sum(r['evaluations'] for r in res)
    print('cfg2 eps', eps, 'eps_md', em, 'batch_s %.3f' % dt, 'evals', ev, sorted(set(r['status_name'] for r in res)), 'max_l1 %.3g' % max(r['l1_final'] for r in res), flush=True)
"
done

"""Throughput mode: B = 16 independent n = 4096 solves sharing one C
(config-3 shape, H/log n = 0.9 pairs, gbar 4096, T 16, L1 1e-6), as (a) the lockstep batch
(MDOT_BATCH_LOCKSTEP=1: one launch per phase for all instances), (b) the worker-stream path (default,
8 workers), (c) one persistent solve after the other.  Host wall
clock around the synchronous calls (after one warm-up each); eps_md in argv[1] (0 = paper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
B = int(os.environ.get("TP_B", "16"))
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
base = S.config3(0, frac=0.9)
C = t(base.C)
pairs = [S.config3(i, frac=0.9) for i in range(B)]
Rb = t(np.stack([p.r for p in pairs])); Cb = t(np.stack([p.c for p in pairs]))
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16)
for em in [float(x) for x in (sys.argv[1:] or ["1e-3", "0"])]:
    opts = lambda: M.options(eps=1e-6, eps_md=em)
    def lock():
        os.environ["MDOT_BATCH_LOCKSTEP"] = "1"
        try:
            return M.mdot_solve_batch(C, Rb, Cb, schedule=sched, options=opts())
        finally:
            del os.environ["MDOT_BATCH_LOCKSTEP"]
    def workers():
        return M.mdot_solve_batch(C, Rb, Cb, schedule=sched, options=opts())
    def seq():
        return [M.mdot_solve(C, Rb[b], Cb[b], schedule=sched, options=opts()) for b in range(B)]
    ref = None
    for name, fn in (("lockstep", lock), ("workers8", workers), ("sequential", seq)):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        costs = np.array([o["cost_unrounded"] for o in out])
        ref = costs if ref is None else ref
        print(f"eps_md {em:g} {name:10s} {dt*1e3:8.1f} ms  evals {sum(o['evaluations'] for o in out):6d}  "
              f"paths {sorted(set(o['control_path'] for o in out))}  ok {all(o['status'] == 0 for o in out)}  "
              f"max L1 {max(o['l1_final'] for o in out):.2e}  max cost rel diff vs lockstep {np.max(np.abs(costs / ref - 1)):.1e}",
              flush=True)

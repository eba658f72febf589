"""Throughput mode A/B (B = TP_B (16) x n = 4096 sharing one C, config-3 shape, gbar 4096,
T 16, L1 1e-6): lockstep batch with decoupled MD steps (MDOT_BATCH_LOCKSTEP=1),
lockstep with synchronous MD steps (+ MDOT_BATCH_SYNC_MD=1), worker streams
(default path); three interleaved rounds, host wall clock per batch after a
warm-up of each."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
base = S.config3(0, frac=0.9)
C = t(base.C)
B = int(os.environ.get("TP_B", "16"))   # the paper runs 32 instances per point
pairs = [S.config3(i, frac=0.9) for i in range(B)]
Rb = t(np.stack([p.r for p in pairs]))
Cb = t(np.stack([p.c for p in pairs]))
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16)
VARIANTS = {"lockstep-decoupled": {"MDOT_BATCH_LOCKSTEP": "1"},
            "lockstep-sync-md": {"MDOT_BATCH_LOCKSTEP": "1", "MDOT_BATCH_SYNC_MD": "1"},
            "workers": {}}


def run(env, em):
    for k in ("MDOT_BATCH_LOCKSTEP", "MDOT_BATCH_SYNC_MD"):
        os.environ.pop(k, None)
    os.environ.update(env)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = M.mdot_solve_batch(C, Rb, Cb, schedule=sched, options=M.options(eps=1e-6, eps_md=em))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


for em in (1e-3, 0.0):
    for name, env in VARIANTS.items():
        run(env, em)   # warm-up
    times = {k: [] for k in VARIANTS}
    for rnd in range(3):
        for name, env in VARIANTS.items():
            dt, out = run(env, em)
            times[name].append(1000 * dt)
            if rnd == 0:
                print(f"eps_md {em:g} {name:20s} evals {sum(o['evaluations'] for o in out):6d} paths "
                      f"{sorted(set(o['control_path'] for o in out))} ok {all(o['status'] == 0 for o in out)} "
                      f"max L1 {max(o['l1_final'] for o in out):.2e}", flush=True)
    for name in VARIANTS:
        ts = times[name]
        print(f"B {B} eps_md {em:g} {name:20s} ms per batch: " + " ".join(f"{x:7.1f}" for x in ts)
              + f"   median {sorted(ts)[1]:7.1f}", flush=True)

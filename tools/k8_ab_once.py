"""Config 2 (64 pairs, n = 784, gbar 4096, T 16) batch time per eps for the
library selected by MDOT_LIB (A/B of K8 compile-time variants); prints the
batch wall time (after one warm-up batch), evaluations and the summed costs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
Cd, Rd, Cmd = t(C), t(R), t(Cm)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
tag = os.path.basename(os.environ.get("MDOT_LIB", "default"))
for eps in (1e-4, 1e-6, 1e-8):
    M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=eps), check=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=eps), check=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{tag:24s} eps {eps:g}  batch {1000 * dt:8.1f} ms  evals {sum(r['evaluations'] for r in res):7d}  "
          f"max evals {max(r['evaluations'] for r in res):6d}  sum cost {sum(r['cost_unrounded'] for r in res):.12g}  "
          f"status {sorted(set(r['status_name'] for r in res))}", flush=True)

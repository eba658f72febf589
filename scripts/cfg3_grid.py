"""Config 3 (n = 4096, H = 0.9 log n, gbar 4096, T 16, L1 1e-6) PNCG time-to-eps
and per-slot phases of the persistent kernel; grid size via MDOT_PERSIST_NCTA."""
import os
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

inst = S.config3(0, frac=0.9)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
C, r, c = t(inst.C), t(inst.r), t(inst.c)
for rep in range(3):
    res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                       options=M.options(eps=1e-6, time_kernels=1))
k = max(1, res["stage_samples"])
print(os.environ.get("MDOT_PERSIST_NCTA", "all"), f"{1000 * res['seconds']:.1f} ms", res["evaluations"],
      [round(1000 * x / k, 2) for x in res["stage_ms"]], res["control_path"])

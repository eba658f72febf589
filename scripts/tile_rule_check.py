"""Row-tile height rule check: PNCG time-to-eps per evaluation for
config-3-shaped instances (H/log n = 0.9, gbar 4096, T 16, L1 1e-6) at several
n, automatic tile height vs MDOT_TILE_M forced (set in the environment)."""
import os
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
for n in [int(x) for x in sys.argv[1].split(",")]:
    inst = S.config3(0, frac=0.9, n=n)
    C, r, c = t(inst.C), t(inst.r), t(inst.c)
    best = None
    for rep in range(3):
        res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                           options=M.options(eps=1e-6, time_kernels=1))
        best = res if best is None or res["seconds"] < best["seconds"] else best
    k = max(1, best["stage_samples"])
    print(n, os.environ.get("MDOT_TILE_M", "auto"), f"{1000 * best['seconds']:.1f} ms", best["evaluations"],
          f"{1e6 * best['seconds'] / best['evaluations']:.2f} us/eval",
          [round(1000 * x / k, 2) for x in best["stage_ms"]], flush=True)

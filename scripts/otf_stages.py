"""Config 5 (n = 65536, d = 16, on-the-fly cost) per-slot stages of the
graph control path (ctrl, prep, K2, finalize; sampled CUDA events) over a
bounded number of evaluations, and wall time per evaluation."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
inst = S.config5(0)
X, Y, r, c = t(inst.X), t(inst.Y), t(inst.r), t(inst.c)
for me in (60, 160):
    res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0),
                       options=M.options(eps=1e-5, time_kernels=1, max_evals=me), check=False)
    k = max(1, res["stage_samples"])
    print(me, res["evaluations"], f"{1000 * res['seconds']:.1f} ms",
          "stages_us", [round(1000 * x / k, 1) for x in res["stage_ms"]], "samples", k, flush=True)

"""Sweep of the persistent kernel's next-pass L2 prefetch depth (MDOT_L2_PREFETCH)
on config 4: time-to-eps and the per-slot phase times."""
import json
import os
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

inst = S.config4(0)
n = inst.n
C = torch.from_numpy(inst.C).cuda()
r = torch.from_numpy(inst.r).cuda()
c = torch.from_numpy(inst.c).cuda()
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
out = {}
vals = sys.argv[1:] or ["0", "3", "6", "9", "12"]
for rep in range(2):
    for pf in vals:
        os.environ["MDOT_L2_PREFETCH"] = pf
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        res = M.mdot_solve(C, r, c, schedule=sched, options=M.options(eps=1e-6, time_kernels=1))
        e1.record()
        torch.cuda.synchronize()
        ns = max(1, res["stage_samples"])
        row = {"ms": round(e0.elapsed_time(e1), 1), "evals": res["evaluations"],
               "phases_us": [round(x / ns * 1e3, 2) for x in res["stage_ms"]]}
        out.setdefault(pf, []).append(row)
        print(pf, row, flush=True)
print("JSON " + json.dumps(out))

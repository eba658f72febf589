"""Repeat the config-4 solve and compare results bit for bit (the solve has no
atomics and fixed reduction orders: it must be deterministic)."""
import os
import sys

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

n = int(os.environ.get("DET_N", "16384"))
inst = S.config4(0, n=n)
C = torch.from_numpy(inst.C).cuda()
r = torch.from_numpy(inst.r).cuda()
c = torch.from_numpy(inst.c).cuda()
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
for cfg in sys.argv[1:]:
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    for k in ("MDOT_L2_PREFETCH", "MDOT_NO_PERSIST"):
        os.environ.pop(k, None)
    os.environ.update(env)
    outs = []
    for rep in range(3):
        U = torch.empty(n, dtype=torch.float64, device="cuda")
        res = M.mdot_solve(C, r, c, schedule=sched, options=M.options(eps=1e-6), u_out=U)
        outs.append((res["evaluations"], res["cost_unrounded"].hex(), float(U.sum())))
    print(cfg, "DETERMINISTIC" if len(set(outs)) == 1 else "DIFFERS", outs, flush=True)

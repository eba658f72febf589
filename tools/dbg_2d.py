import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
DEV = torch.device("cuda:0")
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
n = 800
inst = S.uniform_points_instance(3, n, 2, 34, marg="dirichlet")
sched = M.schedule(M.MDOT_SCHED_FIXED, 512.0, T=2)
rc = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
cc = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
for dc in (1, 0):
    res = M.mdot_solve_sharded_2d(rc, cc, 0, n, 0, n, t(inst.C), t(inst.r), t(inst.c), n=n, schedule=sched,
                                  options=M.options(eps=1e-6, device_control=dc), check=False)
    print(dc, {k: res[k] for k in ("status_name", "control_path", "fallbacks", "evaluations", "l1_final", "cost_unrounded")}, M.mdot_last_error())
res = M.mdot_solve_sharded(cc, 0, n, t(inst.C), t(inst.r), t(inst.c), n=n, schedule=sched, options=M.options(eps=1e-6), check=False)
print("1d", {k: res[k] for k in ("status_name", "control_path", "fallbacks", "evaluations", "l1_final", "cost_unrounded")})

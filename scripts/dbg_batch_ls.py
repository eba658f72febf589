# which config-2 instances fail at eps 1e-8 with eps_md 1e-3 (K8 batch), and do
# the per-instance solver and the oracle agree?
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
res = M.mdot_solve_batch(t(C), t(R), t(Cm), schedule=sched, options=M.options(eps=1e-8, eps_md=1e-3), check=False)
bad = [b for b, r in enumerate(res) if r["status"] != 0]
print("bad", bad, [(res[b]["status_name"], res[b]["md_steps"], res[b]["l1_final"], res[b]["evaluations"]) for b in bad])
for b in bad[:2]:
    for dc in (0, 1):
        r1 = M.mdot_solve(t(C), t(R[b]), t(Cm[b]), schedule=sched, options=M.options(eps=1e-8, eps_md=1e-3, device_control=dc), check=False)
        print("single", b, dc, r1["status_name"], r1["md_steps"], r1["l1_final"], r1["evaluations"], r1["fallbacks"])
    np.save(f"gpurun_out/bad_{b}.npy", np.stack([R[b], Cm[b]]))

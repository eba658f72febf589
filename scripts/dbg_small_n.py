# K8 (small-problem route) on tiny n: status per n, fp32 / fp64 entries
import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, paper_2307_08507_b200 as M
t=lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
rng = np.random.default_rng(0)
for n in (1, 2, 3, 4, 5, 8, 16, 31, 32, 33, 64):
    row = []
    for kind in ("const", "rand"):
        C = np.full((n, n), 0.5, dtype=np.float32) if kind == "const" else rng.uniform(0, 1, (n, n)).astype(np.float32)
        r = rng.dirichlet(np.ones(n)) if n > 1 else np.ones(1)
        c = rng.dirichlet(np.ones(n)) if n > 1 else np.ones(1)
        for eps in (1e-6, 1e-9):
            res = M.mdot_solve(t(C), t(r), t(c), schedule=M.schedule(M.MDOT_SCHED_FIXED, 64.0, T=1), options=M.options(eps=eps), check=False)
            row.append((kind, eps, res["status"], res["evaluations"]))
    print(n, row, flush=True)
import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, paper_2307_08507_b200 as M
t=lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
for n in (1, 2, 3, 5):
    for eps in (1e-6, 1e-9):
        C = np.full((n, n), 0.5, dtype=np.float32); r = np.full(n, 1.0/n); c = np.full(n, 1.0/n)
        res = M.mdot_solve(t(C), t(r), t(c), options=M.options(eps=eps), check=False)
        print(n, eps, res["status"], res["control_path"], res["evaluations"], res["cost_rounded"], flush=True)

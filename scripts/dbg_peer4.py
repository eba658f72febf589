import sys, threading
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
inst = S.config4(0); n = inst.n; G = 4
rows = np.array_split(np.arange(n), G)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
out = [None]*G
def run(k):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        row0, nloc = int(rows[k][0]), len(rows[k])
        C = torch.from_numpy(np.ascontiguousarray(inst.C[row0:row0+nloc])).cuda()
        r = torch.from_numpy(inst.r).cuda(); c = torch.from_numpy(inst.c).cuda()
        comm = M.mdot_comm_create_local("x", G, k, 0); M.mdot_comm_enable_peer(comm, n)
        res = M.mdot_solve_sharded(comm, row0, nloc, C_local=C, r=r, c=c, n=n, schedule=sched, options=M.options(eps=1e-6), check=False)
        s.synchronize(); M.mdot_comm_destroy(comm); out[k] = res
ths = [threading.Thread(target=run, args=(k,)) for k in range(G)]
[t.start() for t in ths]; [t.join() for t in ths]
for o in out: print(o["status_name"], o["control_path"], o["evaluations"], o["fallbacks"], o["l1_final"], o["cost_unrounded"])

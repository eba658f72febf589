"""Fused peer exchange (mdot_comm_enable_peer) emulated on one GPU: the
config-4 solve (n = 16384, gbar 4096, T 16, L1 1e-6) row-sharded over G
virtual ranks whose CTAs share ONE cooperative launch (k_persist_peer), vs
the single-rank persistent kernel (G = 1).  All ranks' K1 work runs on the
same GPU, so the K1 phase stays ~n^2 work per evaluation; what this measures
is the cost of the in-kernel exchange protocol (column totals + row scalars
pushed to every rank's receive block, system-scope flags, rank-ordered
sums, the replicated column finalize) per evaluation, and that the sharded
solve reaches the single-GPU result.  NVLink transfer time is not in it."""
import json
import sys
import threading

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

inst = S.config4(0)
n = inst.n
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=0)
opts = dict(eps=1e-6, time_kernels=1)
dev = torch.device("cuda", 0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
r, c = t(inst.r), t(inst.c)
names = ["ctrl+prep", "k1", "finalize+exchange", "combine"]


def stages(res):
    k = max(1, res["stage_samples"])
    return {nm: round(1000.0 * res["stage_ms"][q] / k, 2) for q, nm in enumerate(names)}


out = {}
C = t(inst.C)
for rep in range(2):
    res = M.mdot_solve(C, r, c, schedule=sched, options=M.options(**opts))
out["G1"] = {"seconds": res["seconds"], "evaluations": res["evaluations"], "cost": res["cost_unrounded"],
             "l1": res["l1_final"], "control_path": res["control_path"], "stage_us": stages(res)}
print("G1", out["G1"], flush=True)
del C
torch.cuda.empty_cache()

for G in (2, 4, 8):
    rows = np.array_split(np.arange(n), G)
    slabs = [t(inst.C[int(rw[0]):int(rw[0]) + len(rw)]) for rw in rows]
    results = [None] * G
    err = [None] * G

    def run(k, reps=2):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                comm = M.mdot_comm_create_local(f"emu{G}", G, k, 0)
                M.mdot_comm_enable_peer(comm, n)
                row0, nloc = int(rows[k][0]), len(rows[k])
                for _ in range(reps):
                    res = M.mdot_solve_sharded(comm, row0, nloc, C_local=slabs[k], r=r, c=c, n=n, schedule=sched,
                                               options=M.options(**opts))
                s.synchronize()
                M.mdot_comm_destroy(comm)
                results[k] = res
        except Exception as e:  # noqa: BLE001
            err[k] = e

    ths = [threading.Thread(target=run, args=(k,)) for k in range(G)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    for e in err:
        if e is not None:
            raise e
    r0 = results[0]
    out[f"G{G}"] = {"seconds": max(x["seconds"] for x in results), "evaluations": r0["evaluations"],
                    "cost": r0["cost_unrounded"], "l1": r0["l1_final"], "control_path": r0["control_path"],
                    "identical_cost_all_ranks": all(x["cost_unrounded"] == r0["cost_unrounded"] for x in results),
                    "rel_cost_vs_G1": abs(r0["cost_unrounded"] - out["G1"]["cost"]) / out["G1"]["cost"],
                    "stage_us_rank0": stages(r0)}
    print(f"G{G}", out[f"G{G}"], flush=True)
    del slabs
    torch.cuda.empty_cache()
print("JSON " + json.dumps(out))

"""One rank's share of the row-sharded config-5 solve (n = 65536, d = 16,
on-the-fly cost): rows [0, n/G) of X on a 1-rank NCCL communicator forced
onto the sharded path (MDOT_SHARDED_SELFTEST), CUDA-graph slots with the NCCL
allreduce of [column totals | row scalars] captured in every slot.  The solve
is cut after a fixed number of evaluations; per-evaluation wall time and the
sampled stage times of the slot are reported.  With one rank the allreduce
is a local copy: the NVLink transfer of a real G-GPU run is not included."""
import json
import os
import sys
import time

os.environ["MDOT_SHARDED_SELFTEST"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
inst = S.config5(0)
n = inst.n
r, c, Y = t(inst.r), t(inst.c), t(inst.Y)
comm = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
out = {}
def run(X, m, evals):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = M.mdot_solve_sharded(comm, 0, m, X_local=X, Y=Y, scale=float(inst.scale), r=r, c=c, n=n,
                               schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                               options=M.options(eps=1e-5, max_evals=evals), check=False)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res


for G in (1, 2, 4, 8):
    m = n // G
    X = t(inst.X[:m])
    run(X, m, 20)
    # fixed costs (allocation, upload, setup, rounding) cancel in the difference
    d_lo, r_lo = run(X, m, 40)
    d_hi, r_hi = run(X, m, 140)
    ev = r_hi["evaluations"] - r_lo["evaluations"]
    out[G] = {"rows": m, "per_eval_ms": 1000.0 * (d_hi - d_lo) / max(1, ev), "evals": ev,
              "control_path": r_hi["control_path"]}
    print(G, out[G], flush=True)
    del X
    torch.cuda.empty_cache()
M.mdot_comm_destroy(comm)
t1 = out[1]["per_eval_ms"]
print("per-evaluation speedup G=8 vs 1 (one rank's work):", t1 / out[8]["per_eval_ms"])
print("JSON " + json.dumps(out))

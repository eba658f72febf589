"""Per-rank work of the row-sharded solve measured on one GPU:
one rank's evaluation kernel on its row slab (rows [0, n/G) of C or X, full
columns) for G = 1, 2, 4, 8, through mdot_solve_sharded on a 1-rank NCCL
communicator forced onto the sharded code path (MDOT_SHARDED_SELFTEST); the
solve is cut after a few evaluations (it cannot converge on a slab) and the
evaluation kernel's mean duration is read from the solver's own CUDA-event
timing.  The per-evaluation allreduce of [n column totals | 16 scalars]
cannot be measured with one GPU."""
import json
import os
import sys

os.environ["MDOT_SHARDED_SELFTEST"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
out = {}
comm = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
for name in ("cfg4", "cfg5"):
    inst = S.config4(0) if name == "cfg4" else S.config5(0)
    n = inst.n
    r, c = t(inst.r), t(inst.c)
    for G in (1, 2, 4, 8):
        m = n // G
        if name == "cfg4":
            kw = dict(C_local=t(inst.C[:m]))
        else:
            kw = dict(X_local=t(inst.X[:m]), Y=t(inst.Y), scale=float(inst.scale))
        res = M.mdot_solve_sharded(comm, 0, m, r=r, c=c, n=n, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=1),
                                   options=M.options(eps=1e-6, max_evals=6, time_kernels=1, device_control=0),
                                   check=False, **kw)
        k = res["kernel_ms"] / max(1, res["kernel_launches"])
        out[f"{name}_G{G}"] = {"rows": m, "eval_kernel_ms": k, "launches": res["kernel_launches"]}
        print(name, G, out[f"{name}_G{G}"], flush=True)
        del kw
        torch.cuda.empty_cache()
M.mdot_comm_destroy(comm)
for name in ("cfg4", "cfg5"):
    t1 = out[f"{name}_G1"]["eval_kernel_ms"]
    out[f"{name}_kernel_speedup"] = {G: t1 / out[f"{name}_G{G}"]["eval_kernel_ms"] for G in (2, 4, 8)}
print("JSON " + json.dumps(out))

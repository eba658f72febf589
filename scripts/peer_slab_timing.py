"""One rank's share of the row-sharded config-4 solve with the fused peer
exchange, measured on one GPU: rows [0, n/G) of C on a 1-rank NCCL
communicator forced onto the sharded path (MDOT_SHARDED_SELFTEST) with
mdot_comm_enable_peer, so every evaluation slot runs the real per-rank code
of k_persist_peer (K1 on the slab, F1, the exchange to itself, F2 over all n
replicated columns).  The solve cannot converge on a slab; it is cut at a
fixed number of evaluations and the device-timed phases per slot are
reported.  Missing from a real G-GPU run: the NVLink store/flag latency
(G x (n + 16) x 8 B per rank per evaluation)."""
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
inst = S.config4(0)
n = inst.n
r, c = t(inst.r), t(inst.c)
names = ["ctrl+prep", "k1", "finalize+exchange", "combine"]
comm = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
M.mdot_comm_enable_peer(comm, n)
out = {}
for G in [int(x) for x in os.environ.get("GS", "1,2,4,8").split(",")]:
    m = n // G
    C = t(inst.C[:m])
    for rep in range(2):
        res = M.mdot_solve_sharded(comm, 0, m, C_local=C, r=r, c=c, n=n,
                                   schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=1),
                                   options=M.options(eps=1e-6, max_evals=400, time_kernels=1), check=False)
    k = max(1, res["stage_samples"])
    st = {nm: round(1000.0 * res["stage_ms"][q] / k, 2) for q, nm in enumerate(names)}
    out[G] = {"rows": m, "control_path": res["control_path"], "slots": k, "stage_us": st,
              "slot_us": round(sum(st.values()), 2), "tile_m": os.environ.get("MDOT_TILE_M", "auto")}
    print(G, out[G], flush=True)
    del C
    torch.cuda.empty_cache()
M.mdot_comm_destroy(comm)
print("JSON " + json.dumps(out))

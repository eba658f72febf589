"""Beyond the BASELINE sizes: n = 32768 dense fp32 C (4 GiB, 2 x config 4 per side) -- one fused
evaluation (graph-path K1) checked on sampled rows / columns against the oracle, and a short
persistent-kernel solve (index arithmetic past 2^31 entries, 128 column tiles)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
t0 = time.time()
inst = S.config4(0, n=n)
print(f"instance n={n} built in {time.time() - t0:.1f} s", flush=True)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
C, r, c = t(inst.C), t(inst.r), t(inst.c)
U = torch.empty(n, dtype=torch.float64, device="cuda")
V = torch.empty_like(U)
gb = 512.0
res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=2), options=M.options(eps=1e-5),
                   u_out=U, v_out=V, check=False)
print("solve", res["status_name"], res["control_path"], res["evaluations"], f"{res['seconds']:.2f} s", res["l1_final"],
      flush=True)
lr, lc, fb = M.mdot_marginals(U, V, gb, C, r, c)
prob = O.OracleProblem(inst)
rng = np.random.default_rng(0)
rows = np.sort(rng.choice(n, 12, replace=False))
cols = np.sort(rng.choice(n, 12, replace=False))
sub = O.log_marginal_subset(prob, U.cpu().numpy(), V.cpu().numpy(), gb, rows=rows, cols=cols)
err_r = np.max(np.abs(np.expm1(lr.cpu().numpy()[rows] - sub["rows"])))
err_c = np.max(np.abs(np.expm1(lc.cpu().numpy()[cols] - sub["cols"])))
print(f"sampled parity: max rel err rows {err_r:.2e} cols {err_c:.2e} (gate 2e-6), fallback {fb}")
assert res["status"] == 0 and err_r <= 2e-6 and err_c <= 2e-6
print("OK")

"""Per-solve time-to-eps variance on config 4, with and without the
nvidia-smi clock sampler running (diagnostic for bench.py)."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

inst = S.config4(0)
n = inst.n
C = torch.from_numpy(inst.C).cuda()
r = torch.from_numpy(inst.r).cuda()
c = torch.from_numpy(inst.c).cuda()
U = torch.empty(n, dtype=torch.float64, device="cuda")
V = torch.empty_like(U)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)


def one(tk):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    res = M.mdot_solve(C, r, c, schedule=sched, options=M.options(eps=1e-6, time_kernels=tk), u_out=U, v_out=V)
    e1.record()
    torch.cuda.synchronize()
    k1 = res["kernel_ms"] / max(1, res["kernel_launches"]) * 1e3
    ph = [round(x, 1) for x in res["stage_ms"]]
    return (round(e0.elapsed_time(e1), 1), round((time.perf_counter() - t0) * 1e3, 1), round(k1, 1),
            res["evaluations"], res["fallbacks"], res["control_path"], ph, round(res["seconds"] * 1e3, 1))


out = {}
for _ in range(2):
    one(1)
out["plain_tk1"] = [one(1) for _ in range(4)]
out["plain_tk0"] = [one(0) for _ in range(4)]
clk = bench.ClockSampler(0)
clk.start()
out["sampler_tk1"] = [one(1) for _ in range(4)]
out["clocks"] = clk.stop()
out["after_tk1"] = [one(1) for _ in range(4)]
print("JSON " + json.dumps(out))
if len(sys.argv) > 1 and sys.argv[1] == "trace":
    import os
    os.environ["MDOT_TRACE"] = "1"
    for _ in range(6):
        print("SOLVE", one(1), file=sys.stderr, flush=True)

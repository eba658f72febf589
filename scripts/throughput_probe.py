"""Throughput-mode probe: B independent n = 4096 solves
sharing one cost C (config 3 shape, H/log n = 0.9 marginal pairs), run
(a) sequentially on the persistent kernel, (b) sequentially on the graph
path, (c) concurrently from B host threads, each on its own CUDA stream
(graph path; the ctypes call releases the GIL)."""
import os
import sys
import threading
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
em = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
base = S.config3(0, frac=0.9)
C = t(base.C)
pairs = [S.config3(i, frac=0.9) for i in range(B)]
R = [t(p.r) for p in pairs]
Cm = [t(p.c) for p in pairs]
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16)


def run_seq():
    out = []
    for b in range(B):
        out.append(M.mdot_solve(C, R[b], Cm[b], schedule=sched, options=M.options(eps=1e-6, eps_md=em)))
    torch.cuda.synchronize()
    return out


def run_threads(nthreads):
    out = [None] * B
    def work(k):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for b in range(k, B, nthreads):
                out[b] = M.mdot_solve(C, R[b], Cm[b], schedule=sched, options=M.options(eps=1e-6, eps_md=em))
            s.synchronize()
    th = [threading.Thread(target=work, args=(k,)) for k in range(nthreads)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    return out


def timed(fn, *a):
    fn(*a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn(*a)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


dt, out = timed(run_seq)
print(f"sequential persistent: {dt*1e3:.1f} ms for {B} solves, evals {sum(o['evaluations'] for o in out)}, "
      f"paths {sorted(set(o['control_path'] for o in out))}", flush=True)
os.environ["MDOT_NO_PERSIST"] = "1"
dt, out = timed(run_seq)
print(f"sequential graph: {dt*1e3:.1f} ms", flush=True)
del os.environ["MDOT_NO_PERSIST"]
Rb = torch.stack(R)
Cb = torch.stack(Cm)
dt, out = timed(lambda: M.mdot_solve_batch(C, Rb, Cb, schedule=sched, options=M.options(eps=1e-6, eps_md=em)))
print(f"mdot_solve_batch grouped (lockstep MD steps): {dt*1e3:.1f} ms ok={all(o['status'] == 0 for o in out)} "
      f"evals {sum(o['evaluations'] for o in out)} paths {sorted(set(o['control_path'] for o in out))}", flush=True)
os.environ["MDOT_NO_GROUPS"] = "1"
for w in (1, 4, 8, 16):
    os.environ["MDOT_BATCH_WORKERS"] = str(w)
    dt, out = timed(lambda: M.mdot_solve_batch(C, Rb, Cb, schedule=sched, options=M.options(eps=1e-6, eps_md=em)))
    print(f"mdot_solve_batch workers={w}: {dt*1e3:.1f} ms ok={all(o['status'] == 0 for o in out)} "
          f"evals {sum(o['evaluations'] for o in out)} paths {sorted(set(o['control_path'] for o in out))}", flush=True)
os.environ["MDOT_NO_PERSIST"] = "1"
for nt in (2, 4, 8, 16):
    if nt > B:
        break
    dt, out = timed(run_threads, nt)
    ok = all(o["status"] == 0 for o in out)
    print(f"{nt} threads graph: {dt*1e3:.1f} ms ok={ok} evals {sum(o['evaluations'] for o in out)}", flush=True)

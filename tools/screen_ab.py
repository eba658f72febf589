"""A/B of the screened on-the-fly evaluation (K2s) against the dense K2 on
config-5-shaped instances: same solve with MDOT_SCREEN=1 / 0 (read at every
solve's setup), cost, evaluations, time-to-eps, the screen statistics.
Usage: python tools/screen_ab.py [n ...]   (default 8192 65536)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as S  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402


def run(inst, screen, recipe="dot", gb=4096.0, T=16, eps=1e-5):
    os.environ["MDOT_SCREEN"] = "1" if screen else "0"
    dev = torch.device("cuda:0")
    X = torch.from_numpy(inst.X).to(dev)
    Y = torch.from_numpy(inst.Y).to(dev)
    r = torch.from_numpy(inst.r).to(dev)
    c = torch.from_numpy(inst.c).to(dev)
    U = torch.empty(inst.n, dtype=torch.float64, device=dev)
    V = torch.empty_like(U)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=T),
                       options=M.options(eps=eps, time_kernels=1), u_out=U, v_out=V, check=False, recipe=recipe)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = M.mdot_last_screen_stats()
    return res, dt, st, U.cpu().numpy(), V.cpu().numpy()


def main():
    ns = [int(a) for a in sys.argv[1:]] or [8192, 65536]
    for n in ns:
        inst = S.config5(0, n=n)
        for rep in range(2 if n <= 16384 else 1):
            out = {}
            for screen in (0, 1):
                res, dt, st, U, V = run(inst, screen)
                out[screen] = (res, U, V)
                k2 = (res["kernel_ms"] / max(res["kernel_launches"], 1))
                print(f"n={n} screen={screen} status={res['status_name']} cost={res['cost_unrounded']:.12g} "
                      f"L1={res['l1_final']:.2e} evals={res['evaluations']} fallbacks={res['fallbacks']} "
                      f"time={dt:.3f}s mean_eval_ms={k2:.3f} stats={st}", flush=True)
                if screen and st["timed"]:
                    print(f"   screened K2s mean {st['ms'] / st['timed']:.3f} ms over {st['timed']} timed, "
                          f"{st['evals']} screened evaluations", flush=True)
            c0, c1 = out[0][0]["cost_unrounded"], out[1][0]["cost_unrounded"]
            print(f"   cost rel diff {abs(c1 - c0) / c0:.2e}  max|dU| {np.abs(out[1][1] - out[0][1]).max():.2e}",
                  flush=True)


if __name__ == "__main__":
    main()

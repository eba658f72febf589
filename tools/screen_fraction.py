"""Config 5: what fraction of the n^2 entries carry mass that a marginal can see?

For MD step t of the config-5 FIXED schedule (gamma_t = 256, gbar_t = 256 t;
Lemma 2: the projection after t steps is the gbar_t problem), solve to L1 1e-5
on the GPU, then for sampled rows i compute log P_ij = U_i + V_j - gbar_t C_ij
(fp64, exact C from the fp32 coordinates) over all j, and count the entries
with log P_ij >= min(log r_i(P), log c_j) - T for several windows T (nats).
Entries below that bound change no row or column total by more than e^-T
relative each.  Also prints evaluations per MD step of the full solve.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as S  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    inst = S.config5(0)
    n = inst.n
    X = torch.from_numpy(inst.X).to(dev)
    Y = torch.from_numpy(inst.Y).to(dev)
    r = torch.from_numpy(inst.r).to(dev)
    c = torch.from_numpy(inst.c).to(dev)
    U = torch.empty(n, dtype=torch.float64, device=dev)
    V = torch.empty(n, dtype=torch.float64, device=dev)
    eps = 1e-5
    # full solve: evaluations per MD step via the trace-free counters
    t0 = time.time()
    res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                       options=M.options(eps=eps), u_out=U, v_out=V, check=False, recipe="dot")
    torch.cuda.synchronize()
    print(f"full solve {time.time() - t0:.2f}s evals {res['evaluations']} iters/step {res['iters_step']}", flush=True)
    rng = np.random.default_rng(1)
    rows = torch.from_numpy(np.sort(rng.choice(n, 256, replace=False))).to(dev)
    Xd = X.double()
    Yd = Y.double()
    ny = (Yd * Yd).sum(1)
    logc = torch.log(c)
    for t in (1, 2, 3, 4, 6, 8, 12, 16):
        gb = 256.0 * t
        res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=t),
                           options=M.options(eps=eps), u_out=U, v_out=V, check=False, recipe="dot")
        torch.cuda.synchronize()
        xs = Xd[rows]
        Cs = ((xs * xs).sum(1)[:, None] + ny[None, :] - 2.0 * xs @ Yd.T).clamp_min(0.0) * inst.scale
        L = U[rows][:, None] + V[None, :] - gb * Cs
        lr = torch.logsumexp(L, 1)
        out = [f"t={t:2d} gbar={gb:6.0f} evals={res['evaluations']:5d} status={res['status_name']}",
               f"max|log r(P)-log r|={float((lr - torch.log(r[rows])).abs().max()):.1e}"]
        for T in (30, 40, 50, 60, 80):
            thr = torch.minimum(lr[:, None], logc[None, :]) - T
            frac = float((L >= thr).double().mean())
            rowonly = float((L >= lr[:, None] - T).double().mean())
            out.append(f"T{T}: {frac:.4%} (row-only {rowonly:.4%})")
        print("  ".join(out), flush=True)


if __name__ == "__main__":
    main()

"""One small invocation of a hot-path kernel family, run by
tests/test_gpu_checked.py against the MDOT_CHECKED build of the library
(device-side bounds / invariant traps, guard bands around every workspace
buffer) and twice in a row (bitwise-identical results: a shared-memory or
cross-CTA race shows up as run-to-run differences).  Prints a digest of the
results; exits non-zero if the call fails."""
import hashlib
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

DEV = torch.device("cuda:0")


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def main(case):
    sched = M.schedule(M.MDOT_SCHED_FIXED, 256.0, T=2)
    opts = M.options(eps=1e-4)
    if case == "persist":          # k_persist: TMA ring, grid barriers, device controller (n = 600, ragged)
        inst = S.uniform_points_instance(3, 600, 2, 0, marg="dirichlet")
        res = M.mdot_solve(t(inst.C), t(inst.r), t(inst.c), schedule=sched, options=opts)
        assert res["control_path"] == 2, res["control_path"]
    elif case == "graph":          # k_ctrl / k_prep / k_eval_tma / k_finalize in CUDA-graph slots
        os.environ["MDOT_NO_PERSIST"] = "1"
        inst = S.uniform_points_instance(3, 600, 2, 1, marg="dirichlet")
        res = M.mdot_solve(t(inst.C), t(inst.r), t(inst.c), schedule=sched, options=opts)
        assert res["control_path"] == 1
    elif case == "k8":             # k_batch_solve: 2-CTA clusters, DSMEM exchange, narrow tail tile
        C, R, Cm = S.config2(0, pairs=2)
        res = M.mdot_solve_batch(t(C), t(R), t(Cm), schedule=sched, options=opts)[0]
    elif case == "otf":            # k_eval_otf<16> + on-the-fly rounding tiles
        inst = S.config5(0, n=600, d=16)
        res = M.mdot_solve(X=t(inst.X), Y=t(inst.Y), scale=inst.scale, r=t(inst.r), c=t(inst.c), schedule=sched,
                           options=opts)
    elif case == "otf_dot":        # k_eval_otf<16, DOT> + dot-form rounding tiles (Z22b), ragged n
        inst = S.config5(0, n=777, d=16)
        res = M.mdot_solve(X=t(inst.X), Y=t(inst.Y), scale=inst.scale, r=t(inst.r), c=t(inst.c), schedule=sched,
                           options=opts, recipe="dot")
    elif case == "round":          # rounding + dense plan output, exact fp64 evaluator
        inst = S.uniform_points_instance(3, 300, 2, 2, marg="dirichlet")
        P = torch.empty((300, 300), dtype=torch.float32, device=DEV)
        U = torch.zeros(300, dtype=torch.float64, device=DEV) + t(np.log(inst.r))
        V = t(np.log(inst.c))
        M.mdot_round(U, V, 64.0, t(inst.C), t(inst.r), t(inst.c), P_out=P)
        res = {"status_name": "MDOT_OK", "cost_rounded": float(P.double().sum().item())}
    elif case == "peer2":          # k_persist_peer: 2 emulated ranks in one cooperative launch
        inst = S.uniform_points_instance(3, 600, 2, 3, marg="dirichlet")
        rows = np.array_split(np.arange(600), 2)
        out = [None, None]

        def run(k):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                r0, nl = int(rows[k][0]), len(rows[k])
                comm = M.mdot_comm_create_local("san", 2, k, 0)
                M.mdot_comm_enable_peer(comm, 600)
                out[k] = M.mdot_solve_sharded(comm, r0, nl, t(inst.C[r0:r0 + nl]), t(inst.r), t(inst.c), n=600,
                                              schedule=sched, options=M.options(eps=1e-4))
                s.synchronize()
                M.mdot_comm_destroy(comm)
        th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        res = out[0]
        assert res["control_path"] == 2
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    dig = hashlib.sha256(repr(sorted((k, v) for k, v in res.items()
                                     if k in ("cost_rounded", "cost_unrounded", "evaluations", "l1_final"))).encode())
    print("case", case, res["status_name"], "digest", dig.hexdigest()[:16], flush=True)
    assert res["status_name"] == "MDOT_OK"


if __name__ == "__main__":
    main(sys.argv[1])

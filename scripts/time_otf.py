"""K2 (on-the-fly cost) per-evaluation kernel time, packed f32x2 kernel vs the
generic scalar kernel (MDOT_OTF_GENERIC), from the solver's own sampled CUDA
events over a bounded number of evaluations."""
import json
import os
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    inst = S.config5(0, n=n, d=d)
    X, Y, r, c = t(inst.X), t(inst.Y), t(inst.r), t(inst.c)
    out = {"n": n, "d": d}
    for name, generic in (("packed", False), ("generic", True)):
        if generic:
            os.environ["MDOT_OTF_GENERIC"] = "1"
        else:
            os.environ.pop("MDOT_OTF_GENERIC", None)
        res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0),
                           options=M.options(eps=1e-5, time_kernels=1, max_evals=40), check=False)
        k1 = res["kernel_ms"] / max(1, res["kernel_launches"])
        out[name] = {"k2_ms": k1, "pairs_per_s": float(n) * n / (k1 / 1e3), "launches": res["kernel_launches"],
                     "cost_unrounded": res["cost_unrounded"], "control_path": res["control_path"]}
        print(name, out[name], flush=True)
    out["speedup"] = out["generic"]["k2_ms"] / out["packed"]["k2_ms"]
    print("JSON " + json.dumps(out))


if __name__ == "__main__":
    main()

"""Write tests/golden/*.json: full fp64 ORACLE solves of the BASELINE configs.

Test infrastructure.  This script calls only `oracle/` (and the input
generators in synthetic.py, which hold none of the method's arithmetic); no
value comes from the CUDA path.  The GPU parity tests gate the CUDA solve's
unrounded cost <C, P(U,V)> at 1e-5 relative against these files (north_star /
DESIGN.md Z20) and its rounded cost with the Z20 rounding allowance.

Usage: python scripts/make_golden.py cfg4 [cfg3_h0.5 cfg3_h0.9 cfg3_h0.99 ...]
       (OMP_NUM_THREADS sets the oracle's threads; config 4 takes ~15-30 min
       on 8 cores).
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synthetic as S  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

# name -> (instance builder, gamma_bar, T, eps, description)
CASES = {
    "cfg4_seed0": (lambda: S.config4(0), 4096.0, 16, 1e-6,
                   "BASELINE config 4: n=16384, X,Y~U[0,1]^2, C=d^2/max fp32, Dirichlet(1), FIXED gbar 4096 T 16, L1 1e-6"),
    "cfg3_h0.5_seed0": (lambda: S.config3(0, frac=0.5), 4096.0, 16, 1e-6,
                        "BASELINE config 3: n=4096, H(r)/log n = 0.5, FIXED gbar 4096 T 16, L1 1e-6"),
    "cfg3_h0.9_seed0": (lambda: S.config3(0, frac=0.9), 4096.0, 16, 1e-6,
                        "BASELINE config 3: n=4096, H(r)/log n = 0.9, FIXED gbar 4096 T 16, L1 1e-6"),
    "cfg3_h0.99_seed0": (lambda: S.config3(0, frac=0.99), 4096.0, 16, 1e-6,
                         "BASELINE config 3: n=4096, H(r)/log n = 0.99, FIXED gbar 4096 T 16, L1 1e-6"),
    "cfg3_h0.5_gb512_T4_seed1": (lambda: S.config3(1, frac=0.5), 512.0, 4, 1e-6,
                                 "BASELINE config 3 secondary: n=4096, H/log n = 0.5, FIXED gbar 512 T 4, L1 1e-6"),
    "cfg2_s0_p0_eps1e-8": (lambda: S.config2_pair(0, 0), 4096.0, 16, 1e-8,
                           "BASELINE config 2: n=784 28x28 grid, blob pair 0 of seed 0, FIXED gbar 4096 T 16, L1 1e-8"),
    "cfg2_s0_p1_eps1e-8": (lambda: S.config2_pair(0, 1), 4096.0, 16, 1e-8,
                           "BASELINE config 2: n=784 28x28 grid, blob pair 1 of seed 0, FIXED gbar 4096 T 16, L1 1e-8"),
}


def sha16(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def run(name):
    build, gb, T, eps, desc = CASES[name]
    inst = build()
    prob = O.OracleProblem(inst)
    t0 = time.time()
    U, V, res, _ = O.mdot(prob, O.schedule_fixed(gb, T=T), O.make_options(eps=eps))
    secs = time.time() - t0
    out = {
        "name": name, "description": desc, "n": int(inst.n), "instance": inst.name,
        "gamma_bar": gb, "T": T, "eps": eps, "projector": "PNCG", "beta": "PPR (Z6)", "c1": 0.1, "c2": 0.4,
        "warm": "scaled (Z4)",
        "status": res["status_name"], "cost_unrounded": res["cost_unrounded"],
        "cost_rounded": res["cost_rounded"], "l1_final": res["l1_final"], "rho_final": res["rho_final"],
        "evaluations": res["evaluations"], "iterations": res["iterations"], "md_steps": res["md_steps"],
        "oracle_seconds": secs, "oracle_threads": os.environ.get("OMP_NUM_THREADS", "default"),
        "generator": "scripts/make_golden.py (calls oracle/ only)",
        "oracle_source_sha16": sha16(os.path.join(ROOT, "oracle", "mdot_oracle.c")),
    }
    os.makedirs(GOLDEN, exist_ok=True)
    with open(os.path.join(GOLDEN, name + ".json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("name", "status", "cost_unrounded", "evaluations", "oracle_seconds")}),
          flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CASES):
        run(nm)

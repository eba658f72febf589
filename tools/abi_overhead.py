"""Per-call overhead of the C ABI entry points at config-4 size: mdot_marginals
(one evaluation) back to back, and the fixed cost of a solve (alloc, input
checks, setup), host wall clock around synchronous calls."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
inst = S.config4(0, n=n)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
C, r, c = t(inst.C), t(inst.r), t(inst.c)
U, V = torch.log(r).clone(), torch.log(c).clone()
lr = torch.empty(n, dtype=torch.float64, device="cuda")
lc = torch.empty_like(lr)
for _ in range(5):
    M.mdot_marginals(U, V, 64.0, C, r, c, lr=lr, lc=lc)
torch.cuda.synchronize()
t0 = time.perf_counter()
K = 100
for _ in range(K):
    M.mdot_marginals(U, V, 64.0, C, r, c, lr=lr, lc=lc)
torch.cuda.synchronize()
print(f"mdot_marginals n={n}: {1e6 * (time.perf_counter() - t0) / K:.1f} us per call")

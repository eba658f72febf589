"""One K2 evaluation at config-5 size (for ncu captures)."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
d = int(sys.argv[2]) if len(sys.argv) > 2 else 16
inst = S.config5(0, n=n, d=d)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
A = t(np.log(inst.r))
B = t(np.log(inst.c))
lr, lc, fb = M.mdot_marginals(A, B, 4096.0, X=t(inst.X), Y=t(inst.Y), scale=inst.scale, r=t(inst.r), c=t(inst.c))
torch.cuda.synchronize()
print("ok", fb)

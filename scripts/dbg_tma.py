import os, sys, time
sys.path.insert(0, '/root/repo')
os.environ['MDOT_DEBUG'] = '1'
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
inst = S.uniform_points_instance(3, 2048, 2, 1, marg="dirichlet")
t = lambda x: torch.from_numpy(x).cuda()
A = torch.from_numpy(np.log(inst.r)).cuda(); B = torch.from_numpy(np.log(inst.c)).cuda()
lr, lc, fb = M.mdot_marginals(A, B, 64.0, t(inst.C), t(inst.r), t(inst.c))
print("ok", fb, lr[:3])

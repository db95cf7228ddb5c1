"""cProfile of one short ML-CPCP solve: where the fixed per-solve host time goes."""
import cProfile
import pstats
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else 'C4'
d, mask = make_config(name); c = CONFIGS[name]; m, n = d.shape
D = torch.from_numpy(d).cuda(); om = pkg.ObservationMask(mask)
lam = 1 / np.sqrt(max(m, n))
opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=c['tol'], max_iters=10,
                       levels=c['n_coarse'], collect_rank=False)
pkg.ml_fwt_solve(D, om, opts)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
pkg.ml_fwt_solve(D, om, opts)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(22)

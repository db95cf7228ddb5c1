"""One ML-CPCP C4 solve (40 iterations) for ncu captures of its kernels."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS
d, mask = make_config("C4"); c = CONFIGS["C4"]; m, n = d.shape
D = torch.from_numpy(d).cuda(); om = pkg.ObservationMask(mask); lam = 1 / np.sqrt(max(m, n))
pkg.ml_fwt_solve(D, om, pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=c["tol"], max_iters=40,
                                        levels=c["n_coarse"], collect_rank=False))
torch.cuda.synchronize()

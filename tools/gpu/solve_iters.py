import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS
name = sys.argv[1]
d, mask = make_config(name); c = CONFIGS[name]; m, n = d.shape
D = torch.from_numpy(d).cuda()
if c['solver'] == 'cpcp':
    lam = 1/np.sqrt(max(m, n))
    st = pkg.ml_fwt_solve(D, pkg.ObservationMask(mask), pkg.CpcpOptions(lambda_l=lam, lambda_s=lam/np.sqrt(max(m, n)), tol=c['tol'], max_iters=int(sys.argv[2]), levels=c['n_coarse'], collect_rank=False, check_every=1))
else:
    st = pkg.ml_ialm_solve(D, pkg.PcpOptions(lam=1/np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'], max_iters=int(sys.argv[2]), check_every=1))
torch.cuda.synchronize(); print('iters', st.iter)

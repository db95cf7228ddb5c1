import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import cpcp as CP
from paper_2206_13369_b200.datasets import make_config, CONFIGS
for name, its in [('C3', 5000), ('C4', 300)]:
    d, mask = make_config(name); c = CONFIGS[name]; m, n = d.shape
    D = torch.from_numpy(d).cuda(); om = pkg.ObservationMask(mask)
    lam = 1/np.sqrt(max(m, n))
    opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam/np.sqrt(max(m, n)), tol=c['tol'], max_iters=its, levels=c['n_coarse'], collect_rank=False)
    pkg.ml_fwt_solve(D, om, pkg.CpcpOptions(lambda_l=lam, lambda_s=lam/np.sqrt(max(m, n)), tol=c['tol'], max_iters=20, levels=c['n_coarse'], collect_rank=False))
    sink = []; CP.TIMING_SINK = sink
    torch.cuda.synchronize(); t = time.time(); st = pkg.ml_fwt_solve(D, om, opts); torch.cuda.synchronize(); dt = time.time() - t
    CP.TIMING_SINK = None
    s = sink[0]; it = s['iters']
    print(name, 'iters', st.iter, 'solve %.3fs' % dt, 'ms/iter %.3f' % (1e3 * dt / st.iter), {k: round(v[0] / it, 4) for k, v in s.items() if isinstance(v, tuple)}, flush=True)

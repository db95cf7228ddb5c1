"""Per-step wall time of the e2e path (pinned host D in, host L/S/Y out)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS
d, _ = make_config('C2'); c = CONFIGS['C2']
opts = pkg.PcpOptions(lam=1/np.sqrt(2000), tol_feasibility=c['tol'], levels=c['n_coarse'])
d_pin = torch.from_numpy(d).pin_memory()
D = d_pin.cuda()
for w in range(2): pkg.ml_ialm_solve(D, opts)
for rep in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = pkg.ml_ialm_solve(d_pin, opts)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print('e2e wall ms %.2f' % ((t1 - t0) * 1e3), type(st.l), st.l.is_pinned(), flush=True)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = pkg.ml_ialm_solve(D, opts)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print('device wall ms %.2f' % ((t1 - t0) * 1e3), flush=True)

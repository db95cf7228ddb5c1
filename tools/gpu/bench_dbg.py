import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.datasets import make_config, CONFIGS
d, _ = make_config('C2'); c = CONFIGS['C2']
D = torch.from_numpy(d).cuda()
opts = pkg.PcpOptions(lam=1/np.sqrt(2000), tol_feasibility=c['tol'], levels=c['n_coarse'])
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device='cuda')
for w in range(3): pkg.ml_ialm_solve(D, opts)
for sinkon in (False, True):
    for rep in range(4):
        P.TIMING_SINK = [] if sinkon else None
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record(); st = pkg.ml_ialm_solve(D, opts); e1.record(); e1.synchronize()
        print('sink', sinkon, 'ev ms %.2f wall ms %.2f' % (e0.elapsed_time(e1), (time.perf_counter()-t0)*1e3), st.iter, flush=True)
P.TIMING_SINK = None

import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS
d, _ = make_config('C2'); c = CONFIGS['C2']
opts = pkg.PcpOptions(lam=1/np.sqrt(2000), tol_feasibility=c['tol'], levels=c['n_coarse'])
d_pin = torch.from_numpy(np.ascontiguousarray(d)).pin_memory()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device='cuda')
for w in range(3): pkg.ml_ialm_solve(d_pin, opts)
for mode in ('flush', 'noflush', 'flush'):
    ts = []
    for rep in range(5):
        if mode == 'flush': flush.fill_(1.0)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = pkg.ml_ialm_solve(d_pin, opts)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print(mode, ['%.1f' % t for t in ts], flush=True)

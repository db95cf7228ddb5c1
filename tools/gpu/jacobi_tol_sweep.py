import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from oracle import mlrpca_oracle as O
from paper_2206_13369_b200.datasets import make_config, CONFIGS
d, _ = make_config('C2'); c = CONFIGS['C2']
ref = O.ml_ialm(d.astype(np.float64), lam=1/np.sqrt(2000), tol=c['tol'], levels=c['n_coarse'])
D = torch.from_numpy(d).cuda()
for jt in [1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4]:
    opts = pkg.PcpOptions(lam=1/np.sqrt(2000), tol_feasibility=c['tol'], levels=c['n_coarse'], jacobi_tol=jt)
    pkg.ml_ialm_solve(D, opts)
    sink = []; P.TIMING_SINK = sink
    torch.cuda.synchronize(); t = time.time(); st = pkg.ml_ialm_solve(D, opts); torch.cuda.synchronize(); dt = time.time() - t
    P.TIMING_SINK = None
    rl = np.linalg.norm(st.l.cpu().numpy() - ref.l) / np.linalg.norm(ref.l); rs = np.linalg.norm(st.s.cpu().numpy() - ref.s) / np.linalg.norm(ref.s)
    s = sink[0]
    print(f'jtol {jt:.0e} iters {st.iter}/{ref.iter} relL {rl:.2e} relS {rs:.2e} rank {st.history[-1].rank_l}/{ref.history[-1].rank_l} solve {dt*1e3:.1f} ms jac/iter {s["jacobi"][0]/s["iters"]:.3f} ms sweeps {np.mean(s["jac_sweeps"]):.2f}', flush=True)
d, _ = make_config('C1'); c = CONFIGS['C1']
ref = O.ml_ialm(d, lam=1/np.sqrt(500), tol=c['tol'], levels=c['n_coarse'])
for jt in [1.4e-14, 1e-13, 1e-12, 1e-11]:
    opts = pkg.PcpOptions(lam=1/np.sqrt(500), tol_feasibility=c['tol'], levels=c['n_coarse'], jacobi_tol=jt)
    sink = []; P.TIMING_SINK = sink
    st = pkg.ml_ialm_solve(d, opts)
    P.TIMING_SINK = None
    rl = np.linalg.norm(st.l - ref.l) / np.linalg.norm(ref.l)
    s = sink[0]
    print(f'C1 jtol {jt:.0e} iters {st.iter}/{ref.iter} relL {rl:.2e} sweeps {np.mean(s["jac_sweeps"]):.2f} jac/iter {s["jacobi"][0]/s["iters"]:.3f} ms', flush=True)

import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import _lib
from paper_2206_13369_b200.datasets import make_config, CONFIGS
lib = _lib.load()
for name in sys.argv[1:]:
    d, _ = make_config(name); c = CONFIGS[name]; m, n = d.shape
    D = torch.from_numpy(d).cuda()
    opts = pkg.PcpOptions(lam=1/np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
    pkg.ml_ialm_solve(D, opts); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    lib.mlr_debug_j2prof(buf)
    buf2 = (ctypes.c_ulonglong * 8)()
    lib.mlr_debug_j2prof2(buf2)
    st = pkg.ml_ialm_solve(D, opts); torch.cuda.synchronize()
    lib.mlr_debug_j2prof(buf)
    lib.mlr_debug_j2prof2(buf2)
    v = list(buf); steps = max(v[5], 1)
    names = ["A_load", "A_Q", "bar1", "B_apply", "bar2", "steps", "A_publish", "A_rounds"]
    print(name, 'iters', st.iter, 'steps', steps, {names[i]: round(v[i] / steps) for i in (0, 7, 1, 6, 2, 3, 4)}, 'total cycles/step', round(sum(v[i] for i in (0,1,2,3,4,6,7)) / steps), flush=True)
    if v[10]:
        print('   pipelined rounds', v[10], 'rotation warp cycles/round', round(v[8]/v[10]), 'update thread', round(v[9]/v[10]), 'incl barrier', round(v[11]/v[10]), flush=True)
    if v[15]:
        print('   worker CTA (last): barrier wait/step', round(v[12] / steps), 'setup+grabs/step', round(v[13] / steps),
              'items/step', round(v[15] / steps, 2), 'cycles/item', round(v[14] / v[15]), flush=True)
        w2 = list(buf2)
        print('   worker setup split/step: qflag+maps', round(w2[0] / steps), 'dmark+critical list', round(w2[1] / steps),
              'to first/next item', round(w2[2] / steps), flush=True)

"""C5 ML-PCP parity numbers against the reference fixture (the gate itself is
tests/test_gpu_large.py::test_c5_ml_ialm_vs_reference_fixture), for both
coarse eigensolvers (MLR_EIG read at plan creation)."""
import os
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import test_gpu_large as T
import torch
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import CONFIGS, make_config

g = T.fixture("c5_pcp")
c = CONFIGS["C5"]
d, _ = make_config("C5", int(g["seed"]))
D = torch.from_numpy(d).cuda()
del d
for eig in sys.argv[1:] or ["trd", "jacobi"]:
    os.environ["MLR_EIG"] = eig
    st = pkg.ml_ialm_solve(D, pkg.PcpOptions(lam=1 / np.sqrt(c["m"]), tol_feasibility=c["tol"], levels=c["n_coarse"]))
    rows = g["rows"]
    lk = T.device_sketches(st.l, "l")
    sk = T.device_sketches(st.s, "s")
    ranks = [h.rank_l for h in st.history]
    print(eig, "iters", st.iter, "ref", int(g["iter"]), "rank column equal", ranks == [int(x) for x in g["h_rank"]],
          "relF rows L %.2e S %.2e" % (T.relf(st.l[rows].cpu().numpy(), g["l_rows"]), T.relf(st.s[rows].cpu().numpy(), g["s_rows"])),
          "sketch L %.2e S %.2e" % (T.relf(lk["l_q"], g["l_q"]), T.relf(sk["s_q"], g["s_q"])), flush=True)

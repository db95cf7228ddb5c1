"""C5 (or another PCP config) solve time, Jacobi sweeps per iteration and
parity against the C5 reference fixture (rank column, relF of the fixed rows
and the L sketch).  Used for the eigensolver experiments in DESIGN.md 4."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2206_13369_b200 as pkg  # noqa: E402
from paper_2206_13369_b200 import pcp as P  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402
from test_gpu_large import device_sketches, relf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
c = CONFIGS[name]
g = np.load(os.path.join(ROOT, "tests", "golden", "c5_pcp.npz")) if name == "C5" else None
d, _ = make_config(name, int(g["seed"]) if g is not None else 0)
D = torch.from_numpy(d).cuda()
opts = pkg.PcpOptions(lam=1 / np.sqrt(c["m"]), tol_feasibility=c["tol"], levels=c["n_coarse"])
pkg.ml_ialm_solve(D, opts)
P.TIMING_SINK = []
torch.cuda.synchronize()
t0 = time.perf_counter()
st = pkg.ml_ialm_solve(D, opts)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
t = P.TIMING_SINK[-1]
ranks = [h.rank_l for h in st.history]
line = (f"{name} env={ {k: v for k, v in os.environ.items() if k.startswith('MLR_')} }: solve {wall * 1e3:.1f} ms, iters {st.iter}, "
        f"sweeps {t['jac_sweeps']} (sum {sum(abs(x) for x in t['jac_sweeps'])}), "
        f"phases { {k: round(v, 1) for k, v in t.items() if isinstance(v, float)} }")
print(line)
if g is not None:
    rows = g["rows"]
    sk = device_sketches(st.l, "l")
    print(f"   ref iters {int(g['iter'])}, rank column equal {ranks == [int(x) for x in g['h_rank']]}, "
          f"ranks {ranks}, relF rows L {relf(st.l[rows].cpu().numpy(), g['l_rows']):.2e} "
          f"S {relf(st.s[rows].cpu().numpy(), g['s_rows']):.2e}, L_q {relf(sk['l_q'], g['l_q']):.2e}")

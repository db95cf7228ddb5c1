"""Numbers behind the full-size parity tests (tests/test_gpu_large.py): the
GPU solve of C5 / C3 / C4 against the reference fixtures (relF of fixed rows
and sketches, iteration counts, rank column, objective vs envelope)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2206_13369_b200 as pkg  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402
from test_gpu_large import device_sketches, relf  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
for name in sys.argv[1:] or ["C5", "C3", "C4"]:
    path = os.path.join(G, f"{name.lower()}_{'pcp' if name == 'C5' else 'cpcp'}.npz")
    if not os.path.exists(path):
        print(name, "fixture missing")
        continue
    g = np.load(path)
    c = CONFIGS[name]
    d, mask = make_config(name, int(g["seed"]))
    D = torch.from_numpy(d).cuda()
    if name == "C5":
        st = pkg.ml_ialm_solve(D, pkg.PcpOptions(lam=1 / np.sqrt(c["m"]), tol_feasibility=c["tol"],
                                                 levels=c["n_coarse"]))
        ranks = [h.rank_l for h in st.history]
        print(f"{name}: iterations {st.iter} (ref {int(g['iter'])}), rank column equal "
              f"{ranks == [int(x) for x in g['h_rank']]}, final rank {ranks[-1]}")
    else:
        cap = int(g["max_iters"])
        st = pkg.ml_fwt_solve(D, pkg.ObservationMask(mask), pkg.CpcpOptions(
            lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=c["tol"], max_iters=cap,
            levels=c["n_coarse"], collect_rank=False))
        eo = np.asarray(g["env_obj"])
        print(f"{name}: iterations {st.iter} (envelope {list(g['env_iter'])}), objective rel diff "
              f"{abs(st.objective_history[-1] - eo[0]) / eo[0]:.2e} (envelope spread {(eo.max() - eo.min()) / eo[0]:.2e})")
    rows = g["rows"]
    for tag, X in (("l", st.l), ("s", st.s)):
        sk = device_sketches(X, tag)
        print(f"   relF {tag.upper()} rows {relf(X[rows].cpu().numpy(), g[tag + '_rows']):.2e} sketch q "
              f"{relf(sk[tag + '_q'], g[tag + '_q']):.2e} p {relf(sk[tag + '_p'], g[tag + '_p']):.2e} fro "
              f"{abs(sk[tag + '_fro'] - float(g[tag + '_fro'])) / float(g[tag + '_fro']):.2e}")
    del D, st
    torch.cuda.empty_cache()

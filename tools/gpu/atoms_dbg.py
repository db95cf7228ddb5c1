import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from oracle import mlrpca_oracle as O
for name in ["atoms_ml_f64", "atoms_full_f64"]:
    g = dict(np.load(f'/root/repo/tests/golden/{name}.npz'))
    nh = int(g["n_coarse"]) or None
    opts = pkg.CpcpOptions(lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=1e-9,
                           max_iters=int(g["max_iters"]), levels=nh, collect_rank=False, track_oracle_atoms=True)
    fn = pkg.fwt_solve if nh is None else pkg.ml_fwt_solve
    st = fn(g["d"], pkg.ObservationMask(g["mask"]), opts)
    r = [np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(st.oracle_atoms, g["atoms"])]
    print(name, st.iter, ["%.1e" % x for x in r])
    print(" obj", np.array(st.objective_history[:6]) / g["h_obj"][:6] - 1)

"""Per-CTA timeline of the cooperative Jacobi (C5) over one sweep: for each
step, every CTA's barrier arrival relative to the previous release, grouped
by role (pair owner / worker) and phase-B items processed; the barrier's own
latency (release - last arrival).  Uses mlr_debug_j2trace (globaltimer)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2206_13369_b200 as pkg  # noqa: E402
from paper_2206_13369_b200 import _lib  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
g0 = int(sys.argv[2]) if len(sys.argv) > 2 else 80
n = int(sys.argv[3]) if len(sys.argv) > 3 else 80
nctas = int(os.environ.get("NCTAS", "296"))
obase = int(os.environ.get("OBASE", "0"))
lib = _lib.load()
d, _ = make_config(name)
c = CONFIGS[name]
D = torch.from_numpy(d).cuda()
opts = pkg.PcpOptions(lam=1 / np.sqrt(c["m"]), tol_feasibility=c["tol"], levels=c["n_coarse"])
pkg.ml_ialm_solve(D, opts)
buf = torch.zeros(n * nctas * 8, dtype=torch.int64, device="cuda")
lib.mlr_debug_j2trace(ctypes.c_void_p(buf.data_ptr()), g0, n)
pkg.ml_ialm_solve(D, opts)
torch.cuda.synchronize()
lib.mlr_debug_j2trace(ctypes.c_void_p(0), 0, 0)
t = buf.cpu().numpy().reshape(n, nctas, 8).astype(np.float64)
owners = (np.arange(nctas) >= obase) & (np.arange(nctas) < obase + 40)
arr_o, arr_w, lat, by_items = [], [], [], {}
for s in range(1, n):
    rel_prev = t[s - 1, :, 1].min()
    if rel_prev == 0 or t[s, :, 0].min() == 0:
        continue
    a = t[s, :, 0] - rel_prev
    arr_o.append(np.median(a[owners]))
    arr_w.append(np.median(a[~owners]))
    lat.append(t[s, :, 1].min() - t[s, :, 0].max())
    last = int(np.argmax(a))
    items = t[s - 1, :, 2]  # items of step s-1 are done before arriving at step s's barrier
    for k in np.unique(items[~owners]):
        by_items.setdefault(int(k), []).append(np.median(a[~owners & (items == k)]))
    if s < 6:
        print(f"step {g0 + s}: last arrival CTA {last} ({'owner' if owners[last] else 'worker'}, items {int(items[last])}) "
              f"at {a.max() / 1e3:.2f} us; owners median {np.median(a[owners]) / 1e3:.2f}, workers median "
              f"{np.median(a[~owners]) / 1e3:.2f}, barrier latency {lat[-1] / 1e3:.2f} us")
print(f"over {len(lat)} steps: owner arrival {np.mean(arr_o) / 1e3:.2f} us, worker arrival {np.mean(arr_w) / 1e3:.2f} us, "
      f"barrier latency {np.mean(lat) / 1e3:.2f} us, step {np.mean([t[s, :, 1].min() - t[s - 1, :, 1].min() for s in range(1, n) if t[s - 1, :, 1].min() > 0]) / 1e3:.2f} us")
for k in sorted(by_items):
    print(f"   workers with {k} items: median arrival {np.mean(by_items[k]) / 1e3:.2f} us")

# owner timeline (median over owners and steps), relative to the previous release
seg = {"start": [], "load/quadrant": [], "rounds+Q": [], "wflag wait": [], "publish->arrive": []}
for s_ in range(1, n):
    rel = t[s_ - 1, :, 1].min()
    if rel == 0:
        continue
    o = t[s_, obase:obase + 40]
    seg["start"].append(np.median(o[:, 3] - rel))
    seg["load/quadrant"].append(np.median(o[:, 4] - o[:, 3]))
    seg["rounds+Q"].append(np.median(o[:, 5] - o[:, 4]))
    w = o[:, 6] > 0
    seg["wflag wait"].append(np.median(o[w, 6] - o[w, 5]) if w.any() else 0.0)
    seg["publish->arrive"].append(np.median(o[:, 0] - np.where(w, o[:, 6], o[:, 5])))
print("owner segments (us):", {k: round(np.mean(v) / 1e3, 2) for k, v in seg.items() if v})

sm = t[1, :, 7].astype(int)
owner_sms = sm[owners]
others = sm[~owners]
shared = sum(1 for x in owner_sms if x in set(others))
print(f"SM placement: {len(set(sm))} distinct SMs for {nctas} CTAs; owners on SMs shared with a worker: {shared} of {owners.sum()}")
if os.environ.get("SMDUMP"):
    for c in range(nctas):
        mates = [int(x) for x in np.nonzero(sm == sm[c])[0] if x != c]
        print(f"cta {c} sm {sm[c]} mates {mates}")

# per-owner rounds+Q time, split by what shares the owner's SM
rq = []
for s_ in range(1, n):
    if t[s_ - 1, :, 1].min() == 0:
        continue
    o = t[s_, obase:obase + 40]
    rq.append(o[:, 5] - o[:, 4])
rq = np.mean(rq, axis=0) / 1e3
own_idx = np.arange(obase, obase + 40)
dbl = np.array([any(owners[x] for x in np.nonzero(sm == sm[c])[0] if x != c) for c in own_idx])
print(f"rounds+Q per owner: owner-mate {rq[dbl].mean() if dbl.any() else float('nan'):.2f} us ({dbl.sum()}), "
      f"worker-mate {rq[~dbl].mean() if (~dbl).any() else float('nan'):.2f} us ({(~dbl).sum()}); max {rq.max():.2f}")

"""The product host loops (run_ialm / run_fwt) driven by the CPU emulation of
the device steps (tests/emu_backend.py): validates the GPU formulation
(Gram-based coarse SVT, exact residual recomputation, coarse QP dots) and the
loop control against the oracle, on CPU."""

import numpy as np
import pytest
import torch

from emu_backend import EmuCpcp, EmuPcp
from oracle import mlrpca_oracle as O
from paper_2206_13369_b200 import api_types as T
from paper_2206_13369_b200 import chain as CH
from paper_2206_13369_b200 import cpcp as C
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.runtime import SINGLE


def run_pcp_emu(d, nh, tol, max_iters=500):
    m, n = d.shape
    be = EmuPcp(CH.build_chain(n, nh), m, m, d.dtype == np.float32, max_iters)
    opts = T.PcpOptions(levels=nh, tol_feasibility=tol, max_iters=max_iters)
    return P.run_ialm(be, SINGLE, torch.from_numpy(d), m, n, opts, 1 / np.sqrt(max(m, n)), 3)


@pytest.mark.parametrize("name", ["pcp_f64_small", "pcp_f64_odd"])
def test_emulated_pcp_matches_golden(golden, name):
    g = golden(name)
    L, S, Y, st, h = run_pcp_emu(g["d"], int(g["n_coarse"]), float(g["tol"]))
    assert st["k"] == int(g["iter"])
    assert np.linalg.norm(L.numpy() - g["l"]) / np.linalg.norm(g["l"]) < 1e-10
    assert np.linalg.norm(S.numpy() - g["s"]) / np.linalg.norm(g["s"]) < 1e-10
    assert np.allclose(h[:, 0], g["h_gap"], rtol=1e-8)
    assert list(h[:, 2].astype(int)) == list(g["h_rank"])
    assert np.isclose(st["mu_final"], float(g["mu"]), rtol=1e-12)


def test_emulated_pcp_max_iters_and_zero():
    d, _ = O.gaussian_rpca(60, 48, 3, 0.1, 2)
    L, S, Y, st, h = run_pcp_emu(d, 12, 1e-12, max_iters=5)
    assert st["k"] == 5 and st["done"] == 2
    z = np.zeros((10, 8))
    be = EmuPcp(CH.build_chain(8, 4), 10, 10, False, 10)
    assert P.run_ialm(be, SINGLE, torch.from_numpy(z), 10, 8, T.PcpOptions(levels=4), 0.3, 2) is None


def test_emulated_pcp_rejects_nonfinite():
    d = np.ones((8, 8))
    d[3, 3] = np.nan
    be = EmuPcp(CH.build_chain(8, 4), 8, 8, False, 10)
    with pytest.raises(ValueError, match="non-finite"):
        P.run_ialm(be, SINGLE, torch.from_numpy(d), 8, 8, T.PcpOptions(levels=4), 0.3, 2)


def test_emulated_fwt_first_iteration_exact_and_envelope(golden):
    g = golden("fwt_f64_small")
    d, mask = g["d"], g["mask"]
    m, n = d.shape
    nh = int(g["n_coarse"])
    ch = CH.build_chain(n, nh)
    be = EmuCpcp(ch, m, m, 0, False, int(g["max_iters"]), 1)
    bits = torch.from_numpy(T.ObservationMask(mask).packed_bits().view(np.int32))
    opts = T.CpcpOptions(lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=float(g["tol"]),
                         max_iters=int(g["max_iters"]), levels=nh, collect_rank=False)
    L, S, st, h, objs = C.run_fwt(be, SINGLE, torch.from_numpy(d), bits, m, opts, 1 / ch.sigma_max(), 4)
    ref = g["h_obj"]
    # iteration 1 follows the reference to rounding; later iterations fork on
    # l1 arg-max ties: envelope gate
    assert abs(objs[0] - ref[0]) <= 1e-12 * ref[0]
    assert abs(st["k"] - int(g["iter"])) <= max(2, int(0.05 * int(g["iter"])))
    assert abs(objs[-1] - ref[-1]) / ref[-1] < 1e-4

"""Row-sharded (N > 1) host path on CPU: two processes over gloo run the
product host loops with the emulated device steps; the all-reduced Gram /
statistics and the gathered l1 arg-max must reproduce the unsharded run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, out_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    from emu_backend import EmuCpcp, EmuPcp
    from oracle import mlrpca_oracle as O
    from paper_2206_13369_b200 import api_types as T
    from paper_2206_13369_b200 import chain as CH
    from paper_2206_13369_b200 import cpcp as C
    from paper_2206_13369_b200 import pcp as P
    from paper_2206_13369_b200.runtime import Comm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm()
        budget = kind.endswith("_budget")
        kind = kind.replace("_budget", "")
        if kind == "pcp":
            d, _ = O.gaussian_rpca(96, 80, 5, 0.1, 21)
            m, n = d.shape
            r0, r1 = rank * m // world, (rank + 1) * m // world
            be = EmuPcp(CH.build_chain(n, 20), r1 - r0, m, False, 200)
            opts = T.PcpOptions(levels=20, tol_feasibility=1e-7, time_budget=1000.0 if budget else None)
            if budget and rank == 1:
                be.clock_skew = 1e6  # only this rank's clock says the budget is spent
            L, S, Y, st, h = P.run_ialm(be, comm, torch.from_numpy(np.ascontiguousarray(d[r0:r1])), m, n, opts,
                                        1 / np.sqrt(max(m, n)), 2)
            out_q.put((rank, r0, L.numpy(), S.numpy(), st["k"], h[:, 0].copy()))
        else:
            d, mask = O.gaussian_rpca(96, 80, 4, 0.1, 22, observe=0.8)
            m, n = d.shape
            r0, r1 = rank * m // world, (rank + 1) * m // world
            ch = CH.build_chain(n, 20)
            be = EmuCpcp(ch, r1 - r0, m, r0, False, 300, world)
            bits = torch.from_numpy(T.ObservationMask(mask[r0:r1]).packed_bits().view(np.int32))
            lam = 1 / np.sqrt(m)
            opts = T.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(m), tol=1e-6, max_iters=300, levels=20,
                                 collect_rank=False, time_budget=1000.0 if budget else None)
            if budget and rank == 1:
                be.clock_skew = 1e6
            L, S, st, h, objs = C.run_fwt(be, comm, torch.from_numpy(np.ascontiguousarray(d[r0:r1])), bits, m,
                                          opts, 1 / ch.sigma_max(), 3)
            out_q.put((rank, r0, L.numpy(), S.numpy(), st["k"], np.array(objs)))
    finally:
        dist.destroy_process_group()


def _run(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def _single(kind):
    return _run(kind, 1)[0]


@pytest.mark.timeout(600)
def test_pcp_row_sharded_matches_single():
    one = _single("pcp")
    two = _run("pcp", 2)
    assert two[0][4] == two[1][4] == one[4]
    L = np.concatenate([r[2] for r in two])
    S = np.concatenate([r[3] for r in two])
    assert np.linalg.norm(L - one[2]) / np.linalg.norm(one[2]) < 1e-10
    assert np.linalg.norm(S - one[3]) / np.linalg.norm(one[3]) < 1e-10
    assert np.allclose(two[0][5], one[5], rtol=1e-9)


@pytest.mark.timeout(600)
def test_cpcp_row_sharded_matches_single():
    one = _single("cpcp")
    two = _run("cpcp", 2)
    assert two[0][4] == two[1][4]
    # both ranks saw the same objective sequence (replicated scalars)
    assert np.array_equal(two[0][5], two[1][5])
    # same algorithm; sums in a different order -> FW-T stays within its envelope
    assert abs(two[0][4] - one[4]) <= max(2, int(0.05 * one[4]))
    # the warm-started power iteration stops on a 1e-6 relative s^2 change, so
    # an ulp-level difference in the summed Gram can move the stop by a pass
    assert abs(two[0][5][0] - one[5][0]) <= 1e-7 * one[5][0]
    assert abs(two[0][5][-1] - one[5][-1]) / one[5][-1] < 1e-4


@pytest.mark.timeout(600)
@pytest.mark.parametrize("kind", ["pcp", "cpcp"])
def test_time_budget_decision_is_collective(kind):
    """One rank's clock passes the budget while the other's does not: the
    budget flags travel in the summed stats, so both ranks stop after the
    same iteration (no hang, no mismatched collective counts)."""
    two = _run(kind + "_budget", 2)
    assert two[0][4] == two[1][4] == 1


@pytest.mark.timeout(600)
@pytest.mark.parametrize("kind", ["pcp", "cpcp"])
def test_replicated_inputs_bitwise_equal(kind, monkeypatch):
    """MLR_VERIFY_REPLICATED=1: every iteration all-gathers a hash of the
    all-reduced Gram (+ arg-max records) and raises if any rank differs."""
    monkeypatch.setenv("MLR_VERIFY_REPLICATED", "1")
    two = _run(kind, 2)
    assert two[0][4] == two[1][4]

"""Row-sharded solvers on the real CUDA kernels: two ranks share cuda:0 and
combine their Gram / statistics / arg-max over gloo (host-staged).  No kernel
waits on another rank, so this checks the sharded host + device logic, not
NVLink performance.  The sharded results must reproduce the one-rank solve."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


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
    import paper_2206_13369_b200 as pkg
    from oracle import mlrpca_oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "pcp":
            d, _ = O.gaussian_rpca(150, 120, 5, 0.1, 31)
            m, n = d.shape
            r0, r1 = rank * m // world, (rank + 1) * m // world
            st = pkg.ml_ialm_solve_rows(torch.from_numpy(np.ascontiguousarray(d[r0:r1])).cuda(),
                                        pkg.PcpOptions(levels=30, tol_feasibility=1e-7), m)
            out_q.put((rank, r0, st.l.cpu().numpy(), st.s.cpu().numpy(), st.iter, [h.feasibility_gap for h in st.history]))
        else:
            d, mask = O.gaussian_rpca(150, 120, 4, 0.1, 32, observe=0.8)
            m, n = d.shape
            r0, r1 = rank * m // world, (rank + 1) * m // world
            lam = 1 / np.sqrt(m)
            st = pkg.ml_fwt_solve_rows(torch.from_numpy(np.ascontiguousarray(d[r0:r1])).cuda(),
                                       pkg.ObservationMask(mask[r0:r1]),
                                       pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(m), tol=1e-6,
                                                       max_iters=300, levels=30, collect_rank=False), m, r0)
            out_q.put((rank, r0, st.l.cpu().numpy(), st.s.cpu().numpy(), st.iter, list(st.objective_history)))
    finally:
        dist.destroy_process_group()


def _run(kind, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _relf(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_pcp_rows_two_ranks_match_one():
    import paper_2206_13369_b200 as pkg
    from oracle import mlrpca_oracle as O
    res = _run("pcp")
    d, _ = O.gaussian_rpca(150, 120, 5, 0.1, 31)
    one = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=30, tol_feasibility=1e-7))
    L = np.concatenate([r[2] for r in res])
    S = np.concatenate([r[3] for r in res])
    assert res[0][4] == res[1][4] == one.iter
    assert _relf(L, one.l) <= 1e-10 and _relf(S, one.s) <= 1e-10


def test_cpcp_rows_two_ranks_match_one():
    import paper_2206_13369_b200 as pkg
    from oracle import mlrpca_oracle as O
    res = _run("cpcp")
    d, mask = O.gaussian_rpca(150, 120, 4, 0.1, 32, observe=0.8)
    m = d.shape[0]
    lam = 1 / np.sqrt(m)
    one = pkg.ml_fwt_solve(d, pkg.ObservationMask(mask), pkg.CpcpOptions(
        lambda_l=lam, lambda_s=lam / np.sqrt(m), tol=1e-6, max_iters=300, levels=30, collect_rank=False))
    obj = res[0][5]
    assert res[0][5] == res[1][5]  # every rank holds the same scalars
    # iteration 1 agrees to rounding; FW-T is chaotic afterwards
    assert abs(obj[0] - one.objective_history[0]) <= 1e-9 * one.objective_history[0]
    assert abs(res[0][4] - one.iter) <= max(2, int(0.05 * one.iter))
    assert abs(obj[-1] - one.objective_history[-1]) / one.objective_history[-1] <= 1e-3


def test_native_nccl_communicator_one_rank():
    """The library's own NCCL communicator (mlr_comm_*: dlopen'd NCCL, unique
    id exchanged through torch.distributed once) drives every collective of
    the row-sharded loops; on the one-GPU box a one-rank NCCL group runs the
    same calls (all-reduce in place, all-gather) and must reproduce the
    single-GPU solves bit for bit."""
    import ctypes
    import paper_2206_13369_b200 as pkg
    from oracle import mlrpca_oracle as O
    from paper_2206_13369_b200 import _lib, runtime

    lib = _lib.load()
    assert lib.mlr_comm_available() == 1
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    os.environ["MLR_FORCE_NATIVE_NCCL"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        c = runtime.Comm()
        assert c.native is not None and lib.mlr_comm_size(c.native) == 1
        x = torch.arange(10, dtype=torch.float64, device="cuda")
        c.sum(x)
        c.max(x)
        out = torch.zeros(10, dtype=torch.float64, device="cuda")
        c.gather(out, x)
        torch.cuda.synchronize()
        assert torch.equal(x, torch.arange(10, dtype=torch.float64, device="cuda")) and torch.equal(out, x)
        d, _ = O.gaussian_rpca(150, 120, 5, 0.1, 31)
        one = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=30, tol_feasibility=1e-7))
        st = pkg.ml_ialm_solve_rows(torch.from_numpy(d).cuda(), pkg.PcpOptions(levels=30, tol_feasibility=1e-7), 150)
        assert st.iter == one.iter and np.array_equal(st.l.cpu().numpy(), one.l)
        d2, mask = O.gaussian_rpca(150, 120, 4, 0.1, 32, observe=0.8)
        lam = 1 / np.sqrt(150)
        opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(150), tol=1e-6, max_iters=300, levels=30,
                               collect_rank=False)
        one2 = pkg.ml_fwt_solve(d2, pkg.ObservationMask(mask), opts)
        st2 = pkg.ml_fwt_solve_rows(torch.from_numpy(d2).cuda(), pkg.ObservationMask(mask), opts, 150, 0)
        assert st2.iter == one2.iter and st2.objective_history == one2.objective_history
    finally:
        os.environ.pop("MLR_FORCE_NATIVE_NCCL", None)
        runtime._NATIVE.clear()
        dist.destroy_process_group()

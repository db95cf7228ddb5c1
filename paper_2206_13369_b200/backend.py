"""CUDA backends: thin objects owning a plan + its torch-allocated buffers and
exposing the per-iteration steps of the C ABI (include/mlr_b200.h).

PyTorch is used only to allocate device memory and to hand out the current
stream; all arithmetic runs in libmlr_b200.so.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _budget(time_budget):
    """None -> -1 (no budget); any other value, including 0, is a budget
    (the reference stops once wall >= budget, pcp.py:295, cpcp.py:451)."""
    return -1.0 if time_budget is None else float(time_budget)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class _Snapshots:
    """Double-buffered pinned host copies of a plan's device state, each
    followed by an event: the host reads batch j's state while batch j + 1
    is already queued, so the GPU never idles on a poll.  Instances are
    pooled (pinned allocation is slow and can stall behind other host work),
    so a solve allocates nothing on the host once warm."""

    _pool: dict = {}
    _lock = threading.Lock()

    def __init__(self, nbytes, device_index):
        self.key = (int(nbytes), int(device_index))  # events belong to one device
        self.buf = [torch.empty(int(nbytes), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.ev = [torch.cuda.Event(), torch.cuda.Event()]
        self.next = 0

    @classmethod
    def get(cls, nbytes):
        key = (int(nbytes), torch.cuda.current_device())
        with cls._lock:
            free = cls._pool.get(key)
            if free:
                snap = free.pop()
                snap.next = 0
                return snap
        return cls(*key)

    def release(self):
        for e in self.ev:
            e.synchronize()  # no copy into these buffers is still in flight
        with self._lock:
            self._pool.setdefault(self.key, []).append(self)

    def take(self, copy_fn):
        i = self.next
        self.next ^= 1
        copy_fn(ctypes.c_void_p(self.buf[i].data_ptr()))
        self.ev[i].record()
        return i

    def wait(self, i):
        self.ev[i].synchronize()
        return ctypes.c_void_p(self.buf[i].data_ptr())


class CudaPcp:
    """Device plan for ML-PCP over one row block of the iterate."""

    def __init__(self, chain, m_local, m_global, f32, max_iters, device):
        self.h = None  # close() is safe even if the constructor fails below
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.f32 = bool(f32)
        self.n = chain.n_fine
        self.nh = chain.n_coarse
        self.m_local = int(m_local)
        self.max_iters = int(max_iters)
        self.chain_h = chain.device_handle(self.device.index)
        lib = self.lib
        nbytes = lib.mlr_pcp_workspace_bytes(self.chain_h, self.m_local, int(self.f32), self.max_iters)
        if nbytes < 0:
            raise _lib.MlrError("mlr_pcp_workspace_bytes failed")
        self.ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _lib.check(lib.mlr_pcp_create(self.chain_h, self.m_local, int(m_global), int(self.f32), self.max_iters,
                                      _ptr(self.ws), ctypes.byref(h)))
        self.h = h
        self.red = torch.zeros(int(lib.mlr_pcp_red_doubles(h)), dtype=torch.float64, device=self.device)
        self.np_ = int(lib.mlr_chain_padded_width(self.chain_h))
        self.stats = torch.zeros(4, dtype=torch.float64, device=self.device)
        self.lz_w = torch.zeros(self.n, dtype=torch.float64, device=self.device)

    def close(self):
        if getattr(self, "_snaps", None) is not None:
            self._snaps.release()
            self._snaps = None
        if self.h is not None:
            self.lib.mlr_pcp_destroy(self.h)
            self.h = None

    __del__ = close

    def input_stats(self, D):
        _lib.check(self.lib.mlr_pcp_input_stats(self.h, _ptr(D), D.stride(0), _ptr(self.stats), _stream()))
        return self.stats

    def lanczos_init(self):
        _lib.check(self.lib.mlr_pcp_lanczos_init(self.h, _stream()))

    def lanczos_matvec(self, D):
        _lib.check(self.lib.mlr_pcp_lanczos_matvec(self.h, _ptr(D), D.stride(0), _ptr(self.lz_w), _stream()))
        return self.lz_w

    def lanczos_update(self, w, tol):
        _lib.check(self.lib.mlr_pcp_lanczos_update(self.h, _ptr(w), float(tol), _stream()))

    def lanczos_run_available(self):
        return bool(self.lib.mlr_pcp_lanczos_run_available(self.h))

    def lanczos_run(self, D, tol):
        _lib.check(self.lib.mlr_pcp_lanczos_run(self.h, _ptr(D), D.stride(0), float(tol), _stream()))

    def lanczos_state(self):
        out = np.zeros(4)
        _lib.check(self.lib.mlr_pcp_lanczos_state(self.h, out.ctypes.data, _stream()))
        return {"k": int(out[0]), "done": int(out[1]), "sigma1": float(out[2]), "theta": float(out[3])}

    def start(self, D, Y0, lam, mu0, rho, tol, max_iters, time_budget, jac_tol, jac_max_sweeps):
        _lib.check(self.lib.mlr_pcp_start(
            self.h, _ptr(D), D.stride(0), _ptr(Y0), Y0.stride(0), _ptr(self.stats), float(lam),
            float(mu0 or 0.0), float(rho), float(tol), int(max_iters), _budget(time_budget),
            float(jac_tol), int(jac_max_sweeps), _stream()))

    def gram(self, with_stats):
        _lib.check(self.lib.mlr_pcp_gram(self.h, _ptr(self.red), int(with_stats), _stream()))

    def stats_slice(self):
        nn = self.np_ * self.np_
        return nn, nn + 4  # Gram, then res^2, sum|S|, nnz, time-budget flag

    def finalize(self):
        _lib.check(self.lib.mlr_pcp_finalize(self.h, _ptr(self.red), _stream()))

    def svt(self):
        _lib.check(self.lib.mlr_pcp_svt(self.h, _ptr(self.red), _stream()))

    def update(self, D, Yin, Yout):
        _lib.check(self.lib.mlr_pcp_update(self.h, _ptr(D), D.stride(0), _ptr(Yin), _ptr(Yout), Yout.stride(0),
                                           _stream()))

    def outputs(self, D, Yprev, L, S):
        _lib.check(self.lib.mlr_pcp_outputs(self.h, _ptr(D), D.stride(0), _ptr(Yprev), Yprev.stride(0), _ptr(L),
                                            _ptr(S), L.stride(0), _stream()))

    def state(self):
        out = np.zeros(16)
        _lib.check(self.lib.mlr_pcp_state(self.h, out.ctypes.data, _stream()))
        return self._state_dict(out)

    @staticmethod
    def _state_dict(out):
        keys = ("k", "done", "status", "rank", "mu", "mu_final", "mu_last", "nuclear", "sigma1", "d_norm",
                "jac_sweeps", "tau", "scale", "lam")
        d = dict(zip(keys, out[:len(keys)].tolist()))
        for k in ("k", "done", "status", "rank", "jac_sweeps"):
            d[k] = int(d[k])
        return d

    def history(self, count):
        out = np.zeros((max(count, 1), 8))
        _lib.check(self.lib.mlr_pcp_history(self.h, int(count), out.ctypes.data, _stream()))
        return out[:count]

    def snapshot(self):
        """Queue a copy of the device state; returns a token for read_snapshot."""
        if getattr(self, "_snaps", None) is None:
            self._snaps = _Snapshots.get(self.lib.mlr_pcp_snapshot_bytes())
        return self._snaps.take(lambda p: _lib.check(self.lib.mlr_pcp_snapshot(self.h, p, _stream())))

    def read_snapshot(self, token):
        """(state dict as state(), lanczos dict as lanczos_state()) of a snapshot."""
        p = self._snaps.wait(token)
        out, lz = np.zeros(16), np.zeros(4)
        _lib.check(self.lib.mlr_pcp_snapshot_read(p, out.ctypes.data, lz.ctypes.data))
        return self._state_dict(out), {"k": int(lz[0]), "done": int(lz[1]), "sigma1": float(lz[2]),
                                       "theta": float(lz[3])}

    def coarse_copy(self, out):
        """out (m_local x n_H) <- the latest coarse iterate L_H = Z."""
        _lib.check(self.lib.mlr_pcp_coarse_copy(self.h, _ptr(out), out.stride(0), _stream()))

    def delta(self, Zk, Zf, out, work):
        """out (one device double) <- <Z_k (G - I), Z_k - Z_f G> over this rank's rows."""
        _lib.check(self.lib.mlr_pcp_delta(self.h, _ptr(Zk), _ptr(Zf), Zk.stride(0), _ptr(out), _ptr(work),
                                          _stream()))

    def set_truncation(self, sv0, cap):
        """Truncated SVT of the full-width ialm_solve (0 restores the full SVT)."""
        _lib.check(self.lib.mlr_pcp_set_truncation(self.h, int(sv0), int(cap)))

    PHASES = ("gram", "pre", "jacobi", "post", "recon", "update", "finalize", "lanczos")

    def set_timing(self, on):
        _lib.check(self.lib.mlr_pcp_set_timing(self.h, int(bool(on))))

    def timing(self):
        """{phase: (total ms, launches)} since the last call (synchronises)."""
        ms = np.zeros(8)
        cnt = np.zeros(8, dtype=np.int32)
        _lib.check(self.lib.mlr_pcp_timing(self.h, ms.ctypes.data, cnt.ctypes.data))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(self.PHASES)}

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)


class CudaCpcp:
    """Device plan for ML-CPCP over one row block."""

    def __init__(self, chain, m_local, m_global, row0, f32, max_iters, world, device):
        self.h = None  # close() is safe even if the constructor fails below
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.f32 = bool(f32)
        self.n = chain.n_fine
        self.nh = chain.n_coarse
        self.m_local = int(m_local)
        self.max_iters = int(max_iters)
        self.chain_h = chain.device_handle(self.device.index)
        lib = self.lib
        nbytes = lib.mlr_cpcp_workspace_bytes(self.chain_h, self.m_local, int(self.f32), self.max_iters)
        self.ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _lib.check(lib.mlr_cpcp_create(self.chain_h, self.m_local, int(m_global), int(row0), int(self.f32),
                                       self.max_iters, int(world), _ptr(self.ws), ctypes.byref(h)))
        self.h = h
        self.np_ = int(lib.mlr_chain_padded_width(self.chain_h))
        self.red = torch.zeros(int(lib.mlr_cpcp_red_doubles(h)), dtype=torch.float64, device=self.device)
        self.amax = torch.zeros(4, dtype=torch.float64, device=self.device)
        self.amax_all = torch.zeros(4 * int(world), dtype=torch.float64, device=self.device)
        self.dots = torch.zeros(3, dtype=torch.float64, device=self.device)
        self.mstats = torch.zeros(4, dtype=torch.float64, device=self.device)
        self.mwork = torch.zeros(int(lib.mlr_matrix_stats_work_doubles()), dtype=torch.float64, device=self.device)

    def close(self):
        if getattr(self, "_snaps", None) is not None:
            self._snaps.release()
            self._snaps = None
        if self.h is not None:
            self.lib.mlr_cpcp_destroy(self.h)
            self.h = None

    __del__ = close

    def input_stats(self, D):
        _lib.check(self.lib.mlr_matrix_stats(D.shape[0], D.shape[1], int(self.f32), _ptr(D), D.stride(0),
                                             _ptr(self.mstats), _ptr(self.mwork), _stream()))
        return self.mstats

    def start(self, D, mask, S, lam_l, lam_s, tol, radius, max_iters, time_budget):
        ldm = mask.shape[1] if mask is not None else 0
        _lib.check(self.lib.mlr_cpcp_start(self.h, _ptr(D), D.stride(0), _ptr(mask), ldm, _ptr(S), S.stride(0),
                                           float(lam_l), float(lam_s), float(tol), float(radius), int(max_iters),
                                           _budget(time_budget), _stream()))

    def gram(self):
        _lib.check(self.lib.mlr_cpcp_gram(self.h, _ptr(self.red), _ptr(self.amax), _stream()))

    def stats_slice(self):
        nn = self.np_ * self.np_
        return nn, nn + 6  # Gram, then 5 stats and the time-budget flag

    def begin(self):
        _lib.check(self.lib.mlr_cpcp_begin(self.h, _ptr(self.red), _ptr(self.amax_all), _stream()))

    def lmo(self):
        _lib.check(self.lib.mlr_cpcp_lmo(self.h, _ptr(self.red), _ptr(self.amax_all), _ptr(self.dots), _stream()))

    def update(self, D, mask, S):
        ldm = mask.shape[1] if mask is not None else 0
        _lib.check(self.lib.mlr_cpcp_update(self.h, _ptr(D), D.stride(0), _ptr(mask), ldm, _ptr(S), S.stride(0),
                                            _ptr(self.dots), _stream()))

    def finalize(self):
        _lib.check(self.lib.mlr_cpcp_finalize(self.h, _ptr(self.red), _stream()))

    def outputs(self, L):
        _lib.check(self.lib.mlr_cpcp_outputs(self.h, _ptr(L), L.stride(0), _stream()))

    def snapshot(self):
        if getattr(self, "_snaps", None) is None:
            self._snaps = _Snapshots.get(self.lib.mlr_cpcp_snapshot_bytes())
        return self._snaps.take(lambda p: _lib.check(self.lib.mlr_cpcp_snapshot(self.h, p, _stream())))

    def read_snapshot(self, token):
        p = self._snaps.wait(token)
        out = np.zeros(32)
        _lib.check(self.lib.mlr_cpcp_snapshot_read(p, out.ctypes.data))
        return self._state_dict(out)

    def state(self):
        out = np.zeros(32)
        _lib.check(self.lib.mlr_cpcp_state(self.h, out.ctypes.data, _stream()))
        return self._state_dict(out)

    @staticmethod
    def _state_dict(out):
        keys = ("k", "done", "status", "t_l", "t_s", "u_l", "u_s", "sigma", "passes", "ga", "gb", "corner_l",
                "corner_s", "i_s", "j_s", "s2", "pd_norm", "sq", "l1", "nnz", "ss", "sr", "r_is", "s_is", "spike",
                "none", "coef")
        d = dict(zip(keys, out[:len(keys)].tolist()))
        for k in ("k", "done", "status", "passes", "corner_l", "corner_s", "i_s", "j_s", "none"):
            d[k] = int(d[k])
        return d

    PHASES = ("gram", "power", "dots", "qp", "unused", "update", "finalize", "unused2")

    def set_timing(self, on):
        _lib.check(self.lib.mlr_cpcp_set_timing(self.h, int(bool(on))))

    def timing(self):
        ms = np.zeros(8)
        cnt = np.zeros(8, dtype=np.int32)
        _lib.check(self.lib.mlr_cpcp_timing(self.h, ms.ctypes.data, cnt.ctypes.data))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(self.PHASES) if not p.startswith("unused")}

    def rank_binding(self):
        """(L_H pointer, its leading dimension, device stop flag, rank slot)."""
        lh, done, slot = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        ld = ctypes.c_int64()
        _lib.check(self.lib.mlr_cpcp_rank_binding(self.h, ctypes.byref(lh), ctypes.byref(ld), ctypes.byref(done),
                                                  ctypes.byref(slot)))
        return lh.value, ld.value, done.value, slot.value

    def atom_copy(self, u, v):
        _lib.check(self.lib.mlr_cpcp_atom_copy(self.h, _ptr(u), _ptr(v), _stream()))

    def atom_dense(self, u, v, out):
        _lib.check(self.lib.mlr_cpcp_atom_dense(self.h, _ptr(u), _ptr(v), _ptr(out), out.stride(0), _stream()))

    def rank_shadow(self, L64):
        _lib.check(self.lib.mlr_cpcp_rank_shadow(self.h, _ptr(L64), L64.stride(0), _stream()))

    def history(self, count):
        out = np.zeros((max(count, 1), 8))
        objs = np.zeros(max(count, 1))
        _lib.check(self.lib.mlr_cpcp_history(self.h, int(count), out.ctypes.data, objs.ctypes.data, _stream()))
        return out[:count], objs[:count]

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)


class CudaSpectrum:
    """Two-pass singular values of a row-sharded tall X (or X C) for the
    reference's numerical-rank telemetry (spectrum plan of the C ABI)."""

    def __init__(self, m_local, n, f32, device, C=None, skip_ptr=None):
        self.h = None  # close() is safe even if the constructor fails below
        self.lib = _lib.load()
        self.device = torch.device(device)
        lib = self.lib
        nbytes = lib.mlr_spec_workspace_bytes(int(m_local), int(n))
        if nbytes < 0:
            raise _lib.MlrError("mlr_spec_workspace_bytes failed")
        self.ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _lib.check(lib.mlr_spec_create(int(m_local), int(n), int(bool(f32)), _ptr(C), C.stride(0) if C is not None else 0,
                                       ctypes.c_void_p(skip_ptr or 0), _ptr(self.ws), ctypes.byref(h), _stream()))
        self.h = h
        nn = int(lib.mlr_spec_red_doubles(h))
        self.np_ = int(round(nn ** 0.5))
        self.red = torch.zeros(nn, dtype=torch.float64, device=self.device)
        self.red2 = torch.zeros(nn, dtype=torch.float64, device=self.device)
        self.C = C  # keep alive until spec_init's copy has run

    def close(self):
        if self.h is not None:
            self.lib.mlr_spec_destroy(self.h)
            self.h = None

    __del__ = close

    def gram(self, x_ptr, ldx):
        _lib.check(self.lib.mlr_spec_gram(self.h, ctypes.c_void_p(x_ptr), int(ldx), _ptr(self.red), _stream()))

    def rotate(self, x_ptr, ldx):
        _lib.check(self.lib.mlr_spec_rotate(self.h, ctypes.c_void_p(x_ptr), int(ldx), _ptr(self.red),
                                            _ptr(self.red2), _stream()))

    def finish(self, rel, sig_out=None, rank_ptr=None, pair_w=None, wsum_out=None):
        _lib.check(self.lib.mlr_spec_finish(self.h, _ptr(self.red2), float(rel), _ptr(sig_out),
                                            ctypes.c_void_p(rank_ptr or 0), _ptr(pair_w), _ptr(wsum_out),
                                            _stream()))


def chain_cholesky(chain, device):
    """Dense lower Cholesky factor of R^T R on the device (n_H x n_H, float64)."""
    lib = _lib.load()
    h = chain.device_handle(torch.device(device).index)
    C = torch.empty((chain.n_coarse, chain.n_coarse), dtype=torch.float64, device=device)
    _lib.check(lib.mlr_chain_cholesky(h, _ptr(C), C.stride(0), _stream()))
    return C

"""ctypes binding of the in-tree CUDA library ``libmlr_b200.so``.

The library is the only compute path: if it is missing or no CUDA device is
present, every solver raises instead of falling back to CPU code.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLR_LIB_PATH") or os.path.join(_HERE, "libmlr_b200.so")  # override: A/B builds

_lib = None


class MlrError(RuntimeError):
    """Error reported by the CUDA library (message from mlr_last_error)."""


_SIGS = {
    "mlr_version": (c_int, []),
    "mlr_last_error": (ctypes.c_char_p, []),
    "mlr_device_count": (c_int, []),
    "mlr_chain_create": (c_int, [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 POINTER(c_void_p)]),
    "mlr_chain_destroy": (c_int, [c_void_p]),
    "mlr_chain_padded_width": (c_int, [c_void_p]),
    "mlr_restrict": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_int64, c_void_p, c_void_p]),
    "mlr_prolong": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_matrix_stats_work_doubles": (c_int64, []),
    "mlr_matrix_stats": (c_int, [c_int64, c_int, c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "mlr_eigh_work_doubles": (c_int64, [c_int]),
    "mlr_eigh_psd": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p, c_void_p,
                             c_void_p]),
    # NCCL communicator (row-sharded solvers)
    "mlr_comm_available": (c_int, []),
    "mlr_comm_unique_id": (c_int, [c_void_p]),
    "mlr_comm_create": (c_int, [c_void_p, c_int, c_int, c_int, POINTER(c_void_p)]),
    "mlr_comm_destroy": (c_int, [c_void_p]),
    "mlr_comm_allreduce": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p]),
    "mlr_comm_allgather": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "mlr_comm_rank": (c_int, [c_void_p]),
    "mlr_comm_size": (c_int, [c_void_p]),
    # exact box QP of the FW-T step (test entry)
    "mlr_box_qp_batch": (c_int, [c_void_p, c_void_p, c_int, c_void_p]),
    # 3xTF32 tcgen05 reconstruction GEMM (test entry)
    "mlr_tc_gemm_tf32x3": (c_int, [c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    # ML-PCP
    "mlr_pcp_workspace_bytes": (c_int64, [c_void_p, c_int64, c_int, c_int]),
    "mlr_pcp_create": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "mlr_pcp_destroy": (c_int, [c_void_p]),
    "mlr_pcp_red_doubles": (c_int64, [c_void_p]),
    "mlr_pcp_input_stats": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "mlr_pcp_lanczos_init": (c_int, [c_void_p, c_void_p]),
    "mlr_pcp_lanczos_matvec": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "mlr_pcp_lanczos_update": (c_int, [c_void_p, c_void_p, c_double, c_void_p]),
    "mlr_pcp_lanczos_state": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_pcp_lanczos_run": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_void_p]),
    "mlr_pcp_lanczos_run_available": (c_int, [c_void_p]),
    "mlr_pcp_start": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_double, c_double,
                              c_double, c_double, c_int, c_double, c_double, c_int, c_void_p]),
    "mlr_pcp_gram": (c_int, [c_void_p, c_void_p, c_int, c_void_p]),
    "mlr_pcp_finalize": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_pcp_svt": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_pcp_update": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_pcp_outputs": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                c_void_p]),
    "mlr_pcp_state": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_pcp_snapshot_bytes": (c_int64, []),
    "mlr_pcp_snapshot": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_pcp_snapshot_read": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_pcp_history": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "mlr_pcp_set_truncation": (c_int, [c_void_p, c_int, c_int]),
    "mlr_pcp_set_timing": (c_int, [c_void_p, c_int]),
    "mlr_pcp_timing": (c_int, [c_void_p, c_void_p, c_void_p]),
    # ML-CPCP
    "mlr_cpcp_workspace_bytes": (c_int64, [c_void_p, c_int64, c_int, c_int]),
    "mlr_cpcp_create": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_int, c_void_p,
                                POINTER(c_void_p)]),
    "mlr_cpcp_destroy": (c_int, [c_void_p]),
    "mlr_cpcp_red_doubles": (c_int64, [c_void_p]),
    "mlr_cpcp_start": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_double,
                               c_double, c_double, c_double, c_int, c_double, c_void_p]),
    "mlr_cpcp_gram": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_begin": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_lmo": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_update": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                c_void_p]),
    "mlr_cpcp_finalize": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_outputs": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_cpcp_state": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_snapshot_bytes": (c_int64, []),
    "mlr_cpcp_snapshot": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_snapshot_read": (c_int, [c_void_p, c_void_p]),
    "mlr_cpcp_history": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_set_timing": (c_int, [c_void_p, c_int]),
    "mlr_cpcp_timing": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mlr_spec_workspace_bytes": (c_int64, [c_int64, c_int]),
    "mlr_spec_create": (c_int, [c_int64, c_int, c_int, c_void_p, c_int64, c_void_p, c_void_p, POINTER(c_void_p),
                                c_void_p]),
    "mlr_spec_destroy": (c_int, [c_void_p]),
    "mlr_spec_red_doubles": (c_int64, [c_void_p]),
    "mlr_spec_gram": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "mlr_spec_rotate": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "mlr_spec_finish": (c_int, [c_void_p, c_void_p, c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "mlr_chain_cholesky": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_pcp_coarse_copy": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_pcp_delta_work_doubles": (c_int64, []),
    "mlr_pcp_delta": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "mlr_frames_to_matrix": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int64, c_void_p]),
    "mlr_matrix_to_frames": (c_int, [c_void_p, c_int64, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "mlr_mask_pack": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    "mlr_cpcp_rank_shadow": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_cpcp_atom_copy": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "mlr_cpcp_atom_dense": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "mlr_cpcp_rank_binding": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_int64), POINTER(c_void_p),
                                      POINTER(c_void_p)]),
}

EXPORTED = tuple(_SIGS)


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises if it cannot."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise MlrError(
            f"CUDA library not built: {p} is missing (run "
            "`python -c 'import __graft_entry__ as g; g.build()'` or "
            "`make -C paper_2206_13369_b200/csrc`)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int):
    if rc != 0:
        msg = load().mlr_last_error()
        raise MlrError(msg.decode() if msg else f"mlr error code {rc}")

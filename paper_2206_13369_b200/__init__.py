"""B200-native multilevel PCP / CPCP (arXiv 2206.13369) hot path.

Drop-in replacements for the reference package's solver entry points
(``mlrpca.ml_ialm_solve`` / ``mlrpca.ml_fwt_solve``) with the same option,
record and state types.  All arithmetic runs in the hand-written sm_100a
CUDA library ``libmlr_b200.so`` (C ABI: ``include/mlr_b200.h``); there is no
CPU fallback.
"""

__version__ = "0.1.0"

from .api_types import (  # noqa: F401
    CpcpOptions,
    CpcpState,
    IterationRecord,
    MultilevelDiagnostics,
    ObservationMask,
    PcpOptions,
    PcpState,
    SvdError,
)
from .chain import LevelError, build_chain, coarse_sizes, select_levels  # noqa: F401
from .cpcp import fwt_solve, ml_fwt_solve, ml_fwt_solve_rows  # noqa: F401
from . import frames  # noqa: F401
from .ops import eigh_psd, matrix_rank, prolong, restrict, singular_values  # noqa: F401
from .pcp import ialm_solve, ml_ialm_solve, ml_ialm_solve_rows  # noqa: F401

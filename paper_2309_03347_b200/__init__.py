"""B200-native (sm_100a, fp64) hot path of arXiv 2309.03347: TT/QTT k-eigenvalue
neutron transport — exact TT matvec, TT rounding, ALS/AMEn local apply and
interfaces, k-eff fixed point — behind the C ABI of include/tt.h.

Importing the package loads libtt.so and fails loudly if it is missing."""
from . import _lib
from ._lib import TTError

_lib.lib()  # raise now if the CUDA library is absent (no CPU fallback)

from .tt import (AlphaResult, KeffResult, alpha_secant, TTMat, TTVec, als_local_apply, als_update_interfaces, amen_mv, amen_solve,  # noqa: E402
                 keff_fixed_point, keff_workspace_bytes, matvec_out, tt_add, tt_copy, tt_dot, tt_matvec, tt_matvec_batched, tt_orthogonalize, tt_round,
                 tt_round_batched, RoundBatch,
                 tt_scale, CORE_DENSE, CORE_DIAG, core_kinds, als_local_apply_structured,
                 als_update_interfaces_structured, set_graph_mode, graph_mode, graph_stats)

__all__ = ["TTError", "TTMat", "TTVec", "tt_matvec", "matvec_out", "tt_add", "tt_scale", "tt_copy", "tt_dot",
           "tt_orthogonalize", "tt_round", "tt_round_batched", "RoundBatch", "als_local_apply", "als_update_interfaces", "amen_mv", "amen_solve",
           "keff_fixed_point", "keff_workspace_bytes", "KeffResult", "alpha_secant", "AlphaResult", "CORE_DENSE", "CORE_DIAG", "core_kinds",
           "als_local_apply_structured", "als_update_interfaces_structured", "set_graph_mode", "graph_mode", "graph_stats"]

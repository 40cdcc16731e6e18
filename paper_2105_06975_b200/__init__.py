"""B200-native (sm_100a, FP64) hot path of arXiv 2105.06975 (Tabeart & Pearson):
the weak-constraint 4D-Var saddle operator A, the preconditioners P_D / P_I with
L_M(k) and correlated R_hat terms, and batched MINRES / GMRES -- behind the C ABI
in include/wf4dvar.h, bound here through ctypes (argument marshalling only).

Importing this package loads libwf4dvar.so and raises if it is missing: there
is no CPU fallback.
"""
from ._lib import (Context, WF4DVarError, make_precond, version, EXPORTED,  # noqa: F401
                   LIB_PATH, LocalGroup, partition, chain_plan, nccl_unique_id, local_windows,
                   global_windows, rblock_plan)

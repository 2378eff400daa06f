"""B200-native SRMDP (Stratified Regression MDP, arXiv 2407.21085) hot path.

The product is the C-ABI library ``libsrmdp_b200.so`` (include/srmdp.h):
fp64 CUDA kernels for sm_100a. ``srmdp`` is a thin ctypes binding with the
same names; it performs argument marshalling only and raises if the
extension is missing (there is no CPU fallback).
"""
from .srmdp import (  # noqa: F401
    SrmdpError, Solver, config_from_workload, library, srmdp_build_info, srmdp_coeffs, srmdp_create,
    srmdp_destroy, srmdp_eval, srmdp_last_error, srmdp_nccl_unique_id, srmdp_reseed, srmdp_shard_plan, srmdp_solve, srmdp_solve_async, srmdp_solve_steps, srmdp_wait, srmdp_step_ms,
    srmdp_table_load, srmdp_table_save,
    srmdp_stats,
)

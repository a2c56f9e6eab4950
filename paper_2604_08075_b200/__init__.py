"""B200-native fleet-sizing sweep for token-budget pool routing (arxiv 2604.08075).

The product is the C-ABI library lib/libfleetplan.so (include/fleet_plan.h,
hand-written sm_100a CUDA in csrc/); this package is its thin ctypes binding.
Importing it without the built library raises: there is no CPU fallback.
"""
from ._abi import (  # noqa: F401
    EXPORTED, FP_CANDIDATE, FP_CAND_FEASIBLE, FP_CAND_HOMO_FEASIBLE, FP_CAND_VALID,
    FP_FLAG_KERNEL_TIMING, FP_FLAG_NO_MASS, FP_FLAG_REPLICATED_GRID, FP_FLAG_CHECK_ORDER, FP_FLAG_COLLECTIVES, FP_FLAG_TIME_TRACE,
    FP_FLAG_P2P, FP_FLAG_SPECULATE, FP_P2P_HANDLE_BYTES, fp_p2p_export, fp_p2p_import,
    FP_KERNEL_EVAL, FP_KERNEL_ROUTE, FP_KERNEL_TRACE, fp_kernel_time, fp_kernel_time_reset, FleetPlan, FleetPlanError, LIB_PATH,
    best_split, desc_from_config, fleet_plan_create, fleet_plan_destroy, fleet_plan_info,
    fp_candidate_range, fp_kernel_launches, fp_merge_best, fp_nccl_get_unique_id,
    fp_shard_range, fp_status_string, route_batch, route_batch_raw, sweep_and_route, sweep_and_route_graph,
    sweep_histogram,
    sweep_thresholds, sweep_thresholds_raw, sweep_and_route_raw, sweep_three_pools, FP_POOL3, calibrate_replay,
    sweep_peak_windows, FP_PEAK,
)

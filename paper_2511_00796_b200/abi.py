"""ctypes mirror of include/gplan.h (the C ABI of libgplan.so).

Also used by the tests to drive the C restatement oracle (oracle/liboracle.so),
which takes the very same input structs.
"""
from __future__ import annotations

import ctypes as C

GP_MAX_TYPES = 8
GP_MAX_STAGES = 32
GP_MAX_ROLLOUT_STAGES = 8

GP_OK, GP_INFEASIBLE, GP_BAND_INFEASIBLE, GP_INVALID, GP_CUDA_ERROR, GP_CAPACITY = range(6)

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class gp_cluster(C.Structure):
    _fields_ = [
        ("n_devices", C.c_int32), ("n_types", C.c_int32), ("n_machines", C.c_int32),
        ("device_type", i32p), ("device_machine", i32p),
        ("device_flops", f64p), ("device_hbm_bw", f64p), ("device_hbm_cap", f64p),
        ("type_flops", f64p), ("type_hbm_bw", f64p), ("type_hbm_cap", f64p),
        ("links", f64p),
    ]


class gp_workload(C.Structure):
    _fields_ = [
        ("model_params_b", C.c_double), ("num_layers", C.c_int32), ("hidden_dim", C.c_int32),
        ("batch_rollouts", C.c_int32), ("prompt_len", C.c_int32), ("mean_len", C.c_double),
        ("bytes_per_param_train", C.c_double), ("bytes_per_param_infer", C.c_double),
        ("reward_cost_const", C.c_double), ("micro_batches", C.c_int32), ("staleness", C.c_int32),
    ]


class gp_calib(C.Structure):
    _fields_ = [
        ("compute_eff", f64p), ("io_eff", f64p),
        ("sync_latency_s", C.c_double), ("stage_latency_penalty", C.c_double),
        ("max_concurrency", C.c_int32), ("activation_coeff", C.c_double),
        ("tp_allreduce_coeff", C.c_double), ("grad_bytes_per_param", C.c_double),
    ]


class gp_train_opts(C.Structure):
    _fields_ = [("max_stages_per_type", C.c_int32), ("device_granularity_limit", C.c_int32)]


class gp_rollout_opts(C.Structure):
    _fields_ = [("max_stages", C.c_int32)]


class gp_gamma(C.Structure):
    _fields_ = [("q", C.c_double), ("r", C.c_double), ("gamma_l", C.c_double), ("gamma_h", C.c_double)]


class gp_part_opts(C.Structure):
    _fields_ = [
        ("exact_threshold", C.c_int32), ("restarts", C.c_int32), ("seed", C.c_uint64),
        ("band_epsilon", C.c_double), ("force_local_search", C.c_int32),
        ("machine_granularity", C.c_int32),
    ]


class gp_stage(C.Structure):
    _fields_ = [("first", C.c_int32), ("count", C.c_int32), ("tp", C.c_int32), ("dp", C.c_int32),
                ("layers", C.c_int32)]


class gp_train_result(C.Structure):
    _fields_ = [
        ("found", C.c_int32), ("n_stages", C.c_int32), ("cost", C.c_double), ("rank", C.c_int64),
        ("layouts", C.c_int64), ("feasible", C.c_int64), ("stage", gp_stage * GP_MAX_STAGES),
    ]


class gp_config(C.Structure):
    _fields_ = [
        ("type_counts", C.c_int32 * GP_MAX_TYPES), ("n_stages", C.c_int32),
        ("tp", C.c_int32 * GP_MAX_ROLLOUT_STAGES), ("throughput", C.c_double),
    ]


class gp_rollout_entry(C.Structure):
    _fields_ = [("config", C.c_int32), ("replicas", C.c_int32), ("workload", C.c_double)]


class gp_rollout_result(C.Structure):
    _fields_ = [
        ("n_entries", C.c_int32), ("makespan", C.c_double), ("total_rollouts", C.c_double),
        ("aggregate", C.c_double), ("states", C.c_int64),
    ]


class gp_partition(C.Structure):
    _fields_ = [("train_offset", C.c_int32), ("train_count", C.c_int32), ("objective", C.c_double),
                ("compute_fraction", C.c_double)]


class gp_exhaustive_result(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32), ("n_train", C.c_int32), ("objective", C.c_double),
        ("partitions", C.c_int64), ("train_candidates", C.c_int64), ("replica_vectors", C.c_int64),
    ]


class gp_sim_plan(C.Structure):
    _fields_ = [
        ("window", C.c_int32), ("staleness", C.c_int32), ("c_train", C.c_double), ("c_update", C.c_double),
        ("c_reward", C.c_double), ("n_entries", C.c_int32), ("configs", C.POINTER(gp_config)),
        ("replicas", i32p), ("n_train", C.c_int32), ("n_rollout", C.c_int32), ("train_ids", i32p),
        ("rollout_ids", i32p), ("device_price", f64p), ("n_buckets", C.c_int32), ("bucket_len", i32p),
        ("bucket_prob", f64p),
    ]


class gp_sim_report(C.Structure):
    _fields_ = [
        ("steps_completed", C.c_int32), ("pad", C.c_int32), ("avg_step_time", C.c_double),
        ("avg_step_time_steady", C.c_double), ("throughput_tokens_per_s", C.c_double),
        ("max_staleness_observed", C.c_int64), ("rollout_stall_time", C.c_double),
        ("trainer_wait_time", C.c_double), ("rollout_busy_time", C.c_double), ("train_busy_time", C.c_double),
        ("sync_time_total", C.c_double), ("reward_time_total", C.c_double), ("rollouts_produced", C.c_int64),
        ("rollouts_consumed", C.c_int64), ("rollouts_pending", C.c_int64), ("rollouts_in_flight", C.c_int64),
        ("tokens_consumed", C.c_int64), ("total_time", C.c_double), ("dollar_cost_per_token", C.c_double),
    ]


def default_train_opts() -> gp_train_opts:
    return gp_train_opts(4, 16)


def default_rollout_opts() -> gp_rollout_opts:
    return gp_rollout_opts(4)


def default_part_opts(seed: int = 0x5EED, restarts: int = 16) -> gp_part_opts:
    return gp_part_opts(12, restarts, seed, 1e-9, 0, 0)


def declare(lib: C.CDLL, prefix: str) -> None:
    """Set argtypes/restype for the gp_* (engine) or or_* (oracle) symbol family."""
    P = C.POINTER
    vp = C.c_void_p
    sigs = {
        "train_space": [vp, i32p, C.c_int32, P(gp_train_opts), P(C.c_int64)],
        "enumerate_configs": [vp, i32p, C.c_int32, P(gp_rollout_opts), P(gp_config), C.c_int32,
                              P(C.c_int32)],
        "rollout_capacities": [vp, i32p, C.c_int32, i32p],
        "partition_candidates": [vp, P(gp_gamma), P(gp_part_opts), C.c_int32, P(gp_partition), i32p,
                                 P(C.c_int32)],
        "partition_objective": [vp, i32p, C.c_int32, f64p, f64p],
    }
    if prefix == "gp":
        sigs.update({
            "ctx_create": [P(gp_cluster), P(gp_workload), P(gp_calib), C.c_int, P(vp)],
            "constrained_search": [vp, i32p, C.c_int32, C.c_int32, P(gp_train_opts),
                                   P(gp_train_result), i32p],
            "constrained_search_range": [vp, i32p, C.c_int32, C.c_int32, P(gp_train_opts), C.c_int64,
                                         C.c_int64, P(gp_train_result), i32p],
            "solve_milp": [vp, P(gp_config), C.c_int32, i32p, C.c_int32, C.c_double, C.c_double,
                           P(gp_rollout_result), P(gp_rollout_entry)],
            "weight_sync_cost": [vp, i32p, C.c_int32, i32p, C.c_int32, i32p, i32p, C.c_int32,
                                 C.c_int32, f64p],
            "train_candidates_search": [vp, i32p, C.c_int32, C.c_int32, P(gp_train_result), i32p],
            "debug_layout_costs": [vp, i32p, C.c_int32, P(gp_train_opts), C.c_int64, C.c_int64, C.c_int32,
                                   f64p, P(C.c_int32)],
            "train_shard_bounds": [vp, i32p, C.c_int32, P(gp_train_opts), C.c_int32, P(C.c_int64)],
            "constrained_search_batch": [vp, C.c_int32, i32p, i32p, C.c_int32, P(gp_train_opts),
                                         P(gp_train_result), i32p],
            "exhaustive_optimum": [vp, C.c_int32, P(gp_exhaustive_result), i32p],
            "simulate": [vp, P(gp_sim_plan), C.c_int32, C.c_int32, P(C.c_uint64), C.c_int32, P(gp_sim_report),
                         i32p, i32p],
        })
    else:  # oracle: cluster/workload/calib pointers instead of a context
        cw = [P(gp_cluster), P(gp_workload)]
        cwk = [P(gp_cluster), P(gp_workload), P(gp_calib)]
        sigs = {
            "train_space": cw + [i32p, C.c_int32, P(gp_train_opts), P(C.c_int64)],
            "constrained_search": cwk + [i32p, C.c_int32, C.c_int32, P(gp_train_opts), C.c_int64,
                                         C.c_int64, P(gp_train_result), i32p],
            "enumerate_configs": cwk + [i32p, C.c_int32, P(gp_rollout_opts), P(gp_config), C.c_int32,
                                        P(C.c_int32)],
            "rollout_capacities": [P(gp_cluster), i32p, C.c_int32, i32p],
            "solve_milp": [P(gp_config), C.c_int32, i32p, C.c_int32, C.c_double, C.c_double,
                           P(gp_rollout_result), P(gp_rollout_entry)],
            "weight_sync_cost": cwk + [i32p, C.c_int32, i32p, C.c_int32, i32p, i32p, C.c_int32,
                                       C.c_int32, f64p],
            "partition_candidates": [P(gp_cluster), P(gp_gamma), P(gp_part_opts), C.c_int32,
                                     P(gp_partition), i32p, P(C.c_int32)],
            "partition_objective": [P(gp_cluster), i32p, C.c_int32, f64p, f64p],
            "train_candidates_search": cwk + [i32p, C.c_int32, C.c_int32, P(gp_train_result), i32p],
            "brute_milp": [P(gp_config), C.c_int32, i32p, C.c_int32, C.c_double, C.c_double, i32p, f64p,
                           i32p, P(C.c_int64)],
            "exhaustive_optimum": cwk + [C.c_int32, P(gp_exhaustive_result), i32p],
        }
    for name, args in sigs.items():
        fn = getattr(lib, f"{prefix}_{name}", None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = C.c_int
    err = getattr(lib, f"{prefix}_last_error")
    err.restype = C.c_char_p
    err.argtypes = []


class gp_sched_opts(C.Structure):
    _fields_ = [
        ("eta_override", C.c_int32), ("stable_iters", C.c_int32), ("iteration_cap", C.c_int32),
        ("stability_tol", C.c_double), ("balance_tol", C.c_double), ("interval_min", C.c_double),
        ("band_widen_step", C.c_double), ("delta_cap", C.c_int32), ("expand_window", C.c_int32),
        ("candidate_width", C.c_int32), ("grid_probes", C.c_int32), ("train", gp_train_opts),
        ("rollout", gp_rollout_opts), ("exact_threshold", C.c_int32), ("restarts", C.c_int32),
        ("seed", C.c_uint64), ("band_epsilon", C.c_double), ("force_local_search", C.c_int32),
        ("machine_granularity", C.c_int32),
    ]


class gp_schedule_result(C.Structure):
    _fields_ = [
        ("window", C.c_int32), ("staleness", C.c_int32), ("iterations_run", C.c_int32),
        ("converged", C.c_int32), ("n_trace", C.c_int32), ("n_train", C.c_int32),
        ("n_rollout", C.c_int32), ("train", gp_train_result), ("rollout", gp_rollout_result),
        ("c_train", C.c_double), ("c_rollout", C.c_double), ("c_reward", C.c_double),
        ("c_update", C.c_double), ("c_infer_total", C.c_double),
        ("evaluated_partitions", C.c_int64), ("evaluated_layouts", C.c_int64),
    ]

"""ctypes mirror of ``include/biscale_gpu.h`` (the C ABI of the sm_100a path).

The layouts below must match the header field for field; ``tests`` check the
struct sizes against the C compiler's (``test_abi_layout``).
"""
from __future__ import annotations

import ctypes as C

BS_MAX_RANK = 4
BS_MAX_K = 16
BS_MAX_CAND = 32
BS_MAX_LEVELS = 32
BS_MAX_LADDER = 64

BS_OK = 0
BS_PARAMETER_ERROR = 1
BS_MODEL_ERROR = 2
BS_SIMULATION_ERROR = 3
BS_CONFIG_ERROR = 4
BS_ACCOUNTING_ERROR = 5
BS_IO_ERROR = 6
BS_INFEASIBLE_ERROR = 7
BS_CUDA_ERROR = 100

AXIS_ROLE = {"sum_len": 0, "n_requests": 1, "tp": 2, "freq_mhz": 3}
BS_AXIS_UNKNOWN = -1

dp = C.POINTER(C.c_double)


class bs_grid(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("role", C.c_int32 * BS_MAX_RANK),
        ("n_knots", C.c_int32 * BS_MAX_RANK),
        ("knots", dp * BS_MAX_RANK),
        ("values", dp),
    ]


class bs_idle_entry(C.Structure):
    _fields_ = [("tp", C.c_int32), ("n", C.c_int32), ("freqs_mhz", dp), ("idle_w", dp)]


class bs_model_set(C.Structure):
    _fields_ = [
        ("latency_prefill", bs_grid),
        ("latency_decode", bs_grid),
        ("power_prefill", bs_grid),
        ("power_decode", bs_grid),
        ("n_idle", C.c_int32),
        ("idle", C.POINTER(bs_idle_entry)),
    ]


class bs_features(C.Structure):
    _fields_ = [("n_requests", C.c_int64), ("sum_len", C.c_int64)]


class bs_scheduler_policy(C.Structure):
    _fields_ = [
        ("max_batch_tokens", C.c_int64),
        ("max_batch_requests", C.c_int64),
        ("kv_capacity_tokens", C.c_int64),
        ("chunking", C.c_int32),
        ("_pad", C.c_int32),
    ]


class bs_mpc_config(C.Structure):
    _fields_ = [
        ("horizon_K", C.c_int32),
        ("ladder_N", C.c_int32),
        ("n_ladder", C.c_int32),
        ("_pad", C.c_int32),
        ("ladder_mhz", dp),
        ("ttft_ms", C.c_double),
        ("tpot_ms", C.c_double),
        ("percentile", C.c_double),
        ("switch_latency_ms", C.c_double),
        ("margin", C.c_double),
    ]


class bs_waiting(C.Structure):
    _fields_ = [("id", C.c_int64), ("arrival_ms", C.c_double), ("total_len", C.c_int64), ("remaining_len", C.c_int64)]


class bs_snapshot(C.Structure):
    _fields_ = [
        ("now_ms", C.c_double),
        ("current_freq_mhz", C.c_double),
        ("target_freq_mhz", C.c_double),
        ("running_work_remaining", C.c_double),
        ("running_features", bs_features),
        ("tp", C.c_int32),
        ("running_active", C.c_int32),
        ("n_waiting", C.c_int32),
        ("n_running", C.c_int32),
        ("waiting", C.POINTER(bs_waiting)),
        ("running_completes", C.POINTER(C.c_uint8)),
        ("running_arrivals_ms", dp),
    ]


class bs_mpc_problem(C.Structure):
    _fields_ = [("snap", bs_snapshot), ("cfg_index", C.c_int32), ("_pad", C.c_int32)]


class bs_level_stats(C.Structure):
    _fields_ = [
        ("level", C.c_int32),
        ("k_prime", C.c_int32),
        ("replaced_mhz", C.c_double),
        ("mutations", C.c_int64),
        ("feasible_mutations", C.c_int64),
        ("accepted", C.c_int32),
        ("_pad", C.c_int32),
    ]


class bs_slice(C.Structure):
    _fields_ = [("digits", C.c_int32), ("_pad", C.c_int32), ("lo", C.c_uint64), ("hi", C.c_uint64)]


class bs_placement_problem(C.Structure):
    _fields_ = [("table", C.c_void_p), ("n", C.c_int32), ("total_gpus", C.c_int32), ("target_rps", C.c_double),
                ("alpha", C.c_double), ("max_throughput", C.c_int32), ("_pad", C.c_int32),
                ("max_freq_mhz", C.c_double), ("counts", C.POINTER(C.c_int64))]


class bs_placement_solution(C.Structure):
    _fields_ = [("status", C.c_int32), ("gpus_used", C.c_int32), ("objective_w", C.c_double),
                ("error", C.c_char * 192)]


class bs_mpc_result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("K", C.c_int32),
        ("feasible", C.c_int32),
        ("n_levels", C.c_int32),
        ("eval_count", C.c_int64),
        ("objective_w", C.c_double),
        ("freqs_mhz", C.c_double * BS_MAX_K),
        ("freq_index", C.c_int32 * BS_MAX_K),
        ("decision_freq_mhz", C.c_double),
        ("feasible_count", C.c_uint64),
        ("trajectories", C.c_uint64),
        ("best_code", C.c_uint64),
        ("levels", bs_level_stats * BS_MAX_LEVELS),
    ]


class bs_projected_batch(C.Structure):
    _fields_ = [
        ("features", bs_features),
        ("work_fraction", C.c_double),
        ("min_completing_arrival_ms", C.c_double),
        ("n_completing", C.c_int32),
        ("_pad", C.c_int32),
    ]


class bs_decode_config(C.Structure):
    _fields_ = [
        ("tbt_slo_ms", C.c_double),
        ("kv_threshold", C.c_double),
        ("margin", C.c_double),
        ("n_ladder", C.c_int32),
        ("_pad", C.c_int32),
        ("ladder_mhz", dp),
    ]


class bs_decode_query(C.Structure):
    _fields_ = [
        ("batch", bs_features),
        ("kv_capacity_tokens", C.c_int64),
        ("kv_used_tokens", C.c_int64),
        ("tp", C.c_int32),
        ("cfg_index", C.c_int32),
    ]


class bs_decode_result(C.Structure):
    _fields_ = [("freq_mhz", C.c_double), ("eval_count", C.c_int64), ("kv_override", C.c_int32), ("status", C.c_int32)]


class bs_request(C.Structure):
    _fields_ = [("id", C.c_int64), ("arrival_ms", C.c_double), ("input_len", C.c_int64), ("output_len", C.c_int64)]


class bs_trace(C.Structure):
    _fields_ = [("n", C.c_int64), ("requests", C.POINTER(bs_request)), ("duration_ms", C.c_double)]


class bs_length_dist(C.Structure):
    _fields_ = [
        ("lognormal", C.c_int32),
        ("n_samples", C.c_int32),
        ("input_mu", C.c_double),
        ("input_sigma", C.c_double),
        ("output_mu", C.c_double),
        ("output_sigma", C.c_double),
        ("sample_input", C.POINTER(C.c_int64)),
        ("sample_output", C.POINTER(C.c_int64)),
    ]


class bs_slo(C.Structure):
    _fields_ = [("ttft_ms", C.c_double), ("tpot_ms", C.c_double), ("percentile", C.c_double)]


class bs_goodput_search(C.Structure):
    _fields_ = [("tolerance_rps", C.c_double), ("probe_count", C.c_int32), ("_pad", C.c_int32), ("seed", C.c_uint64)]


class bs_instance_config(C.Structure):
    _fields_ = [("phase", C.c_int32), ("tp", C.c_int32), ("base_freq_mhz", C.c_double)]


class bs_table_entry(C.Structure):
    _fields_ = [
        ("config", bs_instance_config),
        ("r_c", C.c_double),
        ("e_c", C.c_double),
        ("has_e_c", C.c_int32),
        ("g_c", C.c_int32),
        ("saturated", C.c_int32),
        ("error_code", C.c_int32),
        ("k_star", C.c_int64),
        ("error", C.c_char * 96),
    ]


class bs_sim_summary(C.Structure):
    _fields_ = [("status", C.c_int32), ("meets_slo", C.c_int32), ("completed", C.c_int64),
                ("busy_energy_j", C.c_double), ("idle_energy_j", C.c_double), ("horizon_ms", C.c_double)]


class bs_cluster_instance(C.Structure):
    _fields_ = [("config", bs_instance_config), ("weight", C.c_double)]


class bs_replay_config(C.Structure):
    _fields_ = [
        ("mpc", bs_mpc_config),
        ("decode", bs_decode_config),
        ("policy", bs_scheduler_policy),
        ("slo", bs_slo),
        ("switch_latency_ms", C.c_double),
        ("horizon_ms", C.c_double),
        ("rampup_s", C.c_double),
        ("controlled", C.c_int32),
        ("_pad", C.c_int32),
    ]


class bs_scenario(C.Structure):
    _fields_ = [("trace", bs_trace), ("instances", C.POINTER(bs_cluster_instance)), ("n_instances", C.c_int32),
                ("config", C.c_int32)]


class bs_replay_summary(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("has_p99_ttft", C.c_int32),
        ("has_p99_tpot", C.c_int32),
        ("has_e_first", C.c_int32),
        ("has_e_output", C.c_int32),
        ("_pad", C.c_int32),
        ("horizon_ms", C.c_double),
        ("completed_requests", C.c_int64),
        ("generated_tokens", C.c_int64),
        ("n_batches", C.c_int64),
        ("n_idles", C.c_int64),
        ("n_decisions", C.c_int64),
        ("decisions_by_trigger", C.c_int64 * 3),
        ("p99_ttft_ms", C.c_double),
        ("p99_mean_tpot_ms", C.c_double),
        ("energy_per_first_token_j", C.c_double),
        ("energy_per_output_token_j", C.c_double),
        ("avg_power_prefill_w", C.c_double),
        ("avg_power_decode_w", C.c_double),
        ("prefill_energy_j", C.c_double),
        ("decode_energy_j", C.c_double),
        ("span_ms", C.c_double),
        ("report_completed", C.c_int64),
        ("report_generated", C.c_int64),
        ("ttft_violations", C.c_int64),
        ("tpot_violations", C.c_int64),
    ]


class bs_replay_request(C.Structure):
    _fields_ = [
        ("id", C.c_int64),
        ("prefill_instance", C.c_int32),
        ("decode_instance", C.c_int32),
        ("prefill_done_ms", C.c_double),
        ("decode_first_start_ms", C.c_double),
        ("first_token_ms", C.c_double),
        ("last_token_ms", C.c_double),
        ("max_tbt_ms", C.c_double),
        ("n_tokens", C.c_int64),
        ("completed", C.c_int32),
        ("_pad", C.c_int32),
    ]


class bs_batch_record(C.Structure):
    _fields_ = [("instance", C.c_int32), ("phase", C.c_int32), ("batch_seq", C.c_int64), ("start_ms", C.c_double),
                ("end_ms", C.c_double), ("n_requests", C.c_int64), ("sum_len", C.c_int64), ("freq_mhz", C.c_double),
                ("power_w", C.c_double), ("energy_j", C.c_double)]


class bs_idle_record(C.Structure):
    _fields_ = [("instance", C.c_int32), ("phase", C.c_int32), ("start_ms", C.c_double), ("end_ms", C.c_double),
                ("freq_mhz", C.c_double), ("power_w", C.c_double), ("energy_j", C.c_double)]


class bs_decision_record(C.Structure):
    _fields_ = [("time_ms", C.c_double), ("instance", C.c_int32), ("trigger", C.c_int32),
                ("chosen_freq_mhz", C.c_double), ("feasible", C.c_int32), ("_pad", C.c_int32),
                ("eval_count", C.c_int64)]


class bs_replay_logs(C.Structure):
    _fields_ = [
        ("batches", C.POINTER(bs_batch_record)), ("batch_cap", C.c_int64), ("n_batches", C.c_int64),
        ("idles", C.POINTER(bs_idle_record)), ("idle_cap", C.c_int64), ("n_idles", C.c_int64),
        ("decisions", C.POINTER(bs_decision_record)), ("decision_cap", C.c_int64), ("n_decisions", C.c_int64),
    ]


ctx_t = C.c_void_p
models_t = C.c_void_p

# (name, restype, argtypes) for every exported entry point of the header.
PROTOTYPES = [
    ("bs_abi_version", C.c_int, []),
    ("bs_ctx_create", C.c_int, [C.c_int, C.POINTER(ctx_t)]),
    ("bs_ctx_destroy", None, [ctx_t]),
    ("bs_last_error", C.c_char_p, [ctx_t]),
    ("bs_ctx_info", C.c_int, [ctx_t, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("bs_ctx_set_exhaustive_limits", C.c_int, [ctx_t, C.c_double, C.c_uint64, C.c_uint64]),
    ("bs_ctx_sync", C.c_int, [ctx_t]),
    ("bs_ctx_kernel_launches", C.c_int64, [ctx_t]),
    ("bs_ctx_stats", C.c_int, [ctx_t, C.POINTER(C.c_double), C.c_int]),
    ("bs_ctx_stream", C.c_void_p, [ctx_t]),
    ("bs_ctx_last_transfer", C.c_int, [ctx_t, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("bs_fp64_peak", C.c_int, [ctx_t, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("bs_models_upload", C.c_int, [ctx_t, C.POINTER(bs_model_set), C.POINTER(models_t)]),
    ("bs_models_free", None, [ctx_t, models_t]),
    ("bs_predict", C.c_int, [ctx_t, models_t, C.c_int, C.POINTER(bs_features), C.POINTER(C.c_int32), dp, C.c_int,
                             dp, C.POINTER(C.c_int32), C.POINTER(C.c_uint32)]),
    ("bs_grid_interpolate", C.c_int, [ctx_t, C.POINTER(bs_grid), dp, C.c_int, dp, C.POINTER(C.c_uint32)]),
    ("bs_project_batches", C.c_int, [ctx_t, C.POINTER(bs_mpc_config), C.POINTER(bs_scheduler_policy), C.c_int,
                                     C.POINTER(bs_mpc_problem), C.c_int, C.POINTER(bs_projected_batch),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("bs_mpc_greedy", C.c_int, [ctx_t, models_t, C.POINTER(bs_mpc_config), C.POINTER(bs_scheduler_policy), C.c_int,
                                C.POINTER(bs_mpc_problem), C.c_int, C.POINTER(bs_mpc_result)]),
    ("bs_mpc_exhaustive", C.c_int, [ctx_t, models_t, C.POINTER(bs_mpc_config), C.POINTER(bs_scheduler_policy),
                                    C.c_int, C.POINTER(bs_mpc_problem), C.c_int, C.POINTER(bs_mpc_result)]),
    ("bs_mpc_exhaustive_slice", C.c_int, [ctx_t, models_t, C.POINTER(bs_mpc_config),
                                          C.POINTER(bs_scheduler_policy), C.c_int, C.POINTER(bs_mpc_problem),
                                          C.c_int, C.POINTER(bs_slice), C.POINTER(bs_mpc_result)]),
    ("bs_mpc_plan_create", C.c_int, [ctx_t, models_t, C.POINTER(bs_mpc_config), C.POINTER(bs_scheduler_policy),
                                     C.c_int, C.POINTER(bs_mpc_problem), C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("bs_mpc_plan_run", C.c_int, [ctx_t, C.c_void_p, C.c_int]),
    ("bs_mpc_plan_results", C.c_int, [ctx_t, C.c_void_p, C.POINTER(bs_mpc_result)]),
    ("bs_mpc_plan_kernel_ms", C.c_int, [ctx_t, C.c_void_p, C.POINTER(C.c_float), C.c_int]),
    ("bs_mpc_plan_info", C.c_int, [ctx_t, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("bs_mpc_plan_destroy", None, [ctx_t, C.c_void_p]),
    ("bs_mpc_eval_codes", C.c_int, [ctx_t, models_t, C.POINTER(bs_mpc_config), C.POINTER(bs_scheduler_policy),
                                    C.POINTER(bs_mpc_problem), C.POINTER(C.c_uint64), C.c_int,
                                    C.POINTER(C.c_int32), dp]),
    ("bs_mpc_tables", C.c_int, [ctx_t, models_t, C.POINTER(bs_mpc_config), C.POINTER(bs_scheduler_policy),
                                C.POINTER(bs_mpc_problem), C.POINTER(C.c_int32), C.POINTER(C.c_int32), dp, dp, dp]),
    ("bs_decode_pick", C.c_int, [ctx_t, models_t, C.POINTER(bs_decode_config), C.c_int, C.POINTER(bs_decode_query),
                                 C.c_int, C.POINTER(bs_decode_result)]),
    ("bs_gen_gamma_trace", C.c_int, [C.c_double, C.c_double, C.c_double, C.POINTER(bs_length_dist), C.c_uint64,
                                     C.POINTER(bs_request), C.c_int64, C.POINTER(C.c_int64)]),
    ("bs_downsample_keep", C.c_int, [ctx_t, C.POINTER(bs_trace), C.POINTER(bs_goodput_search), C.c_int64, C.c_int,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    ("bs_goodput_table", C.c_int, [ctx_t, models_t, C.POINTER(bs_trace), C.POINTER(bs_slo),
                                   C.POINTER(bs_scheduler_policy), C.POINTER(bs_goodput_search),
                                   C.POINTER(bs_instance_config), C.c_int, C.POINTER(bs_table_entry)]),
    ("bs_goodput_tables", C.c_int, [ctx_t, models_t, C.POINTER(bs_trace), C.c_int, C.POINTER(bs_slo),
                                    C.POINTER(bs_scheduler_policy), C.POINTER(bs_goodput_search),
                                    C.POINTER(bs_instance_config), C.c_int, C.POINTER(bs_table_entry)]),
    ("bs_simulate_instance", C.c_int, [ctx_t, models_t, C.POINTER(bs_trace), C.c_int, C.POINTER(bs_instance_config),
                                       C.POINTER(bs_scheduler_policy), C.POINTER(bs_slo), C.POINTER(bs_sim_summary)]),
    ("bs_placement_solve", C.c_int, [ctx_t, C.POINTER(bs_table_entry), C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    ("bs_placement_max_throughput", C.c_int, [ctx_t, C.POINTER(bs_table_entry), C.c_int, C.c_int, C.c_double,
                                              C.c_double, C.c_double, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                              C.POINTER(C.c_int32)]),
    ("bs_placement_solve_batch", C.c_int, [ctx_t, C.POINTER(bs_placement_problem), C.c_int,
                                           C.POINTER(bs_placement_solution)]),
    ("bs_replay", C.c_int, [ctx_t, models_t, models_t, C.POINTER(bs_replay_config), C.c_int, C.POINTER(bs_scenario),
                            C.c_int, C.POINTER(bs_replay_summary), C.POINTER(bs_replay_request),
                            C.POINTER(bs_replay_logs)]),
]

/*
 * biscale_gpu.h — C ABI of the B200 (sm_100a) decision-evaluation path of
 * BiScale (arXiv 2602.18755).  Plain C: POD structs, plain pointers and
 * sizes, no torch or CUDA types.  Every entry point returns an int status
 * (BS_OK or one code per exception class of the reference's
 * proj/include/pdsim/errors.hpp:10-56); the message is read back with
 * bs_last_error().
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj/include/pdsim/):
 *
 *   bs_models_upload        ModelSet (perfmodel.hpp:494-503) held by every
 *                           controller as `const ModelSet*` (dvfs.hpp:336)
 *   bs_predict              predict_latency / predict_power
 *                           (perfmodel.hpp:262-272), NdGrid::interpolate
 *                           (perfmodel.hpp:150-193)
 *   bs_project_batches      project_batches (dvfs.hpp:63-100)
 *   bs_mpc_greedy           greedy_freq_select (dvfs.hpp:185-259), i.e.
 *                           PrefillMpcController::run (dvfs.hpp:325-333)
 *   bs_mpc_exhaustive       the exhaustive MPC oracle loop
 *                           (tests/test_dvfs.cpp:74-94,
 *                           tests/acceptance_main.cpp:245-261) over
 *                           meets_slo (dvfs.hpp:105-122) and
 *                           MpcEvaluator::time_weighted_power (dvfs.hpp:163-171)
 *   bs_mpc_eval_codes       meets_slo + time_weighted_power for given
 *                           assignments (per-trajectory parity probe)
 *   bs_mpc_tables           the (k, f) -> (lat, pow) memo of MpcEvaluator::eval
 *                           (dvfs.hpp:150-160)
 *   bs_decode_pick          select_decode_freq_ex (dvfs.hpp:274-293), i.e.
 *                           DecodePolicyController::decide (dvfs.hpp:347-350)
 *   bs_goodput_table        build_config_table (placement.hpp:240-260) over
 *                           evaluate_candidate / max_goodput
 *                           (placement.hpp:154-238); bs_goodput_tables for
 *                           several probe traces in one grid (plan_window of
 *                           every window of run_experiment, runner.hpp:155-172)
 *   bs_placement_solve      solve_placement (placement.hpp:357-416)
 *   bs_placement_max_throughput  solve_max_throughput (placement.hpp:421-499)
 *   bs_replay               simulate_cluster (simulator.hpp:758-893) with the
 *                           TwoTierFactory controllers (dvfs.hpp:370-390),
 *                           trim_steady_state + make_report (metrics.hpp:71-156)
 *
 * Threading: a context is not thread-safe (one per host thread, each with its
 * own CUDA stream).  Uploaded models are immutable; kernels are re-entrant.
 * Ownership: the context owns device memory and streams; the caller owns
 * every host array passed in or out; nothing is retained after return.
 */
#ifndef BISCALE_GPU_H_
#define BISCALE_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_ABI_VERSION 1

/* Hard limits of the device path (validated; ParameterError beyond them). */
#define BS_MAX_RANK 4      /* grid axes: sum_len, n_requests, tp, freq_mhz */
#define BS_MAX_K 16        /* MPC horizon (projected batches) */
#define BS_MAX_CAND 32     /* MPC candidate rungs after ladder.select(N) */
#define BS_MAX_LEVELS 32   /* greedy expansion levels (<= N-2) */
#define BS_MAX_LADDER 64   /* decode ladder rungs */

/* Status codes: one per exception class of errors.hpp. */
enum bs_status {
  BS_OK = 0,
  BS_PARAMETER_ERROR = 1,  /* pdsim::ParameterError  (errors.hpp:10) */
  BS_MODEL_ERROR = 2,      /* pdsim::ModelError      (errors.hpp:15) */
  BS_SIMULATION_ERROR = 3, /* pdsim::SimulationError (errors.hpp:20) */
  BS_CONFIG_ERROR = 4,     /* pdsim::ConfigError     (errors.hpp:25) */
  BS_ACCOUNTING_ERROR = 5, /* pdsim::AccountingError (errors.hpp:30) */
  BS_IO_ERROR = 6,         /* pdsim::IoError         (errors.hpp:40) */
  BS_INFEASIBLE_ERROR = 7, /* pdsim::InfeasibleError (errors.hpp:47) */
  BS_CUDA_ERROR = 100      /* device/runtime failure (no reference analogue) */
};

/* Axis roles: the axis names query_coords understands (perfmodel.hpp:204-207,
 * 241-258).  BS_AXIS_UNKNOWN reproduces "grid: unknown axis" ModelError. */
enum bs_axis_role {
  BS_AXIS_UNKNOWN = -1,
  BS_AXIS_SUM_LEN = 0,
  BS_AXIS_N_REQUESTS = 1,
  BS_AXIS_TP = 2,
  BS_AXIS_FREQ = 3
};

enum bs_phase { BS_PHASE_PREFILL = 0, BS_PHASE_DECODE = 1 };

/* One NdGrid (perfmodel.hpp:116-201): row-major values, last axis fastest. */
typedef struct bs_grid {
  int32_t rank;                    /* 1..BS_MAX_RANK */
  int32_t role[BS_MAX_RANK];       /* enum bs_axis_role per axis */
  int32_t n_knots[BS_MAX_RANK];    /* knots per axis (>= 1, strictly increasing) */
  const double* knots[BS_MAX_RANK];
  const double* values;            /* prod(n_knots) doubles */
} bs_grid;

/* IdlePowerModel::TpEntry (perfmodel.hpp:230-237). */
typedef struct bs_idle_entry {
  int32_t tp;
  int32_t n;
  const double* freqs_mhz;
  const double* idle_w;
} bs_idle_entry;

/* ModelSet (perfmodel.hpp:494-503). */
typedef struct bs_model_set {
  bs_grid latency_prefill;
  bs_grid latency_decode;
  bs_grid power_prefill;
  bs_grid power_decode;
  int32_t n_idle;
  const bs_idle_entry* idle;
} bs_model_set;

/* BatchFeatures (perfmodel.hpp:30-51); only n_requests and sum_len reach the
 * grids (perfmodel.hpp:245-249). */
typedef struct bs_features {
  int64_t n_requests;
  int64_t sum_len;
} bs_features;

/* SchedulerPolicy (scheduler.hpp:11-22). */
typedef struct bs_scheduler_policy {
  int64_t max_batch_tokens;   /* default 8192 */
  int64_t max_batch_requests; /* default 256 */
  int64_t kv_capacity_tokens; /* default 1000000 */
  int32_t chunking;           /* default 1 */
  int32_t _pad;
} bs_scheduler_policy;

/* MpcConfig (dvfs.hpp:17-34) with its SLOSpec (slo.hpp:7-16). */
typedef struct bs_mpc_config {
  int32_t horizon_K;          /* default 8 */
  int32_t ladder_N;           /* default 7 */
  int32_t n_ladder;
  int32_t _pad;
  const double* ladder_mhz;   /* FrequencyLadder::freqs_mhz, strictly increasing */
  double ttft_ms;             /* SLOSpec::ttft_ms, default 600 */
  double tpot_ms;             /* SLOSpec::tpot_ms, default 100 */
  double percentile;          /* SLOSpec::percentile, default 0.99 */
  double switch_latency_ms;   /* default 30 */
  double margin;              /* default 0.05 */
} bs_mpc_config;

/* SnapshotWaiting (controller.hpp:26-31). */
typedef struct bs_waiting {
  int64_t id;
  double arrival_ms;
  int64_t total_len;
  int64_t remaining_len;
} bs_waiting;

/* QueueSnapshot (controller.hpp:45-55) restricted to what the prefill MPC
 * reads (dvfs.hpp:63-122, 325-333): the running batch enters the projection
 * through ids/completes/arrivals/work_remaining/features only. */
typedef struct bs_snapshot {
  double now_ms;
  double current_freq_mhz;
  double target_freq_mhz;
  double running_work_remaining;
  bs_features running_features;
  int32_t tp;
  int32_t running_active;
  int32_t n_waiting;
  int32_t n_running;
  const bs_waiting* waiting;
  const uint8_t* running_completes;  /* n_running flags */
  const double* running_arrivals_ms; /* n_running */
} bs_snapshot;

/* One MPC decision problem: a snapshot plus the index of its controller
 * configuration in the cfgs/policies arrays passed alongside. */
typedef struct bs_mpc_problem {
  bs_snapshot snap;
  int32_t cfg_index;
  int32_t _pad;
} bs_mpc_problem;

/* GreedyLevelStats (dvfs.hpp:124-131). */
typedef struct bs_level_stats {
  int32_t level;
  int32_t k_prime;
  double replaced_mhz;
  int64_t mutations;
  int64_t feasible_mutations;
  int32_t accepted;
  int32_t _pad;
} bs_level_stats;

/* GreedyResult (dvfs.hpp:133-139) / exhaustive result, plus the controller's
 * FreqDecision (controller.hpp:67-71) as PrefillMpcController::run derives it
 * (dvfs.hpp:328-331). */
typedef struct bs_mpc_result {
  int32_t status;             /* per-problem status (bs_status) */
  int32_t K;                  /* projection length; assignment length */
  int32_t feasible;           /* GreedyResult::feasible */
  int32_t n_levels;
  int64_t eval_count;
  double objective_w;
  double freqs_mhz[BS_MAX_K]; /* assignment */
  int32_t freq_index[BS_MAX_K]; /* index into the ascending candidate rungs */
  double decision_freq_mhz;   /* FreqDecision::freq_mhz */
  uint64_t feasible_count;    /* exhaustive: # feasible trajectories */
  uint64_t trajectories;      /* exhaustive: N^K */
  uint64_t best_code;         /* exhaustive: argmin code, batch 0 most significant */
  bs_level_stats levels[BS_MAX_LEVELS]; /* [0, n_levels) written; later entries are left untouched */
} bs_mpc_result;

/* ProjectedBatch (dvfs.hpp:54-59), device-side summary. */
typedef struct bs_projected_batch {
  bs_features features;
  double work_fraction;
  double min_completing_arrival_ms; /* +inf when nothing completes */
  int32_t n_completing;
  int32_t _pad;
} bs_projected_batch;

/* DecodePolicyConfig (dvfs.hpp:36-48). */
typedef struct bs_decode_config {
  double tbt_slo_ms;          /* default 100 */
  double kv_threshold;        /* default 0.9 */
  double margin;              /* default 0 */
  int32_t n_ladder;
  int32_t _pad;
  const double* ladder_mhz;
} bs_decode_config;

/* Inputs of select_decode_freq_ex (dvfs.hpp:274-275): batch features,
 * KVCacheState (controller.hpp:16-24) and tp. */
typedef struct bs_decode_query {
  bs_features batch;
  int64_t kv_capacity_tokens;
  int64_t kv_used_tokens;
  int32_t tp;
  int32_t cfg_index;
} bs_decode_query;

/* DecodeDecision (dvfs.hpp:268-272). */
typedef struct bs_decode_result {
  double freq_mhz;
  int64_t eval_count;
  int32_t kv_override;
  int32_t status;
} bs_decode_result;

/* Request / Trace (workload.hpp:18-50): requests sorted by arrival. */
typedef struct bs_request {
  int64_t id;
  double arrival_ms;
  int64_t input_len;
  int64_t output_len;
} bs_request;

typedef struct bs_trace {
  int64_t n;
  const bs_request* requests;
  double duration_ms;
} bs_trace;

/* LengthDistribution (workload.hpp:54-85): an empirical pool (n_samples > 0)
 * or the lognormal form. */
typedef struct bs_length_dist {
  int32_t lognormal;
  int32_t n_samples;
  double input_mu;
  double input_sigma;
  double output_mu;
  double output_sigma;
  const int64_t* sample_input;
  const int64_t* sample_output;
} bs_length_dist;

/* SLOSpec (slo.hpp:7-16). */
typedef struct bs_slo {
  double ttft_ms;
  double tpot_ms;
  double percentile;
} bs_slo;

/* GoodputSearch (placement.hpp:107-111). */
typedef struct bs_goodput_search {
  double tolerance_rps;  /* default 0.25 */
  int32_t probe_count;   /* default 1 */
  int32_t _pad;
  uint64_t seed;         /* default 0x9e3779b97f4a7c15 */
} bs_goodput_search;

/* InstanceConfig (simulator.hpp:22-31). */
typedef struct bs_instance_config {
  int32_t phase;         /* enum bs_phase */
  int32_t tp;
  double base_freq_mhz;
} bs_instance_config;

/* ConfigTableEntry (placement.hpp:25-34).  error_code: 0 none,
 * BS_MODEL_ERROR (evaluate_candidate's caught ModelError, placement.hpp:233),
 * -1 "no completed request at R_c" (placement.hpp:231); error holds the
 * message. */
typedef struct bs_table_entry {
  bs_instance_config config;
  double r_c;
  double e_c;
  int32_t has_e_c;
  int32_t g_c;
  int32_t saturated;
  int32_t error_code;
  int64_t k_star;
  char error[96];
} bs_table_entry;

typedef struct bs_ctx_s* bs_ctx_t;
typedef struct bs_models_s* bs_models_t;

/* --- context and models ---------------------------------------------------- */

int bs_abi_version(void);
int bs_ctx_create(int device, bs_ctx_t* out);
void bs_ctx_destroy(bs_ctx_t ctx);
/* Message of the last failing call on ctx.  The host-only entry points
 * (bs_gen_gamma_trace, bs_placement_solve, bs_placement_max_throughput)
 * accept ctx == NULL; their messages are then read with bs_last_error(NULL)
 * (per calling thread). */
const char* bs_last_error(bs_ctx_t ctx);
/* Device the context runs on and its SM count (for host-side grid sizing). */
int bs_ctx_info(bs_ctx_t ctx, int* device, int* sm_count);
/* Exhaustive-MPC limits of the context (tuning and test hook; 0 restores a
 * default): the number of prefixes at depth K - 2 above which the sweep walks
 * three bottom levels instead of two (default 2^24), and the frontier
 * capacities in entries -- per BFS ping-pong list (default 2.5e8, 40 B each)
 * and for the final list (default 2e9, 12 B each).  A batch whose frontiers
 * exceed them is split into smaller launches; one decision that exceeds them
 * fails with BS_PARAMETER_ERROR.  Results never depend on these settings. */
int bs_ctx_set_exhaustive_limits(bs_ctx_t ctx, double sweep3_min_prefixes, uint64_t level_cap, uint64_t final_cap);
/* Synchronise the context's stream. */
int bs_ctx_sync(bs_ctx_t ctx);
/* Number of kernels the context launched since creation (instrumentation). */
int64_t bs_ctx_kernel_launches(bs_ctx_t ctx);
/* Instrumentation of the last call that records it (bs_goodput_table:
 * {mask ms, probe ms, energy ms, max events per probe, total events}).
 * Returns the number of values available. */
int bs_ctx_stats(bs_ctx_t ctx, double* out, int n);
/* The context's cudaStream_t (as void*), for event timing by the caller. */
void* bs_ctx_stream(bs_ctx_t ctx);
/* Host<->device bytes moved by the last one-shot entry point. */
int bs_ctx_last_transfer(bs_ctx_t ctx, uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* FP64 issue microbenchmark (independent DADD chains on every SM):
 * measured non-FMA FP64 ops/s, the roofline denominator of the MPC kernels. */
int bs_fp64_peak(bs_ctx_t ctx, double* ops_per_s, double* ms);

/* Validates structure (NdGrid::validate_structure, perfmodel.hpp:127-138)
 * and uploads an immutable device copy. */
int bs_models_upload(bs_ctx_t ctx, const bs_model_set* models, bs_models_t* out);
void bs_models_free(bs_ctx_t ctx, bs_models_t models);

/* --- model queries (parity probes for the interpolator) --------------------- */

/* which: 0 latency_prefill, 1 latency_decode, 2 power_prefill, 3 power_decode.
 * n queries of (features, tp, freq); out values and per-query status
 * (ModelError on non-positive/non-finite, perfmodel.hpp:264,270, or unknown
 * axis, perfmodel.hpp:254); clamp_events: per-query clamp count. */
int bs_predict(bs_ctx_t ctx, bs_models_t models, int which, const bs_features* feats,
               const int32_t* tp, const double* freq_mhz, int n, double* out,
               int32_t* status, uint32_t* clamp_events);

/* Raw NdGrid::interpolate over caller coordinates (no role mapping):
 * coords is n x grid->rank, row-major.  clamp_events per query. */
int bs_grid_interpolate(bs_ctx_t ctx, const bs_grid* grid, const double* coords, int n,
                        double* out, uint32_t* clamp_events);

/* --- prefill MPC ---------------------------------------------------------- */

/* project_batches for each problem: out is n x BS_MAX_K, K per problem in
 * out_K.  Per-problem status in out_status (SimulationError from
 * form_prefill_batch, scheduler.hpp:47). */
int bs_project_batches(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
                       int n_cfgs, const bs_mpc_problem* problems, int n, bs_projected_batch* out,
                       int32_t* out_K, int32_t* out_status);

/* greedy_freq_select for n independent decisions: one warp per decision for
 * batches that fill the GPU, a CTA of 2-16 warps per decision for smaller
 * ones, and a thread-block cluster of 8 CTAs per decision when n x 8 <= SMs
 * (a single controller call).  Results are identical in every mode. */
int bs_mpc_greedy(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                  const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems, int n,
                  bs_mpc_result* out);

/* Exhaustive MPC: every |cand|^K assignment, feasibility by meets_slo,
 * objective by time_weighted_power; argmin over (objective, assignment in
 * lexicographic frequency order, batch 0 most significant) -- the rule
 * dvfs.hpp:243 applies to greedy.  Nothing feasible: all-max, feasible = 0.
 * Requires |cand|^K < 2^62. */
int bs_mpc_exhaustive(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                      const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems,
                      int n, bs_mpc_result* out);

/* One slice of every decision's code space, for splitting a single large
 * decision across GPUs: the assignments whose first `digits`
 * digits (batch 0 most significant, base |cand|) form a number in [lo, hi);
 * digits is 0 (whole tree), 1 or 2, hi <= |cand|^digits.  A projection
 * shorter than `digits` reads its missing digits as 0, so the slices of any
 * partition of [0, |cand|^digits) partition every decision.  Per slice the
 * result holds the slice's feasible count, its (objective, code) minimum
 * (feasible = 0 and the all-max fallback when it has no feasible
 * assignment) and trajectories = eval_count = the slice's size; the
 * decision is the minimum over slices (sharding.argmin_over_ranks) and the
 * feasible counts add up. */
typedef struct bs_slice {
  int32_t digits;
  int32_t _pad;
  uint64_t lo;
  uint64_t hi;
} bs_slice;
int bs_mpc_exhaustive_slice(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                            const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems,
                            int n, const bs_slice* slice, bs_mpc_result* out);

/* Resident batches (the throughput path): upload a batch of problems once
 * (one H2D copy), then enqueue its kernels any number of times on the
 * context stream without host synchronisation, and copy results out.
 * mode: 0 exhaustive, 1 greedy.  bs_mpc_plan_kernel_ms returns the number
 * of phases and their durations from the last run with record_kernel_times
 * (exhaustive: prepare, thresholds, bfs, sweep, finalize; greedy: greedy). */
typedef struct bs_mpc_plan_s* bs_mpc_plan_t;
int bs_mpc_plan_create(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                       const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems, int n,
                       int mode, bs_mpc_plan_t* out);
int bs_mpc_plan_run(bs_ctx_t ctx, bs_mpc_plan_t plan, int record_kernel_times);
int bs_mpc_plan_results(bs_ctx_t ctx, bs_mpc_plan_t plan, bs_mpc_result* out);
int bs_mpc_plan_kernel_ms(bs_ctx_t ctx, bs_mpc_plan_t plan, float* ms, int n_ms);
int bs_mpc_plan_info(bs_ctx_t ctx, bs_mpc_plan_t plan, uint64_t* h2d_bytes, uint64_t* work_capacity);
void bs_mpc_plan_destroy(bs_ctx_t ctx, bs_mpc_plan_t plan);

/* Per-trajectory probe for one problem: codes[i] encodes an assignment with
 * batch 0 as the most significant base-|cand| digit.  out_feasible[i] =
 * meets_slo, out_objective[i] = time_weighted_power. */
int bs_mpc_eval_codes(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfg,
                      const bs_scheduler_policy* policy, const bs_mpc_problem* problem,
                      const uint64_t* codes, int n, int32_t* out_feasible, double* out_objective);

/* The per-(k, f) tables of one problem: lat[k][f] = wf_k * L(k, f),
 * pow[k][f] = P(k, f), energy[k][f] = lat * pow (W ms); each K x n_cand,
 * row-major, with n_cand = |ladder.select(ladder_N)|. */
int bs_mpc_tables(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfg,
                  const bs_scheduler_policy* policy, const bs_mpc_problem* problem, int32_t* out_K,
                  int32_t* out_n_cand, double* lat, double* pow, double* energy);

/* --- decode pick -------------------------------------------------------- */

int bs_decode_pick(bs_ctx_t ctx, bs_models_t models, const bs_decode_config* cfgs, int n_cfgs,
                   const bs_decode_query* queries, int n, bs_decode_result* out);

/* --- workload synthesis (host) -------------------------------------------- */

/* gen_gamma_trace (workload.hpp:95-116), bit-identical to the reference's
 * samplers (rng.hpp).  Writes min(n, capacity) requests (out may be NULL to
 * count) and the total count in *n_out; BS_PARAMETER_ERROR if capacity is
 * too small or an argument is invalid. */
int bs_gen_gamma_trace(double mean_rps, double shape, double duration_ms, const bs_length_dist* lengths,
                       uint64_t seed, bs_request* out, int64_t capacity, int64_t* n_out);

/* --- coarse-tier placement ----------------------------------------------- */

/* goodput_probe_trace (placement.hpp:145-149) = downsample_trace
 * (workload.hpp:120-132) with probe_seed(k, replicate): the kept request
 * indices (increasing) into trace->requests.  kept_idx holds trace->n. */
int bs_downsample_keep(bs_ctx_t ctx, const bs_trace* trace, const bs_goodput_search* search, int64_t k,
                       int replicate, int32_t* kept_idx, int64_t* n_kept);

/* build_config_table (placement.hpp:240-260): for every candidate,
 * max_goodput (154-199) and E_c (217-238).  Candidate order is the
 * caller's (enumerate_candidates, placement.hpp:535-548, gives phase x tp x
 * ladder). */
int bs_goodput_table(bs_ctx_t ctx, bs_models_t models, const bs_trace* base, const bs_slo* slo,
                     const bs_scheduler_policy* policy, const bs_goodput_search* search,
                     const bs_instance_config* cands, int n_cand, bs_table_entry* out);

/* build_config_table for n_tables probe traces (e.g. consecutive windows)
 * in ONE probe grid, long probes of every table first: out is
 * n_tables x n_cand (table-major).  A stream of tables is then bound by the
 * device's throughput, not by each table's longest probe in turn. */
int bs_goodput_tables(bs_ctx_t ctx, bs_models_t models, const bs_trace* bases, int n_tables, const bs_slo* slo,
                      const bs_scheduler_policy* policy, const bs_goodput_search* search,
                      const bs_instance_config* cands, int n_cand, bs_table_entry* out);

/* simulate_instance (simulator.hpp:667-739) at the instance's fixed
 * frequency (no controller) + sim_meets_slo (placement.hpp:119-131) +
 * energy sums, one device thread per trace: n traces share models, config,
 * policy and SLO.  out[i] = {status, meets_slo, completed, busy_j, idle_j,
 * horizon_ms}. */
typedef struct bs_sim_summary {
  int32_t status;
  int32_t meets_slo;
  int64_t completed;
  double busy_energy_j;
  double idle_energy_j;
  double horizon_ms;
} bs_sim_summary;
int bs_simulate_instance(bs_ctx_t ctx, bs_models_t models, const bs_trace* traces, int n,
                         const bs_instance_config* cfg, const bs_scheduler_policy* policy, const bs_slo* slo,
                         bs_sim_summary* out);

/* solve_placement (placement.hpp:357-416) on the device: counts[n]
 * (lexicographically smallest among equal-cost optima), objective, GPUs used.
 * BS_INFEASIBLE_ERROR: bs_last_error is "<binding constraint>|<message>".
 * ctx may be NULL: the calling thread's default context on device 0 is used
 * and the message is read with bs_last_error(NULL). */
int bs_placement_solve(bs_ctx_t ctx, const bs_table_entry* table, int n, int total_gpus, double target_rps,
                       double alpha, int64_t* counts, double* objective_w, int32_t* gpus_used);

/* solve_max_throughput (placement.hpp:421-499), the DistServe-style
 * max-frequency baseline. */
int bs_placement_max_throughput(bs_ctx_t ctx, const bs_table_entry* table, int n, int total_gpus,
                                double target_rps, double alpha, double max_freq_mhz, int64_t* counts,
                                double* objective_w, int32_t* gpus_used);

/* Many placement problems (e.g. every window of run_experiment) in one set
 * of device launches.  max_throughput != 0 selects solve_max_throughput with
 * max_freq_mhz.  Per problem: status (BS_OK, BS_INFEASIBLE_ERROR with error =
 * "<constraint>|<message>", or BS_PARAMETER_ERROR), counts written to the
 * caller's array, objective and GPUs used.  Limits of the device search: at
 * most 256 table entries, 2047 GPUs and 64 non-zero counts per plan. */
typedef struct bs_placement_problem {
  const bs_table_entry* table;
  int32_t n;
  int32_t total_gpus;
  double target_rps;
  double alpha;
  int32_t max_throughput;
  int32_t _pad;
  double max_freq_mhz;
  int64_t* counts; /* out: n entries */
} bs_placement_problem;
typedef struct bs_placement_solution {
  int32_t status;
  int32_t gpus_used;
  double objective_w;
  char error[192];
} bs_placement_solution;
int bs_placement_solve_batch(bs_ctx_t ctx, const bs_placement_problem* problems, int n,
                             bs_placement_solution* out);

/* --- cluster replay ---------------------------------------------------------- */

/* ClusterInstance (simulator.hpp:741-744). */
typedef struct bs_cluster_instance {
  bs_instance_config config;
  double weight; /* routing weight within its phase (RouterState, simulator.hpp:582-598) */
} bs_cluster_instance;

/* What run_policy / run_window_policy (runner.hpp:112-136) fix for one
 * replay: the controllers TwoTierFactory (dvfs.hpp:370-390) builds, the
 * simulator options and the report's SLO and ramp-up. */
typedef struct bs_replay_config {
  bs_mpc_config mpc;           /* PrefillMpcController configuration */
  bs_decode_config decode;     /* DecodePolicyController configuration */
  bs_scheduler_policy policy;  /* every instance's SchedulerPolicy (and the MPC projection's) */
  bs_slo slo;                  /* make_report's SLO (metrics.hpp:121) */
  double switch_latency_ms;    /* SimOptions::switch_latency_ms (simulator.hpp:127) */
  double horizon_ms;           /* SimOptions::horizon_ms; < 0: max(duration, last event) */
  double rampup_s;             /* trim_steady_state ramp-up (metrics.hpp:71) */
  int32_t controlled;          /* 1: TwoTierFactory controllers; 0: nullptr factory (base frequencies) */
  int32_t _pad;
} bs_replay_config;

/* One simulate_cluster call (simulator.hpp:758-893). */
typedef struct bs_scenario {
  bs_trace trace;                       /* requests sorted by arrival */
  const bs_cluster_instance* instances; /* index = instance id */
  int32_t n_instances;
  int32_t config;                       /* index into the bs_replay_config array */
} bs_scenario;

/* SimResult counters and the MetricsReport of
 * make_report(trim_steady_state(sim, rampup_s), slo) (metrics.hpp:71-156).
 * status: BS_OK or the exception class simulate_cluster would throw
 * (message through bs_last_error for the first failing scenario). */
typedef struct bs_replay_summary {
  int32_t status;
  int32_t has_p99_ttft;
  int32_t has_p99_tpot;
  int32_t has_e_first;
  int32_t has_e_output;
  int32_t _pad;
  double horizon_ms;
  int64_t completed_requests;      /* SimResult::completed_requests */
  int64_t generated_tokens;        /* SimResult::generated_tokens */
  int64_t n_batches;
  int64_t n_idles;
  int64_t n_decisions;
  int64_t decisions_by_trigger[3]; /* boundary, arrival, safety */
  /* MetricsReport */
  double p99_ttft_ms;
  double p99_mean_tpot_ms;
  double energy_per_first_token_j;
  double energy_per_output_token_j;
  double avg_power_prefill_w;
  double avg_power_decode_w;
  double prefill_energy_j;
  double decode_energy_j;
  double span_ms;
  int64_t report_completed;
  int64_t report_generated;
  int64_t ttft_violations;
  int64_t tpot_violations;
} bs_replay_summary;

/* RequestRecord (simulator.hpp:59-101), with the token times reduced to
 * what the metrics read.  Absent optionals are NaN. */
typedef struct bs_replay_request {
  int64_t id;
  int32_t prefill_instance;
  int32_t decode_instance;
  double prefill_done_ms;         /* = decode_join_ms */
  double decode_first_start_ms;
  double first_token_ms;          /* token_times_ms.front() */
  double last_token_ms;           /* token_times_ms.back() */
  double max_tbt_ms;              /* RequestRecord::max_tbt_ms */
  int64_t n_tokens;               /* token_times_ms.size() */
  int32_t completed;
  int32_t _pad;
} bs_replay_request;

/* BatchRecord / IdleRecord / DecisionRecord (simulator.hpp:33-57,
 * controller.hpp:100-107) in SimResult order (stable by start, instance). */
typedef struct bs_batch_record {
  int32_t instance;
  int32_t phase;
  int64_t batch_seq;
  double start_ms;
  double end_ms;
  int64_t n_requests;
  int64_t sum_len;
  double freq_mhz;
  double power_w;
  double energy_j;
} bs_batch_record;

typedef struct bs_idle_record {
  int32_t instance;
  int32_t phase;
  double start_ms;
  double end_ms;
  double freq_mhz;
  double power_w;
  double energy_j;
} bs_idle_record;

typedef struct bs_decision_record {
  double time_ms;
  int32_t instance;
  int32_t trigger; /* 0 boundary, 1 arrival, 2 safety */
  double chosen_freq_mhz;
  int32_t feasible;
  int32_t _pad;
  int64_t eval_count;
} bs_decision_record;

/* Optional full logs of one scenario: caller arrays and capacities; the
 * counts are written back (records beyond a capacity are dropped and the
 * count still reports the total). */
typedef struct bs_replay_logs {
  bs_batch_record* batches;
  int64_t batch_cap;
  int64_t n_batches;
  bs_idle_record* idles;
  int64_t idle_cap;
  int64_t n_idles;
  bs_decision_record* decisions;
  int64_t decision_cap;
  int64_t n_decisions;
} bs_replay_logs;

/* simulate_cluster (simulator.hpp:758-893) + trim_steady_state + make_report
 * for n independent scenarios, on the device: prefill instances one CTA each
 * (event loop + block-cooperative greedy MPC per decision), decode instances
 * one warp each (event loop + warp ladder walk per iteration).  sim_models
 * is the simulator's ground truth, ctl_models the controllers' model set
 * (TwoTierFactory's controller_models; may be the same handle).  requests
 * (optional) receives sum(trace.n) records in trace order; logs (optional)
 * one entry per scenario. */
int bs_replay(bs_ctx_t ctx, bs_models_t sim_models, bs_models_t ctl_models, const bs_replay_config* cfgs, int n_cfgs,
              const bs_scenario* scenarios, int n, bs_replay_summary* out, bs_replay_request* requests,
              bs_replay_logs* logs);

#ifdef __cplusplus
}
#endif

#endif /* BISCALE_GPU_H_ */

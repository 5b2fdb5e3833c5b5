/* ref_driver.h -- TEST INFRASTRUCTURE ONLY.  extern "C" wrappers over the
 * unmodified reference (see ref_driver.cpp).  Built into
 * oracle/_ref/libpdsim_ref.so by oracle/Makefile; used by tests/ and by
 * bench.py's cpu_baseline / --impl reference legs only. */
#ifndef PDSIM_REF_DRIVER_H_
#define PDSIM_REF_DRIVER_H_
#include "biscale_gpu.h"
#ifdef __cplusplus
extern "C" {
#endif
/* RunnerConfig (runner.hpp:39-86) as a POD, for ref_run_experiment. */
typedef struct ref_runner_config {
  bs_slo slo;
  int32_t total_gpus;
  int32_t n_tp;
  const int32_t* tp_options;
  const double* ladder;
  int32_t n_ladder;
  int32_t mpc_k;
  bs_scheduler_policy scheduler;
  double alpha;
  double peak_subwindow_s;
  bs_goodput_search search;
  bs_scheduler_policy plan_policy;
  double rampup_s;
  double switch_latency_ms;
  int32_t mpc_n;
  int32_t _pad;
  double mpc_margin;
  double kv_threshold;
  double decode_margin;
} ref_runner_config;

typedef struct ref_window_run {
  int32_t window;
  int32_t policy;
  int32_t gpus_used;
  int32_t slo_pass;
  double objective_w;
  double target_rps;
  bs_replay_summary report; /* SimResult counters + MetricsReport */
} ref_window_run;

const char* ref_last_error(void);
int ref_interpolate(const bs_grid* grid, const double* coords, int n, double* out, uint32_t* clamp_events);
int ref_predict(const bs_model_set* models, int which, const bs_features* feats, const int32_t* tp,
                const double* freq, int n, double* out, int32_t* status);
int ref_synth_model_set(int family, const double* ladder, int n_ladder, const int32_t* tps, int n_tp,
                        const double* prefill_opt, const double* decode_opt, double* lat_p, double* lat_d,
                        double* pow_p, double* pow_d, double* idle_w);
int ref_project(const bs_mpc_config* cfg, const bs_scheduler_policy* policy, const bs_snapshot* snap,
                bs_projected_batch* out, int32_t* out_K);
int ref_greedy(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
               const bs_snapshot* snap, bs_mpc_result* out);
int ref_greedy_batch(const bs_model_set* models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
                     const bs_mpc_problem* problems, int n, bs_mpc_result* out, int n_threads);
int ref_exhaustive(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, bs_mpc_result* out);
int ref_exhaustive_batch(const bs_model_set* models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
                         const bs_mpc_problem* problems, int n, bs_mpc_result* out, int n_threads);
int ref_eval_codes(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, const uint64_t* codes, int n, int32_t* out_feasible,
                   double* out_objective);
int ref_tables(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
               const bs_snapshot* snap, int32_t* out_K, int32_t* out_n_cand, double* lat, double* pow,
               double* energy);
int ref_decode_pick(const bs_model_set* models, const bs_decode_config* cfgs, const bs_decode_query* queries, int n,
                    bs_decode_result* out);
int ref_gen_gamma_trace(double mean_rps, double shape, double duration_ms, const bs_length_dist* lengths,
                        uint64_t seed, bs_request* out, int64_t capacity, int64_t* n_out);
int ref_downsample_keep(const bs_trace* trace, const bs_goodput_search* search, int64_t k, int replicate,
                        int32_t* kept_idx, int64_t* n_kept);
int ref_config_table(const bs_model_set* models, const bs_trace* trace, const bs_slo* slo,
                     const bs_scheduler_policy* policy, const bs_goodput_search* search,
                     const bs_instance_config* cands, int n, bs_table_entry* out);
int ref_solve_placement(const bs_table_entry* table, int n, int total_gpus, double target_rps, double alpha,
                        int64_t* counts, double* objective_w, int32_t* gpus_used);
int ref_simulate(const bs_model_set* models, const bs_trace* traces, int n, const bs_instance_config* cfg,
                 const bs_scheduler_policy* policy, const bs_slo* slo, bs_sim_summary* out);
int ref_solve_max_throughput(const bs_table_entry* table, int n, int total_gpus, double target_rps, double alpha,
                             double max_freq_mhz, int64_t* counts, double* objective_w, int32_t* gpus_used);
int ref_run_experiment(const bs_model_set* models, const bs_trace* trace, double window_ms, const int32_t* policies,
                       int n_policies, const ref_runner_config* cfg, ref_window_run* out, int cap, int* n_out,
                       int32_t* two_tier_slo_pass);
int ref_replay(const bs_model_set* sim_models, const bs_model_set* ctl_models, const bs_replay_config* cfgs,
               const bs_scenario* sc, int n, bs_replay_summary* out, bs_replay_request* requests,
               bs_replay_logs* logs, int n_threads);
#ifdef __cplusplus
}
#endif
#endif

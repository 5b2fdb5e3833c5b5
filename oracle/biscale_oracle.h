/* biscale_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's decision-evaluation algorithms
 * (/root/reference/proj/include/pdsim/), used as the CPU checker for
 * the sm_100a path.  Each function cites the reference file:line it follows.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  Pinned against the reference itself (oracle/_ref) and the
 * reference's own known-answer tests: see tests/test_oracle_*.py.
 *
 * Inputs are the POD structs of include/biscale_gpu.h, so the oracle, the
 * reference driver and the GPU path all see byte-identical problems.
 */
#ifndef BISCALE_ORACLE_H_
#define BISCALE_ORACLE_H_
#include "biscale_gpu.h"
#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* NdGrid::interpolate (perfmodel.hpp:150-193); *clamps += clamp events. */
int orc_interpolate(const bs_grid* grid, const double* coords, double* out, uint32_t* clamps);
/* predict_latency / predict_power / predict_idle_power (perfmodel.hpp:262-288).
 * which: 0 lat prefill, 1 lat decode, 2 pow prefill, 3 pow decode, 4 idle. */
int orc_predict(const bs_model_set* m, int which, const bs_features* f, int tp, double freq, double* out);
int orc_predict_batch(const bs_model_set* m, int which, const bs_features* feats, const int32_t* tp,
                      const double* freq, int n, double* out, int32_t* status);

/* FrequencyLadder::select (perfmodel.hpp:76-91); returns count, -1 on error. */
int orc_ladder_select(const double* ladder, int n_ladder, int n, double* out);

/* synth_model_set (perfmodel.hpp:397-516) with the default knots
 * (perfmodel.hpp:385-386).  opt = {lat_coef, power_a, power_b, mem_knee, idle_frac}. */
int orc_synth_model_set(int family, const double* ladder, int n_ladder, const int32_t* tps, int n_tp,
                        const double* prefill_opt, const double* decode_opt, double* lat_p, double* lat_d,
                        double* pow_p, double* pow_d, double* idle_w);

/* project_batches (dvfs.hpp:63-100) over form_prefill_batch (scheduler.hpp:40-66). */
int orc_project(const bs_mpc_config* cfg, const bs_scheduler_policy* policy, const bs_snapshot* snap,
                bs_projected_batch* out, int32_t* out_K);

/* greedy_freq_select (dvfs.hpp:185-259) + PrefillMpcController::run (325-333). */
int orc_greedy(const bs_model_set* m, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
               const bs_snapshot* snap, bs_mpc_result* out);

/* Exhaustive MPC (tests/test_dvfs.cpp:74-94 loop; pinned lex tie-break). */
int orc_exhaustive(const bs_model_set* m, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, bs_mpc_result* out);

/* meets_slo + time_weighted_power for given codes (batch 0 most significant). */
int orc_eval_codes(const bs_model_set* m, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, const uint64_t* codes, int n, int32_t* out_feasible,
                   double* out_objective);

/* select_decode_freq_ex (dvfs.hpp:274-293). */
int orc_decode_pick(const bs_model_set* m, const bs_decode_config* cfgs, const bs_decode_query* queries, int n,
                    bs_decode_result* out);

#ifdef __cplusplus
}
#endif
#endif

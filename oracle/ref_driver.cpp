// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (oracle).  Wraps the UNMODIFIED
// reference headers (/root/reference/proj/include/pdsim, compiled where they
// lie; nothing is copied) behind extern "C" entry points that take the same
// POD structs as include/biscale_gpu.h, so the parity tests can run the real
// reference on exactly the inputs the GPU path sees.  Built by
// oracle/Makefile into oracle/_ref/libpdsim_ref.so.  Never linked into, or
// called by, the product path.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "pdsim/dvfs.hpp"
#include "pdsim/metrics.hpp"
#include "pdsim/placement.hpp"
#include "pdsim/runner.hpp"
#include "pdsim/simulator.hpp"
#include "pdsim/workload.hpp"

#include "biscale_gpu.h"
#include "ref_driver.h"

using namespace pdsim;

namespace {

const char* role_name(int role) {
  switch (role) {
    case BS_AXIS_SUM_LEN: return kAxisSumLen;
    case BS_AXIS_N_REQUESTS: return kAxisNumRequests;
    case BS_AXIS_TP: return kAxisTp;
    case BS_AXIS_FREQ: return kAxisFreq;
    default: return "unknown";
  }
}

NdGrid to_grid(const bs_grid& g) {
  NdGrid out;
  std::size_t total = 1;
  for (int d = 0; d < g.rank; ++d) {
    Axis a;
    a.name = role_name(g.role[d]);
    a.knots.assign(g.knots[d], g.knots[d] + g.n_knots[d]);
    total *= static_cast<std::size_t>(g.n_knots[d]);
    out.axes.push_back(std::move(a));
  }
  out.values.assign(g.values, g.values + total);
  return out;
}

ModelSet to_models(const bs_model_set& m) {
  ModelSet s;
  s.latency_prefill.phase = Phase::prefill;
  s.latency_prefill.grid = to_grid(m.latency_prefill);
  s.latency_decode.phase = Phase::decode;
  s.latency_decode.grid = to_grid(m.latency_decode);
  s.power_prefill.phase = Phase::prefill;
  s.power_prefill.grid = to_grid(m.power_prefill);
  s.power_decode.phase = Phase::decode;
  s.power_decode.grid = to_grid(m.power_decode);
  for (int i = 0; i < m.n_idle; ++i) {
    IdlePowerModel::TpEntry e;
    e.tp = m.idle[i].tp;
    e.freqs_mhz.assign(m.idle[i].freqs_mhz, m.idle[i].freqs_mhz + m.idle[i].n);
    e.idle_w.assign(m.idle[i].idle_w, m.idle[i].idle_w + m.idle[i].n);
    s.idle.entries.push_back(std::move(e));
  }
  return s;
}

MpcConfig to_mpc(const bs_mpc_config& c) {
  MpcConfig m;
  m.horizon_K = c.horizon_K;
  m.ladder_N = c.ladder_N;
  m.ladder.freqs_mhz.assign(c.ladder_mhz, c.ladder_mhz + c.n_ladder);
  m.slo.ttft_ms = c.ttft_ms;
  m.slo.tpot_ms = c.tpot_ms;
  m.slo.percentile = c.percentile;
  m.switch_latency_ms = c.switch_latency_ms;
  m.margin = c.margin;
  return m;
}

SchedulerPolicy to_policy(const bs_scheduler_policy& p) {
  SchedulerPolicy s;
  s.max_batch_tokens = p.max_batch_tokens;
  s.max_batch_requests = p.max_batch_requests;
  s.kv_capacity_tokens = p.kv_capacity_tokens;
  s.chunking = p.chunking != 0;
  return s;
}

QueueSnapshot to_snapshot(const bs_snapshot& s) {
  QueueSnapshot q;
  q.now_ms = s.now_ms;
  q.phase = Phase::prefill;
  q.tp = s.tp;
  q.current_freq_mhz = s.current_freq_mhz;
  q.target_freq_mhz = s.target_freq_mhz;
  for (int i = 0; i < s.n_waiting; ++i) {
    q.waiting.push_back(SnapshotWaiting{s.waiting[i].id, s.waiting[i].arrival_ms, s.waiting[i].total_len,
                                        s.waiting[i].remaining_len});
  }
  if (s.running_active) {
    q.running.active = true;
    for (int i = 0; i < s.n_running; ++i) {
      q.running.ids.push_back(i);
      q.running.chunk_lens.push_back(0);
      q.running.completes.push_back(s.running_completes[i] != 0);
      q.running.arrivals_ms.push_back(s.running_arrivals_ms[i]);
    }
    q.running.work_remaining = s.running_work_remaining;
    q.running.features.n_requests = s.running_features.n_requests;
    q.running.features.sum_len = s.running_features.sum_len;
  }
  return q;
}

int status_of(const std::exception& e) {
  if (dynamic_cast<const ParameterError*>(&e)) return BS_PARAMETER_ERROR;
  if (dynamic_cast<const ModelError*>(&e)) return BS_MODEL_ERROR;
  if (dynamic_cast<const SimulationError*>(&e)) return BS_SIMULATION_ERROR;
  if (dynamic_cast<const ConfigError*>(&e)) return BS_CONFIG_ERROR;
  if (dynamic_cast<const AccountingError*>(&e)) return BS_ACCOUNTING_ERROR;
  if (dynamic_cast<const IoError*>(&e)) return BS_IO_ERROR;
  if (dynamic_cast<const InfeasibleError*>(&e)) return BS_INFEASIBLE_ERROR;
  return 99;
}

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return BS_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

void fill_result(const GreedyResult& g, const std::vector<double>& cand, const QueueSnapshot& q, double max_mhz,
                 bs_mpc_result* r) {
  std::memset(r, 0, sizeof(*r));
  r->K = static_cast<int32_t>(g.assignment.freqs.size());
  r->feasible = g.feasible ? 1 : 0;
  r->eval_count = g.eval_count;
  r->objective_w = g.objective_w;
  for (std::size_t k = 0; k < g.assignment.freqs.size() && k < BS_MAX_K; ++k) {
    r->freqs_mhz[k] = g.assignment.freqs[k];
    auto it = std::find(cand.begin(), cand.end(), g.assignment.freqs[k]);
    r->freq_index[k] = it == cand.end() ? -1 : static_cast<int32_t>(it - cand.begin());
  }
  r->n_levels = static_cast<int32_t>(g.levels.size());
  for (std::size_t l = 0; l < g.levels.size() && l < BS_MAX_LEVELS; ++l) {
    r->levels[l].level = g.levels[l].level;
    r->levels[l].k_prime = g.levels[l].k_prime;
    r->levels[l].replaced_mhz = g.levels[l].replaced_mhz;
    r->levels[l].mutations = g.levels[l].mutations;
    r->levels[l].feasible_mutations = g.levels[l].feasible_mutations;
    r->levels[l].accepted = g.levels[l].accepted ? 1 : 0;
  }
  // PrefillMpcController::run (dvfs.hpp:328-329)
  r->decision_freq_mhz = g.assignment.freqs.empty() ? (q.target_freq_mhz > 0 ? q.target_freq_mhz : max_mhz)
                                                    : g.assignment.freqs.front();
}

// tw_power exactly as the reference test oracle computes it
// (tests/test_dvfs.cpp:58-67, tests/acceptance_main.cpp:150-160).
double tw_power(const FrequencyAssignment& a, const std::vector<ProjectedBatch>& proj, const QueueSnapshot& q,
                const ModelSet& m) {
  double num = 0.0, den = 0.0;
  for (std::size_t k = 0; k < a.freqs.size(); ++k) {
    double lat = proj[k].work_fraction * predict_latency(m.latency_prefill, proj[k].features, q.tp, a.freqs[k]);
    num += lat * predict_power(m.power_prefill, proj[k].features, q.tp, a.freqs[k]);
    den += lat;
  }
  return den > 0.0 ? num / den : 0.0;
}

// Exhaustive MPC in the shape of the reference oracle loop
// (tests/test_dvfs.cpp:74-94): odometer with digit 0 fastest, meets_slo then
// tw_power per assignment.  The pinned tie-break (objective, then
// lexicographic frequency vector -- dvfs.hpp:243's rule) replaces the
// test's objective-only first-min; feasible assignments are counted.
void exhaustive_one(const ModelSet& m, const MpcConfig& cfg, const SchedulerPolicy& policy, const QueueSnapshot& q,
                    bs_mpc_result* r) {
  cfg.validate();
  std::vector<double> cand = cfg.candidates().freqs_mhz;
  std::vector<ProjectedBatch> proj = project_batches(q, policy, cfg.horizon_K);
  std::memset(r, 0, sizeof(*r));
  const std::size_t K = proj.size();
  r->K = static_cast<int32_t>(K);
  double max_mhz = cand.back();
  if (K == 0) {
    r->feasible = 1;
    r->decision_freq_mhz = q.target_freq_mhz > 0 ? q.target_freq_mhz : max_mhz;
    return;
  }
  std::vector<std::size_t> idx(K, 0);
  bool found = false;
  double best_p = 0.0;
  std::vector<double> best_f;
  std::vector<std::size_t> best_idx;
  std::uint64_t feasible_count = 0, total = 0;
  FrequencyAssignment a;
  a.freqs.resize(K);
  while (true) {
    for (std::size_t k = 0; k < K; ++k) a.freqs[k] = cand[idx[k]];
    ++total;
    if (meets_slo(a, proj, q, m, cfg)) {
      ++feasible_count;
      double p = tw_power(a, proj, q, m);
      if (!found || p < best_p || (p == best_p && detail::lex_less(a.freqs, best_f))) {
        found = true;
        best_p = p;
        best_f = a.freqs;
        best_idx = idx;
      }
    }
    std::size_t d = 0;
    while (d < idx.size() && ++idx[d] == cand.size()) idx[d++] = 0;
    if (d == idx.size()) break;
  }
  r->trajectories = total;
  r->feasible_count = feasible_count;
  r->eval_count = static_cast<int64_t>(total);
  if (!found) {
    best_f.assign(K, max_mhz);
    best_idx.assign(K, cand.size() - 1);
    a.freqs = best_f;
    best_p = tw_power(a, proj, q, m);
  }
  r->feasible = found ? 1 : 0;
  r->objective_w = best_p;
  std::uint64_t code = 0;
  for (std::size_t k = 0; k < K; ++k) {
    r->freqs_mhz[k] = best_f[k];
    r->freq_index[k] = static_cast<int32_t>(best_idx[k]);
    code = code * cand.size() + best_idx[k];
  }
  r->best_code = code;
  r->decision_freq_mhz = best_f.front();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_interpolate(const bs_grid* grid, const double* coords, int n, double* out, uint32_t* clamp_events) {
  return guarded([&] {
    NdGrid g = to_grid(*grid);
    g.validate_structure();
    for (int i = 0; i < n; ++i) {
      std::vector<double> c(coords + static_cast<std::size_t>(i) * grid->rank,
                            coords + static_cast<std::size_t>(i + 1) * grid->rank);
      std::uint64_t before = g.clamp_events.value.load();
      out[i] = g.interpolate(c);
      if (clamp_events) clamp_events[i] = static_cast<uint32_t>(g.clamp_events.value.load() - before);
    }
  });
}

int ref_predict(const bs_model_set* models, int which, const bs_features* feats, const int32_t* tp,
                const double* freq, int n, double* out, int32_t* status) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    for (int i = 0; i < n; ++i) {
      BatchFeatures f;
      f.n_requests = feats[i].n_requests;
      f.sum_len = feats[i].sum_len;
      status[i] = guarded([&] {
        switch (which) {
          case 0: out[i] = predict_latency(m.latency_prefill, f, tp[i], freq[i]); break;
          case 1: out[i] = predict_latency(m.latency_decode, f, tp[i], freq[i]); break;
          case 2: out[i] = predict_power(m.power_prefill, f, tp[i], freq[i]); break;
          case 3: out[i] = predict_power(m.power_decode, f, tp[i], freq[i]); break;
          default: out[i] = predict_idle_power(m.idle, tp[i], freq[i]); break;
        }
      });
      if (status[i] != BS_OK) out[i] = 0.0;
    }
  });
}

int ref_synth_model_set(int family, const double* ladder, int n_ladder, const int32_t* tps, int n_tp,
                        const double* prefill_opt, const double* decode_opt, double* lat_p, double* lat_d,
                        double* pow_p, double* pow_d, double* idle_w) {
  return guarded([&] {
    FrequencyLadder l;
    l.freqs_mhz.assign(ladder, ladder + n_ladder);
    std::vector<int> tp_list(tps, tps + n_tp);
    auto opts = [](const double* o) {
      SynthOptions s;
      s.lat_coef = o[0];
      s.power_a = o[1];
      s.power_b = o[2];
      s.mem_knee_mhz = o[3];
      s.idle_frac = o[4];
      return s;
    };
    ModelSet m = synth_model_set(family == 0 ? SynthFamily::compute_bound : SynthFamily::memory_bound, l, tp_list,
                                 opts(prefill_opt), opts(decode_opt));
    std::copy(m.latency_prefill.grid.values.begin(), m.latency_prefill.grid.values.end(), lat_p);
    std::copy(m.latency_decode.grid.values.begin(), m.latency_decode.grid.values.end(), lat_d);
    std::copy(m.power_prefill.grid.values.begin(), m.power_prefill.grid.values.end(), pow_p);
    std::copy(m.power_decode.grid.values.begin(), m.power_decode.grid.values.end(), pow_d);
    std::size_t o = 0;
    for (const auto& e : m.idle.entries) {
      for (double w : e.idle_w) idle_w[o++] = w;
    }
  });
}

int ref_project(const bs_mpc_config* cfg, const bs_scheduler_policy* policy, const bs_snapshot* snap,
                bs_projected_batch* out, int32_t* out_K) {
  return guarded([&] {
    QueueSnapshot q = to_snapshot(*snap);
    std::vector<ProjectedBatch> proj = project_batches(q, to_policy(*policy), cfg->horizon_K);
    *out_K = static_cast<int32_t>(proj.size());
    for (std::size_t k = 0; k < proj.size() && k < BS_MAX_K; ++k) {
      out[k].features.n_requests = proj[k].features.n_requests;
      out[k].features.sum_len = proj[k].features.sum_len;
      out[k].work_fraction = proj[k].work_fraction;
      out[k].n_completing = static_cast<int32_t>(proj[k].completing_arrivals_ms.size());
      double mn = std::numeric_limits<double>::infinity();
      for (double a : proj[k].completing_arrivals_ms) mn = std::min(mn, a);
      out[k].min_completing_arrival_ms = mn;
    }
  });
}

int ref_greedy(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
               const bs_snapshot* snap, bs_mpc_result* out) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    MpcConfig c = to_mpc(*cfg);
    QueueSnapshot q = to_snapshot(*snap);
    GreedyResult g = greedy_freq_select(q, c, m, to_policy(*policy));
    std::vector<double> cand = c.candidates().freqs_mhz;
    fill_result(g, cand, q, cand.back(), out);
  });
}

// Many greedy decisions spread over host threads (each reference call stays
// single-threaded, as the simulator uses it).  Returns the first failure.
int ref_greedy_batch(const bs_model_set* models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
                     const bs_mpc_problem* problems, int n, bs_mpc_result* out, int n_threads) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    std::atomic<int> next{0};
    auto work = [&] {
      for (;;) {
        int i = next.fetch_add(1);
        if (i >= n) return;
        const bs_mpc_problem& p = problems[i];
        out[i].status = guarded([&] {
          MpcConfig c = to_mpc(cfgs[p.cfg_index]);
          QueueSnapshot q = to_snapshot(p.snap);
          GreedyResult g = greedy_freq_select(q, c, m, to_policy(policies[p.cfg_index]));
          std::vector<double> cand = c.candidates().freqs_mhz;
          fill_result(g, cand, q, cand.back(), &out[i]);
        });
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, n_threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
  });
}

int ref_exhaustive(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, bs_mpc_result* out) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    exhaustive_one(m, to_mpc(*cfg), to_policy(*policy), to_snapshot(*snap), out);
  });
}

int ref_exhaustive_batch(const bs_model_set* models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
                         const bs_mpc_problem* problems, int n, bs_mpc_result* out, int n_threads) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    std::atomic<int> next{0};
    auto work = [&] {
      for (;;) {
        int i = next.fetch_add(1);
        if (i >= n) return;
        const bs_mpc_problem& p = problems[i];
        out[i].status = guarded([&] {
          exhaustive_one(m, to_mpc(cfgs[p.cfg_index]), to_policy(policies[p.cfg_index]), to_snapshot(p.snap),
                         &out[i]);
        });
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, n_threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
  });
}

int ref_eval_codes(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, const uint64_t* codes, int n, int32_t* out_feasible,
                   double* out_objective) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    MpcConfig c = to_mpc(*cfg);
    QueueSnapshot q = to_snapshot(*snap);
    std::vector<double> cand = c.candidates().freqs_mhz;
    std::vector<ProjectedBatch> proj = project_batches(q, to_policy(*policy), c.horizon_K);
    const std::size_t K = proj.size();
    FrequencyAssignment a;
    a.freqs.resize(K);
    for (int i = 0; i < n; ++i) {
      std::uint64_t code = codes[i];
      for (std::size_t k = K; k-- > 0;) {
        a.freqs[k] = cand[code % cand.size()];
        code /= cand.size();
      }
      out_feasible[i] = meets_slo(a, proj, q, m, c) ? 1 : 0;
      detail::MpcEvaluator ev{proj, q, m, c, {}};
      out_objective[i] = ev.time_weighted_power(a);
    }
  });
}

int ref_tables(const bs_model_set* models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
               const bs_snapshot* snap, int32_t* out_K, int32_t* out_n_cand, double* lat, double* pow,
               double* energy) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    MpcConfig c = to_mpc(*cfg);
    QueueSnapshot q = to_snapshot(*snap);
    std::vector<double> cand = c.candidates().freqs_mhz;
    std::vector<ProjectedBatch> proj = project_batches(q, to_policy(*policy), c.horizon_K);
    detail::MpcEvaluator ev{proj, q, m, c, {}};
    *out_K = static_cast<int32_t>(proj.size());
    *out_n_cand = static_cast<int32_t>(cand.size());
    for (std::size_t k = 0; k < proj.size(); ++k) {
      for (std::size_t f = 0; f < cand.size(); ++f) {
        auto [l, p] = ev.eval(k, cand[f]);
        lat[k * cand.size() + f] = l;
        pow[k * cand.size() + f] = p;
        energy[k * cand.size() + f] = l * p;
      }
    }
  });
}

int ref_decode_pick(const bs_model_set* models, const bs_decode_config* cfgs, const bs_decode_query* queries, int n,
                    bs_decode_result* out) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    for (int i = 0; i < n; ++i) {
      const bs_decode_query& qq = queries[i];
      const bs_decode_config& c = cfgs[qq.cfg_index];
      DecodePolicyConfig dc;
      dc.tbt_slo_ms = c.tbt_slo_ms;
      dc.kv_threshold = c.kv_threshold;
      dc.margin = c.margin;
      dc.ladder.freqs_mhz.assign(c.ladder_mhz, c.ladder_mhz + c.n_ladder);
      BatchFeatures f;
      f.n_requests = qq.batch.n_requests;
      f.sum_len = qq.batch.sum_len;
      KVCacheState kv;
      kv.capacity_tokens = qq.kv_capacity_tokens;
      kv.used_tokens = qq.kv_used_tokens;
      std::memset(&out[i], 0, sizeof(out[i]));
      out[i].status = guarded([&] {
        DecodeDecision d = select_decode_freq_ex(f, kv, dc, m, qq.tp);
        out[i].freq_mhz = d.freq_mhz;
        out[i].eval_count = d.eval_count;
        out[i].kv_override = d.kv_override ? 1 : 0;
      });
    }
  });
}

}  // extern "C"

namespace {

Trace to_trace(const bs_trace& t) {
  Trace out;
  out.duration_ms = t.duration_ms;
  for (int64_t i = 0; i < t.n; ++i)
    out.requests.push_back(Request{t.requests[i].id, t.requests[i].arrival_ms, t.requests[i].input_len,
                                   t.requests[i].output_len});
  return out;
}

GoodputSearch to_search(const bs_goodput_search& s) {
  GoodputSearch g;
  g.tolerance_rps = s.tolerance_rps;
  g.probe_count = s.probe_count;
  g.seed = s.seed;
  return g;
}

SLOSpec to_slo(const bs_slo& s) {
  SLOSpec o;
  o.ttft_ms = s.ttft_ms;
  o.tpot_ms = s.tpot_ms;
  o.percentile = s.percentile;
  return o;
}

std::vector<ConfigTableEntry> to_table(const bs_table_entry* t, int n) {
  std::vector<ConfigTableEntry> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    out[i].config = InstanceConfig{t[i].config.phase == BS_PHASE_PREFILL ? Phase::prefill : Phase::decode,
                                   t[i].config.tp, t[i].config.base_freq_mhz};
    out[i].r_c = t[i].r_c;
    if (t[i].has_e_c) out[i].e_c = t[i].e_c;
    out[i].g_c = t[i].g_c;
    out[i].saturated = t[i].saturated != 0;
    out[i].error = t[i].error_code ? std::string(t[i].error) : std::string();
  }
  return out;
}

}  // namespace

extern "C" {

int ref_gen_gamma_trace(double mean_rps, double shape, double duration_ms, const bs_length_dist* lengths,
                        uint64_t seed, bs_request* out, int64_t capacity, int64_t* n_out) {
  return guarded([&] {
    LengthDistribution d;
    if (lengths->n_samples > 0) {
      for (int i = 0; i < lengths->n_samples; ++i)
        d.samples.emplace_back(lengths->sample_input[i], lengths->sample_output[i]);
    } else {
      d.lognormal = LengthDistribution::Lognormal{lengths->input_mu, lengths->input_sigma, lengths->output_mu,
                                                  lengths->output_sigma};
    }
    Trace t = gen_gamma_trace(mean_rps, shape, duration_ms, d, seed);
    *n_out = static_cast<int64_t>(t.requests.size());
    for (std::size_t i = 0; i < t.requests.size() && static_cast<int64_t>(i) < capacity; ++i)
      if (out) out[i] = bs_request{t.requests[i].id, t.requests[i].arrival_ms, t.requests[i].input_len,
                                   t.requests[i].output_len};
  });
}

int ref_downsample_keep(const bs_trace* trace, const bs_goodput_search* search, int64_t k, int replicate,
                        int32_t* kept_idx, int64_t* n_kept) {
  return guarded([&] {
    Trace base = to_trace(*trace);
    Trace probe = goodput_probe_trace(base, to_search(*search), k, replicate);
    std::size_t j = 0;
    int64_t c = 0;
    for (const Request& r : probe.requests) {
      while (j < base.requests.size() && base.requests[j].id != r.id) ++j;
      kept_idx[c++] = static_cast<int32_t>(j++);
    }
    *n_kept = c;
  });
}

int ref_config_table(const bs_model_set* models, const bs_trace* trace, const bs_slo* slo,
                     const bs_scheduler_policy* policy, const bs_goodput_search* search,
                     const bs_instance_config* cands, int n, bs_table_entry* out) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    std::vector<InstanceConfig> cs;
    for (int i = 0; i < n; ++i)
      cs.push_back(InstanceConfig{cands[i].phase == BS_PHASE_PREFILL ? Phase::prefill : Phase::decode, cands[i].tp,
                                  cands[i].base_freq_mhz});
    std::vector<ConfigTableEntry> t =
        build_config_table(cs, to_trace(*trace), to_slo(*slo), m, to_policy(*policy), to_search(*search), true);
    for (int i = 0; i < n; ++i) {
      std::memset(&out[i], 0, sizeof(out[i]));
      out[i].config = cands[i];
      out[i].r_c = t[i].r_c;
      out[i].has_e_c = t[i].e_c.has_value() ? 1 : 0;
      out[i].e_c = t[i].e_c.value_or(0.0);
      out[i].g_c = t[i].g_c;
      out[i].saturated = t[i].saturated ? 1 : 0;
      out[i].k_star = static_cast<int64_t>(std::llround(t[i].r_c / search->tolerance_rps));
      out[i].error_code = t[i].error.empty() ? 0 : (t[i].error == "no completed request at R_c" ? -1 : BS_MODEL_ERROR);
      std::snprintf(out[i].error, sizeof(out[i].error), "%s", t[i].error.c_str());
    }
  });
}

int ref_solve_placement(const bs_table_entry* table, int n, int total_gpus, double target_rps, double alpha,
                        int64_t* counts, double* objective_w, int32_t* gpus_used) {
  try {
    PlacementProblem p{to_table(table, n), total_gpus, target_rps, alpha};
    PlacementPlan plan = solve_placement(p);
    for (int i = 0; i < n; ++i) counts[i] = plan.counts[i];
    *objective_w = plan.objective_w;
    *gpus_used = plan.gpus_used;
    return BS_OK;
  } catch (const InfeasibleError& e) {
    g_err = e.binding_constraint() + "|" + e.what();
    return BS_INFEASIBLE_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

int ref_solve_max_throughput(const bs_table_entry* table, int n, int total_gpus, double target_rps, double alpha,
                             double max_freq_mhz, int64_t* counts, double* objective_w, int32_t* gpus_used) {
  try {
    PlacementProblem p{to_table(table, n), total_gpus, target_rps, alpha};
    PlacementPlan plan = solve_max_throughput(p, max_freq_mhz);
    for (int i = 0; i < n; ++i) counts[i] = plan.counts[i];
    *objective_w = plan.objective_w;
    *gpus_used = plan.gpus_used;
    return BS_OK;
  } catch (const InfeasibleError& e) {
    g_err = e.binding_constraint() + "|" + e.what();
    return BS_INFEASIBLE_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

}  // extern "C"

extern "C" int ref_simulate(const bs_model_set* models, const bs_trace* traces, int n, const bs_instance_config* cfg,
                            const bs_scheduler_policy* policy, const bs_slo* slo, bs_sim_summary* out) {
  return guarded([&] {
    ModelSet m = to_models(*models);
    InstanceConfig ic{cfg->phase == BS_PHASE_PREFILL ? Phase::prefill : Phase::decode, cfg->tp, cfg->base_freq_mhz};
    for (int i = 0; i < n; ++i) {
      std::memset(&out[i], 0, sizeof(out[i]));
      out[i].status = guarded([&] {
        SimResult r = simulate_instance(to_trace(traces[i]), ic, to_policy(*policy), m);
        out[i].meets_slo = sim_meets_slo(r, ic.phase, to_slo(*slo)) ? 1 : 0;
        out[i].completed = r.completed_requests;
        out[i].busy_energy_j = r.busy_energy_j();
        out[i].idle_energy_j = r.idle_energy_j();
        out[i].horizon_ms = r.horizon_ms;
      });
    }
  });
}

// --- cluster replay: simulate_cluster + trim_steady_state + make_report -------

namespace {

void replay_one(const ModelSet& sim_m, const ModelSet& ctl_m, const bs_replay_config& rc, const bs_scenario& sc,
                bs_replay_summary* o, bs_replay_request* req, bs_replay_logs* logs) {
  Trace tr = to_trace(sc.trace);
  ClusterSpec cl;
  for (int i = 0; i < sc.n_instances; ++i) {
    const bs_cluster_instance& ci = sc.instances[i];
    cl.instances.push_back(ClusterInstance{
        InstanceConfig{ci.config.phase == BS_PHASE_PREFILL ? Phase::prefill : Phase::decode, ci.config.tp,
                       ci.config.base_freq_mhz},
        ci.weight});
  }
  SchedulerPolicy pol = to_policy(rc.policy);
  SimOptions opts;
  opts.switch_latency_ms = rc.switch_latency_ms;
  opts.horizon_ms = rc.horizon_ms;
  MpcConfig mpc = to_mpc(rc.mpc);
  DecodePolicyConfig dc;
  dc.tbt_slo_ms = rc.decode.tbt_slo_ms;
  dc.kv_threshold = rc.decode.kv_threshold;
  dc.margin = rc.decode.margin;
  dc.ladder.freqs_mhz.assign(rc.decode.ladder_mhz, rc.decode.ladder_mhz + rc.decode.n_ladder);
  TwoTierFactory factory(mpc, dc, ctl_m, pol);
  SimResult r = simulate_cluster(tr, cl, pol, sim_m, rc.controlled ? &factory : nullptr, opts);
  TrimmedResult view = trim_steady_state(r, rc.rampup_s);
  MetricsReport rep = make_report(view, to_slo(rc.slo), "w", "two-tier");
  o->horizon_ms = r.horizon_ms;
  o->completed_requests = r.completed_requests;
  o->generated_tokens = r.generated_tokens;
  o->n_batches = static_cast<int64_t>(r.batches.size());
  o->n_idles = static_cast<int64_t>(r.idles.size());
  o->n_decisions = static_cast<int64_t>(r.decisions.records.size());
  for (const auto& d : r.decisions.records) o->decisions_by_trigger[static_cast<int>(d.trigger)] += 1;
  o->has_p99_ttft = rep.p99_ttft_ms.has_value();
  o->p99_ttft_ms = rep.p99_ttft_ms.value_or(NAN);
  o->has_p99_tpot = rep.p99_mean_tpot_ms.has_value();
  o->p99_mean_tpot_ms = rep.p99_mean_tpot_ms.value_or(NAN);
  o->has_e_first = rep.energy_per_first_token_j.has_value();
  o->energy_per_first_token_j = rep.energy_per_first_token_j.value_or(NAN);
  o->has_e_output = rep.energy_per_output_token_j.has_value();
  o->energy_per_output_token_j = rep.energy_per_output_token_j.value_or(NAN);
  o->avg_power_prefill_w = rep.avg_power_prefill_w;
  o->avg_power_decode_w = rep.avg_power_decode_w;
  o->prefill_energy_j = rep.prefill_energy_j;
  o->decode_energy_j = rep.decode_energy_j;
  o->span_ms = rep.span_ms;
  o->report_completed = rep.completed_requests;
  o->report_generated = rep.generated_tokens;
  o->ttft_violations = rep.ttft_violations;
  o->tpot_violations = rep.tpot_violations;
  if (req) {
    // SimResult::requests is ordered by id; emit in trace order
    for (int64_t i = 0; i < sc.trace.n; ++i) {
      const int64_t id = sc.trace.requests[i].id;
      auto it = std::lower_bound(r.requests.begin(), r.requests.end(), id,
                                 [](const RequestRecord& a, int64_t v) { return a.id < v; });
      bs_replay_request& q = req[i];
      std::memset(&q, 0, sizeof q);
      q.id = id;
      q.prefill_instance = it->prefill_instance;
      q.decode_instance = it->decode_instance;
      q.prefill_done_ms = it->prefill_done_ms.value_or(NAN);
      q.decode_first_start_ms = it->decode_first_start_ms.value_or(NAN);
      q.first_token_ms = it->token_times_ms.empty() ? NAN : it->token_times_ms.front();
      q.last_token_ms = it->token_times_ms.empty() ? NAN : it->token_times_ms.back();
      q.max_tbt_ms = it->max_tbt_ms().value_or(NAN);
      q.n_tokens = static_cast<int64_t>(it->token_times_ms.size());
      q.completed = it->completed ? 1 : 0;
    }
  }
  if (logs) {
    logs->n_batches = static_cast<int64_t>(r.batches.size());
    for (int64_t k = 0; k < logs->n_batches && k < logs->batch_cap; ++k) {
      const BatchRecord& b = r.batches[k];
      logs->batches[k] = bs_batch_record{b.instance, b.phase == Phase::prefill ? 0 : 1, b.batch_seq, b.start_ms,
                                         b.end_ms, b.features.n_requests, b.features.sum_len, b.freq_mhz, b.power_w,
                                         b.energy_j};
    }
    logs->n_idles = static_cast<int64_t>(r.idles.size());
    for (int64_t k = 0; k < logs->n_idles && k < logs->idle_cap; ++k) {
      const IdleRecord& b = r.idles[k];
      logs->idles[k] = bs_idle_record{b.instance, b.phase == Phase::prefill ? 0 : 1, b.start_ms, b.end_ms,
                                      b.freq_mhz, b.power_w, b.energy_j};
    }
    logs->n_decisions = static_cast<int64_t>(r.decisions.records.size());
    for (int64_t k = 0; k < logs->n_decisions && k < logs->decision_cap; ++k) {
      const DecisionRecord& d = r.decisions.records[k];
      logs->decisions[k] = bs_decision_record{d.time_ms, d.instance, static_cast<int32_t>(d.trigger),
                                              d.chosen_freq_mhz, d.feasible ? 1 : 0, 0, d.eval_count};
    }
  }
}

}  // namespace

extern "C" int ref_replay(const bs_model_set* sim_models, const bs_model_set* ctl_models, const bs_replay_config* cfgs,
                          const bs_scenario* sc, int n, bs_replay_summary* out, bs_replay_request* requests,
                          bs_replay_logs* logs, int n_threads) {
  return guarded([&] {
    const ModelSet sim_m = to_models(*sim_models);
    const ModelSet ctl_m = to_models(ctl_models ? *ctl_models : *sim_models);
    std::vector<int64_t> req_off(static_cast<std::size_t>(n) + 1, 0);
    for (int i = 0; i < n; ++i) req_off[i + 1] = req_off[i] + sc[i].trace.n;
    std::atomic<int> next{0};
    auto work = [&] {
      for (int i = next++; i < n; i = next++) {
        std::memset(&out[i], 0, sizeof out[i]);
        out[i].status = guarded([&] {
          replay_one(sim_m, ctl_m, cfgs[sc[i].config], sc[i], &out[i], requests ? requests + req_off[i] : nullptr,
                     logs ? &logs[i] : nullptr);
        });
      }
    };
    const int t = std::max(1, std::min(n_threads, n));
    std::vector<std::thread> pool;
    for (int k = 1; k < t; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  });
}

// --- run_experiment (runner.hpp:155-172) ------------------------------------------

extern "C" int ref_run_experiment(const bs_model_set* models, const bs_trace* trace, double window_ms,
                                  const int32_t* policies, int n_policies, const ref_runner_config* c,
                                  ref_window_run* out, int cap, int* n_out, int32_t* two_tier_slo_pass) {
  return guarded([&] {
    const ModelSet m = to_models(*models);
    RunnerConfig cfg;
    cfg.slo = to_slo(c->slo);
    cfg.total_gpus = c->total_gpus;
    cfg.tp_options.assign(c->tp_options, c->tp_options + c->n_tp);
    cfg.ladder.freqs_mhz.assign(c->ladder, c->ladder + c->n_ladder);
    cfg.scheduler = to_policy(c->scheduler);
    cfg.plan.alpha = c->alpha;
    cfg.plan.peak_subwindow_s = c->peak_subwindow_s;
    cfg.plan.search = to_search(c->search);
    cfg.plan.policy = to_policy(c->plan_policy);
    cfg.rampup_s = c->rampup_s;
    cfg.switch_latency_ms = c->switch_latency_ms;
    cfg.mpc_horizon_k = c->mpc_k;
    cfg.mpc_ladder_n = c->mpc_n;
    cfg.mpc_margin = c->mpc_margin;
    cfg.kv_threshold = c->kv_threshold;
    cfg.decode_margin = c->decode_margin;
    std::vector<Policy> pols;
    for (int i = 0; i < n_policies; ++i) pols.push_back(static_cast<Policy>(policies[i]));
    ExperimentResult r = run_experiment(to_trace(*trace), window_ms, pols, cfg, m);
    *n_out = static_cast<int>(r.runs.size());
    *two_tier_slo_pass = r.two_tier_slo_pass ? 1 : 0;
    for (int i = 0; i < *n_out && i < cap; ++i) {
      const WindowRun& w = r.runs[static_cast<std::size_t>(i)];
      ref_window_run& o = out[i];
      std::memset(&o, 0, sizeof o);
      o.window = w.window_index;
      o.policy = static_cast<int32_t>(w.policy);
      o.gpus_used = w.plan.gpus_used;
      o.slo_pass = w.slo_pass ? 1 : 0;
      o.objective_w = w.plan.objective_w;
      o.target_rps = w.plan.target_rps;
      bs_replay_summary& s = o.report;
      s.horizon_ms = w.sim.horizon_ms;
      s.completed_requests = w.sim.completed_requests;
      s.generated_tokens = w.sim.generated_tokens;
      s.n_batches = static_cast<int64_t>(w.sim.batches.size());
      s.n_idles = static_cast<int64_t>(w.sim.idles.size());
      s.n_decisions = static_cast<int64_t>(w.sim.decisions.records.size());
      for (const auto& d : w.sim.decisions.records) s.decisions_by_trigger[static_cast<int>(d.trigger)] += 1;
      const MetricsReport& rep = w.report;
      s.has_p99_ttft = rep.p99_ttft_ms.has_value();
      s.p99_ttft_ms = rep.p99_ttft_ms.value_or(NAN);
      s.has_p99_tpot = rep.p99_mean_tpot_ms.has_value();
      s.p99_mean_tpot_ms = rep.p99_mean_tpot_ms.value_or(NAN);
      s.has_e_first = rep.energy_per_first_token_j.has_value();
      s.energy_per_first_token_j = rep.energy_per_first_token_j.value_or(NAN);
      s.has_e_output = rep.energy_per_output_token_j.has_value();
      s.energy_per_output_token_j = rep.energy_per_output_token_j.value_or(NAN);
      s.avg_power_prefill_w = rep.avg_power_prefill_w;
      s.avg_power_decode_w = rep.avg_power_decode_w;
      s.prefill_energy_j = rep.prefill_energy_j;
      s.decode_energy_j = rep.decode_energy_j;
      s.span_ms = rep.span_ms;
      s.report_completed = rep.completed_requests;
      s.report_generated = rep.generated_tokens;
      s.ttft_violations = rep.ttft_violations;
      s.tpot_violations = rep.tpot_violations;
    }
  });
}

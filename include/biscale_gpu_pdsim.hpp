// biscale_gpu_pdsim.hpp — header-only C++ drop-in for the reference's
// controller interface, backed by the sm_100a C ABI (biscale_gpu.h).
//
// Include it from code that already includes the reference's pdsim headers
// (proj/include/pdsim/dvfs.hpp).  It provides:
//
//   pdsim_gpu::Device                   RAII bs_ctx_t (one CUDA stream)
//   pdsim_gpu::DeviceModels             bs_models_upload of a pdsim::ModelSet
//   pdsim_gpu::GpuPrefillMpcController  : pdsim::FreqController
//                                         (replaces PrefillMpcController,
//                                          dvfs.hpp:302-339)
//   pdsim_gpu::GpuDecodePolicyController: pdsim::FreqController
//                                         (replaces DecodePolicyController,
//                                          dvfs.hpp:341-365)
//   pdsim_gpu::GpuTwoTierFactory        : pdsim::ControllerFactory
//                                         (replaces TwoTierFactory,
//                                          dvfs.hpp:370-390; drop-in for
//                                          runner.hpp:118)
//   pdsim_gpu::greedy_freq_select / exhaustive_freq_select /
//   select_decode_freq_ex               batch-of-one wrappers
//   pdsim_gpu::build_config_table       replaces build_config_table
//                                         (placement.hpp:240-260), the call
//                                         in plan_window (placement.hpp:576)
//   pdsim_gpu::solve_placement /        replace solve_placement (357-416) and
//   solve_max_throughput                  solve_max_throughput (421-499)
//   pdsim_gpu::plan_window /            plan_window (placement.hpp:558-582),
//   plan_window_policies                  plan_window_policies (runner.hpp:98-110)
//   pdsim_gpu::run_experiment           run_experiment (runner.hpp:155-172):
//                                         GPU plans + every (window, policy)
//                                         replay in one bs_replay call
//
// Status codes are rethrown as the reference's exception types with the
// library's message.  predicted_latency_ms is evaluated with the reference's
// own predict_latency (the safety deadline relies on exact ties,
// tests/test_simulator.cpp:609-617; the device interpolator is bit-identical
// but a host call avoids a launch on the simulator's critical path).
#pragma once

#include <algorithm>
#include <cstdio>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "biscale_gpu.h"
#include "pdsim/dvfs.hpp"
#include "pdsim/errors.hpp"
#include "pdsim/metrics.hpp"
#include "pdsim/placement.hpp"
#include "pdsim/runner.hpp"

namespace pdsim_gpu {

[[noreturn]] inline void rethrow(int status, const std::string& msg) {
  switch (status) {
    case BS_PARAMETER_ERROR: throw pdsim::ParameterError(msg);
    case BS_MODEL_ERROR: throw pdsim::ModelError(msg);
    case BS_SIMULATION_ERROR: throw pdsim::SimulationError(msg);
    case BS_CONFIG_ERROR: throw pdsim::ConfigError(msg);
    case BS_ACCOUNTING_ERROR: throw pdsim::AccountingError(msg);
    case BS_IO_ERROR: throw pdsim::IoError(msg);
    case BS_INFEASIBLE_ERROR: {
      auto bar = msg.find('|');
      if (bar == std::string::npos) throw pdsim::InfeasibleError("", msg);
      throw pdsim::InfeasibleError(msg.substr(0, bar), msg.substr(bar + 1));
    }
    default: throw std::runtime_error("biscale_gpu: " + msg);
  }
}

class Device {
 public:
  explicit Device(int device = 0) {
    int rc = bs_ctx_create(device, &ctx_);
    if (rc != BS_OK) rethrow(rc, "bs_ctx_create failed: no usable CUDA device (no CPU fallback)");
  }
  ~Device() { bs_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  bs_ctx_t get() const { return ctx_; }
  void check(int rc) const {
    if (rc != BS_OK) rethrow(rc, bs_last_error(ctx_));
  }

 private:
  bs_ctx_t ctx_ = nullptr;
};

namespace detail {

inline int axis_role(const std::string& name) {
  if (name == pdsim::kAxisSumLen) return BS_AXIS_SUM_LEN;
  if (name == pdsim::kAxisNumRequests) return BS_AXIS_N_REQUESTS;
  if (name == pdsim::kAxisTp) return BS_AXIS_TP;
  if (name == pdsim::kAxisFreq) return BS_AXIS_FREQ;
  return BS_AXIS_UNKNOWN;
}

inline bs_grid to_grid(const pdsim::NdGrid& g) {
  bs_grid out{};
  out.rank = static_cast<int32_t>(g.axes.size());
  for (std::size_t d = 0; d < g.axes.size() && d < BS_MAX_RANK; ++d) {
    out.role[d] = axis_role(g.axes[d].name);
    out.n_knots[d] = static_cast<int32_t>(g.axes[d].knots.size());
    out.knots[d] = g.axes[d].knots.data();
  }
  out.values = g.values.data();
  return out;
}

// Owns the marshalled arrays of one QueueSnapshot.
struct SnapshotView {
  std::vector<bs_waiting> waiting;
  std::vector<uint8_t> completes;
  bs_snapshot snap{};

  explicit SnapshotView(const pdsim::QueueSnapshot& q) {
    waiting.reserve(q.waiting.size());
    for (const auto& w : q.waiting) waiting.push_back(bs_waiting{w.id, w.arrival_ms, w.total_len, w.remaining_len});
    snap.now_ms = q.now_ms;
    snap.current_freq_mhz = q.current_freq_mhz;
    snap.target_freq_mhz = q.target_freq_mhz;
    snap.tp = q.tp;
    snap.n_waiting = static_cast<int32_t>(waiting.size());
    snap.waiting = waiting.data();
    snap.running_active = q.running.active ? 1 : 0;
    if (q.running.active) {
      for (bool c : q.running.completes) completes.push_back(c ? 1 : 0);
      snap.n_running = static_cast<int32_t>(completes.size());
      snap.running_completes = completes.data();
      snap.running_arrivals_ms = q.running.arrivals_ms.data();
      snap.running_work_remaining = q.running.work_remaining;
      snap.running_features = bs_features{q.running.features.n_requests, q.running.features.sum_len};
    }
  }
};

inline bs_mpc_config to_mpc(const pdsim::MpcConfig& c) {
  bs_mpc_config o{};
  o.horizon_K = c.horizon_K;
  o.ladder_N = c.ladder_N;
  o.n_ladder = static_cast<int32_t>(c.ladder.freqs_mhz.size());
  o.ladder_mhz = c.ladder.freqs_mhz.data();
  o.ttft_ms = c.slo.ttft_ms;
  o.tpot_ms = c.slo.tpot_ms;
  o.percentile = c.slo.percentile;
  o.switch_latency_ms = c.switch_latency_ms;
  o.margin = c.margin;
  return o;
}

inline bs_scheduler_policy to_policy(const pdsim::SchedulerPolicy& p) {
  bs_scheduler_policy o{};
  o.max_batch_tokens = p.max_batch_tokens;
  o.max_batch_requests = p.max_batch_requests;
  o.kv_capacity_tokens = p.kv_capacity_tokens;
  o.chunking = p.chunking ? 1 : 0;
  return o;
}

inline pdsim::GreedyResult from_result(const bs_mpc_result& r) {
  pdsim::GreedyResult g;
  g.assignment.freqs.assign(r.freqs_mhz, r.freqs_mhz + r.K);
  g.feasible = r.feasible != 0;
  g.eval_count = r.eval_count;
  g.objective_w = r.objective_w;
  for (int l = 0; l < r.n_levels; ++l) {
    pdsim::GreedyLevelStats s;
    s.level = r.levels[l].level;
    s.replaced_mhz = r.levels[l].replaced_mhz;
    s.k_prime = r.levels[l].k_prime;
    s.mutations = r.levels[l].mutations;
    s.feasible_mutations = r.levels[l].feasible_mutations;
    s.accepted = r.levels[l].accepted != 0;
    g.levels.push_back(s);
  }
  return g;
}

}  // namespace detail

// Immutable device copy of a pdsim::ModelSet (perfmodel.hpp:494-503).
class DeviceModels {
 public:
  DeviceModels(const Device& dev, const pdsim::ModelSet& m) : dev_(&dev) {
    bs_model_set s{};
    s.latency_prefill = detail::to_grid(m.latency_prefill.grid);
    s.latency_decode = detail::to_grid(m.latency_decode.grid);
    s.power_prefill = detail::to_grid(m.power_prefill.grid);
    s.power_decode = detail::to_grid(m.power_decode.grid);
    std::vector<bs_idle_entry> idle;
    for (const auto& e : m.idle.entries)
      idle.push_back(bs_idle_entry{e.tp, static_cast<int32_t>(e.freqs_mhz.size()), e.freqs_mhz.data(),
                                   e.idle_w.data()});
    s.n_idle = static_cast<int32_t>(idle.size());
    s.idle = idle.data();
    dev.check(bs_models_upload(dev.get(), &s, &h_));
  }
  ~DeviceModels() { bs_models_free(dev_->get(), h_); }
  DeviceModels(const DeviceModels&) = delete;
  DeviceModels& operator=(const DeviceModels&) = delete;
  bs_models_t get() const { return h_; }
  const Device& device() const { return *dev_; }

 private:
  const Device* dev_;
  bs_models_t h_ = nullptr;
};

// greedy_freq_select (dvfs.hpp:185-259) on the GPU.
inline pdsim::GreedyResult greedy_freq_select(const DeviceModels& dm, const pdsim::QueueSnapshot& q,
                                              const pdsim::MpcConfig& cfg, const pdsim::SchedulerPolicy& policy,
                                              bs_mpc_result* raw = nullptr) {
  detail::SnapshotView v(q);
  bs_mpc_problem p{};
  p.snap = v.snap;
  const bs_mpc_config c = detail::to_mpc(cfg);
  const bs_scheduler_policy pol = detail::to_policy(policy);
  bs_mpc_result r{};
  dm.device().check(bs_mpc_greedy(dm.device().get(), dm.get(), &c, &pol, 1, &p, 1, &r));
  if (raw) *raw = r;
  return detail::from_result(r);
}

// Exhaustive MPC (tests/test_dvfs.cpp:74-94 semantics, lexicographic ties).
inline pdsim::GreedyResult exhaustive_freq_select(const DeviceModels& dm, const pdsim::QueueSnapshot& q,
                                                  const pdsim::MpcConfig& cfg, const pdsim::SchedulerPolicy& policy,
                                                  bs_mpc_result* raw = nullptr) {
  detail::SnapshotView v(q);
  bs_mpc_problem p{};
  p.snap = v.snap;
  const bs_mpc_config c = detail::to_mpc(cfg);
  const bs_scheduler_policy pol = detail::to_policy(policy);
  bs_mpc_result r{};
  dm.device().check(bs_mpc_exhaustive(dm.device().get(), dm.get(), &c, &pol, 1, &p, 1, &r));
  if (raw) *raw = r;
  return detail::from_result(r);
}

// select_decode_freq_ex (dvfs.hpp:274-293) on the GPU.
inline pdsim::DecodeDecision select_decode_freq_ex(const DeviceModels& dm, const pdsim::BatchFeatures& batch,
                                                   const pdsim::KVCacheState& kv,
                                                   const pdsim::DecodePolicyConfig& cfg, int tp) {
  bs_decode_config c{};
  c.tbt_slo_ms = cfg.tbt_slo_ms;
  c.kv_threshold = cfg.kv_threshold;
  c.margin = cfg.margin;
  c.n_ladder = static_cast<int32_t>(cfg.ladder.freqs_mhz.size());
  c.ladder_mhz = cfg.ladder.freqs_mhz.data();
  bs_decode_query q{};
  q.batch = bs_features{batch.n_requests, batch.sum_len};
  q.kv_capacity_tokens = kv.capacity_tokens;
  q.kv_used_tokens = kv.used_tokens;
  q.tp = tp;
  bs_decode_result r{};
  dm.device().check(bs_decode_pick(dm.device().get(), dm.get(), &c, 1, &q, 1, &r));
  pdsim::DecodeDecision d;
  d.freq_mhz = r.freq_mhz;
  d.eval_count = r.eval_count;
  d.kv_override = r.kv_override != 0;
  return d;
}

// PrefillMpcController (dvfs.hpp:302-339) backed by bs_mpc_greedy.
class GpuPrefillMpcController : public pdsim::FreqController {
 public:
  GpuPrefillMpcController(pdsim::MpcConfig cfg, const pdsim::ModelSet& models, const DeviceModels& dm,
                          pdsim::SchedulerPolicy policy)
      : cfg_(std::move(cfg)), models_(&models), dm_(&dm), policy_(policy) {
    cfg_.validate();
    policy_.validate();
    max_mhz_ = cfg_.candidates().max_mhz();
  }

  pdsim::FreqDecision decide(const pdsim::QueueSnapshot& q) override { return run(q); }
  bool reacts_to_arrivals() const override { return true; }
  std::optional<pdsim::FreqDecision> on_arrival(const pdsim::QueueSnapshot& q) override { return run(q); }
  double predicted_latency_ms(const pdsim::BatchFeatures& f, pdsim::Phase phase, int tp,
                              double freq_mhz) const override {
    return pdsim::predict_latency(models_->latency(phase), f, tp, freq_mhz);
  }
  double safety_margin() const override { return cfg_.margin; }
  double max_freq_mhz() const override { return max_mhz_; }

 private:
  pdsim::FreqDecision run(const pdsim::QueueSnapshot& q) const {
    bs_mpc_result r{};
    greedy_freq_select(*dm_, q, cfg_, policy_, &r);
    return pdsim::FreqDecision{r.decision_freq_mhz, r.feasible != 0, r.eval_count};
  }

  pdsim::MpcConfig cfg_;
  const pdsim::ModelSet* models_;
  const DeviceModels* dm_;
  pdsim::SchedulerPolicy policy_;
  double max_mhz_ = 0.0;
};

// DecodePolicyController (dvfs.hpp:341-365) backed by bs_decode_pick.
class GpuDecodePolicyController : public pdsim::FreqController {
 public:
  GpuDecodePolicyController(pdsim::DecodePolicyConfig cfg, const pdsim::ModelSet& models, const DeviceModels& dm)
      : cfg_(std::move(cfg)), models_(&models), dm_(&dm) {
    cfg_.validate();
  }
  pdsim::FreqDecision decide(const pdsim::QueueSnapshot& q) override {
    pdsim::DecodeDecision d = select_decode_freq_ex(*dm_, q.decode_batch, q.kv, cfg_, q.tp);
    return pdsim::FreqDecision{d.freq_mhz, true, d.eval_count};
  }
  double predicted_latency_ms(const pdsim::BatchFeatures& f, pdsim::Phase phase, int tp,
                              double freq_mhz) const override {
    return pdsim::predict_latency(models_->latency(phase), f, tp, freq_mhz);
  }
  double safety_margin() const override { return safety_margin_; }
  double max_freq_mhz() const override { return cfg_.ladder.max_mhz(); }
  void set_safety_margin(double m) { safety_margin_ = m; }

 private:
  pdsim::DecodePolicyConfig cfg_;
  const pdsim::ModelSet* models_;
  const DeviceModels* dm_;
  double safety_margin_ = 0.05;
};

// --- coarse-tier placement ------------------------------------------------------

namespace detail {

struct TraceView {
  std::vector<bs_request> reqs;
  bs_trace t{};
  explicit TraceView(const pdsim::Trace& tr) {
    reqs.reserve(tr.requests.size());
    for (const auto& r : tr.requests) reqs.push_back(bs_request{r.id, r.arrival_ms, r.input_len, r.output_len});
    t.n = static_cast<int64_t>(reqs.size());
    t.requests = reqs.data();
    t.duration_ms = tr.duration_ms;
  }
};

inline bs_table_entry to_entry(const pdsim::ConfigTableEntry& e) {
  bs_table_entry o{};
  o.config = bs_instance_config{e.config.phase == pdsim::Phase::prefill ? BS_PHASE_PREFILL : BS_PHASE_DECODE,
                                e.config.tp, e.config.base_freq_mhz};
  o.r_c = e.r_c;
  o.has_e_c = e.e_c ? 1 : 0;
  o.e_c = e.e_c ? *e.e_c : 0.0;
  o.g_c = e.g_c;
  o.saturated = e.saturated ? 1 : 0;
  o.error_code = e.error.empty() ? 0 : BS_MODEL_ERROR;
  std::snprintf(o.error, sizeof(o.error), "%s", e.error.c_str());
  return o;
}

inline pdsim::ConfigTableEntry from_entry(const bs_table_entry& e) {
  pdsim::ConfigTableEntry o;
  o.config = pdsim::InstanceConfig{e.config.phase == BS_PHASE_PREFILL ? pdsim::Phase::prefill : pdsim::Phase::decode,
                                   e.config.tp, e.config.base_freq_mhz};
  o.r_c = e.r_c;
  if (e.has_e_c) o.e_c = e.e_c;
  o.g_c = e.g_c;
  o.saturated = e.saturated != 0;
  if (e.error_code != 0) o.error = e.error;
  return o;
}

template <class Solve>
pdsim::PlacementPlan solve_with(const pdsim::PlacementProblem& p, Solve&& solve) {
  p.validate();
  std::vector<bs_table_entry> t;
  t.reserve(p.table.size());
  for (const auto& e : p.table) t.push_back(to_entry(e));
  std::vector<int64_t> counts(p.table.size(), 0);
  double obj = 0.0;
  int32_t used = 0;
  int rc = solve(t.data(), static_cast<int>(t.size()), counts.data(), &obj, &used);
  if (rc != BS_OK) rethrow(rc, bs_last_error(nullptr));
  pdsim::PlacementPlan plan;
  plan.counts.assign(counts.begin(), counts.end());
  plan.table = p.table;
  plan.objective_w = obj;
  plan.target_rps = p.target_rps;
  plan.alpha = p.alpha;
  plan.total_gpus = p.total_gpus;
  plan.gpus_used = used;
  plan.instances = pdsim::derive_routing_weights(plan.counts, plan.table);
  return plan;
}

}  // namespace detail

// build_config_table (placement.hpp:240-260) on the GPU: the goodput probes
// of every candidate in one grid, the exact binary-search replay, then E_c.
// Drop-in for the call in plan_window (placement.hpp:576).
inline std::vector<pdsim::ConfigTableEntry> build_config_table(const DeviceModels& dm,
                                                               const std::vector<pdsim::InstanceConfig>& candidates,
                                                               const pdsim::Trace& base, const pdsim::SLOSpec& slo,
                                                               const pdsim::SchedulerPolicy& policy,
                                                               const pdsim::GoodputSearch& search) {
  if (candidates.empty()) throw pdsim::ParameterError("config table: no candidates");
  detail::TraceView tv(base);
  const bs_slo s{slo.ttft_ms, slo.tpot_ms, slo.percentile};
  const bs_scheduler_policy pol = detail::to_policy(policy);
  bs_goodput_search g{};
  g.tolerance_rps = search.tolerance_rps;
  g.probe_count = search.probe_count;
  g.seed = search.seed;
  std::vector<bs_instance_config> cands;
  for (const auto& c : candidates)
    cands.push_back(bs_instance_config{c.phase == pdsim::Phase::prefill ? BS_PHASE_PREFILL : BS_PHASE_DECODE, c.tp,
                                       c.base_freq_mhz});
  std::vector<bs_table_entry> out(candidates.size());
  dm.device().check(bs_goodput_table(dm.device().get(), dm.get(), &tv.t, &s, &pol, &g, cands.data(),
                                     static_cast<int>(cands.size()), out.data()));
  std::vector<pdsim::ConfigTableEntry> table;
  table.reserve(out.size());
  for (const auto& e : out) table.push_back(detail::from_entry(e));
  return table;
}

// build_config_table for several probe traces in one device call
// (bs_goodput_tables): tables[t] belongs to bases[t].
inline std::vector<std::vector<pdsim::ConfigTableEntry>> build_config_tables(
    const DeviceModels& dm, const std::vector<pdsim::InstanceConfig>& candidates,
    const std::vector<const pdsim::Trace*>& bases, const pdsim::SLOSpec& slo, const pdsim::SchedulerPolicy& policy,
    const pdsim::GoodputSearch& search) {
  if (candidates.empty()) throw pdsim::ParameterError("config table: no candidates");
  std::vector<detail::TraceView> tvs;
  tvs.reserve(bases.size());
  std::vector<bs_trace> trs;
  for (const pdsim::Trace* b : bases) {
    tvs.emplace_back(*b);
    trs.push_back(tvs.back().t);
  }
  const bs_slo s{slo.ttft_ms, slo.tpot_ms, slo.percentile};
  const bs_scheduler_policy pol = detail::to_policy(policy);
  bs_goodput_search g{};
  g.tolerance_rps = search.tolerance_rps;
  g.probe_count = search.probe_count;
  g.seed = search.seed;
  std::vector<bs_instance_config> cands;
  for (const auto& c : candidates)
    cands.push_back(bs_instance_config{c.phase == pdsim::Phase::prefill ? BS_PHASE_PREFILL : BS_PHASE_DECODE, c.tp,
                                       c.base_freq_mhz});
  const std::size_t n = cands.size();
  std::vector<bs_table_entry> out(n * bases.size());
  dm.device().check(bs_goodput_tables(dm.device().get(), dm.get(), trs.data(), static_cast<int>(trs.size()), &s,
                                      &pol, &g, cands.data(), static_cast<int>(n), out.data()));
  std::vector<std::vector<pdsim::ConfigTableEntry>> tables(bases.size());
  for (std::size_t t = 0; t < bases.size(); ++t)
    for (std::size_t c = 0; c < n; ++c) tables[t].push_back(detail::from_entry(out[t * n + c]));
  return tables;
}

// solve_placement (placement.hpp:357-416), same fold order and tie-breaks;
// InfeasibleError with the reference's constraint and message.
inline pdsim::PlacementPlan solve_placement(const pdsim::PlacementProblem& p) {
  return detail::solve_with(p, [&](const bs_table_entry* t, int n, int64_t* counts, double* obj, int32_t* used) {
    return bs_placement_solve(nullptr, t, n, p.total_gpus, p.target_rps, p.alpha, counts, obj, used);
  });
}

// solve_max_throughput (placement.hpp:421-499).
inline pdsim::PlacementPlan solve_max_throughput(const pdsim::PlacementProblem& p, double max_freq_mhz) {
  pdsim::PlacementPlan plan =
      detail::solve_with(p, [&](const bs_table_entry* t, int n, int64_t* counts, double* obj, int32_t* used) {
        return bs_placement_max_throughput(nullptr, t, n, p.total_gpus, p.target_rps, p.alpha, max_freq_mhz, counts,
                                           obj, used);
      });
  // the plan carries the restricted table (placement.hpp:423-430, 486)
  for (auto& e : plan.table) {
    if (e.config.base_freq_mhz != max_freq_mhz) {
      e.r_c = 0.0;
      e.e_c.reset();
      e.error = "below maximum frequency";
    }
  }
  plan.instances = pdsim::derive_routing_weights(plan.counts, plan.table);
  return plan;
}

// TwoTierFactory (dvfs.hpp:370-390): drop-in ControllerFactory for
// simulate_cluster / run_policy.
class GpuTwoTierFactory : public pdsim::ControllerFactory {
 public:
  GpuTwoTierFactory(pdsim::MpcConfig mpc, pdsim::DecodePolicyConfig decode, const pdsim::ModelSet& controller_models,
                    const DeviceModels& dm, pdsim::SchedulerPolicy policy)
      : mpc_(std::move(mpc)), decode_(std::move(decode)), models_(&controller_models), dm_(&dm), policy_(policy) {}

  std::unique_ptr<pdsim::FreqController> make(pdsim::Phase phase, int tp, double base_freq_mhz) override {
    (void)tp;
    (void)base_freq_mhz;
    if (phase == pdsim::Phase::prefill)
      return std::make_unique<GpuPrefillMpcController>(mpc_, *models_, *dm_, policy_);
    auto ctl = std::make_unique<GpuDecodePolicyController>(decode_, *models_, *dm_);
    ctl->set_safety_margin(decode_.margin > 0.0 ? decode_.margin : 0.05);
    return ctl;
  }

 private:
  pdsim::MpcConfig mpc_;
  pdsim::DecodePolicyConfig decode_;
  const pdsim::ModelSet* models_;
  const DeviceModels* dm_;
  pdsim::SchedulerPolicy policy_;
};


// --- cluster replay and the window loop -------------------------------------------

// One run_policy (runner.hpp:112-122) + its window report (runner.hpp:131-133),
// as the device replays it.  `sim` carries SimResult's counters and horizon,
// and its records when requested.
struct ReplayRun {
  pdsim::SimResult sim;
  pdsim::MetricsReport report;
  int status = BS_OK;
};

namespace detail {

inline bs_replay_config replay_config(const pdsim::RunnerConfig& cfg, bool controlled, std::vector<double>& keep) {
  bs_replay_config c{};
  keep = cfg.ladder.freqs_mhz;
  if (controlled) {
    c.mpc = to_mpc(cfg.mpc_config());
    c.mpc.ladder_mhz = keep.data();
    const pdsim::DecodePolicyConfig d = cfg.decode_config();
    c.decode.tbt_slo_ms = d.tbt_slo_ms;
    c.decode.kv_threshold = d.kv_threshold;
    c.decode.margin = d.margin;
    c.decode.n_ladder = static_cast<int32_t>(keep.size());
    c.decode.ladder_mhz = keep.data();
    c.controlled = 1;
  }
  c.policy = to_policy(cfg.scheduler);
  c.slo = bs_slo{cfg.slo.ttft_ms, cfg.slo.tpot_ms, cfg.slo.percentile};
  c.switch_latency_ms = cfg.switch_latency_ms;
  c.horizon_ms = -1.0;
  c.rampup_s = cfg.rampup_s;
  return c;
}

inline void fill_run(const bs_replay_summary& o, ReplayRun& r) {
  r.status = o.status;
  r.sim.horizon_ms = o.horizon_ms;
  r.sim.completed_requests = o.completed_requests;
  r.sim.generated_tokens = o.generated_tokens;
  pdsim::MetricsReport& m = r.report;
  if (o.has_p99_ttft) m.p99_ttft_ms = o.p99_ttft_ms;
  if (o.has_p99_tpot) m.p99_mean_tpot_ms = o.p99_mean_tpot_ms;
  if (o.has_e_first) m.energy_per_first_token_j = o.energy_per_first_token_j;
  if (o.has_e_output) m.energy_per_output_token_j = o.energy_per_output_token_j;
  m.avg_power_prefill_w = o.avg_power_prefill_w;
  m.avg_power_decode_w = o.avg_power_decode_w;
  m.prefill_energy_j = o.prefill_energy_j;
  m.decode_energy_j = o.decode_energy_j;
  m.span_ms = o.span_ms;
  m.completed_requests = o.report_completed;
  m.generated_tokens = o.report_generated;
  m.ttft_violations = o.ttft_violations;
  m.tpot_violations = o.tpot_violations;
}

}  // namespace detail

// plan_window (placement.hpp:558-582) with the GPU config table and ILP.
inline pdsim::WindowPlanResult plan_window(const DeviceModels& dm, const pdsim::Trace& history, int total_gpus,
                                           const pdsim::SLOSpec& slo, const pdsim::FrequencyLadder& ladder,
                                           const std::vector<int>& tp_options, const pdsim::PlanOptions& opts = {}) {
  history.validate();
  if (history.requests.empty()) throw pdsim::ParameterError("plan_window: empty history");
  pdsim::Trace predicted = pdsim::predict_next_window(history);
  pdsim::WindowPlanResult res;
  res.predicted_peak_rps = pdsim::peak_rps(predicted, opts.peak_subwindow_s);
  const pdsim::Trace& probe = opts.probe_trace ? *opts.probe_trace : predicted;
  const std::vector<pdsim::InstanceConfig> candidates = pdsim::enumerate_candidates(ladder, tp_options);
  res.table = pdsim_gpu::build_config_table(dm, candidates, probe, slo, opts.policy, opts.search);
  pdsim::PlacementProblem problem{res.table, total_gpus, res.predicted_peak_rps, opts.alpha};
  res.plan = pdsim_gpu::solve_placement(problem);
  return res;
}

// plan_window_policies (runner.hpp:98-110) on the GPU.
inline pdsim::WindowPlans plan_window_policies(const DeviceModels& dm, const pdsim::Trace& history,
                                               const pdsim::RunnerConfig& cfg) {
  cfg.validate();
  pdsim::WindowPlanResult wp = pdsim_gpu::plan_window(dm, history, cfg.total_gpus, cfg.slo, cfg.ladder, cfg.tp_options, cfg.plan);
  pdsim::WindowPlans out;
  out.target_rps = wp.predicted_peak_rps;
  out.table = wp.table;
  out.ilp = wp.plan;
  pdsim::PlacementProblem p{out.table, cfg.total_gpus, out.target_rps, cfg.plan.alpha};
  out.maxfreq = pdsim_gpu::solve_max_throughput(p, cfg.ladder.max_mhz());
  return out;
}

// run_policy + the window report for a batch of (window, plan, policy)
// triples in ONE device call (bs_replay).  Throws like the reference on the
// first failing run.
// records: also fill each SimResult's requests, batches, idles and
// decisions (the reference's CSV writers then produce the same files; a
// request's token_times_ms holds only its first and last emission, which is
// what save_request_csv and the metrics read).
inline std::vector<ReplayRun> replay_policies(const DeviceModels& dm, const std::vector<const pdsim::Trace*>& windows,
                                              const std::vector<const pdsim::PlacementPlan*>& plans,
                                              const std::vector<pdsim::Policy>& policies,
                                              const pdsim::RunnerConfig& cfg, bool records = false) {
  const std::size_t n = windows.size();
  std::vector<double> lad_ctl, lad_fix;
  const bs_replay_config cfgs[2] = {detail::replay_config(cfg, false, lad_fix),
                                    detail::replay_config(cfg, true, lad_ctl)};
  std::vector<detail::TraceView> tvs;
  tvs.reserve(n);
  std::vector<std::vector<bs_cluster_instance>> inst(n);
  std::vector<bs_scenario> sc(n);
  for (std::size_t i = 0; i < n; ++i) {
    tvs.emplace_back(*windows[i]);
    for (const auto& ci : plans[i]->instances)
      inst[i].push_back(bs_cluster_instance{
          bs_instance_config{ci.config.phase == pdsim::Phase::prefill ? BS_PHASE_PREFILL : BS_PHASE_DECODE,
                             ci.config.tp, ci.config.base_freq_mhz},
          ci.weight});
    sc[i].trace = tvs[i].t;
    sc[i].instances = inst[i].data();
    sc[i].n_instances = static_cast<int32_t>(inst[i].size());
    sc[i].config = policies[i] == pdsim::Policy::two_tier ? 1 : 0;
  }
  std::vector<bs_replay_summary> out(n);
  std::vector<bs_replay_request> reqs;
  std::vector<std::vector<bs_batch_record>> bat(records ? n : 0);
  std::vector<std::vector<bs_idle_record>> idl(records ? n : 0);
  std::vector<std::vector<bs_decision_record>> dec(records ? n : 0);
  std::vector<bs_replay_logs> logs(records ? n : 0);
  if (records) {
    std::size_t total = 0;
    for (std::size_t i = 0; i < n; ++i) {
      int64_t cap = 1024;
      for (const auto& r : windows[i]->requests) cap += r.output_len + 4;
      total += windows[i]->requests.size();
      bat[i].resize(static_cast<std::size_t>(cap));
      idl[i].resize(static_cast<std::size_t>(cap));
      dec[i].resize(static_cast<std::size_t>(cap));
      logs[i] = bs_replay_logs{bat[i].data(), cap, 0, idl[i].data(), cap, 0, dec[i].data(), cap, 0};
    }
    reqs.resize(std::max<std::size_t>(total, 1));
  }
  dm.device().check(bs_replay(dm.device().get(), dm.get(), dm.get(), cfgs, 2, sc.data(), static_cast<int>(n),
                              out.data(), records ? reqs.data() : nullptr, records ? logs.data() : nullptr));
  std::vector<ReplayRun> runs(n);
  std::size_t q = 0;
  for (std::size_t i = 0; i < n; ++i) {
    detail::fill_run(out[i], runs[i]);
    if (!records) continue;
    if (logs[i].n_batches > logs[i].batch_cap || logs[i].n_idles > logs[i].idle_cap ||
        logs[i].n_decisions > logs[i].decision_cap)
      throw std::runtime_error("biscale_gpu: replay log capacity exceeded");
    pdsim::SimResult& sim = runs[i].sim;
    for (const auto& ci : plans[i]->instances) sim.instances.push_back(ci.config);
    const auto& rq = windows[i]->requests;
    for (std::size_t k = 0; k < rq.size(); ++k, ++q) {
      const bs_replay_request& r = reqs[q];
      pdsim::RequestRecord rec;
      rec.id = rq[k].id;
      rec.arrival_ms = rq[k].arrival_ms;
      rec.input_len = rq[k].input_len;
      rec.output_len = rq[k].output_len;
      rec.prefill_instance = r.prefill_instance;
      rec.decode_instance = r.decode_instance;
      if (r.prefill_done_ms == r.prefill_done_ms) rec.prefill_done_ms = r.prefill_done_ms;
      if (r.decode_instance >= 0) rec.decode_join_ms = r.prefill_done_ms;
      if (r.decode_first_start_ms == r.decode_first_start_ms) rec.decode_first_start_ms = r.decode_first_start_ms;
      if (r.n_tokens >= 1) rec.token_times_ms.push_back(r.first_token_ms);
      if (r.n_tokens >= 2) rec.token_times_ms.push_back(r.last_token_ms);
      rec.completed = r.completed != 0;
      sim.requests.push_back(std::move(rec));
    }
    std::stable_sort(sim.requests.begin(), sim.requests.end(),
                     [](const pdsim::RequestRecord& a, const pdsim::RequestRecord& b) { return a.id < b.id; });
    auto phase_of = [](int32_t p) { return p == BS_PHASE_PREFILL ? pdsim::Phase::prefill : pdsim::Phase::decode; };
    for (int64_t k = 0; k < logs[i].n_batches; ++k) {
      const bs_batch_record& b = bat[i][static_cast<std::size_t>(k)];
      pdsim::BatchRecord r;
      r.instance = b.instance;
      r.phase = phase_of(b.phase);
      r.batch_seq = b.batch_seq;
      r.start_ms = b.start_ms;
      r.end_ms = b.end_ms;
      r.features.n_requests = b.n_requests;
      r.features.sum_len = b.sum_len;
      r.freq_mhz = b.freq_mhz;
      r.power_w = b.power_w;
      r.energy_j = b.energy_j;
      sim.batches.push_back(std::move(r));
    }
    for (int64_t k = 0; k < logs[i].n_idles; ++k) {
      const bs_idle_record& b = idl[i][static_cast<std::size_t>(k)];
      sim.idles.push_back(pdsim::IdleRecord{b.instance, phase_of(b.phase), b.start_ms, b.end_ms, b.freq_mhz,
                                            b.power_w, b.energy_j});
    }
    for (int64_t k = 0; k < logs[i].n_decisions; ++k) {
      const bs_decision_record& d = dec[i][static_cast<std::size_t>(k)];
      sim.decisions.records.push_back(pdsim::DecisionRecord{d.time_ms, d.instance,
                                                            static_cast<pdsim::Trigger>(d.trigger),
                                                            d.chosen_freq_mhz, d.feasible != 0, d.eval_count});
    }
  }
  return runs;
}

// solve_placement (max_freq[i] < 0) / solve_max_throughput (max_freq[i] =
// the ladder's maximum) for many problems in ONE device call
// (bs_placement_solve_batch).  The first failing problem, in order, throws
// what the reference's call would throw.
inline std::vector<pdsim::PlacementPlan> solve_placements(const Device& dev,
                                                          const std::vector<pdsim::PlacementProblem>& ps,
                                                          const std::vector<double>& max_freq) {
  const std::size_t n = ps.size();
  std::vector<std::vector<bs_table_entry>> tabs(n);
  std::vector<std::vector<int64_t>> counts(n);
  std::vector<bs_placement_problem> in(n);
  for (std::size_t k = 0; k < n; ++k) {
    ps[k].validate();
    for (const auto& e : ps[k].table) tabs[k].push_back(detail::to_entry(e));
    counts[k].assign(ps[k].table.size(), 0);
    in[k] = bs_placement_problem{tabs[k].data(), static_cast<int32_t>(tabs[k].size()), ps[k].total_gpus,
                                 ps[k].target_rps, ps[k].alpha, max_freq[k] >= 0.0 ? 1 : 0, 0,
                                 max_freq[k] >= 0.0 ? max_freq[k] : 0.0, counts[k].data()};
  }
  std::vector<bs_placement_solution> out(n);
  dev.check(bs_placement_solve_batch(dev.get(), in.data(), static_cast<int>(n), out.data()));
  std::vector<pdsim::PlacementPlan> plans(n);
  for (std::size_t k = 0; k < n; ++k) {
    if (out[k].status != BS_OK) rethrow(out[k].status, out[k].error);
    pdsim::PlacementPlan& plan = plans[k];
    plan.counts.assign(counts[k].begin(), counts[k].end());
    plan.table = ps[k].table;
    if (max_freq[k] >= 0.0)  // the restricted table (placement.hpp:423-430, 486)
      for (auto& e : plan.table)
        if (e.config.base_freq_mhz != max_freq[k]) {
          e.r_c = 0.0;
          e.e_c.reset();
          e.error = "below maximum frequency";
        }
    plan.objective_w = out[k].objective_w;
    plan.target_rps = ps[k].target_rps;
    plan.alpha = ps[k].alpha;
    plan.total_gpus = ps[k].total_gpus;
    plan.gpus_used = out[k].gpus_used;
    plan.instances = pdsim::derive_routing_weights(plan.counts, plan.table);
  }
  return plans;
}

// run_experiment (runner.hpp:155-172): window w planned from window w-1 on
// the GPU, then every (window, policy) replayed in one device call.  Result
// as the reference's; runs[i].sim holds SimResult's counters, plus the
// records when `records` (see replay_policies), so the CLI's writers
// (cli.hpp:371-378) produce the reference's files.
inline pdsim::ExperimentResult run_experiment(const DeviceModels& dm, const pdsim::Trace& trace, double window_ms,
                                              const std::vector<pdsim::Policy>& policies,
                                              const pdsim::RunnerConfig& cfg, bool records = false) {
  cfg.validate();
  if (policies.empty()) throw pdsim::ParameterError("no policies selected");
  std::vector<pdsim::Trace> windows = pdsim::split_windows(trace, window_ms);
  // plan_window (placement.hpp:558-582) for every window, all the config
  // tables in one device call (bs_goodput_tables)
  std::vector<pdsim::Trace> predicted;
  for (std::size_t w = 0; w < windows.size(); ++w) {
    const pdsim::Trace& history = w == 0 ? windows[0] : windows[w - 1];
    history.validate();
    if (history.requests.empty()) throw pdsim::ParameterError("plan_window: empty history");
    predicted.push_back(pdsim::predict_next_window(history));
  }
  std::vector<const pdsim::Trace*> probes;
  for (const auto& p : predicted) probes.push_back(cfg.plan.probe_trace ? &*cfg.plan.probe_trace : &p);
  const std::vector<pdsim::InstanceConfig> candidates = pdsim::enumerate_candidates(cfg.ladder, cfg.tp_options);
  std::vector<std::vector<pdsim::ConfigTableEntry>> tables =
      pdsim_gpu::build_config_tables(dm, candidates, probes, cfg.slo, cfg.plan.policy, cfg.plan.search);
  // every window's ILP and max-throughput baseline in one device call
  std::vector<pdsim::WindowPlans> plans(windows.size());
  std::vector<pdsim::PlacementProblem> problems;
  std::vector<double> max_freq;
  for (std::size_t w = 0; w < windows.size(); ++w) {
    pdsim::WindowPlans& wp = plans[w];
    wp.target_rps = pdsim::peak_rps(predicted[w], cfg.plan.peak_subwindow_s);
    wp.table = std::move(tables[w]);
    problems.push_back(pdsim::PlacementProblem{wp.table, cfg.total_gpus, wp.target_rps, cfg.plan.alpha});
    problems.push_back(problems.back());
    max_freq.push_back(-1.0);
    max_freq.push_back(cfg.ladder.max_mhz());
  }
  std::vector<pdsim::PlacementPlan> solved = pdsim_gpu::solve_placements(dm.device(), problems, max_freq);
  for (std::size_t w = 0; w < windows.size(); ++w) {
    plans[w].ilp = std::move(solved[2 * w]);
    plans[w].maxfreq = std::move(solved[2 * w + 1]);
  }
  std::vector<const pdsim::Trace*> wins;
  std::vector<const pdsim::PlacementPlan*> pls;
  std::vector<pdsim::Policy> pols;
  for (std::size_t w = 0; w < windows.size(); ++w)
    for (pdsim::Policy pol : policies) {
      wins.push_back(&windows[w]);
      pls.push_back(pol == pdsim::Policy::maxfreq_distserve ? &plans[w].maxfreq : &plans[w].ilp);
      pols.push_back(pol);
    }
  std::vector<ReplayRun> runs = pdsim_gpu::replay_policies(dm, wins, pls, pols, cfg, records);
  pdsim::ExperimentResult out;
  for (std::size_t i = 0; i < runs.size(); ++i) {
    const std::size_t w = i / policies.size();
    pdsim::WindowRun run;
    run.window_index = static_cast<int>(w);
    run.policy = pols[i];
    run.plan = *pls[i];
    run.sim = std::move(runs[i].sim);
    run.report = runs[i].report;
    run.report.window_id = "w" + std::to_string(w);
    run.report.system = pdsim::policy_name(pols[i]);
    run.slo_pass = (!run.report.p99_ttft_ms || *run.report.p99_ttft_ms <= cfg.slo.ttft_ms) &&
                   (!run.report.p99_mean_tpot_ms || *run.report.p99_mean_tpot_ms <= cfg.slo.tpot_ms);
    if (run.policy == pdsim::Policy::two_tier && !run.slo_pass) out.two_tier_slo_pass = false;
    out.reports.push_back(run.report);
    out.runs.push_back(std::move(run));
  }
  return out;
}

}  // namespace pdsim_gpu

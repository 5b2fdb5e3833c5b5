// experiment_parity.cpp — TEST INFRASTRUCTURE (drop-in proof for the window
// loop).  Runs the reference's run_experiment (runner.hpp:155-172) and
// pdsim_gpu::run_experiment (include/biscale_gpu_pdsim.hpp: GPU config
// tables + ILP per window, every (window, policy) replay in one bs_replay
// call) on the same trace and RunnerConfig, and compares plans, SimResult
// counters, MetricsReports and SLO verdicts run by run.  One JSON line.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pdsim/runner.hpp"

#include "biscale_gpu_pdsim.hpp"

using namespace pdsim;

namespace {

double arg(int argc, char** argv, const char* name, double def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return std::atof(argv[i + 1]);
  return def;
}

bool same_opt(const std::optional<double>& a, const std::optional<double>& b) {
  return a.has_value() == b.has_value() && (!a || *a == *b);
}

bool same_report(const MetricsReport& a, const MetricsReport& b) {
  return a.window_id == b.window_id && a.system == b.system && same_opt(a.p99_ttft_ms, b.p99_ttft_ms) &&
         same_opt(a.p99_mean_tpot_ms, b.p99_mean_tpot_ms) &&
         same_opt(a.energy_per_first_token_j, b.energy_per_first_token_j) &&
         same_opt(a.energy_per_output_token_j, b.energy_per_output_token_j) &&
         a.avg_power_prefill_w == b.avg_power_prefill_w && a.avg_power_decode_w == b.avg_power_decode_w &&
         a.prefill_energy_j == b.prefill_energy_j && a.decode_energy_j == b.decode_energy_j &&
         a.span_ms == b.span_ms && a.completed_requests == b.completed_requests &&
         a.generated_tokens == b.generated_tokens && a.ttft_violations == b.ttft_violations &&
         a.tpot_violations == b.tpot_violations;
}

}  // namespace

int main(int argc, char** argv) {
  const auto seed = static_cast<std::uint64_t>(arg(argc, argv, "--seed", 7));
  const double minutes = arg(argc, argv, "--minutes", 6);
  const double window_s = arg(argc, argv, "--window-s", 120);
  const double rps = arg(argc, argv, "--rps", 8);
  const double shape = arg(argc, argv, "--shape", 1.0);
  const int gpus = static_cast<int>(arg(argc, argv, "--gpus", 8));

  FrequencyLadder ladder;
  for (int i = 0; i < 8; ++i) ladder.freqs_mhz.push_back(360.0 + 210.0 * i);
  SynthOptions pre, dec;
  pre.lat_coef = 366.0;
  pre.power_a = 1e-7;
  pre.power_b = 60.0;
  dec.lat_coef = 6.0;
  dec.power_a = 1e-7;
  dec.power_b = 120.0;
  ModelSet models = synth_model_set(SynthFamily::compute_bound, ladder, {1, 2, 4, 8}, pre, dec);
  LengthDistribution lengths;
  lengths.lognormal = LengthDistribution::Lognormal{6.2, 0.6, 5.3, 0.7};
  Trace trace = gen_gamma_trace(rps, shape, minutes * 60e3, lengths, seed);

  RunnerConfig cfg;
  cfg.total_gpus = gpus;
  cfg.tp_options = {1, 2, 4};
  cfg.ladder = ladder;
  cfg.scheduler.max_batch_tokens = 1024;
  cfg.plan.policy.max_batch_tokens = 1024;
  cfg.rampup_s = 10.0;
  const std::vector<Policy> pols = {Policy::maxfreq_distserve, Policy::place_only, Policy::two_tier};

  auto t0 = std::chrono::steady_clock::now();
  ExperimentResult ref = run_experiment(trace, window_s * 1000.0, pols, cfg, models);
  auto t1 = std::chrono::steady_clock::now();
  pdsim_gpu::Device dev(0);
  pdsim_gpu::DeviceModels dm(dev, models);
  ExperimentResult gpu = pdsim_gpu::run_experiment(dm, trace, window_s * 1000.0, pols, cfg);
  auto t2 = std::chrono::steady_clock::now();

  int mismatch = 0;
  bool counts = ref.runs.size() == gpu.runs.size();
  for (std::size_t i = 0; counts && i < ref.runs.size(); ++i) {
    const WindowRun& a = ref.runs[i];
    const WindowRun& b = gpu.runs[i];
    const bool ok = a.window_index == b.window_index && a.policy == b.policy && a.plan.counts == b.plan.counts &&
                    a.plan.objective_w == b.plan.objective_w && a.plan.gpus_used == b.plan.gpus_used &&
                    a.sim.horizon_ms == b.sim.horizon_ms && a.sim.completed_requests == b.sim.completed_requests &&
                    a.sim.generated_tokens == b.sim.generated_tokens && same_report(a.report, b.report) &&
                    a.slo_pass == b.slo_pass;
    mismatch += ok ? 0 : 1;
  }
  const bool match = counts && mismatch == 0 && ref.two_tier_slo_pass == gpu.two_tier_slo_pass;
  std::printf("{\"runs\": %zu, \"mismatch\": %d, \"two_tier_slo_pass\": %s, \"cpu_s\": %.3f, \"gpu_s\": %.3f, "
              "\"match\": %s}\n",
              ref.runs.size(), mismatch, gpu.two_tier_slo_pass ? "true" : "false",
              std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
              match ? "true" : "false");
  return match ? 0 : 1;
}

// placement_parity.cpp — TEST INFRASTRUCTURE (drop-in proof for the
// placement boundary).  Builds the config table of one trace window twice:
// with the reference's own build_config_table (placement.hpp:240-260,
// std::async per candidate) and with pdsim_gpu::build_config_table (the
// sm_100a path through the C ABI, include/biscale_gpu_pdsim.hpp); then
// solves the placement ILP and the max-throughput baseline from each table
// with the reference and with the shim.  Compares entries, counts,
// objectives and routing weights bit for bit and prints one JSON line.
// Built by oracle/Makefile into oracle/_ref/.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "pdsim/placement.hpp"
#include "pdsim/workload.hpp"

#include "biscale_gpu_pdsim.hpp"

using namespace pdsim;

namespace {

double arg(int argc, char** argv, const char* name, double def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return std::atof(argv[i + 1]);
  return def;
}

bool same_entry(const ConfigTableEntry& a, const ConfigTableEntry& b) {
  return a.config.phase == b.config.phase && a.config.tp == b.config.tp &&
         a.config.base_freq_mhz == b.config.base_freq_mhz && a.r_c == b.r_c && a.e_c == b.e_c && a.g_c == b.g_c &&
         a.saturated == b.saturated && a.error == b.error;
}

bool same_plan(const PlacementPlan& a, const PlacementPlan& b) {
  if (a.counts != b.counts || a.objective_w != b.objective_w || a.gpus_used != b.gpus_used) return false;
  if (a.instances.size() != b.instances.size()) return false;
  for (std::size_t i = 0; i < a.instances.size(); ++i)
    if (a.instances[i].weight != b.instances[i].weight || a.instances[i].config.tp != b.instances[i].config.tp ||
        a.instances[i].config.base_freq_mhz != b.instances[i].config.base_freq_mhz)
      return false;
  return true;
}

template <class F>
std::string outcome(F&& f, PlacementPlan* out) {
  try {
    *out = f();
    return "ok";
  } catch (const InfeasibleError& e) {
    return std::string("infeasible:") + e.what();
  } catch (const std::exception& e) {
    return std::string("error:") + e.what();
  }
}

}  // namespace

int main(int argc, char** argv) {
  const auto seed = static_cast<std::uint64_t>(arg(argc, argv, "--seed", 7));
  const double duration_s = arg(argc, argv, "--duration-s", 600);
  const double rps = arg(argc, argv, "--rps", 12);
  const double shape = arg(argc, argv, "--shape", 0.5);
  const int levels = static_cast<int>(arg(argc, argv, "--levels", 8));
  const int gpus = static_cast<int>(arg(argc, argv, "--gpus", 16));
  const long long mbt = static_cast<long long>(arg(argc, argv, "--max-batch-tokens", 2048));

  // Llama-3.3-70B-shaped synthetic models on an L-level
  // ladder 360 + i (1830 - 360) / (L - 1).
  FrequencyLadder ladder;
  for (int i = 0; i < levels; ++i) ladder.freqs_mhz.push_back(360.0 + i * (1830.0 - 360.0) / (levels - 1));
  SynthOptions pre, dec;
  pre.lat_coef = 366.0;
  pre.power_a = 1e-7;
  pre.power_b = 60.0;
  dec.lat_coef = 6.0;
  dec.power_a = 1e-7;
  dec.power_b = 60.0;
  ModelSet models = synth_model_set(SynthFamily::compute_bound, ladder, {1, 2, 4, 8}, pre, dec);
  LengthDistribution lengths;
  lengths.lognormal = LengthDistribution::Lognormal{6.2, 0.6, 5.3, 0.7};
  Trace base = gen_gamma_trace(rps, shape, duration_s * 1000.0, lengths, seed);

  SLOSpec slo;
  slo.ttft_ms = arg(argc, argv, "--ttft", 600);
  slo.tpot_ms = arg(argc, argv, "--tpot", 100);
  SchedulerPolicy policy;
  policy.max_batch_tokens = mbt;
  GoodputSearch search;
  std::vector<InstanceConfig> cands = enumerate_candidates(ladder, {1, 2, 4, 8});

  auto t0 = std::chrono::steady_clock::now();
  std::vector<ConfigTableEntry> ref = build_config_table(cands, base, slo, models, policy, search, true);
  auto t1 = std::chrono::steady_clock::now();
  pdsim_gpu::Device dev(0);
  pdsim_gpu::DeviceModels dm(dev, models);
  std::vector<ConfigTableEntry> gpu = pdsim_gpu::build_config_table(dm, cands, base, slo, policy, search);
  auto t2 = std::chrono::steady_clock::now();

  int table_mismatch = 0;
  for (std::size_t i = 0; i < cands.size(); ++i) table_mismatch += same_entry(ref[i], gpu[i]) ? 0 : 1;

  PlacementProblem pr{ref, gpus, peak_rps(base, 10.0), 0.05};
  PlacementPlan a, b, c, d;
  std::string oa = outcome([&] { return solve_placement(pr); }, &a);
  std::string ob = outcome([&] { return pdsim_gpu::solve_placement(pr); }, &b);
  std::string oc = outcome([&] { return solve_max_throughput(pr, ladder.max_mhz()); }, &c);
  std::string od = outcome([&] { return pdsim_gpu::solve_max_throughput(pr, ladder.max_mhz()); }, &d);
  const bool ilp_ok = oa == ob && (oa != "ok" || same_plan(a, b));
  const bool mt_ok = oc == od && (oc != "ok" || same_plan(c, d));

  // Error-path parity: a budget too small for the target.
  PlacementProblem tiny{ref, 1, peak_rps(base, 10.0) * 50.0, 0.05};
  std::string ea = outcome([&] { return solve_placement(tiny); }, &a);
  std::string eb = outcome([&] { return pdsim_gpu::solve_placement(tiny); }, &b);

  const bool match = table_mismatch == 0 && ilp_ok && mt_ok && ea == eb;
  std::printf(
      "{\"requests\": %zu, \"candidates\": %zu, \"table_mismatch\": %d, \"ilp\": \"%s\", \"ilp_match\": %s, "
      "\"maxthr_match\": %s, \"error_path\": \"%s\", \"error_match\": %s, \"cpu_s\": %.3f, \"gpu_s\": %.3f, "
      "\"match\": %s}\n",
      base.requests.size(), cands.size(), table_mismatch, oa.c_str(), ilp_ok ? "true" : "false",
      mt_ok ? "true" : "false", ea.substr(0, 60).c_str(), ea == eb ? "true" : "false",
      std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
      match ? "true" : "false");
  return match ? 0 : 1;
}

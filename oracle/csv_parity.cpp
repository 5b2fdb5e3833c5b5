// csv_parity.cpp — TEST INFRASTRUCTURE (output-format drop-in proof, SURVEY.md
// §8f item 2).  Writes the files of the CLI's `run` command (cli.hpp:371-378:
// plan_*.json, requests_*.csv, batches_*.csv, decisions_*.csv, report.csv)
// with the reference's own writers, once from the reference's
// run_experiment and once from pdsim_gpu::run_experiment(records = true),
// and compares them byte for byte.  One JSON line.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>

#include "pdsim/runner.hpp"

#include "biscale_gpu_pdsim.hpp"

using namespace pdsim;

namespace {

double arg(int argc, char** argv, const char* name, double def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return std::atof(argv[i + 1]);
  return def;
}

std::string slurp(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  std::stringstream ss;
  ss << is.rdbuf();
  return ss.str();
}

std::vector<std::string> write_all(const ExperimentResult& r, const std::string& dir) {
  std::filesystem::create_directories(dir);
  std::vector<std::string> names;
  for (const WindowRun& run : r.runs) {
    const std::string tag = "w" + std::to_string(run.window_index) + "_" + policy_name(run.policy);
    save_plan_json(run.plan, dir + "/plan_" + tag + ".json");
    save_request_csv(run.sim, dir + "/requests_" + tag + ".csv");
    save_batch_csv(run.sim, dir + "/batches_" + tag + ".csv");
    save_decision_log_csv(run.sim.decisions, dir + "/decisions_" + tag + ".csv");
    for (const char* k : {"plan_", "requests_", "batches_", "decisions_"})
      names.push_back(std::string(k) + tag + (std::string(k) == "plan_" ? ".json" : ".csv"));
  }
  save_report_csv(r.reports, dir + "/report.csv");
  names.push_back("report.csv");
  return names;
}

}  // namespace

int main(int argc, char** argv) {
  const auto seed = static_cast<std::uint64_t>(arg(argc, argv, "--seed", 7));
  const double minutes = arg(argc, argv, "--minutes", 4);
  const double window_s = arg(argc, argv, "--window-s", 120);
  const double rps = arg(argc, argv, "--rps", 8);
  const std::string out = argc > 1 && argv[argc - 1][0] != '-' ? argv[argc - 1] : "/tmp/csv_parity";

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
  Trace trace = gen_gamma_trace(rps, 1.0, minutes * 60e3, lengths, seed);
  RunnerConfig cfg;
  cfg.total_gpus = 8;
  cfg.tp_options = {1, 2, 4};
  cfg.ladder = ladder;
  cfg.scheduler.max_batch_tokens = 1024;
  cfg.plan.policy.max_batch_tokens = 1024;
  cfg.rampup_s = 10.0;
  const std::vector<Policy> pols = {Policy::maxfreq_distserve, Policy::place_only, Policy::two_tier};

  ExperimentResult ref = run_experiment(trace, window_s * 1000.0, pols, cfg, models);
  pdsim_gpu::Device dev(0);
  pdsim_gpu::DeviceModels dm(dev, models);
  ExperimentResult gpu = pdsim_gpu::run_experiment(dm, trace, window_s * 1000.0, pols, cfg, true);

  const std::vector<std::string> a = write_all(ref, out + "/ref");
  const std::vector<std::string> b = write_all(gpu, out + "/gpu");
  int differ = 0;
  std::string first;
  long long bytes = 0;
  for (const std::string& f : a) {
    const std::string x = slurp(out + "/ref/" + f), y = slurp(out + "/gpu/" + f);
    bytes += static_cast<long long>(x.size());
    if (x != y) {
      ++differ;
      if (first.empty()) first = f;
    }
  }
  const bool match = a == b && differ == 0;
  std::printf("{\"files\": %zu, \"bytes\": %lld, \"differ\": %d, \"first_diff\": \"%s\", \"match\": %s}\n", a.size(),
              bytes, differ, first.c_str(), match ? "true" : "false");
  return match ? 0 : 1;
}

// replay_parity.cpp — TEST INFRASTRUCTURE (drop-in proof for the controller
// boundary).  Runs the reference's own, unmodified simulate_cluster
// (simulator.hpp:758-893, the run_policy shape of runner.hpp:112-122) twice
// on the same trace and cluster: once with pdsim::TwoTierFactory (the CPU
// reference controllers) and once with pdsim_gpu::GpuTwoTierFactory (the
// sm_100a path through the C ABI, include/biscale_gpu_pdsim.hpp), and
// compares the decision logs, batch records and request records bit for bit.
// Prints one JSON line.  Built by oracle/Makefile into oracle/_ref/.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "pdsim/dvfs.hpp"
#include "pdsim/simulator.hpp"
#include "pdsim/workload.hpp"

#include "biscale_gpu_pdsim.hpp"

using namespace pdsim;

namespace {

double arg(int argc, char** argv, const char* name, double def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return std::atof(argv[i + 1]);
  return def;
}

}  // namespace

int main(int argc, char** argv) {
  const auto seed = static_cast<std::uint64_t>(arg(argc, argv, "--seed", 7));
  const double duration_s = arg(argc, argv, "--duration-s", 120);
  const double rps = arg(argc, argv, "--rps", 6);
  const double shape = arg(argc, argv, "--shape", 1.0);
  const int mpc_k = static_cast<int>(arg(argc, argv, "--mpc-k", 8));
  const int mpc_n = static_cast<int>(arg(argc, argv, "--mpc-n", 7));
  const int n_prefill = static_cast<int>(arg(argc, argv, "--prefill", 1));
  const int n_decode = static_cast<int>(arg(argc, argv, "--decode", 1));
  const double ttft = arg(argc, argv, "--ttft", 600);
  const int skip_cpu = static_cast<int>(arg(argc, argv, "--gpu-only", 0));

  // Llama-3.3-70B-shaped synthetic models on the 8-rung H100-style ladder
  // (SURVEY.md §8d).
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
  Trace trace = gen_gamma_trace(rps, shape, duration_s * 1000.0, lengths, seed);

  ClusterSpec cluster;
  for (int i = 0; i < n_prefill; ++i)
    cluster.instances.push_back(ClusterInstance{InstanceConfig{Phase::prefill, 2, ladder.max_mhz()}, 1.0 / n_prefill});
  for (int i = 0; i < n_decode; ++i)
    cluster.instances.push_back(ClusterInstance{InstanceConfig{Phase::decode, 4, ladder.max_mhz()}, 1.0 / n_decode});

  MpcConfig mpc;
  mpc.horizon_K = mpc_k;
  mpc.ladder_N = mpc_n;
  mpc.ladder = ladder;
  mpc.slo.ttft_ms = ttft;
  mpc.switch_latency_ms = 30.0;
  mpc.margin = 0.05;
  DecodePolicyConfig dcfg;
  dcfg.tbt_slo_ms = 100.0;
  dcfg.kv_threshold = 0.9;
  dcfg.ladder = ladder;
  dcfg.margin = 0.05;
  SchedulerPolicy policy;
  policy.max_batch_tokens = 2048;
  SimOptions opts;
  opts.switch_latency_ms = 30.0;

  SimResult cpu;
  double cpu_s = 0.0;
  if (!skip_cpu) {
    TwoTierFactory cpu_factory(mpc, dcfg, models, policy);
    auto t0 = std::chrono::steady_clock::now();
    cpu = simulate_cluster(trace, cluster, policy, models, &cpu_factory, opts);
    cpu_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  pdsim_gpu::Device dev(0);
  pdsim_gpu::DeviceModels dm(dev, models);
  pdsim_gpu::GpuTwoTierFactory gpu_factory(mpc, dcfg, models, dm, policy);
  auto t1 = std::chrono::steady_clock::now();
  SimResult gpu = simulate_cluster(trace, cluster, policy, models, &gpu_factory, opts);
  const double gpu_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();

  std::size_t mismatches = 0;
  std::string first;
  auto miss = [&](const std::string& what) {
    if (mismatches++ == 0) first = what;
  };
  if (!skip_cpu) {
    if (cpu.decisions.records.size() != gpu.decisions.records.size()) miss("decision count");
    for (std::size_t i = 0; i < std::min(cpu.decisions.records.size(), gpu.decisions.records.size()); ++i) {
      const auto& a = cpu.decisions.records[i];
      const auto& b = gpu.decisions.records[i];
      if (a.time_ms != b.time_ms || a.instance != b.instance || a.trigger != b.trigger ||
          a.chosen_freq_mhz != b.chosen_freq_mhz || a.feasible != b.feasible || a.eval_count != b.eval_count)
        miss("decision " + std::to_string(i));
    }
    if (cpu.batches.size() != gpu.batches.size()) miss("batch count");
    for (std::size_t i = 0; i < std::min(cpu.batches.size(), gpu.batches.size()); ++i) {
      const auto& a = cpu.batches[i];
      const auto& b = gpu.batches[i];
      if (a.start_ms != b.start_ms || a.end_ms != b.end_ms || a.freq_mhz != b.freq_mhz || a.power_w != b.power_w ||
          a.energy_j != b.energy_j || a.instance != b.instance)
        miss("batch " + std::to_string(i));
    }
    for (std::size_t i = 0; i < cpu.requests.size(); ++i) {
      const auto& a = cpu.requests[i];
      const auto& b = gpu.requests[i];
      if (a.prefill_done_ms != b.prefill_done_ms || a.token_times_ms != b.token_times_ms || a.completed != b.completed)
        miss("request " + std::to_string(i));
    }
    if (cpu.total_energy_j() != gpu.total_energy_j()) miss("total energy");
  }
  std::size_t prefill_dec = 0, decode_dec = 0;
  for (const auto& r : gpu.decisions.records) {
    if (r.trigger == Trigger::safety) continue;
    (gpu.instances[static_cast<std::size_t>(r.instance)].phase == Phase::prefill ? prefill_dec : decode_dec) += 1;
  }
  std::printf(
      "{\"requests\": %zu, \"decisions\": %zu, \"prefill_decisions\": %zu, \"decode_decisions\": %zu, "
      "\"batches\": %zu, \"match\": %s, \"mismatches\": %zu, \"first_mismatch\": \"%s\", \"cpu_s\": %.6f, "
      "\"gpu_s\": %.6f, \"energy_j\": %.9g, \"checked\": %s}\n",
      trace.requests.size(), gpu.decisions.records.size(), prefill_dec, decode_dec, gpu.batches.size(),
      mismatches == 0 ? "true" : "false", mismatches, first.c_str(), cpu_s, gpu_s, gpu.total_energy_j(),
      skip_cpu ? "false" : "true");
  return mismatches == 0 ? 0 : 1;
}

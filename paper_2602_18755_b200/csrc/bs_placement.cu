// bs_placement.cu — coarse-tier placement search on sm_100a:
// build_config_table (placement.hpp:240-260) = for every candidate,
// max_goodput (154-199) + E_c (217-238); then solve_placement (357-416) and
// solve_max_throughput (421-499).
//
//   mask_kernel    one warp per probe stream (rate step k, replicate j):
//                  mt19937_64 seeded with probe_seed(k, j) (a warp-parallel
//                  twist), keep request i iff uniform01 < min(1, k tol /
//                  rate) (downsample_trace, workload.hpp:120-132); writes the
//                  compacted kept-index list.  Streams depend only on (k, j),
//                  so every candidate shares them.
//   probe_kernel   one thread per (candidate, k, j): the instance event loop
//                  at the candidate's fixed frequency (bs_sim.cuh), stopping
//                  at the first SLO violation when no ModelError can occur
//                  later in the run (all grid values positive, idle entry
//                  present); otherwise the full run with exact error order.
//   host replay    the reference's exact search path over the per-k results
//                  (k_max, then 1, then lo + (hi - lo) / 2): feasibility is
//                  not monotone in k (independent down-samples per k), so
//                  "largest feasible k" would differ.
//   energy_kernel  one thread per candidate with k* > 0: the full run at
//                  (k*, replicate 0) -> busy (+ idle for prefill) / completed.
//   ILP            exact branch and bound (host), reference fold order and
//                  tie-breaks.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "bs_internal.h"
#include "bs_rng.cuh"
#include "bs_sim.cuh"

using namespace bs;

namespace {

constexpr int kMaskWarps = 4;

// --- keep masks ---------------------------------------------------------------

struct MaskParams {
  long long n;            // base requests
  int k_max;
  int reps;
  double tol;
  double base_rate;
  unsigned long long seed;
};

// One warp per stream s = (k - 1) * reps + j.  The mt19937_64 twist in three
// dependency phases (indices [0,156), [156,311), 311) so the warp computes it
// in parallel; outputs are consumed in order, one per request.
// Several tables at once: stream S of the launch belongs to the table t with
// stream_off[t] <= S < stream_off[t + 1]; its kept list starts at
// kept_off[t] + (S - stream_off[t]) * n_t.
__global__ void __launch_bounds__(kMaskWarps * 32) mask_kernel(const MaskParams* mps, int n_tables,
                                                               const long long* stream_off, const long long* kept_off,
                                                               int* kept, long long* kept_count) {
  __shared__ unsigned long long st[kMaskWarps][kMtN];
  __shared__ unsigned long long tmp[kMaskWarps][kMtN];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long S = static_cast<long long>(blockIdx.x) * kMaskWarps + w;
  if (S >= stream_off[n_tables]) return;
  int tb = 0;
  while (stream_off[tb + 1] <= S) ++tb;
  const MaskParams mp = mps[tb];
  const long long s = S - stream_off[tb];
  const long long k = s / mp.reps + 1;
  const int j = s % mp.reps;
  // keep = min(1, k * tol / base_rate)  (placement.hpp:146-147)
  const double kk = __ddiv_rn(__dmul_rn(static_cast<double>(k), mp.tol), mp.base_rate);
  const double keep = kk < 1.0 ? kk : 1.0;
  unsigned long long* mt = st[w];
  unsigned long long* tp = tmp[w];
  if (lane == 0) {
    const unsigned long long seed = probe_seed(mp.seed, k, j);
    mt[0] = seed;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
  }
  __syncwarp();
  int* out = kept + kept_off[tb] + static_cast<size_t>(s) * mp.n;
  long long count = 0;
  for (long long base = 0; base < mp.n; base += kMtN) {
    // twist
    auto f = [&](unsigned long long a, unsigned long long b, unsigned long long c) {
      const unsigned long long x = (a & kMtUpper) | (b & kMtLower);
      unsigned long long xa = x >> 1;
      if (x & 1ull) xa ^= kMtMatrix;
      return c ^ xa;
    };
    for (int i = lane; i < kMtM; i += 32) tp[i] = f(mt[i], mt[i + 1], mt[i + kMtM]);
    __syncwarp();
    for (int i = lane; i < kMtM; i += 32) mt[i] = tp[i];
    __syncwarp();
    for (int i = kMtM + lane; i < kMtN - 1; i += 32) tp[i] = f(mt[i], mt[i + 1], mt[i - kMtM]);
    __syncwarp();
    for (int i = kMtM + lane; i < kMtN - 1; i += 32) mt[i] = tp[i];
    __syncwarp();
    if (lane == 0) mt[kMtN - 1] = f(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
    __syncwarp();
    // outputs in order, 32 at a time
    const long long cnt = (mp.n - base) < kMtN ? (mp.n - base) : kMtN;
    for (int i0 = 0; i0 < cnt; i0 += 32) {
      const int i = i0 + lane;
      bool keepit = false;
      if (i < cnt) {
        const double u = static_cast<double>(Mt64::temper(mt[i]) >> 11) * 0x1.0p-53;
        keepit = u < keep;
      }
      const unsigned mask = __ballot_sync(0xffffffffu, keepit);
      if (keepit) out[count + __popc(mask & ((1u << lane) - 1u))] = static_cast<int>(base + i);
      count += __popc(mask);
    }
    __syncwarp();
  }
  if (lane == 0) kept_count[S] = count;
}

// --- probes ---------------------------------------------------------------------

struct DCand {
  int phase;
  int tp;
  double freq;
  int safe;  // no ModelError possible: early exit allowed
};

struct ProbeOut {
  int status;
  int model_err;
  int meets;
  int empty;
  long long events;  // batches / iterations simulated (instrumentation)
  // energy accounting of the run; complete whenever the probe was feasible
  // (a feasible probe never stops early), which is what E_c needs
  long long completed;
  double busy_j;
  double idle_j;
  long long ns;  // wall time of the probe (%globaltimer; diagnostics)
};

struct TraceDev {
  const double* arrival;
  const long long* input;
  const long long* output;
  double duration_ms;
};

struct PolicyDev {
  long long max_batch_tokens, max_batch_requests, kv_capacity;
  int chunking;
  double ttft, tpot;
};

__device__ __forceinline__ SimParams make_params(const DCand& c, const PolicyDev& pol, int early) {
  SimParams p;
  p.tp = c.tp;
  p.freq = c.freq;
  p.max_batch_tokens = pol.max_batch_tokens;
  p.max_batch_requests = pol.max_batch_requests;
  p.kv_capacity = pol.kv_capacity;
  p.chunking = pol.chunking;
  p.ttft_bound = pol.ttft;
  p.tpot_bound = pol.tpot;
  p.early_exit = early;
  p.search = nullptr;
  p.k = 0;
  return p;
}

// Per-warp shared scratch of the warp-cooperative decode simulator: the
// resident array and the batch-size bracket table (when they fit) and the
// 3 x 32-entry window arrays.
__host__ __device__ inline size_t ntab_bytes(int heap_cap) {
  return (static_cast<size_t>(heap_cap) + 1) * sizeof(double) + ((static_cast<size_t>(heap_cap) + 1 + 15) / 16) * 16;
}

__host__ __device__ inline size_t warp_scratch_bytes(int heap_cap, bool heap_in_smem) {
  return (heap_in_smem ? static_cast<size_t>(heap_cap) * sizeof(Resident) + ntab_bytes(heap_cap) : 0) +
         3 * 32 * sizeof(double);
}

__device__ __forceinline__ WarpScratch carve_scratch(unsigned char* smem, int warp, int heap_cap, bool heap_in_smem,
                                                    Resident* gheap) {
  unsigned char* p = smem + static_cast<size_t>(warp) * warp_scratch_bytes(heap_cap, heap_in_smem);
  WarpScratch ws;
  ws.nfrac = nullptr;
  ws.nlo = nullptr;
  if (heap_in_smem) {
    ws.heap = reinterpret_cast<Resident*>(p);
    p += static_cast<size_t>(heap_cap) * sizeof(Resident);
    ws.nfrac = reinterpret_cast<double*>(p);
    ws.nlo = p + (static_cast<size_t>(heap_cap) + 1) * sizeof(double);
    p += ntab_bytes(heap_cap);
  } else {
    ws.heap = gheap;
  }
  ws.L = reinterpret_cast<double*>(p);
  ws.P = ws.L + 32;
  ws.T = ws.L + 64;
  return ws;
}

// One warp per probe.  Prefill probes run the scalar event loop on lane 0
// (batches are few); decode probes run the warp-cooperative simulator
// (bs_sim.cuh), which evaluates up to 32 iterations' predictions at once.
// Packing 32 probes into one warp instead would serialise their divergent
// paths.
// One probe of a multi-table launch: table, candidate, stream of the table.
struct ProbeId {
  int t;
  int c;
  long long s;
};

// Per-table views of the concatenated inputs.
struct TableDev {
  long long req_off;     // first request in the concatenated trace arrays
  long long n;           // requests of the table's base trace
  long long stream_off;  // first (k, replicate) stream in kept_count
  long long kept_off;    // first kept index slot
  long long probe_off;   // first probe output: + c * n_streams + s
  long long n_streams;
  double duration_ms;
};

#ifndef BS_PROBE_MINB
#define BS_PROBE_MINB 3  // resident CTAs per SM the probe kernel is register-budgeted for (throughput of a stream of tables over the latency of one)
#endif

__global__ void __launch_bounds__(128, BS_PROBE_MINB) probe_kernel(DModels m, TraceDev tr, const TableDev* tabs, const DCand* cands, const int* kept,
                             const long long* kept_count, PolicyDev pol, Resident* heaps, int heap_cap,
                             int heap_in_smem, const ProbeId* order, long long n_probes, ProbeOut* out, int* pst,
                             int reps) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long slot = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (slot >= n_probes) return;
  const ProbeId id = order[slot];  // launch order: the search tree's top levels first, across every table
  const TableDev tb = tabs[id.t];
  const long long cbase = tb.probe_off + static_cast<long long>(id.c) * tb.n_streams;
  const long long gid = cbase + id.s;
  const DCand cd = cands[id.c];
  const SearchView sv{pst + cbase, tb.n_streams / reps, reps};
  const long long k = id.s / reps + 1;
  ProbeOut o;
  o.status = BS_OK;
  o.model_err = 0;
  o.meets = 1;
  o.empty = 0;
  o.events = 0;
  o.completed = 0;
  o.busy_j = 0.0;
  o.idle_j = 0.0;
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  o.ns = 0;
  auto publish = [&](int code) {  // the outcome record first, then its code for the other probes
    out[gid] = o;
    __threadfence();
    *reinterpret_cast<volatile int*>(pst + gid) = code;
  };
  int alive = lane == 0 ? (search_alive(sv, k) ? 1 : 0) : 0;
  alive = __shfl_sync(0xffffffffu, alive, 0);
  if (!alive) {  // off the search path already: never run
    o.status = kSimAborted;
    o.completed = -1;  // marks "skipped at start" in the statistics
    if (lane == 0) publish(kProbeSkipped);
    return;
  }
  const long long nk = kept_count[tb.stream_off + id.s];
  if (nk == 0) {  // placement.hpp:169: an empty probe passes
    o.empty = 1;
    if (lane == 0) publish(kProbePass);
    return;
  }
  SimTrace st;
  st.arrival = tr.arrival + tb.req_off;
  st.input = tr.input + tb.req_off;
  st.output = tr.output + tb.req_off;
  st.kept = kept + tb.kept_off + static_cast<size_t>(id.s) * tb.n;
  st.n = nk;
  st.duration_ms = tb.duration_ms;
  SimParams p = make_params(cd, pol, cd.safe);
  p.search = &sv;
  p.k = k;
  SimOut r;
  if (cd.phase == BS_PHASE_PREFILL) {
    if (lane != 0) return;
    r = simulate_prefill(m, st, p);
  } else {
    const WarpScratch ws =
        carve_scratch(smem, warp, heap_cap, heap_in_smem != 0, heaps + static_cast<size_t>(slot) * heap_cap);
    r = simulate_decode_warp(m, st, p, ws, heap_cap, lane);
    if (lane != 0) return;
  }
  o.status = r.status;
  o.model_err = r.model_err;
  o.meets = r.meets_slo;
  o.events = r.batches;
  o.completed = r.completed;
  o.busy_j = r.busy_j;
  o.idle_j = r.idle_j;
  {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    o.ns = static_cast<long long>(t_end - t_start);
  }
  // feasible(k) (placement.hpp:172-176): SimulationError counts as a failure
  publish(r.status == kSimAborted           ? kProbeSkipped
          : r.status == BS_MODEL_ERROR      ? kProbeErr
          : r.status == BS_PARAMETER_ERROR  ? kProbeErr
          : (r.status == BS_OK && r.meets_slo) ? kProbePass
                                               : kProbeFail);
}

// Whole-trace simulations (bs_simulate_instance): thread i runs trace i.
__global__ void sim_kernel(DModels m, const double* arrival, const long long* input, const long long* output,
                           const int* identity, const long long* meta, const double* durations, int n, DCand cd,
                           PolicyDev pol, Resident* heaps, int heap_cap, int heap_in_smem, SimOut* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per trace
  if (i >= n) return;
  const long long off = meta[i];
  SimTrace st;
  st.arrival = arrival + off;
  st.input = input + off;
  st.output = output + off;
  st.kept = identity;
  st.n = meta[n + i];
  st.duration_ms = durations[i];
  const SimParams p = make_params(cd, pol, 0);
  SimOut r;
  if (cd.phase == BS_PHASE_PREFILL) {
    if (lane != 0) return;
    r = simulate_prefill(m, st, p);
  } else {
    const WarpScratch ws =
        carve_scratch(smem, warp, heap_cap, heap_in_smem != 0, heaps + static_cast<size_t>(i) * heap_cap);
    r = simulate_decode_warp(m, st, p, ws, heap_cap, lane);
    if (lane != 0) return;
  }
  out[i] = r;
}

// --- host helpers ---------------------------------------------------------------

cudaError_t set_smem_limit(const void* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

const char* model_err_msg(int kind) {
  switch (kind) {
    case 1: return "latency model returned non-positive value";
    case 2: return "power model returned non-positive value";
    default: return "idle model: tp not present";
  }
}

int validate_trace(bs_ctx_t ctx, const bs_trace& t) {  // Trace::validate (workload.hpp:37-49)
  double prev = 0.0;
  for (int64_t i = 0; i < t.n; ++i) {
    const bs_request& r = t.requests[i];
    if (r.arrival_ms < 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "trace: negative arrival");
    if (r.input_len < 1 || r.output_len < 1) return set_error(ctx, BS_PARAMETER_ERROR, "trace: lengths must be >= 1");
    if (r.arrival_ms < prev) return set_error(ctx, BS_PARAMETER_ERROR, "trace: arrivals not sorted");
    prev = r.arrival_ms;
  }
  if (t.n > 0 && t.duration_ms < t.requests[t.n - 1].arrival_ms)
    return set_error(ctx, BS_PARAMETER_ERROR, "trace: duration shorter than last arrival");
  return BS_OK;
}



// Replays the reference's binary search (placement.hpp:180-198) over the
// per-k feasibility outcomes; err_k < 0 until a ModelError is met.
struct SearchResult {
  long long k_star = 0;
  bool saturated = false;
  int model_err = 0;  // nonzero: the ModelError kind the reference would raise
};

SearchResult replay_search(long long k_max, const std::function<int(long long)>& outcome) {
  // outcome(k): 1 feasible, 0 infeasible, -kind ModelError
  SearchResult r;
  if (k_max < 1) return r;
  int f = outcome(k_max);
  if (f < 0) {
    r.model_err = -f;
    return r;
  }
  if (f == 1) {
    r.k_star = k_max;
    r.saturated = true;
    return r;
  }
  f = outcome(1);
  if (f < 0) {
    r.model_err = -f;
    return r;
  }
  if (f == 0) return r;
  long long lo = 1, hi = k_max;
  while (hi - lo > 1) {
    const long long mid = lo + (hi - lo) / 2;
    f = outcome(mid);
    if (f < 0) {
      r.model_err = -f;
      r.k_star = 0;
      return r;
    }
    if (f == 1)
      lo = mid;
    else
      hi = mid;
  }
  r.k_star = lo;
  return r;
}

}  // namespace

extern "C" {

int bs_downsample_keep(bs_ctx_t ctx, const bs_trace* trace, const bs_goodput_search* search, int64_t k,
                       int replicate, int32_t* kept_idx, int64_t* n_kept) {
  if (!ctx || !trace || !search) return set_error(ctx, BS_PARAMETER_ERROR, "bs_downsample_keep: null argument");
  if (trace->n <= 0) {
    *n_kept = 0;
    return BS_OK;
  }
  const double base_rate = trace->duration_ms <= 0.0 ? 0.0
                               : static_cast<double>(trace->n) / (trace->duration_ms / 1000.0);
  // one stream: k' = k, reps = replicate + 1, take stream (k, replicate) by
  // running the kernel over [k, k] via k_max = k and reading stream index.
  MaskParams mp;
  mp.n = trace->n;
  mp.k_max = static_cast<int>(k);
  mp.reps = replicate + 1;
  mp.tol = search->tolerance_rps;
  mp.base_rate = base_rate;
  mp.seed = search->seed;
  const long long streams = static_cast<long long>(mp.k_max) * mp.reps;
  const size_t o_c = ((4ull * streams * mp.n + 255) / 256) * 256, o_p = o_c + ((8ull * streams + 255) / 256) * 256;
  char* base = static_cast<char*>(ctx->dev_buf(kSlotMisc, o_p + 512));
  if (!base) return set_error(ctx, BS_CUDA_ERROR, "downsample: allocation failed");
  int* dk = reinterpret_cast<int*>(base);
  long long* dc = reinterpret_cast<long long*>(base + o_c);
  struct {
    MaskParams mp;
    long long so[2];
    long long ko[1];
  } hp{mp, {0, streams}, {0}};
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(base + o_p, &hp, sizeof hp, cudaMemcpyHostToDevice, ctx->stream));
  const MaskParams* dmp = reinterpret_cast<const MaskParams*>(base + o_p);
  const long long* dso = reinterpret_cast<const long long*>(base + o_p + offsetof(decltype(hp), so));
  const long long* dko = reinterpret_cast<const long long*>(base + o_p + offsetof(decltype(hp), ko));
  mask_kernel<<<static_cast<unsigned>((streams + kMaskWarps - 1) / kMaskWarps), kMaskWarps * 32, 0, ctx->stream>>>(
      dmp, 1, dso, dko, dk, dc);
  BS_LAUNCH_CHECK(ctx);
  const long long s = (k - 1) * mp.reps + replicate;
  long long cnt = 0;
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(&cnt, dc + s, 8, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  BS_CUDA_TRY(ctx, cudaMemcpy(kept_idx, dk + s * mp.n, 4ull * cnt, cudaMemcpyDeviceToHost));
  *n_kept = cnt;
  return BS_OK;
}

static int validate_table_args(bs_ctx_t ctx, const bs_slo* slo, const bs_scheduler_policy* policy,
                               const bs_goodput_search* search, const bs_instance_config* cands, int n_cand) {
  if (n_cand < 1) return set_error(ctx, BS_PARAMETER_ERROR, "config table: no candidates");
  if (slo->ttft_ms <= 0.0 || slo->tpot_ms <= 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "slo: bounds must be > 0");
  if (slo->percentile <= 0.0 || slo->percentile > 1.0)
    return set_error(ctx, BS_PARAMETER_ERROR, "slo: percentile must be in (0,1]");
  if (search->tolerance_rps <= 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "goodput: tolerance must be > 0");
  if (search->probe_count < 1) return set_error(ctx, BS_PARAMETER_ERROR, "goodput: probe_count must be >= 1");
  for (int c = 0; c < n_cand; ++c) {  // InstanceConfig::validate via InstanceSim (simulator.hpp:27-30)
    if (cands[c].tp < 1) return set_error(ctx, BS_PARAMETER_ERROR, "instance: tp must be >= 1");
    if (cands[c].base_freq_mhz <= 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "instance: base_freq_mhz must be > 0");
  }
  if (policy->max_batch_tokens < 1) return set_error(ctx, BS_PARAMETER_ERROR, "scheduler: max_batch_tokens must be >= 1");
  if (policy->max_batch_requests < 1)
    return set_error(ctx, BS_PARAMETER_ERROR, "scheduler: max_batch_requests must be >= 1");
  if (policy->kv_capacity_tokens < 1)
    return set_error(ctx, BS_PARAMETER_ERROR, "scheduler: kv_capacity_tokens must be >= 1");
  return BS_OK;
}

int bs_goodput_table(bs_ctx_t ctx, bs_models_t models, const bs_trace* base, const bs_slo* slo,
                     const bs_scheduler_policy* policy, const bs_goodput_search* search,
                     const bs_instance_config* cands, int n_cand, bs_table_entry* out) {
  return bs_goodput_tables(ctx, models, base, 1, slo, policy, search, cands, n_cand, out);
}

int bs_goodput_tables(bs_ctx_t ctx, bs_models_t models, const bs_trace* bases, int n_tables, const bs_slo* slo,
                      const bs_scheduler_policy* policy, const bs_goodput_search* search,
                      const bs_instance_config* cands, int n_cand, bs_table_entry* out) {
  if (!ctx || !models || !bases || !slo || !policy || !search || (!cands && n_cand > 0) || n_tables < 0 ||
      (n_tables > 0 && !out))
    return set_error(ctx, BS_PARAMETER_ERROR, "bs_goodput_table: null argument");
  if (n_tables == 0) return BS_OK;
  int rc = validate_table_args(ctx, slo, policy, search, cands, n_cand);
  if (rc) return rc;
  for (int t = 0; t < n_tables; ++t) {
    rc = validate_trace(ctx, bases[t]);
    if (rc) return rc;
  }
  const int reps = search->probe_count;
  ctx->last_h2d = 0;
  ctx->last_d2h = 0;

  // per table: Trace::mean_rps (workload.hpp:32-35) and k_max (placement.hpp:161-162)
  std::vector<long long> k_max(n_tables), n_of(n_tables);
  std::vector<double> rate(n_tables);
  std::vector<TableDev> tabs(n_tables);
  std::vector<MaskParams> mps(n_tables);
  long long req_total = 0, stream_total = 0, kept_total = 0, probe_total = 0;
  for (int t = 0; t < n_tables; ++t) {
    const bs_trace& b = bases[t];
    n_of[t] = b.n;
    rate[t] = b.duration_ms <= 0.0 ? 0.0 : static_cast<double>(b.n) / (b.duration_ms / 1000.0);
    k_max[t] = static_cast<long long>(std::floor(rate[t] / search->tolerance_rps));
    for (int c = 0; c < n_cand; ++c) {
      bs_table_entry& e = out[static_cast<size_t>(t) * n_cand + c];
      std::memset(&e, 0, sizeof(bs_table_entry));
      e.config = cands[c];
      e.g_c = cands[c].tp;
    }
    const bool active = k_max[t] >= 1 && b.n > 0;  // otherwise r_c = 0 everywhere
    const long long streams = active ? k_max[t] * reps : 0;
    tabs[t] = TableDev{req_total, b.n, stream_total, kept_total, probe_total, streams, b.duration_ms};
    mps[t] = MaskParams{b.n, static_cast<int>(active ? k_max[t] : 0), reps, search->tolerance_rps, rate[t],
                        search->seed};
    req_total += b.n;
    stream_total += streams;
    kept_total += streams * b.n;
    probe_total += streams * n_cand;
  }
  if (probe_total == 0) return BS_OK;

  // per-candidate safety (no ModelError reachable): grids positive, axes
  // known, idle entry for tp present with at least one point
  std::vector<DCand> hc(n_cand);
  std::vector<int> idle_tp_ok(n_cand, 0);
  {
    std::vector<int> ids(models->dm.idle.n_entries), ns(models->dm.idle.n_entries);
    if (models->dm.idle.n_entries > 0) {
      BS_CUDA_TRY(ctx, cudaMemcpy(ids.data(), models->dm.idle.tp, 4ull * ids.size(), cudaMemcpyDeviceToHost));
      BS_CUDA_TRY(ctx, cudaMemcpy(ns.data(), models->dm.idle.n, 4ull * ns.size(), cudaMemcpyDeviceToHost));
    }
    for (int c = 0; c < n_cand; ++c) {
      for (size_t e = 0; e < ids.size(); ++e)
        if (ids[e] == cands[c].tp) {
          idle_tp_ok[c] = ns[e] >= 1;
          break;
        }
      const int gl = cands[c].phase == BS_PHASE_PREFILL ? 0 : 1;
      const int gp = cands[c].phase == BS_PHASE_PREFILL ? 2 : 3;
      hc[c].phase = cands[c].phase;
      hc[c].tp = cands[c].tp;
      hc[c].freq = cands[c].base_freq_mhz;
      hc[c].safe = models->grid_positive[gl] && models->grid_positive[gp] && !models->dm.grid[gl].bad_axis &&
                   !models->dm.grid[gp].bad_axis && idle_tp_ok[c];
    }
  }
  // decode scratch: at most min(max_batch_requests, n, kv / min_need) residents
  long long heap_cap = 1;
  for (int t = 0; t < n_tables; ++t) {
    if (tabs[t].n_streams == 0) continue;
    long long min_need = INT64_MAX;
    for (long long i = 0; i < bases[t].n; ++i)
      min_need = std::min<long long>(min_need, bases[t].requests[i].input_len + bases[t].requests[i].output_len);
    long long hcap = std::min<long long>(policy->max_batch_requests, bases[t].n);
    hcap = std::min<long long>(hcap, std::max<long long>(1, policy->kv_capacity_tokens / std::max(1LL, min_need)));
    heap_cap = std::max(heap_cap, hcap);
  }
  bool any_decode = false;
  for (int c = 0; c < n_cand; ++c) any_decode |= cands[c].phase == BS_PHASE_DECODE;

  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t o_arr = 0, o_in = up(8ull * req_total), o_out = o_in + up(8ull * req_total);
  const size_t o_cand = o_out + up(8ull * req_total);
  const size_t o_tabs = o_cand + up(sizeof(DCand) * n_cand);
  const size_t o_mps = o_tabs + up(sizeof(TableDev) * n_tables);
  const size_t o_soff = o_mps + up(sizeof(MaskParams) * n_tables);
  const size_t o_koff = o_soff + up(8ull * (n_tables + 1));
  const size_t o_order = o_koff + up(8ull * n_tables);
  const size_t in_bytes = o_order + up(sizeof(ProbeId) * probe_total);
  const size_t o_kept = in_bytes, o_kc = o_kept + up(4ull * kept_total), o_probe = o_kc + up(8ull * stream_total);
  const size_t o_pst = o_probe + up(sizeof(ProbeOut) * probe_total);
  const size_t o_heap = o_pst + up(4ull * probe_total);
  // decode residents live in shared memory when they fit (heap_cap <= 1024, see the launch); global
  // heaps only otherwise
  const size_t heap_rows = any_decode && heap_cap > 1024 ? static_cast<size_t>(probe_total) : 0;
  const size_t total = o_heap + up(sizeof(Resident) * heap_rows * heap_cap);
  char* d = static_cast<char*>(ctx->dev_buf(kSlotWork, total));
  char* h = static_cast<char*>(ctx->host_buf(kSlotWork, in_bytes + sizeof(ProbeOut) * probe_total + 256));
  if (!d || !h) return set_error(ctx, BS_CUDA_ERROR, "config table: allocation of %zu bytes failed", total);
  double* ha = reinterpret_cast<double*>(h + o_arr);
  long long* hi = reinterpret_cast<long long*>(h + o_in);
  long long* ho = reinterpret_cast<long long*>(h + o_out);
  for (int t = 0; t < n_tables; ++t)
    for (long long i = 0; i < bases[t].n; ++i) {
      ha[tabs[t].req_off + i] = bases[t].requests[i].arrival_ms;
      hi[tabs[t].req_off + i] = bases[t].requests[i].input_len;
      ho[tabs[t].req_off + i] = bases[t].requests[i].output_len;
    }
  std::memcpy(h + o_cand, hc.data(), sizeof(DCand) * n_cand);
  std::memcpy(h + o_tabs, tabs.data(), sizeof(TableDev) * n_tables);
  std::memcpy(h + o_mps, mps.data(), sizeof(MaskParams) * n_tables);
  {
    long long* so = reinterpret_cast<long long*>(h + o_soff);
    long long* ko = reinterpret_cast<long long*>(h + o_koff);
    for (int t = 0; t < n_tables; ++t) {
      so[t] = tabs[t].stream_off;
      ko[t] = tabs[t].kept_off;
    }
    so[n_tables] = stream_total;
  }
  {  // launch order, across tables: the levels of max_goodput's search tree (k_max; 1; the midpoints of
     // (1, k_max) level by level), so the probes the search needs start first and the deeper ones run
     // only where the published outcomes still leave them on the path; within a level decode probes
     // (the long ones), higher rate steps first
    ProbeId* po = reinterpret_cast<ProbeId*>(h + o_order);
    std::vector<std::vector<std::pair<int, long long>>> by_depth;  // (table, k)
    for (int t = 0; t < n_tables; ++t) {
      const long long km = tabs[t].n_streams / std::max(1, reps);
      if (km < 1) continue;
      auto put = [&](int depth, long long k) {
        if (static_cast<int>(by_depth.size()) <= depth) by_depth.resize(depth + 1);
        by_depth[depth].push_back({t, k});
      };
      put(0, km);
      if (km > 1) put(1, 1);
      std::vector<std::pair<long long, long long>> lv{{1, km}}, nx;
      for (int depth = 2; !lv.empty(); ++depth) {
        nx.clear();
        for (const auto& iv : lv) {
          if (iv.second - iv.first <= 1) continue;
          const long long mid = iv.first + (iv.second - iv.first) / 2;
          put(depth, mid);
          nx.push_back({iv.first, mid});
          nx.push_back({mid, iv.second});
        }
        lv.swap(nx);
      }
    }
    long long w = 0;
    for (auto& lvl : by_depth) {
      std::stable_sort(lvl.begin(), lvl.end(), [](const auto& a, const auto& b) { return a.second > b.second; });
      for (int pass = 0; pass < 2; ++pass)
        for (const auto& tk : lvl)
          for (int c = 0; c < n_cand; ++c) {
            if ((cands[c].phase == BS_PHASE_DECODE) != (pass == 0)) continue;
            for (int j = 0; j < reps; ++j) po[w++] = ProbeId{tk.first, c, (tk.second - 1) * reps + j};
          }
    }
    if (w != probe_total) return set_error(ctx, BS_CUDA_ERROR, "config table: probe order incomplete");
  }
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->last_h2d = in_bytes;
  TraceDev tr{reinterpret_cast<const double*>(d + o_arr), reinterpret_cast<const long long*>(d + o_in),
              reinterpret_cast<const long long*>(d + o_out), 0.0};
  int* dkept = reinterpret_cast<int*>(d + o_kept);
  long long* dkc = reinterpret_cast<long long*>(d + o_kc);
  cudaEvent_t ev[3];
  for (auto& e : ev) BS_CUDA_TRY(ctx, cudaEventCreate(&e));
  BS_CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));
  mask_kernel<<<static_cast<unsigned>((stream_total + kMaskWarps - 1) / kMaskWarps), kMaskWarps * 32, 0,
                ctx->stream>>>(reinterpret_cast<const MaskParams*>(d + o_mps), n_tables,
                               reinterpret_cast<const long long*>(d + o_soff),
                               reinterpret_cast<const long long*>(d + o_koff), dkept, dkc);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaEventRecord(ev[1], ctx->stream));
  PolicyDev pol{policy->max_batch_tokens, policy->max_batch_requests, policy->kv_capacity_tokens, policy->chunking,
                slo->ttft_ms, slo->tpot_ms};
  ProbeOut* dprobe = reinterpret_cast<ProbeOut*>(d + o_probe);
  Resident* dheap = reinterpret_cast<Resident*>(d + o_heap);
  int* dpst = reinterpret_cast<int*>(d + o_pst);
  BS_CUDA_TRY(ctx, cudaMemsetAsync(dpst, 0, 4ull * probe_total, ctx->stream));
  const bool heap_smem = heap_cap <= 1024;
  const size_t smem4 = 4 * warp_scratch_bytes(static_cast<int>(heap_cap), heap_smem);
  BS_CUDA_TRY(ctx, set_smem_limit(reinterpret_cast<const void*>(probe_kernel), smem4));
  probe_kernel<<<static_cast<unsigned>((probe_total * 32 + 127) / 128), 128, smem4, ctx->stream>>>(
      models->dm, tr, reinterpret_cast<const TableDev*>(d + o_tabs), reinterpret_cast<const DCand*>(d + o_cand),
      dkept, dkc, pol, dheap, static_cast<int>(heap_cap), heap_smem ? 1 : 0,
      reinterpret_cast<const ProbeId*>(d + o_order), probe_total, dprobe, dpst, reps);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaEventRecord(ev[2], ctx->stream));
  ProbeOut* hp = reinterpret_cast<ProbeOut*>(h + in_bytes);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(hp, dprobe, sizeof(ProbeOut) * probe_total, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->last_d2h = sizeof(ProbeOut) * probe_total;
  {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    long long mx = 0, sum = 0, skipped = 0, abandoned = 0;
    for (long long i = 0; i < probe_total; ++i) {
      mx = std::max(mx, hp[i].events);
      sum += hp[i].events;
      if (hp[i].status == kSimAborted) (hp[i].completed < 0 ? skipped : abandoned) += 1;
    }
    ctx->stats[0] = a;
    ctx->stats[1] = b;
    ctx->stats[2] = 0.0;
    ctx->stats[3] = static_cast<double>(mx);
    ctx->stats[4] = static_cast<double>(sum);
    ctx->stats[5] = static_cast<double>(probe_total);
    ctx->stats[6] = static_cast<double>(skipped);
    ctx->stats[7] = static_cast<double>(abandoned);
    ctx->n_stats = 8;
    if (std::getenv("BS_DEBUG_PROBES")) {  // the longest probes (diagnostics)
      std::vector<long long> idx(probe_total);
      for (long long i = 0; i < probe_total; ++i) idx[i] = i;
      std::partial_sort(idx.begin(), idx.begin() + std::min<long long>(8, probe_total), idx.end(),
                        [&](long long a, long long b) { return hp[a].ns > hp[b].ns; });
      double ns_ph[2] = {0.0, 0.0};
      long long n_ph[2] = {0, 0};
      for (long long i = 0; i < probe_total; ++i) {
        int t = 0;
        while (t + 1 < n_tables && tabs[t + 1].probe_off <= i) ++t;
        const long long c = (i - tabs[t].probe_off) / tabs[t].n_streams;
        const int ph = cands[c].phase == BS_PHASE_PREFILL ? 0 : 1;
        if (hp[i].ns > 0) {
          ns_ph[ph] += static_cast<double>(hp[i].ns);
          ++n_ph[ph];
        }
      }
      std::fprintf(stderr, "probes run: prefill %lld (%.1f ms total), decode %lld (%.1f ms total)\n", n_ph[0],
                   ns_ph[0] / 1e6, n_ph[1], ns_ph[1] / 1e6);
      for (long long q = 0; q < std::min<long long>(8, probe_total); ++q) {
        const long long i = idx[q];
        int t = 0;
        while (t + 1 < n_tables && tabs[t + 1].probe_off <= i) ++t;
        const long long rel = i - tabs[t].probe_off, c = rel / tabs[t].n_streams, st = rel % tabs[t].n_streams;
        std::fprintf(stderr, "probe t%d c%lld (phase %d tp %d f %.0f) k %lld: %.1f ms, %lld events, status %d meets %d\n",
                     t, c, cands[c].phase, cands[c].tp, cands[c].base_freq_mhz, st / std::max(1, reps) + 1,
                     hp[i].ns / 1e6, hp[i].events, hp[i].status, hp[i].meets);
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }

  for (int t = 0; t < n_tables; ++t) {
    const TableDev& tb = tabs[t];
    if (tb.n_streams == 0) continue;
    const ProbeOut* hpt = hp + tb.probe_off;
    bs_table_entry* ot = out + static_cast<size_t>(t) * n_cand;
    // replay each candidate's search; feasible(k) = every replicate passes
    // (empty probes pass, SimulationError fails, ModelError propagates)
    for (int c = 0; c < n_cand; ++c) {
      auto outcome = [&](long long k) -> int {
        for (int j = 0; j < reps; ++j) {
          const ProbeOut& p = hpt[static_cast<size_t>(c) * tb.n_streams + (k - 1) * reps + j];
          if (p.status == kSimAborted) return -101;  // the path never leaves the probes that ran
          if (p.empty) continue;
          if (p.status == BS_MODEL_ERROR) return -p.model_err;
          if (p.status == BS_PARAMETER_ERROR) return -100;
          if (p.status != BS_OK || !p.meets) return 0;
        }
        return 1;
      };
      const SearchResult sr = replay_search(k_max[t], outcome);
      if (sr.model_err == 100) return set_error(ctx, BS_CUDA_ERROR, "config table: device resident scratch too small");
      if (sr.model_err == 101) return set_error(ctx, BS_CUDA_ERROR, "config table: search path reached a pruned probe");
      if (sr.model_err) {
        ot[c].error_code = BS_MODEL_ERROR;
        std::snprintf(ot[c].error, sizeof ot[c].error, "%s", model_err_msg(sr.model_err));
        if (sr.model_err == 3)
          std::snprintf(ot[c].error, sizeof ot[c].error, "idle model: tp %d not present", cands[c].tp);
        continue;
      }
      ot[c].k_star = sr.k_star;
      ot[c].r_c = static_cast<double>(sr.k_star) * search->tolerance_rps;  // placement.hpp:182, 197
      ot[c].saturated = sr.saturated ? 1 : 0;
      if (ot[c].r_c <= 0.0) continue;
      // E_c at (k*, replicate 0) (placement.hpp:227-231): that probe passed, so it never stopped early
      // and its run is exactly simulate_instance on the same probe trace -- reuse its energy accounting.
      // An empty probe trace only records the idle span [0, duration] (simulator.hpp:731-733).
      const ProbeOut& e = hpt[static_cast<size_t>(c) * tb.n_streams + (sr.k_star - 1) * reps];
      if (e.empty) {
        if (!idle_tp_ok[c]) {  // evaluate_candidate's catch (placement.hpp:233-236): r_c = 0, saturated kept
          ot[c].error_code = BS_MODEL_ERROR;
          ot[c].r_c = 0.0;
          std::snprintf(ot[c].error, sizeof ot[c].error, "idle model: tp %d not present", cands[c].tp);
        } else {
          ot[c].error_code = -1;
          std::snprintf(ot[c].error, sizeof ot[c].error, "no completed request at R_c");
        }
        continue;
      }
      if (e.status != BS_OK || !e.meets) return set_error(ctx, BS_CUDA_ERROR, "config table: inconsistent probe at k*");
      // energy_per_request (placement.hpp:205-213)
      if (e.completed < 1) {
        ot[c].error_code = -1;
        std::snprintf(ot[c].error, sizeof ot[c].error, "no completed request at R_c");
        continue;
      }
      double en = e.busy_j;
      if (cands[c].phase == BS_PHASE_PREFILL) en = en + e.idle_j;
      ot[c].e_c = en / static_cast<double>(e.completed);
      ot[c].has_e_c = 1;
    }
  }
  return BS_OK;
}

int bs_simulate_instance(bs_ctx_t ctx, bs_models_t models, const bs_trace* traces, int n,
                         const bs_instance_config* cfg, const bs_scheduler_policy* policy, const bs_slo* slo,
                         bs_sim_summary* out) {
  if (!ctx || !models || (!traces && n > 0) || !cfg || !policy || !slo || !out)
    return set_error(ctx, BS_PARAMETER_ERROR, "bs_simulate_instance: null argument");
  if (n <= 0) return BS_OK;
  if (cfg->tp < 1) return set_error(ctx, BS_PARAMETER_ERROR, "instance: tp must be >= 1");
  if (cfg->base_freq_mhz <= 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "instance: base_freq_mhz must be > 0");
  long long total = 0, max_n = 1, min_need = INT64_MAX;
  for (int i = 0; i < n; ++i) {
    int rc = validate_trace(ctx, traces[i]);
    if (rc) return rc;
    total += traces[i].n;
    max_n = std::max<long long>(max_n, traces[i].n);
    for (int64_t r = 0; r < traces[i].n; ++r)
      min_need = std::min<long long>(min_need, traces[i].requests[r].input_len + traces[i].requests[r].output_len);
  }
  long long heap_cap = std::min<long long>(policy->max_batch_requests, max_n);
  if (min_need != INT64_MAX)
    heap_cap = std::min<long long>(heap_cap, std::max<long long>(1, policy->kv_capacity_tokens / std::max(1LL, min_need)));
  heap_cap = std::max<long long>(heap_cap, 1);
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t o_arr = 0, o_in = up(8ull * total + 8), o_out = o_in + up(8ull * total + 8);
  const size_t o_idx = o_out + up(8ull * total + 8), o_meta = o_idx + up(4ull * max_n);
  const size_t in_bytes = o_meta + up(sizeof(long long) * 2 * n + sizeof(double) * n);
  const size_t o_heap = in_bytes, o_res = o_heap + up(sizeof(Resident) * heap_cap * n);
  const size_t all = o_res + up(sizeof(SimOut) * n);
  char* d = static_cast<char*>(ctx->dev_buf(kSlotWork, all));
  char* h = static_cast<char*>(ctx->host_buf(kSlotWork, all));
  if (!d || !h) return set_error(ctx, BS_CUDA_ERROR, "simulate_instance: allocation failed");
  double* ha = reinterpret_cast<double*>(h + o_arr);
  long long* hi = reinterpret_cast<long long*>(h + o_in);
  long long* ho = reinterpret_cast<long long*>(h + o_out);
  int* hx = reinterpret_cast<int*>(h + o_idx);
  long long* hm = reinterpret_cast<long long*>(h + o_meta);  // offsets[n], counts[n]
  double* hd = reinterpret_cast<double*>(h + o_meta + sizeof(long long) * 2 * n);
  long long off = 0;
  for (int i = 0; i < n; ++i) {
    hm[i] = off;
    hm[n + i] = traces[i].n;
    hd[i] = traces[i].duration_ms;
    for (int64_t r = 0; r < traces[i].n; ++r) {
      ha[off + r] = traces[i].requests[r].arrival_ms;
      hi[off + r] = traces[i].requests[r].input_len;
      ho[off + r] = traces[i].requests[r].output_len;
    }
    off += traces[i].n;
  }
  for (long long r = 0; r < max_n; ++r) hx[r] = static_cast<int>(r);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  DCand cd{cfg->phase, cfg->tp, cfg->base_freq_mhz, 0};
  PolicyDev pol{policy->max_batch_tokens, policy->max_batch_requests, policy->kv_capacity_tokens, policy->chunking,
                slo->ttft_ms, slo->tpot_ms};
  const bool heap_smem = heap_cap <= 1024;
  const size_t smem4 = 4 * warp_scratch_bytes(static_cast<int>(heap_cap), heap_smem);
  BS_CUDA_TRY(ctx, set_smem_limit(reinterpret_cast<const void*>(sim_kernel), smem4));
  sim_kernel<<<(n * 32 + 127) / 128, 128, smem4, ctx->stream>>>(
      models->dm, reinterpret_cast<const double*>(d + o_arr), reinterpret_cast<const long long*>(d + o_in),
      reinterpret_cast<const long long*>(d + o_out), reinterpret_cast<const int*>(d + o_idx),
      reinterpret_cast<const long long*>(d + o_meta), reinterpret_cast<const double*>(d + o_meta + sizeof(long long) * 2 * n),
      n, cd, pol, reinterpret_cast<Resident*>(d + o_heap), static_cast<int>(heap_cap), heap_smem ? 1 : 0,
      reinterpret_cast<SimOut*>(d + o_res));
  BS_LAUNCH_CHECK(ctx);
  const SimOut* hr = reinterpret_cast<const SimOut*>(h + o_res);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(h + o_res, d + o_res, sizeof(SimOut) * n, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; ++i) {
    out[i].status = hr[i].status;
    out[i].meets_slo = hr[i].status == BS_OK ? hr[i].meets_slo : 0;
    out[i].completed = hr[i].completed;
    out[i].busy_energy_j = hr[i].busy_j;
    out[i].idle_energy_j = hr[i].idle_j;
    out[i].horizon_ms = hr[i].horizon_ms;
  }
  return BS_OK;
}

}  // extern "C"

// bs_mpc.cu — prefill MPC on sm_100a: projection, (k, f) tables, the
// exhaustive rollout (prefix compaction + leaf sweep + 128-bit argmin) and
// the greedy level search.  Reference: proj/include/pdsim/dvfs.hpp.
//
// Data flow for one batch of decisions (all on one stream, no host sync
// until the final copy-out):
//   prepare_kernel   1 CTA / problem: project_batches (dvfs.hpp:63-100) by
//                    one thread, then the K x N (lat, pow) tables by all
//                    threads through the bit-exact interpolator; resets the
//                    argmin slot and expands the first three levels (N^2
//                    prefixes, then their passing children) straight into
//                    the depth-3 list.
//   bfs_node_kernel  x (max depth of final nodes - 2): level-synchronous
//                    expansion of every feasible prefix of every decision,
//                    one thread per node (its passing children are a sorted
//                    prefix), compacted with block-aggregated appends
//                    (meets_slo fails at the first violated batch, so
//                    violated prefixes have no feasible completion and are
//                    dropped for good).
//   sweep_kernel     one thread per final node sweeps its bottom 2 (or 3)
//                    levels in increasing code order with a division-free
//                    objective filter; (objective, code) minima merge
//                    through a 128-bit CAS.  See bs_exhaustive.cuh.
//   finalize_kernel  1 thread / problem: decode the argmin code.
#include <algorithm>
#include <cstddef>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include <cooperative_groups.h>

#include "bs_internal.h"
#include "bs_sim.cuh"

using namespace bs;

namespace {

constexpr int kPrepThreads = 128;  // K x N <= 128 table entries in one pass; 4 CTAs / SM
constexpr double kFilterScale = 1.0 + 0x1p-50;  // C in the filter bound
constexpr double kFilterMinBest = 0x1p-100;
constexpr double kFilterMinDen = 0x1p-900;

#include "bs_mpc_core.cuh"
#include "bs_greedy_warp.cuh"

#include "bs_exhaustive.cuh"

__global__ void finalize_kernel(const DTables* __restrict__ tables, const DMpcCfg* cfgs, const DProblem* probs,
                                const Key128* best, const unsigned long long* feas, DMpcOut* out, int n, DSlice sl) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the sweep's results (programmatic dependent launch)
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const DTables* T = &tables[d];
  DMpcOut o;
  memset(&o, 0, sizeof o);
  o.status = T->status;
  o.K = T->K;
  if (o.status == BS_OK && T->K > 0) {
    const int K = T->K, nc = T->nc;
    o.feasible_count = feas[d];
    o.eval_count = static_cast<long long>(slice_size(sl, K, nc));  // nc^K unsliced
    if (best[d].obj != ~0ull) {
      o.feasible = 1;
      o.objective = __longlong_as_double(static_cast<long long>(best[d].obj));
      unsigned long long code = best[d].code;
      o.best_code = code;
      // code / nc by a multiply-high with ceil(2^64 / nc): exact for codes < 2^58
      const unsigned long long M = nc > 1 ? ~0ull / static_cast<unsigned>(nc) + 1 : 0ull;
      for (int k = K - 1; k >= 0; --k) {
        const unsigned long long q = nc == 1 ? code : code < (1ull << 58) ? __umul64hi(code, M) : code / nc;
        o.idx[k] = static_cast<unsigned char>(code - q * static_cast<unsigned long long>(nc));
        code = q;
      }
    } else {  // nothing feasible: all-max and its objective
      o.feasible = 0;
      double num = 0.0, den = 0.0;
      unsigned long long code = 0;
      for (int k = 0; k < K; ++k) {
        o.idx[k] = static_cast<unsigned char>(nc - 1);
        num = __dadd_rn(num, T->E[k][nc - 1]);
        den = __dadd_rn(den, T->A[k][nc - 1]);
        code = code * nc + (nc - 1);
      }
      o.best_code = code;
      o.objective = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
    }
  } else if (o.status == BS_OK) {
    o.feasible = 1;
  }
  out[d] = o;
  (void)cfgs;
  (void)probs;
}

// ---------------------------------------------------------------------------
// greedy_freq_select (dvfs.hpp:185-259): one CTA per decision.
// ---------------------------------------------------------------------------
// One warp per decision (greedy_warp, bs_greedy_warp.cuh): per-warp
// dynamic shared memory holds the greedy state, the result and the compact
// (k, f) tables.
constexpr int kGreedyWarps = 4;

__host__ __device__ inline size_t greedy_warp_bytes(int max_h, int max_nc) {
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  return a16(sizeof(WGreedyShared)) + a16(sizeof(DMpcOut)) + a16(8 * wtable_doubles(max_h, max_nc));
}

__global__ void __launch_bounds__(kGreedyWarps * 32) greedy_kernel(DModels m, const DMpcCfg* cfgs,
                                                                  const DProblem* probs, const DWaiting* W,
                                                                  const DRunning* R, DMpcOut* out, DLevel* levels,
                                                                  int n, int max_h, int max_nc, const DFastPair* fg,
                                                                  int lv_stride) {
  extern __shared__ __align__(16) unsigned char gdsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int d = blockIdx.x * kGreedyWarps + wib;
  if (d >= n) return;
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  unsigned char* base = gdsm + static_cast<size_t>(wib) * greedy_warp_bytes(max_h, max_nc);
  WGreedyShared& S = *reinterpret_cast<WGreedyShared*>(base);
  DMpcOut* o = reinterpret_cast<DMpcOut*>(base + a16(sizeof(WGreedyShared)));
  double* tab = reinterpret_cast<double*>(base + a16(sizeof(WGreedyShared)) + a16(sizeof(DMpcOut)));
  const DProblem pr = probs[d];
  const DMpcCfg& c = cfgs[pr.cfg];
  if (lane == 0) wtables_bind(S.T, tab, c.horizon, c.nc);
  __syncwarp();
  const DFastPair* fp = fg ? fg + pr.fgi : nullptr;
  greedy_warp(m, pr, c, W + pr.wait_off, R + pr.run_off, S, o, levels + static_cast<size_t>(d) * lv_stride,
              fp ? fp->lat : nullptr, fp ? fp->pw : nullptr, fp && fp->share);
  if (lane == 0) out[d] = *o;
}

// One decision per CTA of NW warps (greedy_coop): batches too small to fill
// the GPU one warp per decision give each decision more warps, down to a
// single controller call (n = 1) spread over 16 warps.
template <int NW>
__global__ void __launch_bounds__(32 * NW) greedy_coop_kernel(DModels m, const DMpcCfg* cfgs, const DProblem* probs,
                                                             const DWaiting* W, const DRunning* R, DMpcOut* out,
                                                             DLevel* levels, int n, int max_h, int max_nc,
                                                             const DFastPair* fg, int lv_stride) {
  extern __shared__ __align__(16) unsigned char gdsm[];
  const int d = blockIdx.x;
  if (d >= n) return;
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  WGreedyShared& S = *reinterpret_cast<WGreedyShared*>(gdsm);
  DMpcOut* o = reinterpret_cast<DMpcOut*>(gdsm + a16(sizeof(WGreedyShared)));
  double* tab = reinterpret_cast<double*>(gdsm + a16(sizeof(WGreedyShared)) + a16(sizeof(DMpcOut)));
  const DProblem pr = probs[d];
  const DMpcCfg& c = cfgs[pr.cfg];
  if (threadIdx.x == 0) wtables_bind(S.T, tab, c.horizon, c.nc);
  __syncthreads();
  const DFastPair* fp = fg ? fg + pr.fgi : nullptr;
  greedy_coop<NW>(m, pr, c, W + pr.wait_off, R + pr.run_off, S, o, levels + static_cast<size_t>(d) * lv_stride,
                  fp ? fp->lat : nullptr, fp ? fp->pw : nullptr, fp && fp->share);
  if (threadIdx.x == 0) out[d] = *o;
}

// One decision per thread-block cluster of CL CTAs of NW warps (one CTA per
// SM): the latency of a single controller call, a level's mutations spread
// over CL SMs (greedy_coop<NW, CL>).
constexpr int kGreedyCluster = 8;

template <int NW, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(32 * NW)
    greedy_cluster_kernel(DModels m, const DMpcCfg* cfgs, const DProblem* probs, const DWaiting* W,
                          const DRunning* R, DMpcOut* out, DLevel* levels, int n, int max_h, int max_nc,
                          const DFastPair* fg, int lv_stride) {
  extern __shared__ __align__(16) unsigned char gdsm[];
  const int d = blockIdx.x / CL;  // uniform over the cluster (the grid is n x CL)
  const int rank = static_cast<int>(cooperative_groups::this_cluster().block_rank());
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  WGreedyShared& S = *reinterpret_cast<WGreedyShared*>(gdsm);
  DMpcOut* o = reinterpret_cast<DMpcOut*>(gdsm + a16(sizeof(WGreedyShared)));
  double* tab = reinterpret_cast<double*>(gdsm + a16(sizeof(WGreedyShared)) + a16(sizeof(DMpcOut)));
  if (d < n) {
    const DProblem pr = probs[d];
    const DMpcCfg& c = cfgs[pr.cfg];
    if (threadIdx.x == 0) wtables_bind(S.T, tab, c.horizon, c.nc);
    __syncthreads();
    const DFastPair* fp = fg ? fg + pr.fgi : nullptr;
    greedy_coop<NW, CL>(m, pr, c, W + pr.wait_off, R + pr.run_off, S, o,
                        levels + static_cast<size_t>(d) * lv_stride, fp ? fp->lat : nullptr, fp ? fp->pw : nullptr,
                        fp && fp->share);
    if (threadIdx.x == 0 && rank == 0) out[d] = *o;
  }
  cooperative_groups::this_cluster().sync();  // no CTA leaves while another may read its shared memory
}

// ---------------------------------------------------------------------------
// parity probes
// ---------------------------------------------------------------------------
__global__ void tables_only_kernel(DModels m, const DMpcCfg* cfgs, const DProblem* probs, const DWaiting* W,
                                   const DRunning* R, DTables* tables) {
  __shared__ int s_status;
  const DProblem pr = probs[blockIdx.x];
  build_tables(m, pr, cfgs[pr.cfg], W + pr.wait_off, R + pr.run_off, &tables[blockIdx.x], &s_status);
  if (threadIdx.x == 0) tables[blockIdx.x].status = s_status;
}

__global__ void eval_codes_kernel(const DTables* T, const DMpcCfg* cfgs, const DProblem* probs,
                                  const unsigned long long* codes, int n, int32_t* feas, double* obj) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const DProblem pr = probs[0];
  const DMpcCfg& c = cfgs[pr.cfg];
  unsigned char idx[kMaxK];
  unsigned long long code = codes[i];
  for (int k = T->K - 1; k >= 0; --k) {
    idx[k] = static_cast<unsigned char>(code % c.nc);
    code /= c.nc;
  }
  double o = 0.0;
  int err;
  const int ok = eval_assignment(*T, pr, c, idx, &o, &err);
  feas[i] = ok;
  obj[i] = tw_objective(*T, idx);
}

__global__ void project_kernel(const DMpcCfg* cfgs, const DProblem* probs, const DWaiting* W, const DRunning* R,
                               DTables* tables, int n) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const DProblem pr = probs[d];
  tables[d].status = project_dev(pr, cfgs[pr.cfg], W + pr.wait_off, R + pr.run_off, &tables[d]);
}

// ---------------------------------------------------------------------------
// host glue
// ---------------------------------------------------------------------------

void expand_result(const DMpcOut& o, const DLevel* lv, const DMpcCfg& c, double target_freq, bs_mpc_result* r,
                   bool exhaustive) {
  // everything before the level list; levels[n_levels..) are not written
  // (GreedyResult::levels has n_levels entries, dvfs.hpp:133-139)
  std::memset(r, 0, offsetof(bs_mpc_result, levels));
  r->status = o.status;
  r->K = o.K;
  if (o.status != BS_OK) {
    r->n_levels = o.n_levels;  // carries the ModelError kind for the message
    return;
  }
  r->feasible = o.feasible;
  r->eval_count = o.eval_count;
  r->objective_w = o.objective;
  r->feasible_count = o.feasible_count;
  r->best_code = o.best_code;
  if (exhaustive && o.K > 0) r->trajectories = static_cast<uint64_t>(o.eval_count);
  for (int k = 0; k < o.K; ++k) {
    r->freq_index[k] = o.idx[k];
    r->freqs_mhz[k] = c.cand[o.idx[k]];
  }
  if (lv) {
    r->n_levels = o.n_levels;
    for (int l = 0; l < o.n_levels; ++l) {
      r->levels[l].level = l + 1;
      r->levels[l].k_prime = lv[l].k_prime;
      r->levels[l].replaced_mhz = lv[l].replaced_mhz;
      r->levels[l].mutations = lv[l].mutations;
      r->levels[l].feasible_mutations = lv[l].feasible_mutations;
      r->levels[l].accepted = lv[l].accepted;
    }
  }
  // PrefillMpcController::run (dvfs.hpp:328-329)
  r->decision_freq_mhz = o.K == 0 ? (target_freq > 0 ? target_freq : c.max_mhz) : r->freqs_mhz[0];
}

int report_status(bs_ctx_t ctx, const bs_mpc_result* out, int n) {
  for (int i = 0; i < n; ++i) {
    if (out[i].status == BS_OK) continue;
    switch (out[i].status) {
      case BS_SIMULATION_ERROR:
        return set_error(ctx, BS_SIMULATION_ERROR, "scheduler: queued request with no remaining tokens");
      case BS_MODEL_ERROR:
        return set_error(ctx, BS_MODEL_ERROR, "%s model returned non-positive value",
                         out[i].n_levels == -2 ? "power" : "latency");
      default:
        return set_error(ctx, out[i].status, "mpc: problem %d failed with status %d", i, out[i].status);
    }
  }
  return BS_OK;
}

enum Mode { kExhaustive = 0, kGreedy = 1 };
constexpr int kOverflowStatus = BS_CUDA_ERROR + 1;  // internal: frontier capacity exceeded
constexpr int kNumEvents = 6;  // exhaustive phases: prepare, seed, bfs, sweep, finalize

// One batch of MPC decisions resident in HBM: packed problems, scratch, and
// results.  Used by the one-shot entry points (buffers borrowed from the
// context) and by bs_mpc_plan (buffers owned by the plan).
struct MpcRun {
  int mode = kExhaustive;
  int n = 0;
  PackedProblems pk;
  std::vector<DMpcCfg> hc;          // host copy of configurations
  std::vector<int> cfg_of;          // per-problem configuration index
  std::vector<double> target;       // per-problem target_freq (controller fallback)
  int max_nc = 1;                   // largest candidate count in the batch
  int lv_stride = BS_MAX_LEVELS;    // greedy level records per problem: max(1, max_nc - 2) (dvfs.hpp:205)
  int bfs_levels = 0;               // deepest final-node depth over the batch
  unsigned long long cap_level = 0;  // BFS list capacity (per ping-pong buffer)
  unsigned long long cap_final = 0;  // final list capacity
  DTables* dT = nullptr;
  DThr* dThr = nullptr;  // leaf-count thresholds per decision (exhaustive)
  int* dThrList = nullptr;  // decisions that need them (prepare_kernel -> thr_kernel)
  ExCtl* dCtl = nullptr;
  Key128* dBest = nullptr;
  unsigned long long* dFeas = nullptr;
  void* dLev[2] = {nullptr, nullptr};
  void* dFin = nullptr;
  DMpcOut* dOut = nullptr;
  DLevel* dLv = nullptr;
  int bfs_grid = 0, sweep_grid2 = 0, sweep_grid3 = 0;
  bool sweep3 = false;  // some decision may sweep three levels (sweep_levels)
  double sweep3_min = BS_SWEEP3_MIN;  // the context's threshold (bs_ctx_set_exhaustive_limits)
  DSlice slice{};                     // the code-space slice of every decision (digits 0: whole trees)
  ExCtl ctl_host{};  // counters of an overflowed run (exact totals of the levels before the first overflow)
  const DFastPair* dFG = nullptr;       // reduced grids per (configuration, tp) pair (pk.fg_pairs)
  std::vector<DFastPair> hFG;           // their host build
  cudaEvent_t ev[kNumEvents] = {};
  bool have_events = false;
  bool contig = false;  // dLv = dOut + levels_off(n) (greedy one-shot)
};

size_t up256(size_t x) { return (x + 255) / 256 * 256; }
size_t tables_bytes(int n) { return sizeof(DTables) * static_cast<size_t>(n); }
size_t best_bytes(int n) { return (sizeof(Key128) + 8ull) * static_cast<size_t>(n); }
size_t out_bytes(int n) { return sizeof(DMpcOut) * static_cast<size_t>(n); }
size_t levels_bytes(int n, int stride) { return sizeof(DLevel) * static_cast<size_t>(stride) * static_cast<size_t>(n); }
// greedy one-shot results: [out | overflow flag | levels], device and host alike
size_t levels_off(int n) { return (out_bytes(n) + 64 + 255) / 256 * 256; }
size_t result_region(int n, int stride) { return levels_off(n) + levels_bytes(n, stride); }

// Device scratch layout of an exhaustive run (offsets from one base).
struct ExLayout {
  size_t tables = 0, thr = 0, thr_list = 0, ctl = 0, best = 0, lev0 = 0, lev1 = 0, fin = 0, out = 0, total = 0;
};

ExLayout ex_layout(const MpcRun& r, size_t start) {
  ExLayout L;
  size_t o = start;
  L.tables = o;
  o += up256(tables_bytes(r.n));
  L.thr = o;
  o += up256(sizeof(DThr) * static_cast<size_t>(r.n));
  L.thr_list = o;
  o += up256(4ull * static_cast<size_t>(r.n));
  L.ctl = o;
  o += up256(sizeof(ExCtl));
  L.best = o;
  o += up256(best_bytes(r.n));
  L.lev0 = o;
  o += up256(frontier_bytes(r.cap_level));
  L.lev1 = o;
  o += up256(frontier_bytes(r.cap_level));
  L.fin = o;
  o += up256(final_bytes(r.cap_final));
  L.out = o;
  o += up256(out_bytes(r.n));
  L.total = o;
  return L;
}

void bind_exhaustive(MpcRun* r, char* base, const ExLayout& L) {
  r->dT = reinterpret_cast<DTables*>(base + L.tables);
  r->dThr = reinterpret_cast<DThr*>(base + L.thr);
  r->dThrList = reinterpret_cast<int*>(base + L.thr_list);
  r->dCtl = reinterpret_cast<ExCtl*>(base + L.ctl);
  r->dBest = reinterpret_cast<Key128*>(base + L.best);
  r->dFeas = reinterpret_cast<unsigned long long*>(r->dBest + r->n);
  r->dLev[0] = base + L.lev0;
  r->dLev[1] = base + L.lev1;
  r->dFin = base + L.fin;
  r->dOut = reinterpret_cast<DMpcOut*>(base + L.out);
}

constexpr size_t kMaxExhaustiveScratch = 48ull << 30;

// Packs the problems (one H2D copy), validates configurations and sizes the
// exhaustive frontiers from the horizons (K <= horizon_K).
// Frontier capacities: the worst case (every prefix feasible), clamped to a
// scratch budget; a run whose appends overflow is re-run with capacities
// from the observed counts, or split (one_shot).
// (defaults of the context's limits, bs_ctx_s::ex_final_cap / ex_level_cap)

int run_pack(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies, int n_cfgs,
             const bs_mpc_problem* problems, int n, int mode, MpcRun* run, unsigned long long cap_level_hint = 0,
             unsigned long long cap_final_hint = 0) {
  run->mode = mode;
  run->n = n;
  run->sweep3_min = ctx->ex_sweep3_min;
  if (n > (1 << 24)) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: at most 2^24 problems per call");
  int rc = pack_problems(ctx, cfgs, policies, n_cfgs, problems, n, &run->pk);
  if (rc) return rc;
  run->hc.resize(n_cfgs);
  for (int c = 0; c < n_cfgs; ++c) {
    rc = pack_mpc_cfg(ctx, cfgs[c], policies[c], &run->hc[c]);
    if (rc) return rc;
    if (mode == kExhaustive) {
      double space = 1.0;
      for (int k = 0; k < run->hc[c].horizon; ++k) space *= run->hc[c].nc;
      if (space >= 4.0e18)
        return set_error(ctx, BS_PARAMETER_ERROR, "mpc exhaustive: %d^%d trajectories exceed the 2^62 code space",
                         run->hc[c].nc, run->hc[c].horizon);
    }
  }
  run->max_nc = 1;
  for (const DMpcCfg& c : run->hc) run->max_nc = std::max(run->max_nc, c.nc);
  run->lv_stride = std::min(BS_MAX_LEVELS, std::max(1, run->max_nc - 2));
  run->cfg_of.resize(n);
  run->target.resize(n);
  run->cap_level = 0;
  run->cap_final = 0;
  run->bfs_levels = 0;
  run->sweep3 = false;
  for (int i = 0; i < n; ++i) {
    run->cfg_of[i] = problems[i].cfg_index;
    run->target[i] = problems[i].snap.target_freq_mhz;
    if (mode != kExhaustive) continue;
    const DMpcCfg& c = run->hc[problems[i].cfg_index];
    const int FD = c.horizon - sweep_levels(c.horizon, c.nc, ctx->ex_sweep3_min);
    run->bfs_levels = std::max(run->bfs_levels, FD);
    // a shorter projection (K < horizon) may take three levels where the horizon takes two
    for (int K = 3; K <= c.horizon; ++K)
      if (sweep_levels(K, c.nc, ctx->ex_sweep3_min) == 3) run->sweep3 = true;
    run->cap_final += ipow(static_cast<unsigned long long>(c.nc), FD);
    run->cap_level += ipow(static_cast<unsigned long long>(c.nc), FD > 0 ? FD - 1 : 0);
  }
  if (mode == kExhaustive) {
    if (cap_level_hint) run->cap_level = std::min(run->cap_level, cap_level_hint);
    if (cap_final_hint) run->cap_final = std::min(run->cap_final, cap_final_hint);
    run->cap_level = std::min(run->cap_level, ctx->ex_level_cap);
    run->cap_final = std::min(run->cap_final, ctx->ex_final_cap);
    run->cap_level = std::max<unsigned long long>(run->cap_level, static_cast<unsigned long long>(n));
    run->cap_final = std::max<unsigned long long>(run->cap_final, static_cast<unsigned long long>(n));
    const ExLayout L = ex_layout(*run, 0);
    if (L.total > kMaxExhaustiveScratch)
      return set_error(ctx, BS_PARAMETER_ERROR,
                       "mpc exhaustive: batch needs %.1f GB of frontier scratch; split it into smaller calls",
                       L.total / 1e9);
  }
  return BS_OK;
}

// The reduced grids of every (configuration, tp) pair of a packed batch,
// built on the host from the models' mirror (fast_grid2) with device
// pointers; copied into `dst` (device) on the context stream.
int upload_fast_pairs(bs_ctx_t ctx, bs_models_t models, MpcRun* run, DFastPair* dst) {
  const auto& pairs = run->pk.fg_pairs;
  run->hFG.assign(pairs.size(), DFastPair{});
  for (size_t p = 0; p < pairs.size(); ++p) {
    const DMpcCfg& c = run->hc[pairs[p].first];
    const int tp = pairs[p].second;
    DFastPair& fp = run->hFG[p];
    std::memset(&fp, 0, sizeof fp);
    fp.share = 1;
    for (int f = 0; f < c.nc; ++f) {
      fp.lat[f] = fast_grid2(models->hgrid[0], models->dm.grid[0], tp, c.cand[f]);
      fp.pw[f] = fast_grid2(models->hgrid[2], models->dm.grid[2], tp, c.cand[f]);
      if (!fast_same_brackets(fp.lat[0], fp.lat[f]) || !fast_same_brackets(fp.pw[0], fp.pw[f])) fp.share = 0;
    }
  }
  if (!pairs.empty()) {  // staged through pinned memory: an asynchronous copy
    const size_t bytes = sizeof(DFastPair) * pairs.size();
    void* h = ctx->host_buf(kSlotFastGrids, bytes);
    if (!h) return set_error(ctx, BS_CUDA_ERROR, "mpc: pinned staging of the reduced grids failed");
    std::memcpy(h, run->hFG.data(), bytes);
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(dst, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  run->dFG = pairs.empty() ? nullptr : dst;
  return BS_OK;
}

#define BS_REC(i)                                                         \
  do {                                                                    \
    if (timing) BS_CUDA_TRY(ctx, cudaEventRecord(run->ev[i], ctx->stream)); \
  } while (0)

int grid_for(bs_ctx_t ctx, const void* kernel, int threads) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1) b = 1;
  return ctx->sm_count * b;
}

// A launch with programmatic stream serialization (the kernel calls
// griddepcontrol.wait before reading its predecessor's results).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Enqueues the kernels of one run on the context stream (no host sync).
int run_enqueue(bs_ctx_t ctx, bs_models_t models, MpcRun* run, bool timing) {
  const int n = run->n;
  if (n == 0) return BS_OK;
  const PackedProblems& pk = run->pk;
  if (timing && !run->have_events) {
    for (auto& e : run->ev) BS_CUDA_TRY(ctx, cudaEventCreate(&e));
    run->have_events = true;
  }
  BS_REC(0);
  if (run->mode == kGreedy) {
    // warps per decision: one, unless the batch leaves the GPU's warp slots
    // (16 per SM here) idle -- then up to 16 per decision (one per CTA)
    const long long slots = 16ll * ctx->sm_count;
    int nw = 1;
    while (nw < 16 && static_cast<long long>(n) * nw * 2 <= slots) nw *= 2;
    const size_t one = greedy_warp_bytes(pk.max_horizon, pk.max_nc);
    if (nw == 1) {
      const size_t smem = kGreedyWarps * one;
      if (smem > ctx->greedy_smem[0]) {
        BS_CUDA_TRY(ctx, cudaFuncSetAttribute(greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem)));
        ctx->greedy_smem[0] = smem;
      }
      greedy_kernel<<<(n + kGreedyWarps - 1) / kGreedyWarps, kGreedyWarps * 32, smem, ctx->stream>>>(
          models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running, run->dOut, run->dLv, n, pk.max_horizon,
          pk.max_nc, run->dFG, run->lv_stride);
    } else {
      auto go = [&](auto kernel, int slot) -> int {
        if (one > ctx->greedy_smem[slot]) {
          BS_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(one)));
          ctx->greedy_smem[slot] = one;
        }
        kernel<<<n, 32 * nw, one, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running,
                                                 run->dOut, run->dLv, n, pk.max_horizon, pk.max_nc, run->dFG,
                                                 run->lv_stride);
        return BS_OK;
      };
      int rc = BS_OK;
      if (ctx->greedy_no_cluster < 0) ctx->greedy_no_cluster = std::getenv("BS_GREEDY_NO_CLUSTER") ? 1 : 0;
      if (nw == 16 && static_cast<long long>(n) * kGreedyCluster <= ctx->sm_count && !ctx->greedy_no_cluster) {
        // a handful of decisions: one cluster of kGreedyCluster SMs each
        auto kern = greedy_cluster_kernel<16, kGreedyCluster>;
        if (one > ctx->greedy_smem[5]) {
          BS_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(one)));
          ctx->greedy_smem[5] = one;
        }
        kern<<<n * kGreedyCluster, 32 * 16, one, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting,
                                                                pk.running, run->dOut, run->dLv, n, pk.max_horizon,
                                                                pk.max_nc, run->dFG, run->lv_stride);
      } else {
        switch (nw) {
          case 2: rc = go(greedy_coop_kernel<2>, 1); break;
          case 4: rc = go(greedy_coop_kernel<4>, 2); break;
          case 8: rc = go(greedy_coop_kernel<8>, 3); break;
          default: rc = go(greedy_coop_kernel<16>, 4); break;
        }
      }
      if (rc) return rc;
    }
    BS_LAUNCH_CHECK(ctx);
    BS_REC(1);
    return BS_OK;
  }
  if (!run->bfs_grid) {  // occupancy queries once per context
    if (!ctx->grid_cache[0]) {
#ifdef BS_SWEEP_CARVEOUT
      // A/B: the L1 / shared-memory split of the list kernels (percent shared)
      cudaFuncSetAttribute(reinterpret_cast<const void*>(sweep_kernel<kSweepMinB2, kSweep2>),
                           cudaFuncAttributePreferredSharedMemoryCarveout, BS_SWEEP_CARVEOUT);
      cudaFuncSetAttribute(reinterpret_cast<const void*>(sweep_kernel<kSweepMinB3, kSweep3>),
                           cudaFuncAttributePreferredSharedMemoryCarveout, BS_SWEEP_CARVEOUT);
      cudaFuncSetAttribute(reinterpret_cast<const void*>(bfs_node_kernel),
                           cudaFuncAttributePreferredSharedMemoryCarveout, BS_SWEEP_CARVEOUT);
#endif
      ctx->grid_cache[0] = grid_for(ctx, reinterpret_cast<const void*>(bfs_node_kernel), 256);
      ctx->grid_cache[1] = grid_for(ctx, reinterpret_cast<const void*>(sweep_kernel<kSweepMinB2, kSweep2>), 256);
      ctx->grid_cache[2] = grid_for(ctx, reinterpret_cast<const void*>(sweep_kernel<kSweepMinB3, kSweep3>), 256);
    }
    run->bfs_grid = ctx->grid_cache[0];
    run->sweep_grid2 = ctx->grid_cache[1];
    run->sweep_grid3 = ctx->grid_cache[2];
  }
  const Frontier lev[2] = {frontier_at(run->dLev[0], run->cap_level), frontier_at(run->dLev[1], run->cap_level)};
  const FinalList fin = final_at(run->dFin, run->cap_final);
  BS_CUDA_TRY(ctx, cudaMemsetAsync(run->dCtl, 0, sizeof(ExCtl), ctx->stream));
  prepare_kernel<<<n, kPrepThreads, 0, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running,
                                                      run->dT, run->dThr, run->dCtl, n, run->dFG, run->dBest,
                                                      run->dFeas, lev[0],
                                                      lev[1], fin, run->cap_level, run->cap_final,
                                                      run->sweep3_min, run->slice, run->dThrList);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(1);
  BS_CUDA_TRY(ctx, launch_pdl(thr_kernel, dim3(2 * ctx->sm_count), dim3(kPrepThreads), ctx->stream, run->dT,
                              run->dThr, static_cast<const ExCtl*>(run->dCtl), static_cast<const int*>(run->dThrList),
                              n));
  BS_LAUNCH_CHECK(ctx);
  BS_REC(2);  // the roots and first two levels are expanded by prepare_kernel; thresholds by thr_kernel
  // The kernels after prepare are launched as programmatic dependents: each
  // may be scheduled while its predecessor drains and waits for it in
  // griddepcontrol.wait before touching its data (phase events, when
  // recorded, serialise them again).
  for (int k = 3; k < run->bfs_levels; ++k) {  // depths up to 3 come from prepare_kernel
    BS_CUDA_TRY(ctx, launch_pdl(bfs_node_kernel, dim3(run->bfs_grid), dim3(256), ctx->stream,
                                static_cast<const DTables*>(run->dT), k, run->dCtl, lev[k & 1], lev[(k + 1) & 1], fin,
                                run->cap_level, run->cap_final, static_cast<const DThr*>(run->dThr), run->dFeas, n));
    BS_LAUNCH_CHECK(ctx);
  }
  BS_REC(3);
  if (run->sweep3)
    BS_CUDA_TRY(ctx, launch_pdl(sweep_kernel<kSweepMinB3, kSweep3>, dim3(run->sweep_grid3), dim3(256), ctx->stream,
                                static_cast<const DTables*>(run->dT), static_cast<const DThr*>(run->dThr),
                                static_cast<const ExCtl*>(run->dCtl), fin, run->dBest, run->dFeas, run->cap_final));
  else
    BS_CUDA_TRY(ctx, launch_pdl(sweep_kernel<kSweepMinB2, kSweep2>, dim3(run->sweep_grid2), dim3(256), ctx->stream,
                                static_cast<const DTables*>(run->dT), static_cast<const DThr*>(run->dThr),
                                static_cast<const ExCtl*>(run->dCtl), fin, run->dBest, run->dFeas, run->cap_final));
  BS_LAUNCH_CHECK(ctx);
  BS_REC(4);
  BS_CUDA_TRY(ctx, launch_pdl(finalize_kernel, dim3((n + 127) / 128), dim3(128), ctx->stream,
                              static_cast<const DTables*>(run->dT), static_cast<const DMpcCfg*>(pk.cfgs),
                              static_cast<const DProblem*>(pk.problems), static_cast<const Key128*>(run->dBest),
                              static_cast<const unsigned long long*>(run->dFeas), run->dOut, n, run->slice));
  BS_LAUNCH_CHECK(ctx);
  BS_REC(5);
  return BS_OK;
}

// Copies results back, syncs, expands.  Batches of >= 512 problems are
// copied in up to 4 slices, each followed by an event, so the expansion of a
// slice overlaps the D2H copy of the next.
// Problems per host-pool chunk of the result expansion; minimum problems per slice.
#ifndef BS_RESULT_GRAIN
#define BS_RESULT_GRAIN 256
#endif
#ifndef BS_RESULT_SLICE
#define BS_RESULT_SLICE 256
#endif
#ifndef BS_RESULT_SLICES_MAX
#define BS_RESULT_SLICES_MAX 4
#endif

static_assert(BS_RESULT_SLICES_MAX >= 1 && BS_RESULT_SLICES_MAX <= 4, "bs_ctx_s::slice_ev holds 4 events");

int run_results(bs_ctx_t ctx, MpcRun* run, bs_mpc_result* out) {
  const int n = run->n;
  if (n == 0) return BS_OK;
  const int stride = run->lv_stride;
  DMpcOut* hOut = static_cast<DMpcOut*>(ctx->host_buf(kSlotOut, result_region(n, stride)));
  DLevel* hLv = nullptr;
  if (!hOut) return set_error(ctx, BS_CUDA_ERROR, "mpc: host allocation failed");
  unsigned long long* hOverflow = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(hOut) + out_bytes(n));
  *hOverflow = 0;
  if (run->mode == kGreedy) {
    hLv = reinterpret_cast<DLevel*>(reinterpret_cast<char*>(hOut) + levels_off(n));
  } else {  // the overflow flag first: it is checked before any slice is expanded
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(hOverflow, &run->dCtl->overflow, 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  const int n_slices = std::max(1, std::min(BS_RESULT_SLICES_MAX, n / BS_RESULT_SLICE));
  auto slice_lo = [&](int sl) { return static_cast<int>(static_cast<long long>(n) * sl / n_slices); };
  if (n_slices > 1)  // the context's slice events, created on first use and reused by every call
    for (int sl = 0; sl < n_slices; ++sl)
      if (!ctx->slice_ev[sl]) BS_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->slice_ev[sl], cudaEventDisableTiming));
  for (int sl = 0; sl < n_slices; ++sl) {
    const int lo = slice_lo(sl), hi = slice_lo(sl + 1);
    if (hLv && run->contig && n_slices == 1) {  // results, flag and level records in one copy
      BS_CUDA_TRY(ctx, cudaMemcpyAsync(hOut, run->dOut, result_region(n, stride), cudaMemcpyDeviceToHost,
                                       ctx->stream));
      break;
    }
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(hOut + lo, run->dOut + lo, out_bytes(hi - lo), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    if (hLv)
      BS_CUDA_TRY(ctx, cudaMemcpyAsync(hLv + static_cast<size_t>(lo) * stride, run->dLv + static_cast<size_t>(lo) * stride,
                                       levels_bytes(hi - lo, stride), cudaMemcpyDeviceToHost, ctx->stream));
    if (n_slices > 1) BS_CUDA_TRY(ctx, cudaEventRecord(ctx->slice_ev[sl], ctx->stream));
  }
  ctx->last_d2h = out_bytes(n) + (hLv ? levels_bytes(n, stride) : 8);
  for (int sl = 0; sl < n_slices; ++sl) {
    if (n_slices > 1)
      BS_CUDA_TRY(ctx, cudaEventSynchronize(ctx->slice_ev[sl]));
    else
      BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (sl == 0 && run->mode == kExhaustive && *hOverflow) {
      BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      BS_CUDA_TRY(ctx, cudaMemcpy(&run->ctl_host, run->dCtl, sizeof(ExCtl), cudaMemcpyDeviceToHost));
      return set_error(ctx, kOverflowStatus, "mpc exhaustive: %llu frontier appends exceeded the capacity of this "
                       "batch; split it into smaller calls", *hOverflow);
    }
    const int s_lo = slice_lo(sl), s_hi = slice_lo(sl + 1);
    parallel_chunks(ctx, s_hi - s_lo, BS_RESULT_GRAIN, [&](int lo, int hi) {
      for (int i = s_lo + lo; i < s_lo + hi; ++i)
        expand_result(hOut[i], hLv ? hLv + static_cast<size_t>(i) * stride : nullptr, run->hc[run->cfg_of[i]],
                      run->target[i], &out[i], run->mode == kExhaustive);
    });
  }
  return report_status(ctx, out, n);
}

int one_shot(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
             int n_cfgs, const bs_mpc_problem* problems, int n, bs_mpc_result* out, int mode,
             const DSlice& slice = DSlice{}) {
  if (!ctx || !models) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: null context or models");
  unsigned long long cap_level = 0, cap_final = 0;  // 0: worst case (clamped)
  const bool dbg_t = std::getenv("BS_DEBUG_TIMING") != nullptr;  // host phase timings (diagnostics)
  auto now_us = []() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  for (int attempt = 0;; ++attempt) {
    MpcRun run;
    const double t0 = dbg_t ? now_us() : 0.0;
    int rc = run_pack(ctx, cfgs, policies, n_cfgs, problems, n, mode, &run, cap_level, cap_final);
    run.slice = slice;
    const double t1 = dbg_t ? now_us() : 0.0;
    if (rc) return rc;
    ctx->last_h2d = run.pk.h2d_bytes;
    ctx->last_d2h = 0;
    if (n == 0) return BS_OK;
    {
      DFastPair* dfg = static_cast<DFastPair*>(
          ctx->dev_buf(kSlotFastGrids, sizeof(DFastPair) * std::max<size_t>(run.pk.fg_pairs.size(), 1)));
      if (!dfg) return set_error(ctx, BS_CUDA_ERROR, "mpc: allocation of the reduced grids failed");
      // the reduced grids depend only on (models, candidate rungs, tp) per pair:
      // a call with the same pairs as the context's last upload (a controller
      // deciding again) reuses them
      std::string key(reinterpret_cast<const char*>(&models->serial), sizeof models->serial);
      key.append(reinterpret_cast<const char*>(&dfg), sizeof dfg);
      for (const auto& pr : run.pk.fg_pairs) {
        const DMpcCfg& c = run.hc[pr.first];
        key.append(reinterpret_cast<const char*>(&pr.second), sizeof pr.second);
        key.append(reinterpret_cast<const char*>(&c.nc), sizeof c.nc);
        key.append(reinterpret_cast<const char*>(c.cand), sizeof(double) * c.nc);
      }
      if (key != ctx->fg_key) {
        rc = upload_fast_pairs(ctx, models, &run, dfg);
        if (rc) return rc;
        ctx->fg_key = key;
        ctx->last_h2d += sizeof(DFastPair) * run.pk.fg_pairs.size();
      } else {
        run.dFG = run.pk.fg_pairs.empty() ? nullptr : dfg;
      }
    }
    if (mode == kExhaustive) {
      const ExLayout L = ex_layout(run, 0);
      char* base = static_cast<char*>(ctx->dev_buf(kSlotWork, L.total));
      if (!base) return set_error(ctx, BS_CUDA_ERROR, "mpc exhaustive: device allocation of %zu bytes failed", L.total);
      bind_exhaustive(&run, base, L);
    } else {
      // results and level records in one region: one D2H copy for small batches
      char* g = static_cast<char*>(ctx->dev_buf(kSlotOut, result_region(n, run.lv_stride)));
      if (!g) return set_error(ctx, BS_CUDA_ERROR, "mpc greedy: allocation failed");
      run.dOut = reinterpret_cast<DMpcOut*>(g);
      run.dLv = reinterpret_cast<DLevel*>(g + levels_off(n));
      run.contig = true;
    }
    const double t2 = dbg_t ? now_us() : 0.0;
    rc = run_enqueue(ctx, models, &run, false);
    if (rc) return rc;
    const double t3 = dbg_t ? now_us() : 0.0;
    if (dbg_t) cudaStreamSynchronize(ctx->stream);
    const double t4 = dbg_t ? now_us() : 0.0;
    rc = run_results(ctx, &run, out);
    if (dbg_t)
      std::fprintf(stderr, "bs_mpc one_shot us: pack %.1f upload %.1f enqueue %.1f device %.1f results %.1f\n", t1 - t0,
                   t2 - t1, t3 - t2, t4 - t3, now_us() - t4);
    if (rc != kOverflowStatus) return rc;
    // Overflow: counts up to the first overflowing level are exact totals;
    // retry with room for them, or split the batch when they exceed the budget.
    unsigned long long need_level = 0;
    for (int k = 0; k <= kMaxK; ++k) need_level = std::max(need_level, run.ctl_host.level_count[k]);
    const unsigned long long need_final = run.ctl_host.final_count;
    const unsigned long long grow_level = need_level + need_level / 4 + 1024;
    const unsigned long long grow_final = need_final + need_final / 4 + 1024;
    const bool fits = grow_level <= ctx->ex_level_cap && grow_final <= ctx->ex_final_cap;
    if (fits && attempt < kMaxK + 2 && (grow_level > run.cap_level || grow_final > run.cap_final)) {
      cap_level = std::max(grow_level, run.cap_level);
      cap_final = std::max(grow_final, run.cap_final);
      continue;
    }
    if (n == 1) return set_error(ctx, BS_PARAMETER_ERROR, "mpc exhaustive: one decision exceeds the frontier budget");
    // split into pieces sized from the observed (lower-bound) need
    const double over = std::max(static_cast<double>(grow_level) / ctx->ex_level_cap,
                                 static_cast<double>(grow_final) / ctx->ex_final_cap);
    const int pieces = std::min(n, std::max(2, static_cast<int>(std::ceil(over * 1.25))));
    uint64_t h2d = ctx->last_h2d, d2h = ctx->last_d2h;
    for (int p = 0; p < pieces; ++p) {
      const int a = static_cast<int>(static_cast<long long>(n) * p / pieces);
      const int b = static_cast<int>(static_cast<long long>(n) * (p + 1) / pieces);
      rc = one_shot(ctx, models, cfgs, policies, n_cfgs, problems + a, b - a, out + a, mode, slice);
      if (rc) return rc;
      h2d += ctx->last_h2d;
      d2h += ctx->last_d2h;
    }
    ctx->last_h2d = h2d;
    ctx->last_d2h = d2h;
    return BS_OK;
  }
}

}  // namespace

struct bs_mpc_plan_s {
  MpcRun run;
  void* mem = nullptr;
  bs_models_t models = nullptr;
};

extern "C" {

int bs_project_batches(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies, int n_cfgs,
                       const bs_mpc_problem* problems, int n, bs_projected_batch* out, int32_t* out_K,
                       int32_t* out_status) {
  if (!ctx) return BS_PARAMETER_ERROR;
  PackedProblems pk;
  int rc = pack_problems(ctx, cfgs, policies, n_cfgs, problems, n, &pk);
  if (rc) return rc;
  if (n == 0) return BS_OK;
  DTables* dT = static_cast<DTables*>(ctx->dev_buf(kSlotTables, sizeof(DTables) * n));
  DTables* hT = static_cast<DTables*>(ctx->host_buf(kSlotTables, sizeof(DTables) * n));
  if (!dT || !hT) return set_error(ctx, BS_CUDA_ERROR, "allocation failed");
  project_kernel<<<(n + 63) / 64, 64, 0, ctx->stream>>>(pk.cfgs, pk.problems, pk.waiting, pk.running, dT, n);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(hT, dT, sizeof(DTables) * n, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; ++i) {
    out_K[i] = hT[i].K;
    out_status[i] = hT[i].status;
    for (int k = 0; k < hT[i].K; ++k) {
      bs_projected_batch& b = out[static_cast<size_t>(i) * BS_MAX_K + k];
      b.features.n_requests = hT[i].n_req[k];
      b.features.sum_len = hT[i].sum_len[k];
      b.work_fraction = hT[i].wf[k];
      b.min_completing_arrival_ms = hT[i].minarr[k];
      b.n_completing = hT[i].ncomp[k];
    }
  }
  return BS_OK;
}

int bs_mpc_exhaustive(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                      const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems, int n,
                      bs_mpc_result* out) {
  return one_shot(ctx, models, cfgs, policies, n_cfgs, problems, n, out, kExhaustive);
}

int bs_mpc_exhaustive_slice(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                            const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems, int n,
                            const bs_slice* slice, bs_mpc_result* out) {
  if (!slice) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_exhaustive_slice: null slice");
  if (slice->digits < 0 || slice->digits > 2)
    return set_error(ctx, BS_PARAMETER_ERROR, "mpc slice: digits must be 0, 1 or 2 (got %d)", slice->digits);
  DSlice s{};
  s.digits = slice->digits;
  s.lo = slice->lo;
  s.hi = slice->hi;
  if (s.digits > 0) {
    if (s.lo > s.hi) return set_error(ctx, BS_PARAMETER_ERROR, "mpc slice: bad range [%llu, %llu)", s.lo, s.hi);
    for (int c = 0; c < n_cfgs; ++c) {
      double cand[BS_MAX_CAND];
      const int nc = ladder_select(ctx, cfgs[c].ladder_mhz, cfgs[c].n_ladder, cfgs[c].ladder_N, cand, BS_MAX_CAND);
      if (nc < 0) return nc;
      if (static_cast<double>(s.hi) > std::pow(static_cast<double>(nc), s.digits))
        return set_error(ctx, BS_PARAMETER_ERROR, "mpc slice: hi %llu exceeds %d^%d leading-digit values", s.hi, nc,
                         s.digits);
    }
  }
  return one_shot(ctx, models, cfgs, policies, n_cfgs, problems, n, out, kExhaustive, s);
}

int bs_mpc_greedy(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
                  int n_cfgs, const bs_mpc_problem* problems, int n, bs_mpc_result* out) {
  return one_shot(ctx, models, cfgs, policies, n_cfgs, problems, n, out, kGreedy);
}

int bs_mpc_plan_create(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs,
                       const bs_scheduler_policy* policies, int n_cfgs, const bs_mpc_problem* problems, int n,
                       int mode, bs_mpc_plan_t* out) {
  if (!ctx || !models || !out) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_plan_create: null argument");
  if (mode != kExhaustive && mode != kGreedy) return set_error(ctx, BS_PARAMETER_ERROR, "mpc plan: bad mode");
  *out = nullptr;
  auto* plan = new bs_mpc_plan_s();
  plan->models = models;
  MpcRun& run = plan->run;
  int rc = run_pack(ctx, cfgs, policies, n_cfgs, problems, n, mode, &run);
  if (rc) {
    delete plan;
    return rc;
  }
  const size_t fg_bytes = up256(sizeof(DFastPair) * run.pk.fg_pairs.size());
  const size_t blob = up256(run.pk.h2d_bytes) + fg_bytes;
  size_t total = blob, o_o = 0, o_l = 0;
  ExLayout L;
  if (mode == kExhaustive) {
    L = ex_layout(run, blob);
    total = L.total;
  } else {
    o_l = total;
    total += up256(levels_bytes(n, run.lv_stride));
    o_o = total;
    total += up256(out_bytes(n));
  }
  if (cudaMalloc(&plan->mem, total) != cudaSuccess) {
    delete plan;
    return set_error(ctx, BS_CUDA_ERROR, "mpc plan: cudaMalloc(%zu) failed", total);
  }
  char* m = static_cast<char*>(plan->mem);
  if (cudaMemcpyAsync(m, run.pk.base, run.pk.h2d_bytes, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    cudaFree(plan->mem);
    delete plan;
    return set_error(ctx, BS_CUDA_ERROR, "mpc plan: staging copy failed");
  }
  run.pk.rebase(m);
  if (upload_fast_pairs(ctx, models, &run, reinterpret_cast<DFastPair*>(m + up256(run.pk.h2d_bytes))) != BS_OK ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    cudaFree(plan->mem);
    delete plan;
    return set_error(ctx, BS_CUDA_ERROR, "mpc plan: reduced-grid upload failed");
  }
  if (mode == kExhaustive) {
    bind_exhaustive(&run, m, L);
  } else {
    run.dOut = reinterpret_cast<DMpcOut*>(m + o_o);
    run.dLv = reinterpret_cast<DLevel*>(m + o_l);
  }
  *out = plan;
  return BS_OK;
}

int bs_mpc_plan_run(bs_ctx_t ctx, bs_mpc_plan_t plan, int record_kernel_times) {
  if (!ctx || !plan) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_plan_run: null argument");
  return run_enqueue(ctx, plan->models, &plan->run, record_kernel_times != 0);
}

int bs_mpc_plan_results(bs_ctx_t ctx, bs_mpc_plan_t plan, bs_mpc_result* out) {
  if (!ctx || !plan) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_plan_results: null argument");
  const int rc = run_results(ctx, &plan->run, out);
  if (std::getenv("BS_DEBUG_COUNTS") && plan->run.mode == kExhaustive) {  // list sizes of the last run (diagnostics)
    ExCtl c;
    if (cudaMemcpy(&c, plan->run.dCtl, sizeof c, cudaMemcpyDeviceToHost) == cudaSuccess) {
      std::fprintf(stderr, "bs_mpc lists:");
      for (int k = 0; k <= kMaxK; ++k)
        if (c.level_count[k]) std::fprintf(stderr, " depth%d=%llu", k, c.level_count[k]);
      std::fprintf(stderr, " final=%llu overflow=%llu\n", c.final_count, c.overflow);
#ifdef BS_SWEEP_STATS
      std::fprintf(stderr, "bs_mpc sweep: nodes %llu children %llu rows evaluated %llu leaves %llu divisions %llu "
                   "depth-(K-2) nodes counted by thresholds %llu / walked %llu; final nodes without a feasible "
                   "leaf %llu\n",
                   c.st_nodes, c.st_children, c.st_rows_eval, c.st_leaves_eval, c.st_div, c.st_thr_nodes,
                   c.st_slow_nodes, c.st_empty_nodes);
#endif
    }
  }
  // a resident plan's frontiers are fixed at creation: report an overflow as
  // a parameter problem of the batch (one-shot calls re-run or split instead)
  return rc == kOverflowStatus ? set_error(ctx, BS_PARAMETER_ERROR, "%s", ctx->err.c_str()) : rc;
}

int bs_mpc_plan_kernel_ms(bs_ctx_t ctx, bs_mpc_plan_t plan, float* ms, int n_ms) {
  if (!ctx || !plan || !ms) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_plan_kernel_ms: null argument");
  MpcRun& run = plan->run;
  if (!run.have_events) return set_error(ctx, BS_PARAMETER_ERROR, "mpc plan: no timed run recorded");
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const int phases = run.mode == kGreedy ? 1 : kNumEvents - 1;
  for (int i = 0; i < n_ms; ++i) {
    ms[i] = 0.0f;
    if (i < phases) BS_CUDA_TRY(ctx, cudaEventElapsedTime(&ms[i], run.ev[i], run.ev[i + 1]));
  }
  return phases;
}

int bs_mpc_plan_info(bs_ctx_t ctx, bs_mpc_plan_t plan, uint64_t* h2d_bytes, uint64_t* work_capacity) {
  if (!ctx || !plan) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_plan_info: null argument");
  if (h2d_bytes) *h2d_bytes = plan->run.pk.h2d_bytes;
  if (work_capacity) *work_capacity = plan->run.cap_final;
  return BS_OK;
}

void bs_mpc_plan_destroy(bs_ctx_t ctx, bs_mpc_plan_t plan) {
  (void)ctx;
  if (!plan) return;
  if (plan->run.have_events)
    for (auto& e : plan->run.ev) cudaEventDestroy(e);
  if (plan->mem) cudaFree(plan->mem);
  delete plan;
}

int bs_mpc_tables(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                  const bs_mpc_problem* problem, int32_t* out_K, int32_t* out_n_cand, double* lat, double* pow,
                  double* energy) {
  if (!ctx || !models) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_tables: null context or models");
  bs_mpc_problem p = *problem;
  p.cfg_index = 0;
  PackedProblems pk;
  int rc = pack_problems(ctx, cfg, policy, 1, &p, 1, &pk);
  if (rc) return rc;
  DTables* dT = static_cast<DTables*>(ctx->dev_buf(kSlotTables, sizeof(DTables)));
  DTables* hT = static_cast<DTables*>(ctx->host_buf(kSlotTables, sizeof(DTables)));
  if (!dT || !hT) return set_error(ctx, BS_CUDA_ERROR, "allocation failed");
  tables_only_kernel<<<1, kPrepThreads, 0, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running, dT);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(hT, dT, sizeof(DTables), cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (hT->status != BS_OK) return set_error(ctx, hT->status, "mpc tables: projection failed");
  *out_K = hT->K;
  *out_n_cand = hT->nc;
  for (int k = 0; k < hT->K; ++k)
    for (int f = 0; f < hT->nc; ++f) {
      lat[k * hT->nc + f] = hT->A[k][f];
      pow[k * hT->nc + f] = hT->P[k][f];
      energy[k * hT->nc + f] = hT->E[k][f];
    }
  return BS_OK;
}

int bs_mpc_eval_codes(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                      const bs_mpc_problem* problem, const uint64_t* codes, int n, int32_t* out_feasible,
                      double* out_objective) {
  if (!ctx || !models) return set_error(ctx, BS_PARAMETER_ERROR, "bs_mpc_eval_codes: null context or models");
  bs_mpc_problem p = *problem;
  p.cfg_index = 0;
  PackedProblems pk;
  int rc = pack_problems(ctx, cfg, policy, 1, &p, 1, &pk);
  if (rc) return rc;
  if (n <= 0) return BS_OK;
  DTables* dT = static_cast<DTables*>(ctx->dev_buf(kSlotTables, sizeof(DTables)));
  const size_t bytes = static_cast<size_t>(n) * (8 + 4 + 8);
  char* d = static_cast<char*>(ctx->dev_buf(kSlotMisc, bytes));
  char* h = static_cast<char*>(ctx->host_buf(kSlotMisc, bytes));
  if (!dT || !d || !h) return set_error(ctx, BS_CUDA_ERROR, "allocation failed");
  std::memcpy(h, codes, 8ull * n);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
  tables_only_kernel<<<1, kPrepThreads, 0, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running, dT);
  BS_LAUNCH_CHECK(ctx);
  eval_codes_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
      dT, pk.cfgs, pk.problems, reinterpret_cast<const unsigned long long*>(d), n,
      reinterpret_cast<int32_t*>(d + 16ull * n), reinterpret_cast<double*>(d + 8ull * n));
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(h + 8ull * n, d + 8ull * n, 12ull * n, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  std::memcpy(out_objective, h + 8ull * n, 8ull * n);
  std::memcpy(out_feasible, h + 16ull * n, 4ull * n);
  return BS_OK;
}

}  // extern "C"

// bs_mpc.cu — prefill MPC on sm_100a: projection, (k, f) tables, the
// exhaustive rollout (prefix compaction + leaf sweep + 128-bit argmin) and
// the greedy level search.  Reference: proj/include/pdsim/dvfs.hpp.
//
// Data flow for one batch of decisions (all on one stream, no host sync
// until the final copy-out):
//   prepare_kernel   1 CTA / problem: project_batches (dvfs.hpp:63-100) by
//                    one thread, then the K x N (lat, pow) tables by all
//                    threads through the bit-exact interpolator.
//   seed_kernel      1 thread / problem: reset argmin slots, seed the roots.
//   bfs_kernel       x (max depth of final nodes): level-synchronous
//                    expansion of every feasible prefix of every decision,
//                    compacted with warp-aggregated appends (meets_slo fails
//                    at the first violated batch, so violated prefixes have
//                    no feasible completion and are dropped for good).
//   sweep_kernel     one thread per final node sweeps its bottom 2 (or 3)
//                    levels in increasing code order with a division-free
//                    objective filter; (objective, code) minima merge
//                    through a 128-bit CAS.  See bs_exhaustive.cuh.
//   finalize_kernel  1 thread / problem: decode the argmin code.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "bs_internal.h"

using namespace bs;

namespace {

constexpr int kPrepThreads = 256;
constexpr int kGreedyThreads = 256;
constexpr double kFilterScale = 1.0 + 0x1p-50;  // C in the filter bound
constexpr double kFilterMinBest = 0x1p-100;
constexpr double kFilterMinDen = 0x1p-900;

// ---------------------------------------------------------------------------
// projection: project_batches (dvfs.hpp:63-100) over form_prefill_batch
// (scheduler.hpp:40-66).  Only the queue head can be partially consumed (a
// partial chunk ends a batch), so the state is (head, head_remaining).
// ---------------------------------------------------------------------------
__device__ int project_dev(const DProblem& pr, const DMpcCfg& c, const DWaiting* W, const DRunning* R, DTables* T) {
  int K = 0;
  if (pr.run_active) {
    T->n_req[0] = pr.run_n;
    T->sum_len[0] = pr.run_sum;
    T->wf[0] = pr.run_wr;
    double mn = INFINITY;
    int nc = 0;
    for (int i = 0; i < pr.n_run; ++i) {
      if (R[i].completes) {
        const double a = R[i].arrival;
        mn = a < mn ? a : mn;
        ++nc;
      }
    }
    T->minarr[0] = mn;
    T->ncomp[0] = nc;
    K = 1;
  }
  int head = 0;
  long long head_rem = pr.n_wait > 0 ? W[0].remaining : 0;
  while (head < pr.n_wait && K < c.horizon) {
    long long tokens = 0, npick = 0, sum = 0;
    int consumed = 0, ncomp = 0;
    double mn = INFINITY;
    long long partial_rem = -1;
    for (int i = head; i < pr.n_wait; ++i) {
      if (npick >= c.max_batch_requests) break;
      const long long rem = i == head ? head_rem : W[i].remaining;
      if (rem <= 0) {
        T->K = K;
        return BS_SIMULATION_ERROR;  // scheduler.hpp:47
      }
      long long take;
      if (c.chunking) {
        const long long room = c.max_batch_tokens - tokens;
        if (room <= 0) break;
        take = rem < room ? rem : room;
        tokens += take;
      } else {
        if (rem > c.max_batch_tokens) {
          if (npick == 0) {
            ++npick;
            sum += rem;
            ++ncomp;
            const double a = W[i].arrival;
            mn = a < mn ? a : mn;
            ++consumed;
          }
          break;
        }
        if (tokens + rem > c.max_batch_tokens) break;
        take = rem;
        tokens += rem;
      }
      ++npick;
      sum += take;
      if (take == rem) {
        ++ncomp;
        const double a = W[i].arrival;
        mn = a < mn ? a : mn;
        ++consumed;
      } else {
        partial_rem = rem - take;
        break;
      }
    }
    T->n_req[K] = npick;
    T->sum_len[K] = sum;
    T->wf[K] = 1.0;
    T->minarr[K] = mn;
    T->ncomp[K] = ncomp;
    ++K;
    head += consumed;
    if (partial_rem >= 0) {
      head_rem = partial_rem;
    } else if (head < pr.n_wait) {
      head_rem = W[head].remaining;
    }
  }
  T->K = K;
  return BS_OK;
}

// Tables for one problem, written by a CTA.  Projection by thread 0.
__device__ void build_tables(const DModels& m, const DProblem& pr, const DMpcCfg& c, const DWaiting* W,
                             const DRunning* R, DTables* T, int* s_status) {
  if (threadIdx.x == 0) {
    T->nc = c.nc;
    T->ttft = c.ttft;
    int st = project_dev(pr, c, W, R, T);
    if (st == BS_OK && (m.grid[0].bad_axis || m.grid[2].bad_axis) && T->K > 0) st = BS_MODEL_ERROR;
    *s_status = st;
    for (int k = 0; k < kMaxK; ++k) {
      T->bad_lat[k] = 0u;
      T->bad_pow[k] = 0u;
    }
  }
  __syncthreads();
  const int K = T->K;
  const int nc = c.nc;
  if (*s_status != BS_OK) return;
  for (int e = threadIdx.x; e < K * nc; e += blockDim.x) {
    const int k = e / nc, f = e - k * nc;
    const Query q = make_query(T->n_req[k], T->sum_len[k], pr.tp, c.cand[f]);
    const double L = interp(m.grid[0], q, nullptr);
    const double P = interp(m.grid[2], q, nullptr);
    if (!model_value_ok(L)) atomicOr(&T->bad_lat[k], 1u << f);
    if (!model_value_ok(P)) atomicOr(&T->bad_pow[k], 1u << f);
    const double A = __dmul_rn(T->wf[k], L);                               // dvfs.hpp:112-113, 154-155
    T->A[k][f] = A;
    T->P[k][f] = P;
    T->E[k][f] = __dmul_rn(A, P);                                          // dvfs.hpp:167
    T->B0[k][f] = __dmul_rn(A, c.one_plus_margin);                         // dvfs.hpp:115
    T->B1[k][f] = __dmul_rn(__dadd_rn(A, c.switch_ms), c.one_plus_margin);  // dvfs.hpp:114-115
    if (k == 0) T->T1[f] = __dadd_rn(pr.now, c.cand[f] != pr.cur_freq ? T->B1[0][f] : T->B0[0][f]);
  }
  __syncthreads();
  // per-level sorted order of the switched steps: one thread per (k, f)
  // computes its rank (ties by index), then scatters
  int finite = 1;
  for (int e = threadIdx.x; e < K * nc; e += blockDim.x) {
    const int k = e / nc, f = e - k * nc;
    const double* key = k == 0 ? T->T1 : T->B1[k];
    const double v = key[f];
    if (!isfinite(v) || !isfinite(T->B0[k][f])) finite = 0;
    int r = 0;
    for (int g = 0; g < nc; ++g) {
      const double w = key[g];
      r += (w < v || (w == v && g < f)) ? 1 : 0;
    }
    T->sb[k][r] = v;
    T->ord[k][r] = static_cast<unsigned char>(f);
    T->rank[k][f] = static_cast<unsigned char>(r);
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double amax = 0.0, pmin = INFINITY;
    for (int f = 0; f < nc; ++f) {
      amax = T->A[k][f] > amax ? T->A[k][f] : amax;
      pmin = T->P[k][f] < pmin ? T->P[k][f] : pmin;
    }
    T->amax[k] = amax;
    T->pmin_lo[k] = __dmul_rn(pmin, 1.0 - 0x1p-50);
  }
  const int all_finite = __syncthreads_and(finite);
  if (threadIdx.x == 0) {
    int ok = 1;
    for (int k = 0; k < K; ++k)
      for (int f = 0; f < nc; ++f) {
        const double A = T->A[k][f];
        if (!(A >= 0.0) || !isfinite(A) || !isfinite(T->E[k][f])) ok = 0;
      }
    T->filter_ok = ok;
    T->sorted_ok = all_finite && isfinite(T->ttft);
  }
  __syncthreads();
}

#include "bs_exhaustive.cuh"

__global__ void finalize_kernel(const DTables* __restrict__ tables, const DMpcCfg* cfgs, const DProblem* probs,
                                const Key128* best, const unsigned long long* feas, DMpcOut* out, int n) {
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
    o.eval_count = static_cast<long long>(ipow(static_cast<unsigned long long>(nc), K));
    if (best[d].obj != ~0ull) {
      o.feasible = 1;
      o.objective = __longlong_as_double(static_cast<long long>(best[d].obj));
      unsigned long long code = best[d].code;
      o.best_code = code;
      for (int k = K - 1; k >= 0; --k) {
        o.idx[k] = static_cast<unsigned char>(code % nc);
        code /= nc;
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

// Evaluates one assignment (ascending candidate indices).  Returns
// 0 infeasible, 1 feasible; *err = 0 none, 1 latency, 2 power -- the first
// ModelError the reference would raise (meets_slo's predict_latency calls
// in k order up to the first violation, then time_weighted_power's
// predict_latency/predict_power pairs in k order).
__device__ int eval_assignment(const DTables& T, const DProblem& pr, const DMpcCfg& c, const unsigned char* idx,
                               double* obj, int* err) {
  *err = 0;
  double t = pr.now;
  const int K = T.K;
  bool feas = true;
  for (int k = 0; k < K; ++k) {
    const int f = idx[k];
    if ((T.bad_lat[k] >> f) & 1u) {
      *err = 1;
      return 0;
    }
    const bool sw = k == 0 ? (c.cand[f] != pr.cur_freq) : (f != idx[k - 1]);
    t = __dadd_rn(t, sw ? T.B1[k][f] : T.B0[k][f]);
    if (__dsub_rn(t, T.minarr[k]) > T.ttft) {
      feas = false;
      break;
    }
  }
  if (!feas) return 0;
  double num = 0.0, den = 0.0;
  for (int k = 0; k < K; ++k) {
    const int f = idx[k];
    if ((T.bad_lat[k] >> f) & 1u) {
      *err = 1;
      return 1;
    }
    if ((T.bad_pow[k] >> f) & 1u) {
      *err = 2;
      return 1;
    }
    num = __dadd_rn(num, T.E[k][f]);
    den = __dadd_rn(den, T.A[k][f]);
  }
  *obj = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
  return 1;
}

// objective only (tw_power of an assignment, errors ignored)
__device__ double tw_objective(const DTables& T, const unsigned char* idx) {
  double num = 0.0, den = 0.0;
  for (int k = 0; k < T.K; ++k) {
    num = __dadd_rn(num, T.E[k][idx[k]]);
    den = __dadd_rn(den, T.A[k][idx[k]]);
  }
  return den > 0.0 ? __ddiv_rn(num, den) : 0.0;
}

__global__ void __launch_bounds__(kGreedyThreads) greedy_kernel(DModels m, const DMpcCfg* cfgs, const DProblem* probs,
                                                                const DWaiting* W, const DRunning* R, DMpcOut* out,
                                                                DLevel* levels, int n) {
  __shared__ DTables T;
  __shared__ int s_status;
  __shared__ unsigned char cur[kMaxK];
  __shared__ int pos[kMaxK];
  __shared__ int s_np;
  __shared__ unsigned long long s_wbo[kGreedyThreads / 32], s_wbc[kGreedyThreads / 32];
  __shared__ unsigned long long s_feas;
  __shared__ unsigned long long s_err;  // min over (code << 2 | type) of erroring mutations
  const int d = blockIdx.x;
  if (d >= n) return;
  const DProblem pr = probs[d];
  const DMpcCfg& c = cfgs[pr.cfg];
  build_tables(m, pr, c, W + pr.wait_off, R + pr.run_off, &T, &s_status);
  DMpcOut* o = &out[d];
  DLevel* lv = levels + static_cast<size_t>(d) * BS_MAX_LEVELS;
  const int K = T.K, nc = c.nc;
  if (threadIdx.x == 0) {
    memset(o, 0, sizeof *o);
    o->status = s_status;
    o->K = K;
  }
  if (s_status != BS_OK) return;
  if (K == 0) {  // dvfs.hpp:194-197
    if (threadIdx.x == 0) o->feasible = 1;
    return;
  }
  // all-max initialization (dvfs.hpp:201-205)
  __shared__ int s_init_feas;
  __shared__ double s_obj;
  if (threadIdx.x == 0) {
    for (int k = 0; k < K; ++k) cur[k] = static_cast<unsigned char>(nc - 1);
    double obj = 0.0;
    int err;
    const int feas = eval_assignment(T, pr, c, cur, &obj, &err);
    if (!feas && !err) {
      // infeasible: objective still computed (dvfs.hpp:204), may raise
      for (int k = 0; k < K && !err; ++k) {
        if ((T.bad_lat[k] >> (nc - 1)) & 1u) err = 1;
        else if ((T.bad_pow[k] >> (nc - 1)) & 1u) err = 2;
      }
      obj = tw_objective(T, cur);
    }
    if (err) o->status = BS_MODEL_ERROR;
    s_init_feas = feas;
    s_obj = obj;
    o->feasible = feas;
    o->eval_count = 1;
    o->objective = obj;
  }
  __syncthreads();
  if (o->status != BS_OK) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (s_init_feas && nc > 1) {
    const int last_level = nc >= 3 ? nc - 2 : 1;
    // avail (descending) position j <-> ascending index nc - 1 - j
    for (int l = 1; l <= last_level; ++l) {
      const int target = nc - l;  // avail[l-1]
      const int r1 = nc - 1 - l;  // avail[l]
      const int r2 = l + 1 < nc ? nc - 2 - l : -1;
      const unsigned long long base = r2 >= 0 ? 3ull : 2ull;
      if (threadIdx.x == 0) {
        int np = 0;
        for (int k = 0; k < K; ++k)
          if (cur[k] == target) pos[np++] = k;
        s_np = np;
        s_feas = 0;
        s_err = ~0ull;
      }
      __syncthreads();
      const int np = s_np;
      if (np == 0) break;  // dvfs.hpp:222
      const unsigned long long combos = ipow(base, np);
      unsigned char mut[kMaxK];
      for (int k = 0; k < K; ++k) mut[k] = cur[k];
      unsigned long long bo = ~0ull, bc = ~0ull, feas = 0, errkey = ~0ull;
      for (unsigned long long code = 1 + threadIdx.x; code < combos; code += blockDim.x) {
        unsigned long long cc = code, lex = 0;
        for (int i = 0; i < np; ++i) {  // digit i -> pos[i], least significant first (dvfs.hpp:233-237)
          const unsigned long long digit = cc % base;
          cc /= base;
          mut[pos[i]] = static_cast<unsigned char>(digit == 0 ? target : (digit == 1 ? r1 : r2));
        }
        // lexicographic key of the frequency vector: positions in batch
        // order, smaller frequency (larger digit) first
        for (int i = 0; i < np; ++i) {
          const unsigned char v = mut[pos[i]];
          const unsigned long long digit = v == target ? 0 : (v == r1 ? 1 : 2);
          lex = lex * base + (base - 1 - digit);
        }
        double obj = 0.0;
        int err;
        const int ok = eval_assignment(T, pr, c, mut, &obj, &err);
        if (err) {
          const unsigned long long ek = (code << 2) | static_cast<unsigned long long>(err);
          errkey = ek < errkey ? ek : errkey;
          continue;
        }
        if (!ok) continue;
        ++feas;
        const unsigned long long ob = static_cast<unsigned long long>(__double_as_longlong(obj));
        if (key_less(ob, lex, bo, bc)) {
          bo = ob;
          bc = lex;
        }
      }
      // block reduction of (obj, lex), feasible count, first error
#pragma unroll
      for (int of = 16; of > 0; of >>= 1) {
        const unsigned long long oo = __shfl_xor_sync(0xffffffffu, bo, of);
        const unsigned long long oc = __shfl_xor_sync(0xffffffffu, bc, of);
        if (key_less(oo, oc, bo, bc)) {
          bo = oo;
          bc = oc;
        }
        feas += __shfl_xor_sync(0xffffffffu, feas, of);
        const unsigned long long oe = __shfl_xor_sync(0xffffffffu, errkey, of);
        errkey = oe < errkey ? oe : errkey;
      }
      if (lane == 0) {
        s_wbo[warp] = bo;
        s_wbc[warp] = bc;
        atomicAdd(&s_feas, feas);
        atomicMin(&s_err, errkey);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
          if (key_less(s_wbo[w], s_wbc[w], bo, bc)) {
            bo = s_wbo[w];
            bc = s_wbc[w];
          }
        // every mutation of the level is evaluated before acceptance
        o->eval_count += static_cast<long long>(combos - 1);
        DLevel L;
        L.k_prime = np;
        L.replaced_mhz = c.cand[target];
        L.mutations = static_cast<long long>(combos - 1);
        L.feasible_mutations = static_cast<long long>(s_feas);
        L.accepted = 0;
        if (s_err != ~0ull) {
          o->status = BS_MODEL_ERROR;
          o->n_levels = -static_cast<int>(s_err & 3ull);  // error type for the message
        } else {
          // improved iff best_p < cur or (== and lex_less(best, cur)); every
          // mutation is lexicographically below the current assignment
          const double bp = __longlong_as_double(static_cast<long long>(bo));
          if (bo != ~0ull && bp <= s_obj) {
            // decode the lex key back into digits
            unsigned long long lx = bc;
            for (int i = np - 1; i >= 0; --i) {
              const unsigned long long digit = base - 1 - (lx % base);
              lx /= base;
              cur[pos[i]] = static_cast<unsigned char>(digit == 0 ? target : (digit == 1 ? r1 : r2));
            }
            s_obj = bp;
            o->objective = bp;
            L.accepted = 1;
          }
          lv[o->n_levels] = L;
          o->n_levels += 1;
        }
        s_feas = L.accepted;  // broadcast acceptance
      }
      __syncthreads();
      if (o->status != BS_OK || s_feas == 0) break;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && o->status == BS_OK) {
    for (int k = 0; k < K; ++k) o->idx[k] = cur[k];
  }
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
  std::memset(r, 0, sizeof *r);
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
  int bfs_levels = 0;               // deepest final-node depth over the batch
  unsigned long long cap_level = 0;  // BFS list capacity (per ping-pong buffer)
  unsigned long long cap_final = 0;  // final list capacity
  DTables* dT = nullptr;
  ExCtl* dCtl = nullptr;
  Key128* dBest = nullptr;
  unsigned long long* dFeas = nullptr;
  void* dLev[2] = {nullptr, nullptr};
  void* dFin = nullptr;
  DMpcOut* dOut = nullptr;
  DLevel* dLv = nullptr;
  int bfs_grid = 0, sweep_grid = 0;
  cudaEvent_t ev[kNumEvents] = {};
  bool have_events = false;
};

size_t up256(size_t x) { return (x + 255) / 256 * 256; }
size_t tables_bytes(int n) { return sizeof(DTables) * static_cast<size_t>(n); }
size_t best_bytes(int n) { return (sizeof(Key128) + 8ull) * static_cast<size_t>(n); }
size_t out_bytes(int n) { return sizeof(DMpcOut) * static_cast<size_t>(n); }
size_t levels_bytes(int n) { return sizeof(DLevel) * BS_MAX_LEVELS * static_cast<size_t>(n); }

// Device scratch layout of an exhaustive run (offsets from one base).
struct ExLayout {
  size_t tables = 0, ctl = 0, best = 0, lev0 = 0, lev1 = 0, fin = 0, out = 0, total = 0;
};

ExLayout ex_layout(const MpcRun& r, size_t start) {
  ExLayout L;
  size_t o = start;
  L.tables = o;
  o += up256(tables_bytes(r.n));
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
  r->dCtl = reinterpret_cast<ExCtl*>(base + L.ctl);
  r->dBest = reinterpret_cast<Key128*>(base + L.best);
  r->dFeas = reinterpret_cast<unsigned long long*>(r->dBest + r->n);
  r->dLev[0] = base + L.lev0;
  r->dLev[1] = base + L.lev1;
  r->dFin = base + L.fin;
  r->dOut = reinterpret_cast<DMpcOut*>(base + L.out);
}

constexpr size_t kMaxExhaustiveScratch = 24ull << 30;

// Packs the problems (one H2D copy), validates configurations and sizes the
// exhaustive frontiers from the horizons (K <= horizon_K).
int run_pack(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies, int n_cfgs,
             const bs_mpc_problem* problems, int n, int mode, MpcRun* run) {
  run->mode = mode;
  run->n = n;
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
  run->cfg_of.resize(n);
  run->target.resize(n);
  run->cap_level = 0;
  run->cap_final = 0;
  run->bfs_levels = 0;
  for (int i = 0; i < n; ++i) {
    run->cfg_of[i] = problems[i].cfg_index;
    run->target[i] = problems[i].snap.target_freq_mhz;
    if (mode != kExhaustive) continue;
    const DMpcCfg& c = run->hc[problems[i].cfg_index];
    const int FD = c.horizon - sweep_levels(c.horizon, c.nc);
    run->bfs_levels = std::max(run->bfs_levels, FD);
    run->cap_final += ipow(static_cast<unsigned long long>(c.nc), FD);
    run->cap_level += ipow(static_cast<unsigned long long>(c.nc), FD > 0 ? FD - 1 : 0);
  }
  if (mode == kExhaustive) {
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

#define BS_REC(i)                                                         \
  do {                                                                    \
    if (timing) BS_CUDA_TRY(ctx, cudaEventRecord(run->ev[i], ctx->stream)); \
  } while (0)

int grid_for(bs_ctx_t ctx, const void* kernel, int threads) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1) b = 1;
  return ctx->sm_count * b;
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
    greedy_kernel<<<n, kGreedyThreads, 0, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running,
                                                         run->dOut, run->dLv, n);
    BS_LAUNCH_CHECK(ctx);
    BS_REC(1);
    return BS_OK;
  }
  if (!run->bfs_grid) {
    run->bfs_grid = grid_for(ctx, reinterpret_cast<const void*>(bfs_kernel), 256);
    run->sweep_grid = grid_for(ctx, reinterpret_cast<const void*>(sweep_kernel), 256);
  }
  const Frontier lev[2] = {frontier_at(run->dLev[0], run->cap_level), frontier_at(run->dLev[1], run->cap_level)};
  const FinalList fin = final_at(run->dFin, run->cap_final);
  prepare_kernel<<<n, kPrepThreads, 0, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running,
                                                      run->dT, run->dCtl, n);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(1);
  seed_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(run->dT, n, run->dBest, run->dFeas, run->dCtl, lev[0], fin,
                                                        run->cap_level, run->cap_final);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(2);
  for (int k = 0; k < run->bfs_levels; ++k) {
    bfs_kernel<<<run->bfs_grid, 256, 0, ctx->stream>>>(run->dT, k, run->dCtl, lev[k & 1], lev[(k + 1) & 1], fin,
                                                       run->max_nc, run->cap_level, run->cap_final);
    BS_LAUNCH_CHECK(ctx);
  }
  BS_REC(3);
  sweep_kernel<<<run->sweep_grid, 256, 0, ctx->stream>>>(run->dT, run->dCtl, fin, run->dBest, run->dFeas);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(4);
  finalize_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(run->dT, pk.cfgs, pk.problems, run->dBest, run->dFeas,
                                                            run->dOut, n);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(5);
  return BS_OK;
}

// Copies results back (one or two D2H copies), syncs, expands.
int run_results(bs_ctx_t ctx, MpcRun* run, bs_mpc_result* out) {
  const int n = run->n;
  if (n == 0) return BS_OK;
  DMpcOut* hOut = static_cast<DMpcOut*>(ctx->host_buf(kSlotOut, out_bytes(n) + 64));
  DLevel* hLv = nullptr;
  if (!hOut) return set_error(ctx, BS_CUDA_ERROR, "mpc: host allocation failed");
  unsigned long long* hOverflow = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(hOut) + out_bytes(n));
  *hOverflow = 0;
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(hOut, run->dOut, out_bytes(n), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->last_d2h = out_bytes(n);
  if (run->mode == kGreedy) {
    hLv = static_cast<DLevel*>(ctx->host_buf(kSlotLevels, levels_bytes(n)));
    if (!hLv) return set_error(ctx, BS_CUDA_ERROR, "mpc: host allocation failed");
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(hLv, run->dLv, levels_bytes(n), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->last_d2h += levels_bytes(n);
  } else {
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(hOverflow, &run->dCtl->overflow, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->last_d2h += 8;
  }
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (*hOverflow)
    return set_error(ctx, BS_CUDA_ERROR, "mpc exhaustive: %llu frontier appends overflowed (capacity bug)",
                     *hOverflow);
  for (int i = 0; i < n; ++i)
    expand_result(hOut[i], hLv ? hLv + static_cast<size_t>(i) * BS_MAX_LEVELS : nullptr, run->hc[run->cfg_of[i]],
                  run->target[i], &out[i], run->mode == kExhaustive);
  return report_status(ctx, out, n);
}

int one_shot(bs_ctx_t ctx, bs_models_t models, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies,
             int n_cfgs, const bs_mpc_problem* problems, int n, bs_mpc_result* out, int mode) {
  if (!ctx || !models) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: null context or models");
  MpcRun run;
  int rc = run_pack(ctx, cfgs, policies, n_cfgs, problems, n, mode, &run);
  if (rc) return rc;
  ctx->last_h2d = run.pk.h2d_bytes;
  ctx->last_d2h = 0;
  if (n == 0) return BS_OK;
  if (mode == kExhaustive) {
    const ExLayout L = ex_layout(run, 0);
    char* base = static_cast<char*>(ctx->dev_buf(kSlotWork, L.total));
    if (!base) return set_error(ctx, BS_CUDA_ERROR, "mpc exhaustive: device allocation of %zu bytes failed", L.total);
    bind_exhaustive(&run, base, L);
  } else {
    run.dOut = static_cast<DMpcOut*>(ctx->dev_buf(kSlotOut, out_bytes(n)));
    run.dLv = static_cast<DLevel*>(ctx->dev_buf(kSlotLevels, levels_bytes(n)));
    if (!run.dOut || !run.dLv) return set_error(ctx, BS_CUDA_ERROR, "mpc greedy: allocation failed");
  }
  rc = run_enqueue(ctx, models, &run, false);
  if (rc) return rc;
  return run_results(ctx, &run, out);
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
  const size_t blob = up256(run.pk.h2d_bytes);
  size_t total = blob, o_o = 0, o_l = 0;
  ExLayout L;
  if (mode == kExhaustive) {
    L = ex_layout(run, blob);
    total = L.total;
  } else {
    o_l = total;
    total += up256(levels_bytes(n));
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
  return run_results(ctx, &plan->run, out);
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

// bs_mpc.cu — prefill MPC on sm_100a: projection, (k, f) tables, the
// exhaustive rollout (prefix compaction + leaf sweep + 128-bit argmin) and
// the greedy level search.  Reference: proj/include/pdsim/dvfs.hpp.
//
// Data flow for one batch of decisions (all on one stream, no host sync
// until the final copy-out):
//   prepare_kernel   1 CTA / problem: project_batches (dvfs.hpp:63-100) by
//                    one thread, then the K x N (lat, pow) tables by all
//                    threads through the bit-exact interpolator.
//   scan_kernel      1 CTA: exclusive scan of per-problem prefix counts,
//                    reset of argmin slots and counters.
//   prefix_kernel    grid-stride over every (problem, prefix of depth P):
//                    walk P levels, drop infeasible prefixes (meets_slo
//                    returns false at the first violation, so a violated
//                    prefix has no feasible completion), append survivors.
//   leaf_kernel      persistent, dynamically scheduled over the survivors:
//                    each thread sweeps the N^I completions of its prefix
//                    in increasing code order, with a division-free
//                    objective filter, and merges its (objective, code)
//                    minimum through a 128-bit CAS.
//   finalize_kernel  1 thread / problem: decode the argmin code.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "bs_internal.h"

using namespace bs;

namespace {

constexpr int kPrepThreads = 256;
constexpr int kLeafThreads = 256;
constexpr int kGreedyThreads = 256;
constexpr double kFilterScale = 1.0 + 0x1p-50;  // C in the filter bound
constexpr double kFilterMinBest = 0x1p-100;
constexpr double kFilterMinDen = 0x1p-900;
constexpr unsigned long long kItemPrefixBits = 44;

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

// Prefix depth of the exhaustive tree: the leaf sweep covers I = K - P
// levels per thread.
__host__ __device__ inline int prefix_depth(int K, int nc) {
  if (K <= 2) return 0;
  int P = K - 2;
  double np = 1.0;
  for (int i = 0; i < P; ++i) np *= nc;
  if (np > 16777216.0) P = K - 3;
  return P;
}

__host__ __device__ inline unsigned long long ipow(unsigned long long b, int e) {
  unsigned long long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
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
  if (threadIdx.x == 0) {
    int ok = 1;
    for (int k = 0; k < K; ++k)
      for (int f = 0; f < nc; ++f) {
        const double A = T->A[k][f];
        if (!(A >= 0.0) || !isfinite(A) || !isfinite(T->E[k][f])) ok = 0;
      }
    T->filter_ok = ok;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// exhaustive: prepare / scan / prefix / leaf / finalize
// ---------------------------------------------------------------------------
struct ExCtl {
  unsigned long long total_prefixes;
  unsigned long long work_count;  // survivors appended
  unsigned long long work_next;   // leaf scheduler cursor
};

__global__ void __launch_bounds__(kPrepThreads) prepare_kernel(DModels m, const DMpcCfg* cfgs, const DProblem* probs,
                                                               const DWaiting* W, const DRunning* R, DTables* tables,
                                                               unsigned long long* counts, int n) {
  __shared__ int s_status;
  const int d = blockIdx.x;
  if (d >= n) return;
  const DProblem pr = probs[d];
  const DMpcCfg& c = cfgs[pr.cfg];
  DTables* T = &tables[d];
  build_tables(m, pr, c, W + pr.wait_off, R + pr.run_off, T, &s_status);
  if (threadIdx.x == 0) {
    int st = s_status;
    if (st == BS_OK) {
      unsigned any = 0;
      for (int k = 0; k < T->K; ++k) any |= T->bad_lat[k] | T->bad_pow[k];
      if (any) st = BS_MODEL_ERROR;
    }
    T->status = st;
    unsigned long long np = 0;
    if (st == BS_OK && T->K > 0) np = ipow(static_cast<unsigned long long>(c.nc), prefix_depth(T->K, c.nc));
    counts[d] = np;
  }
}

// Single CTA: exclusive scan of counts (in place -> offsets), slot reset.
__global__ void __launch_bounds__(1024) scan_kernel(unsigned long long* counts, int n, Key128* best,
                                                    unsigned long long* feas, ExCtl* ctl) {
  __shared__ unsigned long long s_carry;
  __shared__ unsigned long long s_warp[32];
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    unsigned long long v = i < n ? counts[i] : 0ull;
    if (i < n) {
      best[i].obj = ~0ull;
      best[i].code = ~0ull;
      feas[i] = 0ull;
    }
    // inclusive warp scan
    unsigned long long x = v;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    const unsigned long long excl = s_carry + (warp > 0 ? s_warp[warp - 1] : 0ull) + x - v;
    if (i < n) counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctl->total_prefixes = s_carry;
    ctl->work_count = 0;
    ctl->work_next = 0;
  }
}

// State after levels [0, P) of code prefix p (digits MSD first).
struct PrefixState {
  double t, num, den;
  int last;
  bool ok;
};

__device__ __forceinline__ PrefixState walk_prefix(const DTables* __restrict__ T, int nc, int P,
                                                   unsigned long long p, bool check) {
  PrefixState s;
  s.t = 0.0;
  s.num = 0.0;
  s.den = 0.0;
  s.last = -1;
  s.ok = true;
  unsigned long long div = ipow(static_cast<unsigned long long>(nc), P > 0 ? P - 1 : 0);
  const double ttft = T->ttft;
  for (int k = 0; k < P; ++k) {
    const int f = static_cast<int>(p / div);
    p -= static_cast<unsigned long long>(f) * div;
    div /= static_cast<unsigned long long>(nc);
    if (k == 0) {
      s.t = T->T1[f];
    } else {
      s.t = __dadd_rn(s.t, f == s.last ? T->B0[k][f] : T->B1[k][f]);
    }
    s.num = __dadd_rn(s.num, T->E[k][f]);
    s.den = __dadd_rn(s.den, T->A[k][f]);
    s.last = f;
    if (check && __dsub_rn(s.t, T->minarr[k]) > ttft) {
      s.ok = false;
      return s;
    }
  }
  return s;
}

__device__ __forceinline__ int find_problem(const unsigned long long* offsets, int n, unsigned long long idx) {
  int lo = 0, hi = n - 1;  // last d with offsets[d] <= idx
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (offsets[mid] <= idx)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) prefix_kernel(const DTables* __restrict__ tables,
                                                     const unsigned long long* __restrict__ offsets, int n,
                                                     ExCtl* ctl, unsigned long long* __restrict__ work,
                                                     unsigned long long capacity) {
  const unsigned long long total = ctl->total_prefixes;
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (unsigned long long base = static_cast<unsigned long long>(blockIdx.x) * blockDim.x; base < total;
       base += stride) {
    const unsigned long long idx = base + threadIdx.x;
    bool keep = false;
    unsigned long long item = 0;
    if (idx < total) {
      const int d = find_problem(offsets, n, idx);
      const unsigned long long p = idx - offsets[d];
      const DTables* T = &tables[d];
      const int P = prefix_depth(T->K, T->nc);
      const PrefixState s = walk_prefix(T, T->nc, P, p, true);
      keep = s.ok;
      item = (static_cast<unsigned long long>(d) << kItemPrefixBits) | p;
    }
    // warp-aggregated append
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask == 0u) continue;
    unsigned long long slot0 = 0;
    if (lane == __ffs(mask) - 1) slot0 = atomicAdd(&ctl->work_count, static_cast<unsigned long long>(__popc(mask)));
    slot0 = __shfl_sync(0xffffffffu, slot0, __ffs(mask) - 1);
    if (keep) {
      const unsigned long long slot = slot0 + __popc(mask & ((1u << lane) - 1u));
      if (slot < capacity) work[slot] = item;
    }
  }
}

// Leaf sweep state per thread.
struct LeafAcc {
  double best;                // local minimum objective (+inf: none)
  unsigned long long code;    // its code
  double thr_scaled;          // fl(min(local, global hint) * C), +inf disables
  unsigned long long count;   // feasible leaves
};

__device__ __forceinline__ void set_threshold(LeafAcc& a, double hint) {
  // hint is NaN while the slot still holds its (~0, ~0) reset value
  const double thr = (a.best < hint || hint != hint) ? a.best : hint;
  a.thr_scaled = thr >= kFilterMinBest ? __dmul_rn(thr, kFilterScale) : (thr == 0.0 ? 0.0 : INFINITY);
}

// Last level (k = K - 1) for one state: sweep f = 0..nc-1.
__device__ __forceinline__ void sweep_last(const DTables* __restrict__ T, int k, int nc, double t, double num,
                                           double den, int last, unsigned long long code_base, bool filt,
                                           double hint, LeafAcc& a) {
  const double ttft = T->ttft;
  const double m = T->minarr[k];
  const double* __restrict__ B0 = T->B0[k];
  const double* __restrict__ B1 = T->B1[k];
  const double* __restrict__ E = T->E[k];
  const double* __restrict__ A = T->A[k];
#pragma unroll 4
  for (int f = 0; f < nc; ++f) {
    double tl;
    if (k == 0)
      tl = T->T1[f];
    else
      tl = __dadd_rn(t, f == last ? B0[f] : B1[f]);
    if (__dsub_rn(tl, m) > ttft) continue;  // dvfs.hpp:117
    a.count += 1;
    const double nl = __dadd_rn(num, E[f]);
    const double dl = __dadd_rn(den, A[f]);
    if (filt && nl > __dmul_rn(a.thr_scaled, dl)) continue;  // provably > current best
    const double obj = dl > 0.0 ? __ddiv_rn(nl, dl) : 0.0;  // dvfs.hpp:170
    const unsigned long long code = code_base + static_cast<unsigned long long>(f);
    if (obj < a.best || (obj == a.best && code < a.code)) {
      a.best = obj;
      a.code = code;
      set_threshold(a, hint);
    }
  }
}

__device__ __forceinline__ void sweep_two(const DTables* __restrict__ T, int k, int nc, double t, double num,
                                          double den, int last, unsigned long long code_base, double hint,
                                          LeafAcc& a) {
  const double ttft = T->ttft;
  const double m = T->minarr[k];
  for (int g = 0; g < nc; ++g) {
    double t2;
    if (k == 0)
      t2 = T->T1[g];
    else
      t2 = __dadd_rn(t, g == last ? T->B0[k][g] : T->B1[k][g]);
    if (__dsub_rn(t2, m) > ttft) continue;
    const double n2 = __dadd_rn(num, T->E[k][g]);
    const double d2 = __dadd_rn(den, T->A[k][g]);
    const bool filt = T->filter_ok && d2 >= kFilterMinDen;
    sweep_last(T, k + 1, nc, t2, n2, d2, g, (code_base + static_cast<unsigned long long>(g)) * nc, filt, hint, a);
  }
}

__global__ void __launch_bounds__(kLeafThreads) leaf_kernel(const DTables* __restrict__ tables, ExCtl* ctl,
                                                            const unsigned long long* __restrict__ work,
                                                            Key128* best, unsigned long long* feas) {
  __shared__ unsigned long long s_base;
  const unsigned long long count = ctl->work_count;
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (threadIdx.x == 0) s_base = atomicAdd(&ctl->work_next, static_cast<unsigned long long>(blockDim.x));
    __syncthreads();
    const unsigned long long base = s_base;
    __syncthreads();
    if (base >= count) break;
    const unsigned long long wi = base + threadIdx.x;
    int d = -1;
    LeafAcc a;
    a.best = INFINITY;
    a.code = ~0ull;
    a.count = 0;
    if (wi < count) {
      const unsigned long long item = work[wi];
      d = static_cast<int>(item >> kItemPrefixBits);
      const unsigned long long p = item & ((1ull << kItemPrefixBits) - 1ull);
      const DTables* T = &tables[d];
      const int K = T->K, nc = T->nc;
      const int P = prefix_depth(K, nc);
      const PrefixState s = walk_prefix(T, nc, P, p, false);
      const double hint = __longlong_as_double(static_cast<long long>(
          *reinterpret_cast<volatile unsigned long long*>(&best[d].obj)));
      set_threshold(a, hint);
      const int I = K - P;
      if (I == 1) {
        const bool filt = T->filter_ok && (P == 0 || s.den >= kFilterMinDen);
        sweep_last(T, P, nc, s.t, s.num, s.den, s.last, p * nc, filt, hint, a);
      } else if (I == 2) {
        sweep_two(T, P, nc, s.t, s.num, s.den, s.last, p * nc, hint, a);
      } else {  // I == 3
        const double ttft = T->ttft;
        for (int e = 0; e < nc; ++e) {
          double t3;
          if (P == 0)
            t3 = T->T1[e];
          else
            t3 = __dadd_rn(s.t, e == s.last ? T->B0[P][e] : T->B1[P][e]);
          if (__dsub_rn(t3, T->minarr[P]) > ttft) continue;
          sweep_two(T, P + 1, nc, t3, __dadd_rn(s.num, T->E[P][e]), __dadd_rn(s.den, T->A[P][e]), e,
                    (p * nc + static_cast<unsigned long long>(e)) * nc, hint, a);
        }
      }
    }
    // Merge: warp-level when the whole warp works on one problem.
    const int d0 = __shfl_sync(0xffffffffu, d, 0);
    const bool uniform = __all_sync(0xffffffffu, d == d0) && d0 >= 0;
    if (uniform) {
      unsigned long long c = a.count;
      unsigned long long bo = a.best < INFINITY ? static_cast<unsigned long long>(__double_as_longlong(a.best)) : ~0ull;
      unsigned long long bc = a.code;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        const unsigned long long oo = __shfl_xor_sync(0xffffffffu, bo, o);
        const unsigned long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (key_less(oo, oc, bo, bc)) {
          bo = oo;
          bc = oc;
        }
      }
      if (lane == 0) {
        if (c) atomicAdd(&feas[d0], c);
        if (bo != ~0ull) atomic_min_key(&best[d0], bo, bc);
      }
    } else if (d >= 0) {
      if (a.count) atomicAdd(&feas[d], a.count);
      if (a.best < INFINITY)
        atomic_min_key(&best[d], static_cast<unsigned long long>(__double_as_longlong(a.best)), a.code);
    }
  }
}

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
constexpr int kNumEvents = 6;

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
  unsigned long long capacity = 0;  // exhaustive worklist capacity
  DTables* dT = nullptr;
  unsigned long long* dCounts = nullptr;
  ExCtl* dCtl = nullptr;
  Key128* dBest = nullptr;
  unsigned long long* dFeas = nullptr;
  unsigned long long* dWork = nullptr;
  DMpcOut* dOut = nullptr;
  DLevel* dLv = nullptr;
  cudaEvent_t ev[kNumEvents] = {};
  bool have_events = false;
};

size_t tables_bytes(int n) { return sizeof(DTables) * static_cast<size_t>(n); }
size_t counts_bytes(int n) { return ((8ull * n + 63) / 64) * 64 + sizeof(ExCtl) + 64; }
size_t best_bytes(int n) { return (sizeof(Key128) + 8ull) * static_cast<size_t>(n); }
size_t out_bytes(int n) { return sizeof(DMpcOut) * static_cast<size_t>(n); }
size_t levels_bytes(int n) { return sizeof(DLevel) * BS_MAX_LEVELS * static_cast<size_t>(n); }

// Packs the problems (one H2D copy) and validates configurations.
int run_pack(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies, int n_cfgs,
             const bs_mpc_problem* problems, int n, int mode, MpcRun* run) {
  run->mode = mode;
  run->n = n;
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
  run->cfg_of.resize(n);
  run->target.resize(n);
  run->capacity = 0;
  for (int i = 0; i < n; ++i) {
    run->cfg_of[i] = problems[i].cfg_index;
    run->target[i] = problems[i].snap.target_freq_mhz;
    const DMpcCfg& c = run->hc[problems[i].cfg_index];
    if (mode == kExhaustive) run->capacity += ipow(static_cast<unsigned long long>(c.nc), prefix_depth(c.horizon, c.nc));
  }
  if (n > (1 << 19)) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: at most 2^19 problems per call");
  return BS_OK;
}

void run_bind_exhaustive(MpcRun* run, void* tables, void* counts, void* best, void* work, void* out) {
  const int n = run->n;
  run->dT = static_cast<DTables*>(tables);
  run->dCounts = static_cast<unsigned long long*>(counts);
  run->dCtl = reinterpret_cast<ExCtl*>(static_cast<char*>(counts) + ((8ull * n + 63) / 64) * 64);
  run->dBest = static_cast<Key128*>(best);
  run->dFeas = reinterpret_cast<unsigned long long*>(run->dBest + n);
  run->dWork = static_cast<unsigned long long*>(work);
  run->dOut = static_cast<DMpcOut*>(out);
}

#define BS_REC(i)                                                         \
  do {                                                                    \
    if (timing) BS_CUDA_TRY(ctx, cudaEventRecord(run->ev[i], ctx->stream)); \
  } while (0)

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
  prepare_kernel<<<n, kPrepThreads, 0, ctx->stream>>>(models->dm, pk.cfgs, pk.problems, pk.waiting, pk.running,
                                                      run->dT, run->dCounts, n);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(1);
  scan_kernel<<<1, 1024, 0, ctx->stream>>>(run->dCounts, n, run->dBest, run->dFeas, run->dCtl);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(2);
  prefix_kernel<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(run->dT, run->dCounts, n, run->dCtl, run->dWork,
                                                             run->capacity);
  BS_LAUNCH_CHECK(ctx);
  BS_REC(3);
  leaf_kernel<<<ctx->sm_count * 8, kLeafThreads, 0, ctx->stream>>>(run->dT, run->dCtl, run->dWork, run->dBest,
                                                                   run->dFeas);
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
  DMpcOut* hOut = static_cast<DMpcOut*>(ctx->host_buf(kSlotOut, out_bytes(n)));
  DLevel* hLv = nullptr;
  if (!hOut) return set_error(ctx, BS_CUDA_ERROR, "mpc: host allocation failed");
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(hOut, run->dOut, out_bytes(n), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->last_d2h = out_bytes(n);
  if (run->mode == kGreedy) {
    hLv = static_cast<DLevel*>(ctx->host_buf(kSlotLevels, levels_bytes(n)));
    if (!hLv) return set_error(ctx, BS_CUDA_ERROR, "mpc: host allocation failed");
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(hLv, run->dLv, levels_bytes(n), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->last_d2h += levels_bytes(n);
  }
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
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
    void* t = ctx->dev_buf(kSlotTables, tables_bytes(n));
    void* c = ctx->dev_buf(kSlotCounts, counts_bytes(n));
    void* b = ctx->dev_buf(kSlotBest, best_bytes(n));
    void* w = ctx->dev_buf(kSlotWork, 8ull * run.capacity + 8);
    void* o = ctx->dev_buf(kSlotOut, out_bytes(n));
    if (!t || !c || !b || !w || !o)
      return set_error(ctx, BS_CUDA_ERROR, "mpc exhaustive: device allocation failed (%llu work items)",
                       run.capacity);
    run_bind_exhaustive(&run, t, c, b, w, o);
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
  const size_t a = 256;
  auto up = [a](size_t x) { return (x + a - 1) / a * a; };
  const size_t blob = up(run.pk.h2d_bytes);
  size_t total = blob;
  size_t o_t = 0, o_c = 0, o_b = 0, o_w = 0, o_o = 0, o_l = 0;
  if (mode == kExhaustive) {
    o_t = total;
    total += up(tables_bytes(n));
    o_c = total;
    total += up(counts_bytes(n));
    o_b = total;
    total += up(best_bytes(n));
    o_w = total;
    total += up(8ull * run.capacity + 8);
  } else {
    o_l = total;
    total += up(levels_bytes(n));
  }
  o_o = total;
  total += up(out_bytes(n));
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
    run_bind_exhaustive(&run, m + o_t, m + o_c, m + o_b, m + o_w, m + o_o);
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
  if (work_capacity) *work_capacity = plan->run.capacity;
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

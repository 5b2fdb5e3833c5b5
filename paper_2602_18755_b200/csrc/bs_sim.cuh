// bs_sim.cuh — device restatement of one simulated instance at a fixed
// frequency (no controller: no switches, no safety deadline), the case every
// goodput probe and E_c evaluation of the placement search runs
// (placement.hpp:166-178, 228-230 -> simulate_instance, simulator.hpp:667-739).
//
// Each function is a single sequential event loop (one GPU thread per
// probe); probes are independent, so a grid of (candidate x rate step x
// replicate) probes runs them all at once.  Arithmetic follows the reference
// op for op in FP64 without contraction:
//   t_done  = seg_start + 1.0 * L                     (simulator.hpp:362)
//   energy  = p * (to - from) / 1000.0                (simulator.hpp:210, 225)
//   sums    in record order                           (simulator.hpp:108-122)
//   ttft    = done - arrival; decode gaps token-to-token (simulator.hpp:69-89)
#pragma once

#include "bs_device.cuh"

namespace bs {

// A probe's requests: the kept indices (increasing) into the base trace.
struct SimTrace {
  const double* arrival;
  const long long* input;
  const long long* output;
  const int* kept;  // kept[i] = base index of the i-th kept request
  long long n;      // number of kept requests
  double duration_ms;
};

// Goodput-search pruning.  max_goodput (placement.hpp:154-199) visits k_max,
// then 1, then lo + (hi - lo) / 2 until hi - lo <= 1; which k it visits
// depends only on the outcomes along that path.  A probe grid evaluates all k
// at once, so every probe publishes its outcome, and a probe whose k can no
// longer be on the path, given the outcomes published so far, is skipped (at
// start) or abandoned (polled during the run).  Outcomes only accumulate and
// each is final, so "off the path" is final too, and the probes the host
// replay reads (the path, and (k*, replicate 0) for E_c) always run to their
// exact end.
enum : int { kProbePending = 0, kProbePass = 1, kProbeFail = 2, kProbeErr = 3, kProbeSkipped = 4 };
constexpr int kSimAborted = -7;  // SimOut.status of an abandoned probe

struct SearchView {
  const int* st;  // outcome codes of one candidate's probes, index (k - 1) * reps + j
  long long k_max;
  int reps;
};

// feasible(k) of max_goodput as far as published: every replicate in order
// (placement.hpp:165-178): 1 pass, 0 fail, -1 ModelError, 2 not known yet.
__device__ __forceinline__ int search_outcome(const SearchView& v, long long k) {
  const volatile int* s = v.st + (k - 1) * v.reps;
  for (int j = 0; j < v.reps; ++j) {
    const int c = s[j];
    if (c == kProbePass) continue;
    if (c == kProbeFail) return 0;
    if (c == kProbeErr) return -1;
    return 2;
  }
  return 1;
}

// Can the reference's search still visit k?  Walks the path through the
// published outcomes; an unknown outcome leaves every k of its open interval
// possible.
__device__ inline bool search_alive(const SearchView& v, long long k) {
  if (k == v.k_max) return true;
  int o = search_outcome(v, v.k_max);
  if (o == 2) return true;
  if (o != 0) return false;  // saturated, or a ModelError ended the search
  if (k == 1) return true;
  o = search_outcome(v, 1);
  if (o == 2) return true;
  if (o != 1) return false;
  long long lo = 1, hi = v.k_max;
  while (hi - lo > 1) {
    if (k <= lo || k >= hi) return false;
    const long long mid = lo + (hi - lo) / 2;
    if (k == mid) return true;
    o = search_outcome(v, mid);
    if (o == 2) return true;
    if (o < 0) return false;
    if (o == 1)
      lo = mid;
    else
      hi = mid;
  }
  return false;
}

struct SimParams {
  int tp;
  double freq;
  long long max_batch_tokens;
  long long max_batch_requests;
  long long kv_capacity;
  int chunking;
  double ttft_bound;
  double tpot_bound;
  int early_exit;  // stop at the first SLO violation (feasibility only)
  const SearchView* search;  // non-null: abandon the run once rate step k is off the search path
  long long k;
};

constexpr int kSearchPollPrefill = 64;  // batches between polls (scalar event loop)
constexpr int kSearchPollDecode = 8;    // event windows between polls (warp simulator)

struct SimOut {
  int status;      // BS_OK, BS_SIMULATION_ERROR, BS_MODEL_ERROR
  int model_err;   // 1 latency, 2 power, 3 idle (ModelError kind)
  int meets_slo;   // sim_meets_slo (placement.hpp:119-131)
  long long completed;
  double busy_j;   // SimResult::busy_energy_j
  double idle_j;   // SimResult::idle_energy_j
  double horizon_ms;
  long long batches;
};

// Resident of a decode instance: retires at the end of iteration `retire`.
struct Resident {
  long long retire;
  long long need;  // input + output (KV reservation and final context)
};

__device__ __forceinline__ void heap_push(Resident* h, int& n, Resident r) {
  int i = n++;
  while (i > 0) {
    const int p = (i - 1) >> 1;
    if (h[p].retire <= r.retire) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = r;
}

__device__ __forceinline__ Resident heap_pop(Resident* h, int& n) {
  const Resident top = h[0];
  const Resident last = h[--n];
  int i = 0;
  for (;;) {
    int c = 2 * i + 1;
    if (c >= n) break;
    if (c + 1 < n && h[c + 1].retire < h[c].retire) ++c;
    if (last.retire <= h[c].retire) break;
    h[i] = h[c];
    i = c;
  }
  if (n > 0) h[i] = last;
  return top;
}

// A grid specialised to one instance.  tp and freq_mhz are constant for a
// whole simulation, so their bracketing (lo, frac) is computed once.  An axis
// whose frac is exactly 0 (a fixed value on a knot -- ladder rungs always
// are) or that has a single knot contributes the factor 1.0 - 0 = 1.0 to
// every low corner and weight 0 to every high corner, which
// NdGrid::interpolate then skips (perfmodel.hpp:183-190); at the last knot
// (frac exactly 1) the roles swap.  Dropping such axes therefore leaves every
// weight product, the corner order and the sum bit-identical while the
// corner loop shrinks from 2^D to 2^(active axes).
// sum_len / n_requests are bracketed per call by binary search (the index
// std::upper_bound finds).
struct FastGrid {
  int na;                      // active axes, in axis order
  int bad;
  int role[kMaxRank];          // role of each active axis
  int n[kMaxRank];
  const double* knots[kMaxRank];
  long long stride[kMaxRank];  // row-major stride of each active axis
  int fixed[kMaxRank];         // 1: tp / freq (lo, frac below)
  int lo[kMaxRank];
  double frac[kMaxRank];
  long long base;              // flat offset of the dropped axes' lo
  const double* values;
};

__host__ __device__ __forceinline__ void bracket(const double* k, int n, double x, int* lo, double* frac) {
  const double k0 = k[0], kn = k[n - 1];
  if (x < k0 || x > kn) x = x < k0 ? k0 : (kn < x ? kn : x);
  if (n == 1) {
    *lo = 0;
    *frac = 0.0;
    return;
  }
  int a = 0, b = n;  // first index with k[i] > x
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (x < k[mid])
      b = mid;
    else
      a = mid + 1;
  }
  int hi = a < 1 ? 1 : (a > n - 1 ? n - 1 : a);
  *lo = hi - 1;
#ifdef __CUDA_ARCH__
  *frac = __ddiv_rn(__dsub_rn(x, k[hi - 1]), __dsub_rn(k[hi], k[hi - 1]));
#else  // the same correctly rounded IEEE operations on the host (-ffp-contract=off)
  *frac = (x - k[hi - 1]) / (k[hi] - k[hi - 1]);
#endif
}

// rd: the grid whose knots are read (the device grid, or its host mirror);
// st: the grid whose pointers the FastGrid keeps (always the device grid).
__host__ __device__ inline FastGrid fast_grid2(const DGrid& rd, const DGrid& st_grid, int tp, double freq) {
  const DGrid& g = rd;
  FastGrid f;
  f.na = 0;
  f.bad = g.bad_axis;
  f.values = st_grid.values;
  f.base = 0;
  long long stride[kMaxRank];
  long long st = 1;
  for (int d = g.rank - 1; d >= 0; --d) {
    stride[d] = st;
    st *= g.n[d];
  }
  for (int d = 0; d < g.rank; ++d) {
    if (g.n[d] == 1) continue;  // single knot: lo 0, factor 1.0, high corners weight 0
    const bool fixed_axis = g.role[d] == BS_AXIS_TP || g.role[d] == BS_AXIS_FREQ;
    int lo = 0;
    double fr = 0.0;
    if (fixed_axis) {
      bracket(g.knots[d], g.n[d], g.role[d] == BS_AXIS_TP ? static_cast<double>(tp) : freq, &lo, &fr);
      if (fr == 0.0) {  // on a knot: drop the axis, keep its lo in the base offset
        f.base += lo * stride[d];
        continue;
      }
      if (fr == 1.0) {  // on the axis' last knot (hi = lo + 1, frac 1): every low corner has weight
        // 1 - 1 = 0 and is skipped, every high corner's weight is multiplied by exactly 1.0 -- drop
        // the axis with its high knot in the base offset (same values, same corner order)
        f.base += (lo + 1) * stride[d];
        continue;
      }
    }
    const int a = f.na++;
    f.role[a] = g.role[d];
    f.n[a] = g.n[d];
    f.knots[a] = st_grid.knots[d];
    f.stride[a] = stride[d];
    f.fixed[a] = fixed_axis ? 1 : 0;
    f.lo[a] = lo;
    f.frac[a] = fr;
  }
  return f;
}

__device__ __forceinline__ FastGrid fast_grid(const DGrid& g, int tp, double freq) { return fast_grid2(g, g, tp, freq); }

// bracket() as a branch-free search: std::upper_bound's index in a sorted
// knot vector (the number of knots k with !(x < k)) by halving steps whose
// count depends on n only, so the lanes of a warp never diverge.
__device__ __forceinline__ void bracket_count(const double* __restrict__ k, int n, double x, int* lo, double* frac) {
  const double k0 = __ldg(k), kn = __ldg(k + n - 1);
  if (!(x < kn)) {  // at or beyond the last knot: the last interval, (kn - kp) / (kn - kp) == 1 exactly
    const double d = __dsub_rn(kn, __ldg(k + n - 2));
    if (d > 0.0 && d < INFINITY) {
      *lo = n - 2;
      *frac = 1.0;
      return;
    }
  }
  if (x < k0 || x > kn) x = x < k0 ? k0 : (kn < x ? kn : x);
  int base = 0;
  for (int len = n; len > 1;) {
    const int half = len >> 1;
    base = !(x < __ldg(k + base + half)) ? base + half : base;
    len -= half;
  }
  const int cnt = base + (!(x < __ldg(k + base)) ? 1 : 0);
  const int hi = cnt < 1 ? 1 : (cnt > n - 1 ? n - 1 : cnt);
  *lo = hi - 1;
  const double klo = __ldg(k + hi - 1), khi = __ldg(k + hi);
  *frac = __ddiv_rn(__dsub_rn(x, klo), __dsub_rn(khi, klo));
}

// The (lo, frac) of every active axis of a FastGrid at one query.
struct FastBrk {
  int lo[kMaxRank];
  double frac[kMaxRank];
};

__device__ __forceinline__ void fast_brackets(const FastGrid& g, long long n_req, long long sum_len, FastBrk& b) {
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a >= g.na) break;
    if (g.fixed[a]) {
      b.lo[a] = g.lo[a];
      b.frac[a] = g.frac[a];
    } else {  // active varying axes have >= 2 knots (single-knot axes are dropped)
      bracket_count(g.knots[a], g.n[a], static_cast<double>(g.role[a] == BS_AXIS_SUM_LEN ? sum_len : n_req),
                    &b.lo[a], &b.frac[a]);
    }
  }
}

// The corner sum of NdGrid::interpolate over the active axes.
__device__ __forceinline__ double fast_corners(const FastGrid& g, const FastBrk& b) {
  double acc = 0.0;
  if (g.na == 2) {  // the common case: (sum_len, n_requests) with tp and freq on knots
    const double w0[2] = {__dsub_rn(1.0, b.frac[0]), b.frac[0]};
    const double w1[2] = {__dsub_rn(1.0, b.frac[1]), b.frac[1]};
#pragma unroll
    for (int mask = 0; mask < 4; ++mask) {
      const int h0 = mask & 1, h1 = mask >> 1;
      const double weight = __dmul_rn(__dmul_rn(1.0, w0[h0]), w1[h1]);
      const long long flat = g.base + (b.lo[0] + h0) * g.stride[0] + (b.lo[1] + h1) * g.stride[1];
      if (weight != 0.0) acc = __dadd_rn(acc, __dmul_rn(weight, __ldg(g.values + flat)));
    }
    return acc;
  }
  if (g.na == 1) {  // e.g. prefill power over sum_len
    const double w0[2] = {__dsub_rn(1.0, b.frac[0]), b.frac[0]};
#pragma unroll
    for (int h0 = 0; h0 < 2; ++h0) {
      const double weight = __dmul_rn(1.0, w0[h0]);
      const long long flat = g.base + (b.lo[0] + h0) * g.stride[0];
      if (weight != 0.0) acc = __dadd_rn(acc, __dmul_rn(weight, __ldg(g.values + flat)));
    }
    return acc;
  }
  const int corners = 1 << g.na;
  for (int mask = 0; mask < corners; ++mask) {
    double weight = 1.0;
    long long flat = g.base;
#pragma unroll
    for (int a = 0; a < kMaxRank; ++a) {
      if (a >= g.na) break;
      const int high = (mask >> a) & 1;
      weight = __dmul_rn(weight, high ? b.frac[a] : __dsub_rn(1.0, b.frac[a]));
      flat += (b.lo[a] + high) * g.stride[a];
    }
    if (weight != 0.0) acc = __dadd_rn(acc, __dmul_rn(weight, __ldg(g.values + flat)));
  }
  return acc;
}

__device__ __forceinline__ double fast_interp(const FastGrid& g, long long n_req, long long sum_len) {
  FastBrk b;
  fast_brackets(g, n_req, sum_len, b);
  return fast_corners(g, b);
}

// fast_brackets in two parts: the fixed axes and the n_requests axis (fixed
// over a decode event window, where the batch size is constant), then the
// sum_len axis per query.  Together they equal fast_brackets.
__device__ __forceinline__ void fast_brackets_nreq(const FastGrid& g, long long n_req, FastBrk& b) {
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a >= g.na) break;
    if (g.fixed[a]) {
      b.lo[a] = g.lo[a];
      b.frac[a] = g.frac[a];
    } else if (g.role[a] != BS_AXIS_SUM_LEN) {
      bracket_count(g.knots[a], g.n[a], static_cast<double>(n_req), &b.lo[a], &b.frac[a]);
    }
  }
}

__device__ __forceinline__ void fast_brackets_sum(const FastGrid& g, long long sum_len, FastBrk& b) {
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a >= g.na) break;
    if (!g.fixed[a] && g.role[a] == BS_AXIS_SUM_LEN)
      bracket_count(g.knots[a], g.n[a], static_cast<double>(sum_len), &b.lo[a], &b.frac[a]);
  }
}

// Two reductions of the same grid whose active axes, knots and fixed-axis
// brackets coincide (only the dropped axes' offsets differ, e.g. the same tp
// at two on-knot frequencies): brackets of one serve the other.
__host__ __device__ inline bool fast_same_brackets(const FastGrid& a, const FastGrid& b) {
  if (a.na != b.na || a.bad != b.bad || a.values != b.values) return false;
  for (int i = 0; i < a.na; ++i) {
    if (a.role[i] != b.role[i] || a.n[i] != b.n[i] || a.knots[i] != b.knots[i] || a.stride[i] != b.stride[i] ||
        a.fixed[i] != b.fixed[i])
      return false;
    if (a.fixed[i] && (a.lo[i] != b.lo[i] || a.frac[i] != b.frac[i])) return false;
  }
  return true;
}

// Same bracket inputs (active axes, their knots and the fixed axes'
// brackets) regardless of values, strides and offsets: one FastBrk serves
// both reductions (e.g. the latency grids of two rungs, or of the simulator's
// and the controller's models when they share knot storage).
__host__ __device__ inline bool fast_same_axes(const FastGrid& a, const FastGrid& b) {
  if (a.na != b.na || a.bad != b.bad) return false;
  for (int i = 0; i < a.na; ++i) {
    if (a.role[i] != b.role[i] || a.n[i] != b.n[i] || a.knots[i] != b.knots[i] || a.fixed[i] != b.fixed[i])
      return false;
    if (a.fixed[i] && (a.lo[i] != b.lo[i] || a.frac[i] != b.frac[i])) return false;
  }
  return true;
}

// fast_brackets by one warp (all lanes call it with the same query): lane i
// tests knot i of each varying axis and a ballot counts the knots <= x, the
// same (lo, frac) as bracket_count.  Lane 0 stores into `out` (shared memory).
__device__ __forceinline__ void warp_brackets(const FastGrid& g, long long n_req, long long sum_len, FastBrk* out) {
  const int lane = threadIdx.x & 31;
  for (int a = 0; a < g.na; ++a) {
    int lo;
    double fr;
    if (g.fixed[a]) {
      lo = g.lo[a];
      fr = g.frac[a];
    } else {
      const double* __restrict__ k = g.knots[a];
      const int n = g.n[a];
      double x = static_cast<double>(g.role[a] == BS_AXIS_SUM_LEN ? sum_len : n_req);
      const double k0 = __ldg(k), kn = __ldg(k + n - 1);
      if (x < k0 || x > kn) x = x < k0 ? k0 : (kn < x ? kn : x);
      int cnt = 0;
      for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        cnt += __popc(__ballot_sync(0xffffffffu, i < n && !(x < __ldg(k + i))));
      }
      const int hi = cnt < 1 ? 1 : (cnt > n - 1 ? n - 1 : cnt);
      lo = hi - 1;
      const double klo = __ldg(k + hi - 1), khi = __ldg(k + hi);
      fr = __ddiv_rn(__dsub_rn(x, klo), __dsub_rn(khi, klo));
    }
    if (lane == 0) {
      out->lo[a] = lo;
      out->frac[a] = fr;
    }
  }
  __syncwarp();
}

// predict_latency / predict_power at the instance's (tp, freq); false on
// ModelError (perfmodel.hpp:264, 270).
__device__ __forceinline__ bool predict_at(const FastGrid& g, long long n_req, long long sum_len, double* out) {
  if (g.bad) return false;
  const double v = fast_interp(g, n_req, sum_len);
  *out = v;
  return model_value_ok(v);
}

// simulate_prefill_instance (simulator.hpp:278-409) without a controller,
// followed by simulate_instance's accounting (667-739).
__device__ inline SimOut simulate_prefill(const DModels& m, const SimTrace& tr, const SimParams& p) {
  SimOut o;
  o.status = BS_OK;
  o.model_err = 0;
  o.meets_slo = 1;
  o.completed = 0;
  o.busy_j = 0.0;
  o.idle_j = 0.0;
  o.batches = 0;
  const FastGrid lat = fast_grid(m.grid[0], p.tp, p.freq);
  const FastGrid pw = fast_grid(m.grid[2], p.tp, p.freq);
  double idle_w = 0.0;
  const bool have_idle = idle_power(m.idle, p.tp, p.freq, &idle_w);
  double now = 0.0;
  long long arr = 0;    // next kept request not yet queued
  long long qhead = 0;  // queue = kept [qhead, arr)
  long long head_rem = 0;
  bool active = false;
  double seg_start = 0.0, t_done = 0.0, bp = 0.0;
  long long b_end = 0;     // batch covers queue entries [qhead, b_end)
  bool b_partial = false;  // last entry only partially taken
  long long b_rem_after = 0;

  auto record_idle = [&](double from, double to) -> bool {
    if (to <= from) return true;
    if (!have_idle) {
      o.status = BS_MODEL_ERROR;
      o.model_err = 3;
      return false;
    }
    o.idle_j = __dadd_rn(o.idle_j, __ddiv_rn(__dmul_rn(idle_w, __dsub_rn(to, from)), 1000.0));
    return true;
  };

  int poll = 0;
  for (;;) {
    if (!active && qhead < arr) {
      if (p.search && ++poll == kSearchPollPrefill) {
        poll = 0;
        if (!search_alive(*p.search, p.k)) {
          o.status = kSimAborted;
          return o;
        }
      }
      while (arr < tr.n && tr.arrival[tr.kept[arr]] <= now) ++arr;  // simulator.hpp:350-353
      // form_prefill_batch (scheduler.hpp:40-66) over the queue
      long long tokens = 0, npick = 0, sum = 0;
      b_partial = false;
      b_end = qhead;
      for (long long i = qhead; i < arr; ++i) {
        if (npick >= p.max_batch_requests) break;
        const long long rem = i == qhead ? head_rem : tr.input[tr.kept[i]];
        if (rem <= 0) {
          o.status = BS_SIMULATION_ERROR;
          o.meets_slo = 0;
          return o;
        }
        if (p.chunking) {
          const long long room = p.max_batch_tokens - tokens;
          if (room <= 0) break;
          const long long take = rem < room ? rem : room;
          ++npick;
          sum += take;
          tokens += take;
          if (take < rem) {
            b_partial = true;
            b_rem_after = rem - take;
            b_end = i + 1;
            break;
          }
          b_end = i + 1;
        } else {
          if (rem > p.max_batch_tokens) {
            if (npick == 0) {
              ++npick;
              sum += rem;
              b_end = i + 1;
            }
            break;
          }
          if (tokens + rem > p.max_batch_tokens) break;
          ++npick;
          sum += rem;
          tokens += rem;
          b_end = i + 1;
        }
      }
      double L;
      if (!predict_at(lat, npick, sum, &L)) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 1;
        return o;
      }
      if (!predict_at(pw, npick, sum, &bp)) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 2;
        return o;
      }
      seg_start = now;
      t_done = __dadd_rn(seg_start, __dmul_rn(1.0, L));
      active = true;
      continue;
    }
    const double t_arr = arr < tr.n ? fmax(tr.arrival[tr.kept[arr]], now) : INFINITY;
    if (active && t_done <= t_arr) {
      if (t_done > seg_start) {  // record_segment (simulator.hpp:213-228)
        o.busy_j = __dadd_rn(o.busy_j, __ddiv_rn(__dmul_rn(bp, __dsub_rn(t_done, seg_start)), 1000.0));
        ++o.batches;
      }
      // completions: every fully taken entry of [qhead, b_end)
      const long long full_end = b_partial ? b_end - 1 : b_end;
      for (long long i = qhead; i < full_end; ++i) {
        const double ttft = __dsub_rn(t_done, tr.arrival[tr.kept[i]]);
        if (ttft > p.ttft_bound) {
          o.meets_slo = 0;
          if (p.early_exit) return o;
        }
      }
      o.completed += full_end - qhead;
      qhead = full_end;
      if (b_partial) {
        head_rem = b_rem_after;
      } else if (qhead < tr.n) {
        head_rem = tr.input[tr.kept[qhead]];
      }
      active = false;
      now = t_done;
      continue;
    }
    if (t_arr == INFINITY) break;
    if (!active && !record_idle(now, t_arr)) return o;
    now = fmax(now, t_arr);
    if (arr == qhead && !active) head_rem = tr.input[tr.kept[arr]];
    ++arr;
  }
  o.horizon_ms = fmax(tr.duration_ms, now);  // simulator.hpp:731
  record_idle(now, o.horizon_ms);
  return o;
}

// simulate_decode_instance (simulator.hpp:441-578) without a controller.
// `heap` is per-thread scratch with room for max_batch_requests residents.
__device__ inline SimOut simulate_decode(const DModels& m, const SimTrace& tr, const SimParams& p, Resident* heap,
                                  int heap_cap) {
  SimOut o;
  o.status = BS_OK;
  o.model_err = 0;
  o.meets_slo = 1;
  o.completed = 0;
  o.busy_j = 0.0;
  o.idle_j = 0.0;
  o.batches = 0;
  const FastGrid lat = fast_grid(m.grid[1], p.tp, p.freq);
  const FastGrid pw = fast_grid(m.grid[3], p.tp, p.freq);
  double idle_w = 0.0;
  const bool have_idle = idle_power(m.idle, p.tp, p.freq, &idle_w);
  double now = 0.0;
  long long arr = 0;    // next kept request not yet in `waiting`
  long long whead = 0;  // waiting = kept [whead, arr), FIFO admission
  int n_res = 0;
  long long sum_ctx = 0, reserved = 0, it = 0;
  bool active = false;
  double seg_start = 0.0, t_done = 0.0, bp = 0.0, prev_end = 0.0;
  int n_new = 0;            // residents admitted before the running iteration
  double new_min_arr = 0.0;  // smallest arrival among them (first-token gap)

  auto record_idle = [&](double from, double to) -> bool {
    if (to <= from) return true;
    if (!have_idle) {
      o.status = BS_MODEL_ERROR;
      o.model_err = 3;
      return false;
    }
    o.idle_j = __dadd_rn(o.idle_j, __ddiv_rn(__dmul_rn(idle_w, __dsub_rn(to, from)), 1000.0));
    return true;
  };

  while (arr < tr.n || whead < arr || n_res > 0) {
    if (!active) {
      while (arr < tr.n && tr.arrival[tr.kept[arr]] <= now) ++arr;  // simulator.hpp:516-518
      // admit (simulator.hpp:455-470)
      n_new = 0;
      while (whead < arr) {
        const int r = tr.kept[whead];
        const long long need = tr.input[r] + tr.output[r];
        if (need > p.kv_capacity) {
          o.status = BS_SIMULATION_ERROR;
          o.meets_slo = 0;
          return o;
        }
        if (n_res >= p.max_batch_requests) break;
        if (reserved + need > p.kv_capacity) break;
        if (n_res >= heap_cap) {
          o.status = BS_PARAMETER_ERROR;  // device scratch too small (host sizes it to max_batch_requests)
          return o;
        }
        Resident rs;
        rs.retire = it + tr.output[r] - 1;
        rs.need = need;
        heap_push(heap, n_res, rs);
        reserved += need;
        sum_ctx += tr.input[r];
        const double a = tr.arrival[r];
        new_min_arr = n_new == 0 ? a : (a < new_min_arr ? a : new_min_arr);
        ++n_new;
        ++whead;
      }
      if (n_res == 0) {
        if (arr >= tr.n && whead >= arr) break;
        if (whead < arr) {  // simulator.hpp:522-526
          o.status = BS_SIMULATION_ERROR;
          o.meets_slo = 0;
          return o;
        }
        const double t_next = fmax(tr.arrival[tr.kept[arr]], now);
        if (!record_idle(now, t_next)) return o;  // idle_until without pending switches
        now = t_next;
        continue;
      }
      double L;
      if (!predict_at(lat, n_res, sum_ctx, &L)) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 1;
        return o;
      }
      if (!predict_at(pw, n_res, sum_ctx, &bp)) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 2;
        return o;
      }
      seg_start = now;
      t_done = __dadd_rn(seg_start, __dmul_rn(1.0, L));
      active = true;
      continue;
    }
    const double t_arr = arr < tr.n ? fmax(tr.arrival[tr.kept[arr]], now) : INFINITY;
    if (t_done <= t_arr) {
      if (t_done > seg_start) {
        o.busy_j = __dadd_rn(o.busy_j, __ddiv_rn(__dmul_rn(bp, __dsub_rn(t_done, seg_start)), 1000.0));
        ++o.batches;
      }
      // token gaps (RequestRecord::max_tbt_ms, simulator.hpp:81-89)
      if (n_res > n_new && __dsub_rn(t_done, prev_end) > p.tpot_bound) {
        o.meets_slo = 0;
        if (p.early_exit) return o;
      }
      if (n_new > 0 && __dsub_rn(t_done, new_min_arr) > p.tpot_bound) {
        o.meets_slo = 0;
        if (p.early_exit) return o;
      }
      n_new = 0;
      sum_ctx += n_res;  // every resident emits a token
      while (n_res > 0 && heap[0].retire <= it) {
        const Resident r = heap_pop(heap, n_res);
        reserved -= r.need;
        sum_ctx -= r.need;
        ++o.completed;
      }
      ++it;
      prev_end = t_done;
      active = false;
      now = t_done;
      continue;
    }
    if (t_arr == INFINITY) {
      o.status = BS_SIMULATION_ERROR;  // "decode: event starvation"
      o.meets_slo = 0;
      return o;
    }
    ++arr;
    now = t_arr;
  }
  o.horizon_ms = fmax(tr.duration_ms, now);
  record_idle(now, o.horizon_ms);
  return o;
}

// Warp-cooperative simulate_decode_instance (simulator.hpp:441-578), no
// controller, bit-identical to simulate_decode.
//
// The batch only gains members at an admission, and admissions happen only at
// the first boundary after an arrival (or, while a request waits for KV room,
// after a retirement).  Between two such points the composition of every
// future iteration is known in advance: a resident admitted at iteration i
// with o output tokens retires at the end of iteration i + o - 1, so the
// batch size n and summed context s of iteration it0 + l follow from the
// residents sorted by retirement (n = residents not yet retired, s = the
// context at it0 plus every token generated since, minus the retired
// residents' final contexts).  The 32 lanes derive those features for 32
// consecutive iterations with warp scans, evaluate the latency and power
// interpolations in parallel, lane 0 runs the only truly serial part (the
// FP64 chain t_done = t_start + 1.0 * L), and the warp locates the first
// iteration whose end reaches the next arrival (the window stops there),
// checks every token gap and accumulates the energy terms in record order.
// All lanes hold the same scalar state (redundant, divergence-free); the
// residents (an array sorted by retirement) and the per-chunk arrays live in
// the warp's shared memory.
struct WarpScratch {
  Resident* heap;  // heap_cap entries: the residents, ascending retirement
  double* L;       // 32
  double* P;       // 32
  double* T;       // 32
  double* nfrac;   // heap_cap + 1 entries (or null): the n_requests axis bracket of every batch size
  unsigned char* nlo;
};

// fast_brackets with the n_requests axis (active axis `na`) read from the
// per-simulation table (the same bracket_count results, computed once).
__device__ __forceinline__ void fast_brackets_ntab(const FastGrid& g, long long n_req, long long sum_len, FastBrk& b,
                                                   int na, const unsigned char* nlo, const double* nfrac) {
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a >= g.na) break;
    if (g.fixed[a]) {
      b.lo[a] = g.lo[a];
      b.frac[a] = g.frac[a];
    } else if (a == na) {
      b.lo[a] = nlo[n_req];
      b.frac[a] = nfrac[n_req];
    } else {
      bracket_count(g.knots[a], g.n[a], static_cast<double>(g.role[a] == BS_AXIS_SUM_LEN ? sum_len : n_req),
                    &b.lo[a], &b.frac[a]);
    }
  }
}

// Insert r after every resident retiring no later (warp-cooperative).
__device__ __forceinline__ void res_insert(Resident* a, int n, Resident r, int lane) {
  int pos = 0;
  for (int b = 0; b < n; b += 32) {
    const int j = b + lane;
    const unsigned le = __ballot_sync(0xffffffffu, j < n && !(r.retire < a[j].retire));
    pos += __popc(le);
    if (le != 0xffffffffu) break;
  }
  for (int top = n; top > pos; top -= 32) {  // shift [pos, n) up by one, highest first
    const int j = top - 1 - lane;
    const bool act = j >= pos;
    Resident v;
    if (act) v = a[j];
    __syncwarp();
    if (act) a[j + 1] = v;
    __syncwarp();
  }
  if (lane == 0) a[pos] = r;
  __syncwarp();
}

// Retire every resident with retire <= last_it (a prefix of the array);
// returns how many, their summed needs in *need_sum.
__device__ __forceinline__ int res_retire(Resident* a, int n, long long last_it, long long* need_sum, int lane) {
  int c = 0;
  long long s = 0;
  for (int b = 0; b < n; b += 32) {
    const int j = b + lane;
    const bool r = j < n && a[j].retire <= last_it;
    long long v = r ? a[j].need : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    s += v;
    const unsigned m = __ballot_sync(0xffffffffu, r);
    c += __popc(m);
    if (m != 0xffffffffu) break;
  }
  if (c > 0) {
    for (int b = 0; b < n - c; b += 32) {  // shift the survivors down, lowest first
      const int j = b + lane;
      const bool act = j < n - c;
      Resident v;
      if (act) v = a[j + c];
      __syncwarp();
      if (act) a[j] = v;
      __syncwarp();
    }
  }
  *need_sum = s;
  return c;
}

__device__ inline SimOut simulate_decode_warp(const DModels& m, const SimTrace& tr, const SimParams& p, WarpScratch ws,
                                       int heap_cap, int lane) {
  SimOut o;
  o.status = BS_OK;
  o.model_err = 0;
  o.meets_slo = 1;
  o.completed = 0;
  o.busy_j = 0.0;
  o.idle_j = 0.0;
  o.batches = 0;
  const FastGrid lat = fast_grid(m.grid[1], p.tp, p.freq);
  const FastGrid pw = fast_grid(m.grid[3], p.tp, p.freq);
  const bool share = fast_same_axes(lat, pw);  // one bracket set serves both models
  double idle_w = 0.0;
  const bool have_idle = idle_power(m.idle, p.tp, p.freq, &idle_w);
  double now = 0.0;
  long long arr = 0, whead = 0;
  int n_res = 0;
  long long sum_ctx = 0, reserved = 0, it = 0;
  double prev_end = 0.0;
  Resident* res = ws.heap;
  // the n_requests axis's bracket for every batch size 1..heap_cap, once per
  // simulation (the latency grid's; the power grid shares it when share)
  int na = -1;
  if (ws.nfrac && share && !lat.bad)
    for (int a = 0; a < lat.na; ++a)
      if (!lat.fixed[a] && lat.role[a] == BS_AXIS_N_REQUESTS && lat.n[a] <= 255) na = a;
  if (na >= 0) {
    for (int v = 1 + lane; v <= heap_cap; v += 32) {
      int lo;
      double fr;
      bracket_count(lat.knots[na], lat.n[na], static_cast<double>(v), &lo, &fr);
      ws.nlo[v] = static_cast<unsigned char>(lo);
      ws.nfrac[v] = fr;
    }
    __syncwarp();
  }

  auto record_idle = [&](double from, double to) -> bool {
    if (to <= from) return true;
    if (!have_idle) {
      o.status = BS_MODEL_ERROR;
      o.model_err = 3;
      return false;
    }
    o.idle_j = __dadd_rn(o.idle_j, __ddiv_rn(__dmul_rn(idle_w, __dsub_rn(to, from)), 1000.0));
    return true;
  };

  // the next not-yet-pulled request (index arr), cached: its arrival is read
  // once per request instead of at every event window
  double a_nx = INFINITY;
  auto refresh_next = [&]() { a_nx = arr < tr.n ? tr.arrival[tr.kept[arr]] : INFINITY; };
  refresh_next();
  int poll = 0;
  while (arr < tr.n || whead < arr || n_res > 0) {
    if (p.search && ++poll == kSearchPollDecode) {  // warp-uniform: lane 0's view decides
      poll = 0;
      int alive = lane == 0 ? (search_alive(*p.search, p.k) ? 1 : 0) : 0;
      alive = __shfl_sync(0xffffffffu, alive, 0);
      if (!alive) {
        o.status = kSimAborted;
        return o;
      }
    }
    // ---- boundary: pull arrivals, admit (simulator.hpp:515-519, 455-470)
    while (arr < tr.n && a_nx <= now) {
      ++arr;
      refresh_next();
    }
    int n_new = 0;
    double new_min_arr = 0.0;
    while (whead < arr) {
      const int r = tr.kept[whead];
      const long long need = tr.input[r] + tr.output[r];
      if (need > p.kv_capacity) {
        o.status = BS_SIMULATION_ERROR;
        o.meets_slo = 0;
        return o;
      }
      if (n_res >= p.max_batch_requests) break;
      if (reserved + need > p.kv_capacity) break;
      if (n_res >= heap_cap) {
        o.status = BS_PARAMETER_ERROR;
        return o;
      }
      Resident rs;
      rs.retire = it + tr.output[r] - 1;
      rs.need = need;
      res_insert(res, n_res, rs, lane);
      n_res += 1;
      reserved += need;
      sum_ctx += tr.input[r];
      const double a = tr.arrival[r];
      new_min_arr = n_new == 0 ? a : (a < new_min_arr ? a : new_min_arr);
      ++n_new;
      ++whead;
    }
    if (n_res == 0) {
      if (arr >= tr.n && whead >= arr) break;
      if (whead < arr) {
        o.status = BS_SIMULATION_ERROR;
        o.meets_slo = 0;
        return o;
      }
      const double t_next = fmax(a_nx, now);
      if (!record_idle(now, t_next)) return o;
      now = t_next;
      continue;
    }
    // ---- the event window: from iteration it to the next admission point.
    // Every arrival stops the window at the first boundary it has reached
    // (pulling it early changes nothing; a request too large for the KV cache
    // must stop it, admit throws, simulator.hpp:459-462).  While a request
    // waits for KV room the window also stops at the next retirement.
    const bool blocked = whead < arr;
    const double t_a = a_nx;
    bool first_chunk = true, cut = false;
    long long it0 = it;
    while (!cut) {
      // how many iterations this chunk may cover: the batch empties after the
      // last retirement; lanes see at most 32 retirements before their start
      long long lim = res[n_res - 1].retire - it0 + 1;
      if (n_res > 32) lim = min(lim, res[32].retire - it0 + 1);
      if (blocked) lim = min(lim, res[0].retire - it0 + 1);
      const int mcount = lim < 32 ? static_cast<int>(lim) : 32;
      // composition of iteration it0 + lane: residents retired before it
      const long long rl = lane < n_res ? res[lane].retire : LLONG_MAX;
      long long ndp = lane < n_res ? res[lane].need : 0;  // -> inclusive prefix of needs
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, ndp, o2);
        if (lane >= o2) ndp += v;
      }
      int cend = 0;  // residents retiring by the end of iteration it0 + lane (capped at 32)
      {
        const long long x = it0 + lane;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const long long v = __shfl_sync(0xffffffffu, rl, cend + step - 1);
          if (v <= x) cend += step;
        }
        const long long v = __shfl_sync(0xffffffffu, rl, cend < 31 ? cend : 31);
        if (cend == 31 && v <= x) cend = 32;
      }
      int cbeg = __shfl_up_sync(0xffffffffu, cend, 1);
      if (lane == 0) cbeg = 0;
      const int nl = n_res - cbeg;
      const long long ndb = __shfl_sync(0xffffffffu, ndp, (cbeg - 1) & 31);
      const long long gone = cbeg > 0 ? ndb : 0;
      int ninc = nl;  // inclusive prefix of the batch sizes
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, ninc, o2);
        if (lane >= o2) ninc += v;
      }
      // parallel: predictions of iterations it0 .. it0 + mcount - 1; latency
      // is needed for every iteration (t_done), power only for a segment of
      // positive length (record_segment returns before exec_power when
      // to <= from, simulator.hpp:214-215)
      bool bad = false, pbad = false;
      if (lane < mcount) {
        const long long s = sum_ctx + static_cast<long long>(ninc - nl) - gone;
        double Lv = 0.0, Pv = 0.0;
        FastBrk bl;
        if (lat.bad) {
          bad = true;
        } else {
          if (na >= 0)
            fast_brackets_ntab(lat, nl, s, bl, na, ws.nlo, ws.nfrac);
          else
            fast_brackets(lat, nl, s, bl);
          Lv = fast_corners(lat, bl);
          bad = !model_value_ok(Lv);
        }
        if (pw.bad) {
          pbad = true;
        } else {
          if (share) {
            Pv = fast_corners(pw, bl);
          } else {
            FastBrk bp;
            fast_brackets(pw, nl, s, bp);
            Pv = fast_corners(pw, bp);
          }
          pbad = !model_value_ok(Pv);
        }
        ws.L[lane] = Lv;
        ws.P[lane] = Pv;
      }
      const unsigned badm = __ballot_sync(0xffffffffu, bad);
      const unsigned pbadm = __ballot_sync(0xffffffffu, pbad);
      const int first_bad = badm ? __ffs(badm) - 1 : mcount;
      // serial: end times of the chunk's iterations (simulator.hpp:362, 537)
      __syncwarp();
      if (lane == 0) {  // 1.0 * L == L exactly, so the chain is one DADD per iteration
        double t = now;
#pragma unroll 8
        for (int l = 0; l < first_bad; ++l) {
          t = __dadd_rn(t, ws.L[l]);
          ws.T[l] = t;
        }
      }
      __syncwarp();
      // where does the window stop?  at the first iteration whose end reaches
      // the next arrival, or at a model error
      bool stop_here = false;
      if (lane < first_bad) stop_here = ws.T[lane] >= t_a;
      const unsigned stopm = __ballot_sync(0xffffffffu, stop_here);
      int last = first_bad - 1;  // last iteration simulated in this chunk
      if (stopm) last = min(last, __ffs(stopm) - 1);
      // token gaps (max_tbt_ms, simulator.hpp:81-89) for iterations 0..last;
      // a resident of iteration l > 0 also produced a token in iteration l - 1
      bool viol = false;
      if (lane <= last) {
        const double t_start = lane == 0 ? now : ws.T[lane - 1];
        const double te = ws.T[lane];
        if (lane == 0 && first_chunk) {
          if (n_res > n_new && __dsub_rn(te, prev_end) > p.tpot_bound) viol = true;
          if (n_new > 0 && __dsub_rn(te, new_min_arr) > p.tpot_bound) viol = true;
        } else if (__dsub_rn(te, t_start) > p.tpot_bound) {
          viol = true;
        }
      }
      const unsigned violm = __ballot_sync(0xffffffffu, viol);
      if (violm) {
        o.meets_slo = 0;
        if (p.early_exit) return o;
      }
      // energy of the segments, in record order (simulator.hpp:213-228):
      // each lane forms its segment's energy term; lane 0 adds them in record
      // order (the only serial part)
      bool seg = false;
      if (lane <= last) {
        const double t_start = lane == 0 ? now : ws.T[lane - 1];
        const double te = ws.T[lane];
        seg = te > t_start;
        ws.L[lane] = seg ? __ddiv_rn(__dmul_rn(ws.P[lane], __dsub_rn(te, t_start)), 1000.0) : 0.0;
      }
      const unsigned segm = __ballot_sync(0xffffffffu, seg);
      const unsigned perrm = segm & pbadm;
      const int perr = perrm ? __ffs(perrm) - 1 : -1;
      __syncwarp();
      if (lane == 0) {  // a skipped segment's term is +0.0 and busy >= +0.0: adding it is exact
        double busy = o.busy_j;
        const int upto = perr >= 0 ? perr - 1 : last;
#pragma unroll 8
        for (int l = 0; l <= upto; ++l) busy = __dadd_rn(busy, ws.L[l]);
        ws.P[0] = busy;
      }
      __syncwarp();
      o.busy_j = ws.P[0];
      o.batches += __popc(segm & (perr >= 0 ? ((1u << perr) - 1u) : 0xffffffffu));
      __syncwarp();
      if (perr >= 0) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 2;
        return o;
      }
      int retired = 0;
      if (last >= 0) {
        const double t_end = ws.T[last];
        sum_ctx += __shfl_sync(0xffffffffu, ninc, last);
        it0 += last + 1;
        now = t_end;
        prev_end = t_end;
        __syncwarp();
        // retirements at the ends of the chunk's iterations (simulator.hpp:546-555)
        long long freed = 0;
        retired = res_retire(res, n_res, it0 - 1, &freed, lane);
        n_res -= retired;
        reserved -= freed;
        sum_ctx -= freed;
        o.completed += retired;
      }
      __syncwarp();
      if (first_bad < mcount && last == first_bad - 1 && !stopm) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 1;
        return o;
      }
      first_chunk = false;
      cut = stopm != 0 || n_res == 0 || (blocked && retired > 0);
    }
    it = it0;
  }
  o.horizon_ms = fmax(tr.duration_ms, now);
  record_idle(now, o.horizon_ms);
  return o;
}

}  // namespace bs

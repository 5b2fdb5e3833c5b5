// bs_device.cuh — device-side data layout and the bit-exact FP64 model
// evaluation shared by every sm_100a kernel of the decision path.
//
// Every translation unit is compiled with --fmad=false: the reference is
// built without FMA contraction, so each DMUL/DADD here must
// round exactly where the reference's C++ rounds.  Never --use_fast_math.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "biscale_gpu.h"

namespace bs {

constexpr int kMaxRank = BS_MAX_RANK;
constexpr int kMaxK = BS_MAX_K;
constexpr int kMaxCand = BS_MAX_CAND;

// ---------------------------------------------------------------------------
// Models in HBM.  One DGrid per NdGrid (perfmodel.hpp:116-201): knots and
// row-major values live in one immutable device allocation per ModelSet.
// ---------------------------------------------------------------------------
struct DGrid {
  int rank;
  int role[kMaxRank];
  int n[kMaxRank];
  const double* knots[kMaxRank];
  const double* values;
  int bad_axis;  // an axis name query_coords rejects (perfmodel.hpp:254)
};

struct DIdle {
  int n_entries;
  const int* tp;
  const int* n;
  const int* off;
  const double* freqs;
  const double* watts;
};

struct DModels {
  DGrid grid[4];  // 0 lat prefill, 1 lat decode, 2 pow prefill, 3 pow decode
  DIdle idle;
};

// Coordinates by axis role: {sum_len, n_requests, tp, freq_mhz}, the mapping
// of query_coords (perfmodel.hpp:241-258): int64 features cast to double.
struct Query {
  double c[4];
};

__device__ __forceinline__ Query make_query(int64_t n_requests, int64_t sum_len, int tp, double freq) {
  Query q;
  q.c[BS_AXIS_SUM_LEN] = static_cast<double>(sum_len);
  q.c[BS_AXIS_N_REQUESTS] = static_cast<double>(n_requests);
  q.c[BS_AXIS_TP] = static_cast<double>(tp);
  q.c[BS_AXIS_FREQ] = freq;
  return q;
}

// NdGrid::interpolate (perfmodel.hpp:150-193), same op order:
// per axis clamp (counted) -> upper_bound -> hi = clamp(hi, 1, n-1) ->
// frac = (x - k_lo) / (k_hi - k_lo); corners mask = 0..2^D-1, weight the
// product over axes in ascending order, single-knot high corner -> 0,
// acc += w * v skipped when w == 0.
__device__ __forceinline__ double interp_coords(const DGrid& g, const double* x_by_axis, unsigned* clamps) {
  int lo[kMaxRank];
  double frac[kMaxRank];
  const int dims = g.rank;
#pragma unroll
  for (int d = 0; d < kMaxRank; ++d) {
    if (d >= dims) break;
    const double* k = g.knots[d];
    const int n = g.n[d];
    double x = x_by_axis[d];
    const double k0 = k[0], kn = k[n - 1];
    if (x < k0 || x > kn) {
      if (clamps) *clamps += 1;
      x = x < k0 ? k0 : (kn < x ? kn : x);
    }
    if (n == 1) {
      lo[d] = 0;
      frac[d] = 0.0;
      continue;
    }
    int hi = 0;
    while (hi < n && !(x < k[hi])) ++hi;  // std::upper_bound
    hi = hi < 1 ? 1 : (hi > n - 1 ? n - 1 : hi);
    lo[d] = hi - 1;
    frac[d] = __ddiv_rn(__dsub_rn(x, k[lo[d]]), __dsub_rn(k[hi], k[lo[d]]));
  }
  double acc = 0.0;
  const int corners = 1 << dims;
  for (int mask = 0; mask < corners; ++mask) {
    double weight = 1.0;
    long long flat = 0;
#pragma unroll
    for (int d = 0; d < kMaxRank; ++d) {
      if (d >= dims) break;
      const int high = (mask >> d) & 1;
      if (high && g.n[d] == 1) {
        weight = 0.0;
        break;
      }
      weight = __dmul_rn(weight, high ? frac[d] : __dsub_rn(1.0, frac[d]));
      flat = flat * g.n[d] + (lo[d] + high);
    }
    if (weight != 0.0) acc = __dadd_rn(acc, __dmul_rn(weight, g.values[flat]));
  }
  return acc;
}

__device__ __forceinline__ double interp(const DGrid& g, const Query& q, unsigned* clamps) {
  double x[kMaxRank];
#pragma unroll
  for (int d = 0; d < kMaxRank; ++d) {
    if (d < g.rank) x[d] = q.c[g.role[d] < 0 ? 0 : g.role[d]];
  }
  return interp_coords(g, x, clamps);
}

// predict_latency / predict_power validity test (perfmodel.hpp:264, 270).
__device__ __forceinline__ bool model_value_ok(double v) { return v > 0.0 && isfinite(v); }

// predict_idle_power (perfmodel.hpp:274-288): 1-D lerp lo + t * (hi - lo).
// Returns false when the tp entry is missing or empty (ModelError).
__device__ __forceinline__ bool idle_power(const DIdle& m, int tp, double freq, double* out) {
  for (int i = 0; i < m.n_entries; ++i) {
    if (m.tp[i] != tp) continue;
    const int n = m.n[i];
    if (n < 1) return false;
    const double* f = m.freqs + m.off[i];
    const double* w = m.watts + m.off[i];
    double x = freq < f[0] ? f[0] : (f[n - 1] < freq ? f[n - 1] : freq);
    if (n == 1) {
      *out = w[0];
      return true;
    }
    int hi = 0;
    while (hi < n && !(x < f[hi])) ++hi;
    hi = hi < 1 ? 1 : (hi > n - 1 ? n - 1 : hi);
    const int lo = hi - 1;
    const double t = __ddiv_rn(__dsub_rn(x, f[lo]), __dsub_rn(f[hi], f[lo]));
    *out = __dadd_rn(w[lo], __dmul_rn(t, __dsub_rn(w[hi], w[lo])));
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Packed MPC problems (host -> HBM in one copy).
// ---------------------------------------------------------------------------
struct DMpcCfg {
  int horizon;
  int nc;  // |ladder.select(ladder_N)|
  double cand[kMaxCand];
  double ttft;
  double switch_ms;
  double one_plus_margin;  // (1.0 + margin), the same double the reference forms
  double max_mhz;
  long long max_batch_tokens;
  long long max_batch_requests;
  int chunking;
  int _pad;
};

struct DWaiting {
  long long id;
  double arrival;
  long long total;
  long long remaining;
};

struct DRunning {
  double arrival;
  long long completes;
};

struct DProblem {
  double now;
  double cur_freq;
  double target_freq;
  double run_wr;
  long long run_n;
  long long run_sum;
  long long wait_off;
  long long run_off;
  int tp;
  int run_active;
  int n_wait;
  int n_run;  // < 0: the running batch is summarised by run_minarr / run_ncomp
  int cfg;
  int run_ncomp;      // completing members of the running batch (when n_run < 0)
  double run_minarr;  // their smallest arrival, +inf if none (when n_run < 0)
  int fgi;            // index of the problem's (configuration, tp) reduced-grid pair
  int _pad2;
};

// Per-problem projection + (k, f) tables, built on device.
//   A[k][f]  = wf_k * L(k, f)                     (MpcEvaluator lat)
//   P[k][f]  = P(k, f)                             (MpcEvaluator pow)
//   E[k][f]  = A * P                               (num term)
//   B0[k][f] = A * (1 + margin)                    (no switch)
//   B1[k][f] = (A + switch) * (1 + margin)         (switch charged)
//   T1[f]    = now + (cand[f] != current ? B1 : B0)[0][f]
//   minarr[k]= min completing arrival (+inf if none): monotone-subtraction
//              reduction of meets_slo's per-request test (SURVEY.md appx. 5)
struct __align__(16) SRec {
  double sb, E, A, th0n;  // th0n: the next level's non-switching threshold of this child's rung (thn below)
};

struct DTables {
  int K;
  int nc;
  int status;
  int filter_ok;  // every A >= 0 and finite: the division filter is exact
  unsigned bad_lat[kMaxK];  // bit f: predict_latency(k, f) would throw
  unsigned bad_pow[kMaxK];
  long long n_req[kMaxK];
  long long sum_len[kMaxK];
  double wf[kMaxK];
  double minarr[kMaxK];
  int ncomp[kMaxK];
  double T1[kMaxCand];
  double ttft;
  double A[kMaxK][kMaxCand];
  double P[kMaxK][kMaxCand];
  double E[kMaxK][kMaxCand];
  double B0[kMaxK][kMaxCand];
  double B1[kMaxK][kMaxCand];
  // Per level, the candidates sorted by their switched step (B1; T1 at level
  // 0), ascending, ties by index.  fl(fl(t + b) - m) is monotone in b, so the
  // children of any node that pass meets_slo's check at level k form a
  // prefix of this order (the non-switching child f == last, whose step is
  // B0, is tested on its own).  sorted_ok = every key finite.
  double sb[kMaxK][kMaxCand];
  unsigned char ord[kMaxK][kMaxCand];
  unsigned char rank[kMaxK][kMaxCand];
  // The same order as records for the sweep's children loop (one vector
  // load per child, independent of the index load): srec[k][j] = {sb[k][j],
  // E[k][f], A[k][f], B0[k+1][f]} and sinfo[k][j] = f | rank[k+1][f] << 8
  // with f = ord[k][j] (next-level fields 0 at the last level).
  SRec srec[kMaxK][kMaxCand];
  unsigned short sinfo[kMaxK][kMaxCand];
  int sorted_ok;
  // Per-step thresholds (levels >= 1, set by prepare_kernel): a node with
  // clock t passes level k's check with the switched step of sorted position
  // j iff t <= thsw[k][j] (non-increasing in j), with rung f's non-switching
  // step iff t <= th0[k][f] -- the suprema of meets_slo's monotone test
  // (step_thresholds), so each check is one comparison.
  double thsw[kMaxK][kMaxCand];
  double th0[kMaxK][kMaxCand];
  int thr_ok;  // exhaustive search: the two bottom levels' leaf-count thresholds are built (DThr, bs_exhaustive.cuh)
  int fuse;    // exhaustive search: the BFS settles dominated final nodes (thr_kernel)
  int n_ok3;   // exhaustive search: feasible depth-3 prefixes (prepare_kernel)
  int FD;  // exhaustive search: depth of the final nodes, K - sweep_levels(K, nc) (set by prepare_kernel)
  unsigned nc_magic;  // ceil(2^32 / nc): code / nc by a multiply-high for codes < 2^27 (set by prepare_kernel)
  // Per-level bounds for the leaf-row skip: amax = max_f A, pmin_lo =
  // fl(min_f P * (1 - 2^-50)) <= min_f P * (1 - u).
  double amax[kMaxK];
  double pmin_lo[kMaxK];
  // Node bound of the argmin seed (exhaustive search, set by prepare_kernel;
  // nb_R = +inf disables it): a node at depth K-2 with (num, den) has every
  // leaf worse than the seed when fl(num - fl(nb_beta den)) > fl(nb_R + fl(num 2^-40)).
  double nb_beta;
  double nb_R;
  // exact completion bounds (leaf_exists_bounds, exhaustive search): a node
  // at depth d (1 <= d <= K-2) with clock t and last digit l has a feasible
  // leaf iff t <= rexist[d][l]
  double rexist[kMaxK][kMaxCand];
  int rex_ok;
  int _pad_rex;
};

// Compact per-problem result written by the device; the host expands it
// into bs_mpc_result.
struct DMpcOut {
  int status;
  int K;
  int feasible;
  int n_levels;
  long long eval_count;
  double objective;
  unsigned long long feasible_count;
  unsigned long long best_code;
  unsigned char idx[kMaxK];
};

struct DLevel {
  int k_prime;
  int accepted;
  double replaced_mhz;
  long long mutations;
  long long feasible_mutations;
};

// 128-bit (objective bits, code) key; objectives are >= 0 so their IEEE
// bit patterns order like the values.
struct __align__(16) Key128 {
  unsigned long long obj;
  unsigned long long code;
};

__device__ __forceinline__ bool key_less(unsigned long long ao, unsigned long long ac, unsigned long long bo,
                                         unsigned long long bc) {
  return ao < bo || (ao == bo && ac < bc);
}

__device__ __forceinline__ Key128 atomic_cas128(Key128* addr, Key128 cmp, Key128 val) {
  unsigned long long o0, o1;
  asm volatile(
      "{\n .reg .b128 c, v, r;\n mov.b128 c, {%2, %3};\n mov.b128 v, {%4, %5};\n"
      " atom.global.cas.b128 r, [%6], c, v;\n mov.b128 {%0, %1}, r;\n}"
      : "=l"(o0), "=l"(o1)
      : "l"(cmp.obj), "l"(cmp.code), "l"(val.obj), "l"(val.code), "l"(addr)
      : "memory");
  Key128 r;
  r.obj = o0;
  r.code = o1;
  return r;
}

// Lexicographic atomic min on (obj, code).  Slots start at (~0, ~0).  Keys
// only decrease, so a plain 64-bit read of the objective half is a safe
// early-out when it is already strictly smaller; the pair itself is only
// ever read through the 128-bit CAS (a two-half read could tear).
__device__ __forceinline__ void atomic_min_key(Key128* addr, unsigned long long obj, unsigned long long code) {
  const unsigned long long hint = *reinterpret_cast<volatile unsigned long long*>(&addr->obj);
  if (obj > hint) return;
  Key128 cur;
  cur.obj = ~0ull;
  cur.code = ~0ull;
  while (key_less(obj, code, cur.obj, cur.code)) {
    Key128 val;
    val.obj = obj;
    val.code = code;
    Key128 old = atomic_cas128(addr, cur, val);
    if (old.obj == cur.obj && old.code == cur.code) return;
    cur = old;
  }
}

}  // namespace bs

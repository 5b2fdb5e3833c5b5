// bs_ilp.cu — the coarse-tier ILPs of the placement search on sm_100a:
// solve_placement (placement.hpp:357-416, branch and bound over instance
// counts) and solve_max_throughput (placement.hpp:421-499, the DistServe-style
// max-frequency baseline), for a batch of problems (e.g. every window of a
// run_experiment) in one set of launches.
//
// The search space is the reference's: count vectors n[0..N) over the table
// in table order, n_i in [0, floor(gpus_left / g_i)] for usable entries and 0
// otherwise, visited in lexicographic order (n_0 most significant, ascending).
// States are the reference's left folds: cost += (n e_c) r_c, r_phase += n r_c,
// gpus_left -= n g_c, in table order, with the same pruning tests at every
// node (deficit lower bound with suffix minima of e_c, GPU lower bound with
// suffix maxima of r_c / g_c; placement.hpp:297-311).
//
//   ilp_frontier_kernel   1 CTA / problem: suffix minima / maxima, then a
//                         level-synchronous expansion of the tree from the
//                         root into an ordered frontier of subtree roots
//                         (children of node j before those of node j + 1, in
//                         ascending n: frontier order = lexicographic order).
//                         Entries a node cannot take (unusable, or g_c >
//                         gpus_left) are passed through with the node-entry
//                         tests applied at every depth, as the recursion does.
//   ilp_subtree_kernel    1 thread / frontier node.  Placement: depth-first
//                         walk of its subtree (explicit stack; states stored
//                         only at non-zero choices, since n = 0 leaves every
//                         fold unchanged) against a per-problem key (cost,
//                         frontier index) merged by a 128-bit atomic min: the
//                         lexicographically first minimum-cost vector is the
//                         reference's strict-< first minimum in DFS order.  A
//                         subtree is cut when its lower bound exceeds the key's
//                         cost, or equals it and the key's subtree does not come
//                         later (placement.hpp:306's `lb >= best_cost`, refined
//                         by subtree order so ties keep the lexicographic rule).
//                         Max-throughput: every leaf, counted, then written in
//                         order as (score, GPUs used).
//   ilp_scan_kernel       max-throughput: per-problem exclusive scan of the
//                         subtrees' leaf counts (leaf list offsets).
//   ilp_finish_kernel     1 thread / problem.  Placement: the key's subtree is
//                         walked again with the optimum as the bound to recover
//                         its lexicographically first optimal vector.
//                         Max-throughput: the reference's `better` rule
//                         (1e-12 score window, then fewer GPUs; not transitive,
//                         so applied in leaf order by one thread), then the
//                         winner's vector by walking its subtree to its ordinal.
//
// Exactness: FP64 without FMA (--fmad=false), every fold and test in the
// reference's operand order.  The pruning bounds are those of the reference;
// the frontier merely changes which valid bound is current when a subtree is
// visited, which cannot change the optimum or its lexicographic tie-break.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "bs_internal.h"

using namespace bs;

namespace {

constexpr int kIlpThreads = 256;       // frontier / scan / finish CTAs
constexpr int kIlpSubThreads = 128;    // subtree walkers per CTA
constexpr int kIlpMaxEntries = 256;    // table entries per problem
constexpr int kIlpMaxNz = 64;          // non-zero counts on one path (<= total_gpus / min g_c)
constexpr int kIlpMaxLevels = 32;      // frontier expansion levels recorded
constexpr double kInf = INFINITY;

// Fold state of a node: what dfs() carries (placement.hpp:297).
struct IlpSt {
  double cost, rp, rd;
  int gl;  // gpus_left
  int _pad;
};

// Per-problem description (host-packed).
struct DIlpProb {
  int n;           // table entries
  int total_gpus;
  int mode;        // 0 solve_placement, 1 solve_max_throughput
  int e_off;       // entries at [e_off, e_off + n) of the entry arrays
  double need;     // (1 + alpha) * target_rps
  long long f_off;  // frontier region: nodes [f_off, f_off + f_cap)
  int f_cap;
  int c_off;       // output counts at [c_off, c_off + n)
};

// Entry arrays (SoA) and per-problem suffix arrays (n + 1 each at s_off = e_off + problem).
struct DIlpEntries {
  const double* r;      // R_c (restricted to max-frequency rows in mode 1)
  const double* e;      // E_c (0 when absent)
  const int* g;         // G_c
  const int* ph;        // phase
  const int* use;       // usable()
  double* min_e_p;      // suffix minima / maxima, placement.hpp:371-390
  double* min_e_d;
  double* max_rpg_p;
  double* max_rpg_d;
};

// Per-problem results and bookkeeping.
struct DIlpOut {
  Key128 best;          // placement: (cost bits, frontier index)
  int n_front;          // frontier nodes
  int n_levels;         // expansion levels recorded
  int status;           // 0 ok, 1 infeasible, 2 leaf capacity exceeded, 3 frontier state overflow
  int gpus_used;
  double objective;
  double cut;                   // placement: cost of a known feasible leaf (a strict bound; +inf: none)
  unsigned long long leaves;    // max-throughput: feasible leaves enumerated
  unsigned long long leaf_off;  // their offset in the leaf list
  unsigned long long leaf_best; // the selected leaf (ordinal in the problem's list; ~0: none)
};

// Frontier node storage (per problem region of f_cap nodes; two ping-pong
// lists and kIlpMaxLevels expansion records).
struct DFront {
  IlpSt* st[2];
  int* dep[2];
  int* rec_parent;  // [level * cap + j]: parent index in the previous level (-1: root)
  int* rec_n;       // count chosen at rec_entry (0: none)
  int* rec_entry;   // entry index of the choice (-1: carried leaf)
  unsigned* leaf_cnt;  // max-throughput: leaves per subtree
};

__device__ __forceinline__ double pos_part(double x) { return 0.0 < x ? x : 0.0; }  // std::max(0.0, x)

struct View {
  int n, mode;
  double need;
  double cut;  // placement: subtrees whose lower bound exceeds it hold no optimum
  const double* r;
  const double* e;
  const int* g;
  const int* ph;
  const int* use;
  const double* mep;
  const double* med;
  const double* mrp;
  const double* mrd;
};

__device__ __forceinline__ View view_of(const DIlpProb& P, const DIlpEntries& E, int p) {
  View v;
  v.n = P.n;
  v.mode = P.mode;
  v.need = P.need;
  v.cut = INFINITY;
  v.r = E.r + P.e_off;
  v.e = E.e + P.e_off;
  v.g = E.g + P.e_off;
  v.ph = E.ph + P.e_off;
  v.use = E.use + P.e_off;
  const long long s = static_cast<long long>(P.e_off) + p;  // n + 1 suffix slots per problem
  v.mep = E.min_e_p + s;
  v.med = E.min_e_d + s;
  v.mrp = E.max_rpg_p + s;
  v.mrd = E.max_rpg_d + s;
  return v;
}

// Node-entry tests of dfs(i, ...) (placement.hpp:297-321) without the bound
// test.  Returns 0 pruned, 1 interior node, 2 feasible leaf (i == n); lb out.
__device__ __forceinline__ int node_test(const View& v, int i, const IlpSt& s, double* lb_out) {
  if (v.mode == 1) {  // solve_max_throughput enumerates without pruning (placement.hpp:446-476)
    if (i < v.n) return 1;
    if (s.rp < v.need - 1e-9 || s.rd < v.need - 1e-9) return 0;
    return 2;
  }
  const double def_p = pos_part(v.need - s.rp);
  const double def_d = pos_part(v.need - s.rd);
  if (def_p > 0.0 && v.mep[i] == kInf) return 0;
  if (def_d > 0.0 && v.med[i] == kInf) return 0;
  double lb = s.cost;
  if (def_p > 0.0) lb = lb + def_p * v.mep[i];
  if (def_d > 0.0) lb = lb + def_d * v.med[i];
  *lb_out = lb;
  if (lb > v.cut) return 0;  // above a known feasible leaf's cost: no optimum below
  double gn = 0.0;
  if (def_p > 0.0) gn = gn + def_p / v.mrp[i];
  if (def_d > 0.0) gn = gn + def_d / v.mrd[i];
  if (gn > static_cast<double>(s.gl) + 1e-9) return 0;
  if (i == v.n) return (def_p > 1e-9 || def_d > 1e-9) ? 0 : 2;
  return 1;
}

__device__ __forceinline__ int max_count(const View& v, int i, int gl) { return v.use[i] ? gl / v.g[i] : 0; }

// Child n of a node at entry i (placement.hpp:323-330 / 468-473).
__device__ __forceinline__ IlpSt child(const View& v, int i, const IlpSt& s, int n) {
  IlpSt c;
  const double add_r = static_cast<double>(n) * v.r[i];
  c.gl = s.gl - n * v.g[i];
  if (v.mode == 0) {
    const double add_cost = static_cast<double>(n) * v.e[i] * v.r[i];
    c.cost = s.cost + add_cost;
  } else {
    c.cost = s.cost;
  }
  c.rp = s.rp + (v.ph[i] == BS_PHASE_PREFILL ? add_r : 0.0);
  c.rd = s.rd + (v.ph[i] == BS_PHASE_DECODE ? add_r : 0.0);
  c._pad = 0;
  return c;
}

// Bound test of the placement search against a key read from `slot`:
// true = cut.  Keys only decrease, so a stale cost that is already below lb
// is a valid cut; an equal cost needs the (cost, index) pair, read atomically.
__device__ __forceinline__ bool bound_cut(double lb, int my_idx, Key128* slot) {
  const unsigned long long hint = *reinterpret_cast<volatile unsigned long long*>(&slot->obj);
  if (hint == ~0ull) return false;  // nothing found yet
  const double bc = __longlong_as_double(static_cast<long long>(hint));
  if (lb > bc) return true;
  if (lb < bc) return false;
  Key128 cur;
  cur.obj = hint;
  cur.code = ~0ull;
  cur = atomic_cas128(slot, cur, cur);  // consistent snapshot (a CAS that never changes the value)
  const double c2 = __longlong_as_double(static_cast<long long>(cur.obj));
  return lb > c2 || (lb == c2 && cur.code <= static_cast<unsigned long long>(my_idx));
}

// Walks from node (i0, s0) down through entries it cannot take (one child,
// n = 0, every node-entry test applied) to the first entry with a choice, a
// leaf, or a cut.  Returns the node_test code at the stopping depth.
__device__ __forceinline__ int advance(const View& v, int& i, const IlpSt& s, double* lb) {
  for (;;) {
    const int t = node_test(v, i, s, lb);
    if (t != 1) return t;
    if (max_count(v, i, s.gl) > 0) return 1;
    ++i;
  }
}

// --- frontier ---------------------------------------------------------------------

__device__ __forceinline__ DFront front_at(char* base, int cap) {
  DFront f;
  char* p = base;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  f.st[0] = reinterpret_cast<IlpSt*>(take(sizeof(IlpSt) * cap));
  f.st[1] = reinterpret_cast<IlpSt*>(take(sizeof(IlpSt) * cap));
  f.dep[0] = reinterpret_cast<int*>(take(4ull * cap));
  f.dep[1] = reinterpret_cast<int*>(take(4ull * cap));
  f.rec_parent = reinterpret_cast<int*>(take(4ull * cap * kIlpMaxLevels));
  f.rec_n = reinterpret_cast<int*>(take(4ull * cap * kIlpMaxLevels));
  f.rec_entry = reinterpret_cast<int*>(take(4ull * cap * kIlpMaxLevels));
  f.leaf_cnt = reinterpret_cast<unsigned*>(take(4ull * cap));
  return f;
}

__host__ __device__ inline size_t front_bytes(int cap) {
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  return 2 * up(sizeof(IlpSt) * cap) + 2 * up(4ull * cap) + 3 * up(4ull * cap * kIlpMaxLevels) + up(4ull * cap);
}

// Exclusive block scan of one unsigned per thread (blockDim == kIlpThreads);
// returns the block total.  Every thread must call it.
__device__ unsigned block_scan(unsigned x, unsigned* excl) {
  constexpr int nw = kIlpThreads / 32;
  __shared__ unsigned ws[nw + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned acc = 0;
    for (int k = 0; k < nw; ++k) {
      const unsigned t = ws[k];
      ws[k] = acc;
      acc += t;
    }
    ws[nw] = acc;
  }
  __syncthreads();
  *excl = ws[w] + inc - x;
  const unsigned total = ws[nw];
  __syncthreads();
  return total;
}

// One CTA per problem: suffix arrays, then the frontier.
__global__ void __launch_bounds__(kIlpThreads) ilp_frontier_kernel(const DIlpProb* probs, DIlpEntries E, DIlpOut* outs,
                                                                   char* front_base, int target) {
  const int p = blockIdx.x;
  const DIlpProb P = probs[p];
  DIlpOut* o = &outs[p];
  View v = view_of(P, E, p);
  if (threadIdx.x == 0) {  // placement.hpp:371-390 (solve_max_throughput does not use them)
    double* mep = E.min_e_p + P.e_off + p;
    double* med = E.min_e_d + P.e_off + p;
    double* mrp = E.max_rpg_p + P.e_off + p;
    double* mrd = E.max_rpg_d + P.e_off + p;
    mep[P.n] = kInf;
    med[P.n] = kInf;
    mrp[P.n] = 0.0;
    mrd[P.n] = 0.0;
    for (int i = P.n - 1; i >= 0; --i) {
      double a = mep[i + 1], b = med[i + 1], c = mrp[i + 1], d = mrd[i + 1];
      if (v.use[i]) {
        const double rpg = v.r[i] / static_cast<double>(v.g[i]);
        if (v.ph[i] == BS_PHASE_PREFILL) {
          a = v.e[i] < a ? v.e[i] : a;  // std::min(a, e): e when e < a
          c = c < rpg ? rpg : c;        // std::max(c, rpg)
        } else {
          b = v.e[i] < b ? v.e[i] : b;
          d = d < rpg ? rpg : d;
        }
      }
      mep[i] = a;
      med[i] = b;
      mrp[i] = c;
      mrd[i] = d;
    }
    o->best.obj = ~0ull;
    o->best.code = ~0ull;
    o->status = 0;
    o->leaves = 0;
    o->leaf_off = 0;
    o->cut = INFINITY;
  }
  __syncthreads();
  __threadfence_block();
  if (P.mode == 0) {  // a feasible leaf to bound the search: one prefill and one decode entry
    __shared__ double s_min[kIlpThreads / 32];
    double best = INFINITY;
    for (int e = threadIdx.x; e < P.n * P.n; e += blockDim.x) {
      const int i = e / P.n, j = e - i * P.n;
      if (!v.use[i] || !v.use[j] || v.ph[i] != BS_PHASE_PREFILL || v.ph[j] != BS_PHASE_DECODE) continue;
      // the fewest instances whose goodput fold n r_c (r + 0 * ... = r) reaches need
      auto fewest = [&](int x) {
        double q = ceil(v.need / v.r[x]);
        long long n = q > 4096.0 ? 4097 : static_cast<long long>(q);
        while (n > 1 && static_cast<double>(n - 1) * v.r[x] >= v.need) --n;
        while (n <= 4096 && static_cast<double>(n) * v.r[x] < v.need) ++n;
        return n;
      };
      const long long ni = fewest(i), nj = fewest(j);
      if (ni > 4096 || nj > 4096 || ni * v.g[i] + nj * v.g[j] > P.total_gpus) continue;
      // the leaf's cost fold in table order (other entries add (0 e) r = 0)
      const int a = i < j ? i : j, b = i < j ? j : i;
      const long long na = i < j ? ni : nj, nb = i < j ? nj : ni;
      double c = 0.0 + static_cast<double>(na) * v.e[a] * v.r[a];
      c = c + static_cast<double>(nb) * v.e[b] * v.r[b];
      best = c < best ? c : best;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, best, off);
      best = y < best ? y : best;
    }
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kIlpThreads / 32; ++w) best = s_min[w] < best ? s_min[w] : best;
      o->cut = s_min[0] < best ? s_min[0] : best;
    }
    __syncthreads();
    v.cut = o->cut;
  }
  DFront F = front_at(front_base + P.f_off, P.f_cap);
  __shared__ int s_cnt, s_lv;
  if (threadIdx.x == 0) {  // level 0: the root, advanced to its first choice
    IlpSt s{0.0, 0.0, 0.0, P.total_gpus, 0};
    int i = 0;
    double lb;
    const int t = advance(v, i, s, &lb);
    s_cnt = t ? 1 : 0;
    F.st[0][0] = s;
    F.dep[0][0] = i;
    F.rec_parent[0] = -1;
    F.rec_n[0] = 0;
    F.rec_entry[0] = -1;
    s_lv = 0;
  }
  __syncthreads();
  // Expansion levels: every interior node into its surviving children
  // (ascending n), carried leaves as they are, until the frontier reaches
  // `target` nodes or the next level would not fit.
  for (;;) {
    const int cnt = s_cnt, lv = s_lv, cur = lv & 1;
    if (cnt == 0 || cnt >= target || lv + 1 >= kIlpMaxLevels) break;
    // pass 1: children (before their own tests) per node; total must fit the region
    unsigned tot_raw = 0;
    {
      __shared__ unsigned s_raw;
      if (threadIdx.x == 0) s_raw = 0;
      __syncthreads();
      unsigned mine = 0;
      for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        const int i = F.dep[cur][j];
        mine += i >= P.n ? 1u : static_cast<unsigned>(max_count(v, i, F.st[cur][j].gl) + 1);
      }
      atomicAdd(&s_raw, mine);
      __syncthreads();
      tot_raw = s_raw;
      __syncthreads();
    }
    if (tot_raw > static_cast<unsigned>(P.f_cap) || tot_raw == static_cast<unsigned>(cnt)) break;  // full / nothing to expand
    // pass 2 (counts of survivors) and pass 3 (writes), chunk by chunk in node order
    unsigned base = 0;
    for (int c0 = 0; c0 < cnt; c0 += blockDim.x) {
      const int j = c0 + threadIdx.x;
      unsigned keep = 0;
      IlpSt s{};
      int i = 0, mx = 0;
      if (j < cnt) {
        s = F.st[cur][j];
        i = F.dep[cur][j];
        if (i >= P.n) {
          keep = 1;
        } else {
          mx = max_count(v, i, s.gl);
          for (int n = 0; n <= mx; ++n) {
            int ci = i + 1;
            double lb;
            if (advance(v, ci, child(v, i, s, n), &lb)) ++keep;
          }
        }
      }
      unsigned off;
      const unsigned tot = block_scan(keep, &off);
      if (j < cnt) {
        unsigned w = base + off;
        const int nl = lv + 1, nx = nl & 1;
        if (i >= P.n) {
          F.st[nx][w] = s;
          F.dep[nx][w] = i;
          F.rec_parent[nl * P.f_cap + w] = j;
          F.rec_n[nl * P.f_cap + w] = 0;
          F.rec_entry[nl * P.f_cap + w] = -1;
        } else {
          for (int n = 0; n <= mx; ++n) {
            int ci = i + 1;
            double lb;
            const IlpSt cs = child(v, i, s, n);
            if (!advance(v, ci, cs, &lb)) continue;
            F.st[nx][w] = cs;
            F.dep[nx][w] = ci;
            F.rec_parent[nl * P.f_cap + w] = j;
            F.rec_n[nl * P.f_cap + w] = n;
            F.rec_entry[nl * P.f_cap + w] = i;
            ++w;
          }
        }
      }
      base += tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_cnt = static_cast<int>(base);
      s_lv = lv + 1;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    o->n_front = s_cnt;
    o->n_levels = s_lv;
    if (s_cnt == 0) o->status = 1;
  }
}

// --- subtree walks ------------------------------------------------------------------

// Explicit-stack DFS of one subtree in lexicographic order.  visit(i, s)
// is called at every feasible leaf (node_test == 2) and returns false to stop
// the walk; cut(lb) decides the bound test at interior nodes and leaves.
// Returns false when the walk was stopped by visit.
template <typename Cut, typename Visit>
__device__ bool walk_subtree(const View& v, int i0, const IlpSt& s0, Cut&& cut, Visit&& visit, int* path_n,
                             bool* overflow) {
  unsigned frame[kIlpMaxEntries];  // entry (10 bits) | current n (11 bits) | state slot (11 bits)
  IlpSt ss[kIlpMaxNz + 1];
  int nf = 0, sp = 0;
  ss[0] = s0;
  int i = i0;
  for (;;) {
    // descend from node (i, ss[sp])
    for (;;) {
      double lb = 0.0;
      const IlpSt& s = ss[sp];
      const int t = node_test(v, i, s, &lb);
      if (t == 0 || (v.mode == 0 && cut(lb))) break;
      if (t == 2) {
        if (!visit(ss[sp])) return false;
        break;
      }
      const int mx = max_count(v, i, s.gl);
      if (mx > 0) {
        frame[nf] = static_cast<unsigned>(i) | (static_cast<unsigned>(sp) << 21);
        ++nf;
        if (path_n) path_n[i] = 0;
      }
      ++i;  // child n = 0: every fold unchanged
    }
    // backtrack: the deepest frame with an untried sibling
    for (;;) {
      if (nf == 0) return true;
      const unsigned f = frame[nf - 1];
      const int fi = static_cast<int>(f & 0x3ffu);
      const int fn = static_cast<int>((f >> 10) & 0x7ffu);
      const int fs = static_cast<int>(f >> 21);
      const int mx = max_count(v, fi, ss[fs].gl);
      if (fn < mx) {
        const int nn = fn + 1;
        if (fs + 1 > kIlpMaxNz) {
          *overflow = true;
          return false;
        }
        frame[nf - 1] = static_cast<unsigned>(fi) | (static_cast<unsigned>(nn) << 10) | (static_cast<unsigned>(fs) << 21);
        ss[fs + 1] = child(v, fi, ss[fs], nn);
        sp = fs + 1;
        i = fi + 1;
        if (path_n) path_n[fi] = nn;
        break;
      }
      if (path_n) path_n[fi] = 0;
      --nf;
    }
  }
}

// stage 0: placement B&B walks / max-throughput leaf counts; stage 1:
// max-throughput leaf writes.
__global__ void __launch_bounds__(kIlpSubThreads) ilp_subtree_kernel(const DIlpProb* probs, DIlpEntries E,
                                                                     DIlpOut* outs, char* front_base, int stage,
                                                                     double* leaf_score, int* leaf_used,
                                                                     unsigned long long leaf_cap) {
  const int p = blockIdx.y;
  const DIlpProb P = probs[p];
  DIlpOut* o = &outs[p];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int nfront = o->n_front;
  if (j >= nfront || o->status) return;
  if (stage == 1 && P.mode == 0) return;
  View v = view_of(P, E, p);
  if (P.mode == 0) v.cut = o->cut;
  DFront F = front_at(front_base + P.f_off, P.f_cap);
  const int cur = o->n_levels & 1;
  const IlpSt s0 = F.st[cur][j];
  const int i0 = F.dep[cur][j];
  bool overflow = false;
  if (P.mode == 0) {
    Key128* slot = &o->best;
    walk_subtree(
        v, i0, s0, [&](double lb) { return bound_cut(lb, j, slot); },
        [&](const IlpSt& s) {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(s.cost));
          atomic_min_key(slot, bits, static_cast<unsigned long long>(j));
          return true;
        },
        nullptr, &overflow);
  } else if (stage == 0) {
    unsigned cnt = 0;
    walk_subtree(
        v, i0, s0, [](double) { return false; },
        [&](const IlpSt& s) {
          if (P.total_gpus - s.gl > 0) ++cnt;  // used <= 0 is skipped (placement.hpp:450-451)
          return true;
        },
        nullptr, &overflow);
    F.leaf_cnt[j] = cnt;
  } else {
    unsigned long long w = o->leaf_off + F.leaf_cnt[j];  // leaf_cnt holds the exclusive scan after ilp_scan_kernel
    walk_subtree(
        v, i0, s0, [](double) { return false; },
        [&](const IlpSt& s) {
          const int used = P.total_gpus - s.gl;
          if (used <= 0) return true;
          if (w < leaf_cap) {  // placement.hpp:452
            leaf_score[w] = (s.rd < s.rp ? s.rd : s.rp) / static_cast<double>(used);  // std::min(rp, rd) / used
            leaf_used[w] = used;
          }
          ++w;
          return true;
        },
        nullptr, &overflow);
  }
  if (overflow) o->status = 3;
}

// Max-throughput: per-problem exclusive scan of the subtrees' leaf counts
// (in place) and the problem's leaf-list offset.
__global__ void __launch_bounds__(kIlpThreads) ilp_scan_kernel(const DIlpProb* probs, DIlpOut* outs,
                                                               char* front_base, unsigned long long leaf_cap) {
  const int p = blockIdx.x;
  const DIlpProb P = probs[p];
  DIlpOut* o = &outs[p];
  if (P.mode != 1 || o->status) return;
  DFront F = front_at(front_base + P.f_off, P.f_cap);
  const int nfront = o->n_front;
  unsigned long long base = 0;
  for (int c0 = 0; c0 < nfront; c0 += blockDim.x) {
    const int j = c0 + threadIdx.x;
    const unsigned x = j < nfront ? F.leaf_cnt[j] : 0u;
    unsigned off;
    const unsigned tot = block_scan(x, &off);
    if (j < nfront) F.leaf_cnt[j] = static_cast<unsigned>(base + off);
    base += tot;
  }
  if (threadIdx.x == 0) o->leaves = base;
}

// Leaf-list offsets of the max-throughput problems, in problem order.
__global__ void ilp_offsets_kernel(const DIlpProb* probs, DIlpOut* outs, int np) {
  unsigned long long acc = 0;
  for (int p = 0; p < np; ++p) {
    if (probs[p].mode != 1 || outs[p].status) continue;
    outs[p].leaf_off = acc;
    acc += outs[p].leaves;
  }
}

// Prefix counts of frontier node j (the choices recorded by the expansion).
__device__ void frontier_prefix(const DFront& F, const DIlpProb& P, int levels, int j, long long* counts) {
  for (int lv = levels; lv >= 1; --lv) {
    const int e = F.rec_entry[lv * P.f_cap + j];
    if (e >= 0) counts[e] = F.rec_n[lv * P.f_cap + j];
    j = F.rec_parent[lv * P.f_cap + j];
  }
}

__global__ void ilp_finish_kernel(const DIlpProb* probs, DIlpEntries E, DIlpOut* outs, char* front_base,
                                  const double* leaf_score, const int* leaf_used, unsigned long long leaf_cap,
                                  long long* counts_out) {
  const int p = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const DIlpProb P = probs[p];
  DIlpOut* o = &outs[p];
  const View v = view_of(P, E, p);
  DFront F = front_at(front_base + P.f_off, P.f_cap);
  long long* counts = counts_out + P.c_off;
  if (P.mode == 1 && o->status == 0 && o->leaf_off + o->leaves <= leaf_cap) {
    // the reference's `better` rule in leaf order (placement.hpp:448-461),
    // 32 leaves at a time: the first leaf of a group that is better than the
    // current best (in order) updates it, and the scan resumes after it --
    // the same sequence of updates as one thread walking every leaf
    bool found = false;
    double best_score = -1.0;
    int best_gpus = 0;
    unsigned long long best_k = 0;
    const unsigned long long L = o->leaves;
    for (unsigned long long k = 0; k < L;) {
      const unsigned long long idx = k + static_cast<unsigned long long>(lane);
      bool better = false;
      double score = 0.0;
      int used = 0;
      if (idx < L) {
        score = leaf_score[o->leaf_off + idx];
        used = leaf_used[o->leaf_off + idx];
        better = !found || score > best_score + 1e-12 || (fabs(score - best_score) <= 1e-12 && used < best_gpus);
      }
      const unsigned m = __ballot_sync(0xffffffffu, better);
      if (!m) {
        k += 32;
        continue;
      }
      const int first = __ffs(m) - 1;
      best_score = __shfl_sync(0xffffffffu, score, first);
      best_gpus = __shfl_sync(0xffffffffu, used, first);
      best_k = k + static_cast<unsigned long long>(first);
      found = true;
      k = best_k + 1;
    }
    if (lane == 0) {
      o->leaf_best = found ? best_k : ~0ull;
    }
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < P.n; ++i) counts[i] = 0;
  if (o->status) return;
  const int cur = o->n_levels & 1;
  int jw = -1;
  unsigned long long ordinal = 0;
  if (P.mode == 0) {
    if (o->best.obj == ~0ull) {
      o->status = 1;  // InfeasibleError("capacity", ...) (placement.hpp:394-401)
      return;
    }
    jw = static_cast<int>(o->best.code);
  } else {
    if (o->leaf_off + o->leaves > leaf_cap) {
      o->status = 2;
      return;
    }
    const unsigned long long best_k = o->leaf_best;  // the warp's scan above
    if (best_k == ~0ull) {
      o->status = 1;
      return;
    }
    // the subtree holding leaf best_k: the last j with leaf_cnt[j] (exclusive scan) <= best_k
    int lo = 0, hi = o->n_front - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (F.leaf_cnt[mid] <= best_k) lo = mid;
      else hi = mid - 1;
    }
    jw = lo;
    ordinal = best_k - F.leaf_cnt[jw];
  }
  frontier_prefix(F, P, o->n_levels, jw, counts);
  // walk the winner's subtree again: the first optimal leaf (placement) or the
  // ordinal-th counted leaf (max-throughput), and take its path
  int path[kIlpMaxEntries];
  for (int i = 0; i < P.n; ++i) path[i] = 0;
  const IlpSt s0 = F.st[cur][jw];
  const int i0 = F.dep[cur][jw];
  const double target = __longlong_as_double(static_cast<long long>(o->best.obj));
  bool overflow = false, got = false;
  unsigned long long seen = 0;
  IlpSt fin{};
  walk_subtree(
      v, i0, s0, [&](double lb) { return lb > target; },
      [&](const IlpSt& s) {
        if (P.mode == 0) {
          if (s.cost == target) {
            got = true;
            fin = s;
            return false;
          }
          return true;
        }
        if (P.total_gpus - s.gl <= 0) return true;
        if (seen++ == ordinal) {
          got = true;
          fin = s;
          return false;
        }
        return true;
      },
      path, &overflow);
  if (!got || overflow) {
    o->status = 3;
    return;
  }
  for (int i = i0; i < P.n; ++i) counts[i] = path[i];
  o->gpus_used = P.total_gpus - fin.gl;
  o->objective = fin.cost;
}

}  // namespace

namespace bs {

// The host side of one batch: validation, packing, launches, results.
struct IlpProblemIn {
  const bs_table_entry* table;
  int n;
  int total_gpus;
  double target_rps;
  double alpha;
  int mode;
  double max_freq_mhz;
};

struct IlpResultOut {
  int status;  // BS_OK or BS_INFEASIBLE_ERROR / BS_PARAMETER_ERROR
  std::string error;
  std::vector<long long> counts;
  double objective = 0.0;
  int gpus_used = 0;
};

static bool usable_entry(const bs_table_entry& e) { return e.error_code == 0 && e.r_c > 0.0 && e.has_e_c; }

// Largest goodput reachable with each GPU budget, one phase's usable entries
// (an unbounded knapsack over budgets); the smallest budget reaching `need`
// (min_gpus_for_phase, placement.hpp:339-351 -- only for the message of an
// infeasible problem).
static int phase_gpu_floor(const std::vector<bs_table_entry>& t, const std::vector<char>& use, int phase, double need,
                           int budget) {
  std::vector<double> reach(static_cast<size_t>(budget) + 1, 0.0);
  for (int b = 1; b <= budget; ++b) {
    double v = 0.0;
    for (size_t k = 0; k < t.size(); ++k)
      if (use[k] && t[k].config.phase == phase && t[k].g_c <= b) v = std::max(v, reach[b - t[k].g_c] + t[k].r_c);
    reach[b] = std::max(reach[b - 1], v);
    if (reach[b] >= need - 1e-9) return b;
  }
  return -1;
}

static std::string capacity_message(const std::vector<bs_table_entry>& t, const std::vector<char>& use, double need,
                                    int total) {
  auto s = [&](int g) { return g < 0 ? ">" + std::to_string(total) : std::to_string(g); };
  return "prefill needs " + s(phase_gpu_floor(t, use, BS_PHASE_PREFILL, need, total)) + " GPUs, decode needs " +
         s(phase_gpu_floor(t, use, BS_PHASE_DECODE, need, total)) + ", available " + std::to_string(total);
}

int ilp_solve_batch(bs_ctx_t ctx, const std::vector<IlpProblemIn>& in, std::vector<IlpResultOut>& res) {
  const int np = static_cast<int>(in.size());
  res.assign(np, IlpResultOut{});
  // host side: PlacementProblem::validate (placement.hpp:42-51), restriction
  // (placement.hpp:423-430), the no-usable-entry errors (364-367 / 436-441)
  std::vector<std::vector<bs_table_entry>> tabs(np);
  std::vector<std::vector<char>> uses(np);
  std::vector<int> live;
  for (int p = 0; p < np; ++p) {
    const IlpProblemIn& q = in[p];
    IlpResultOut& r = res[p];
    r.status = BS_OK;
    if (q.total_gpus < 1) r.status = BS_PARAMETER_ERROR, r.error = "placement: total_gpus must be >= 1";
    else if (q.target_rps <= 0.0) r.status = BS_PARAMETER_ERROR, r.error = "placement: target_rps must be > 0";
    else if (q.alpha < 0.0) r.status = BS_PARAMETER_ERROR, r.error = "placement: alpha must be >= 0";
    for (int i = 0; i < q.n && r.status == BS_OK; ++i) {
      const bs_table_entry& e = q.table[i];
      if (e.g_c != e.config.tp) r.status = BS_PARAMETER_ERROR, r.error = "placement: G_c must equal tp";
      else if (e.r_c < 0.0) r.status = BS_PARAMETER_ERROR, r.error = "placement: R_c must be >= 0";
      else if (e.r_c > 0.0 && e.has_e_c && e.e_c <= 0.0)
        r.status = BS_PARAMETER_ERROR, r.error = "placement: E_c must be > 0";
    }
    if (r.status) continue;
    tabs[p].assign(q.table, q.table + q.n);
    if (q.mode == 1)
      for (auto& e : tabs[p])
        if (e.config.base_freq_mhz != q.max_freq_mhz) {
          e.r_c = 0.0;
          e.has_e_c = 0;
        }
    uses[p].resize(q.n);
    bool hp = false, hd = false;
    int min_g = 1 << 30, n_use = 0;
    for (int i = 0; i < q.n; ++i) {
      uses[p][i] = usable_entry(tabs[p][i]);
      if (!uses[p][i]) continue;
      (tabs[p][i].config.phase == BS_PHASE_PREFILL ? hp : hd) = true;
      min_g = std::min(min_g, tabs[p][i].g_c);
      ++n_use;
    }
    const char* mx = q.mode == 1 ? " max-frequency" : "";
    if (!hp) {
      r.status = BS_INFEASIBLE_ERROR;
      r.error = std::string("goodput-prefill|no usable") + mx + " prefill configuration" + (q.mode ? "" : " in the table");
      continue;
    }
    if (!hd) {
      r.status = BS_INFEASIBLE_ERROR;
      r.error = std::string("goodput-decode|no usable") + mx + " decode configuration" + (q.mode ? "" : " in the table");
      continue;
    }
    if (q.n > kIlpMaxEntries || std::min(n_use, q.total_gpus / std::max(1, min_g)) > kIlpMaxNz || q.total_gpus > 2047) {
      r.status = BS_PARAMETER_ERROR;
      r.error = "placement: problem exceeds the device search limits (<= 256 entries, <= 2047 GPUs, <= 64 "
                "non-zero counts per plan)";
      continue;
    }
    live.push_back(p);
  }
  if (live.empty()) return BS_OK;
  const int nl = static_cast<int>(live.size());
  // frontier capacity per problem: enough subtrees to spread one problem over
  // the GPU, fewer per problem in large batches
  int f_cap = std::max(1024, std::min(16384, (1 << 20) / nl));
  const int target = std::max(256, f_cap / 4);
  // pack
  std::vector<DIlpProb> hp(nl);
  std::vector<double> hr, he;
  std::vector<int> hg, hph, hu;
  long long f_off = 0;
  int c_off = 0;
  for (int k = 0; k < nl; ++k) {
    const int p = live[k];
    const IlpProblemIn& q = in[p];
    DIlpProb& d = hp[k];
    d.n = q.n;
    d.total_gpus = q.total_gpus;
    d.mode = q.mode;
    d.e_off = static_cast<int>(hr.size());
    d.need = (1.0 + q.alpha) * q.target_rps;  // placement.hpp:369 / 443
    d.f_off = f_off;
    d.f_cap = f_cap;
    d.c_off = c_off;
    f_off += static_cast<long long>((front_bytes(f_cap) + 255) / 256 * 256);
    c_off += q.n;
    for (int i = 0; i < q.n; ++i) {
      const bs_table_entry& e = tabs[p][i];
      hr.push_back(e.r_c);
      he.push_back(e.has_e_c ? e.e_c : 0.0);  // e.e_c.value_or(0.0)
      hg.push_back(e.g_c);
      hph.push_back(e.config.phase);
      hu.push_back(uses[p][i] ? 1 : 0);
    }
  }
  const size_t ne = hr.size();
  const unsigned long long leaf_cap = 1ull << 22;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  // one device region: probs | r | e | g | ph | use | 4 suffix arrays | outs | counts | leaves | frontiers
  const size_t o_prob = 0, o_r = o_prob + up(sizeof(DIlpProb) * nl), o_e = o_r + up(8 * ne),
               o_g = o_e + up(8 * ne), o_ph = o_g + up(4 * ne), o_u = o_ph + up(4 * ne), o_s = o_u + up(4 * ne),
               o_out = o_s + 4 * up(8 * (ne + nl)), o_cnt = o_out + up(sizeof(DIlpOut) * nl),
               o_ls = o_cnt + up(8ull * c_off), o_lu = o_ls + up(8ull * leaf_cap), o_f = o_lu + up(4ull * leaf_cap),
               total = o_f + static_cast<size_t>(f_off);
  const size_t h2d = o_s;  // problems + entry arrays
  char* d = static_cast<char*>(ctx->dev_buf(kSlotIlp, total));
  char* h = static_cast<char*>(ctx->host_buf(kSlotIlp, std::max<size_t>(h2d, up(sizeof(DIlpOut) * nl) + 8ull * c_off)));
  if (!d || !h) return set_error(ctx, BS_CUDA_ERROR, "placement: ILP scratch allocation (%zu bytes) failed", total);
  std::memcpy(h + o_prob, hp.data(), sizeof(DIlpProb) * nl);
  std::memcpy(h + o_r, hr.data(), 8 * ne);
  std::memcpy(h + o_e, he.data(), 8 * ne);
  std::memcpy(h + o_g, hg.data(), 4 * ne);
  std::memcpy(h + o_ph, hph.data(), 4 * ne);
  std::memcpy(h + o_u, hu.data(), 4 * ne);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, h2d, cudaMemcpyHostToDevice, ctx->stream));
  DIlpEntries E;
  E.r = reinterpret_cast<const double*>(d + o_r);
  E.e = reinterpret_cast<const double*>(d + o_e);
  E.g = reinterpret_cast<const int*>(d + o_g);
  E.ph = reinterpret_cast<const int*>(d + o_ph);
  E.use = reinterpret_cast<const int*>(d + o_u);
  E.min_e_p = reinterpret_cast<double*>(d + o_s);
  E.min_e_d = reinterpret_cast<double*>(d + o_s + up(8 * (ne + nl)));
  E.max_rpg_p = reinterpret_cast<double*>(d + o_s + 2 * up(8 * (ne + nl)));
  E.max_rpg_d = reinterpret_cast<double*>(d + o_s + 3 * up(8 * (ne + nl)));
  const DIlpProb* dP = reinterpret_cast<const DIlpProb*>(d + o_prob);
  DIlpOut* dO = reinterpret_cast<DIlpOut*>(d + o_out);
  long long* dC = reinterpret_cast<long long*>(d + o_cnt);
  double* dLS = reinterpret_cast<double*>(d + o_ls);
  int* dLU = reinterpret_cast<int*>(d + o_lu);
  char* dF = d + o_f;
  BS_CUDA_TRY(ctx, cudaMemsetAsync(dO, 0, sizeof(DIlpOut) * nl, ctx->stream));
  ilp_frontier_kernel<<<nl, kIlpThreads, 0, ctx->stream>>>(dP, E, dO, dF, target);
  BS_LAUNCH_CHECK(ctx);
  const dim3 sg((f_cap + kIlpSubThreads - 1) / kIlpSubThreads, nl);
  ilp_subtree_kernel<<<sg, kIlpSubThreads, 0, ctx->stream>>>(dP, E, dO, dF, 0, dLS, dLU, leaf_cap);
  BS_LAUNCH_CHECK(ctx);
  bool any_mt = false;
  for (const auto& q : hp) any_mt |= q.mode == 1;
  if (any_mt) {
    ilp_scan_kernel<<<nl, kIlpThreads, 0, ctx->stream>>>(dP, dO, dF, leaf_cap);
    BS_LAUNCH_CHECK(ctx);
    ilp_offsets_kernel<<<1, 1, 0, ctx->stream>>>(dP, dO, nl);
    BS_LAUNCH_CHECK(ctx);
    ilp_subtree_kernel<<<sg, kIlpSubThreads, 0, ctx->stream>>>(dP, E, dO, dF, 1, dLS, dLU, leaf_cap);
    BS_LAUNCH_CHECK(ctx);
  }
  ilp_finish_kernel<<<nl, 32, 0, ctx->stream>>>(dP, E, dO, dF, dLS, dLU, leaf_cap, dC);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(h, dO, sizeof(DIlpOut) * nl, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(h + up(sizeof(DIlpOut) * nl), dC, 8ull * c_off, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const DIlpOut* ho = reinterpret_cast<const DIlpOut*>(h);
  const long long* hc = reinterpret_cast<const long long*>(h + up(sizeof(DIlpOut) * nl));
  for (int k = 0; k < nl; ++k) {
    const int p = live[k];
    const IlpProblemIn& q = in[p];
    IlpResultOut& r = res[p];
    const DIlpOut& o = ho[k];
    if (o.status == 1) {
      r.status = BS_INFEASIBLE_ERROR;
      r.error = "capacity|" + capacity_message(tabs[p], uses[p], hp[k].need, q.total_gpus);
      continue;
    }
    if (o.status) {
      r.status = BS_PARAMETER_ERROR;
      r.error = o.status == 2 ? "placement: max-throughput enumeration exceeds the device leaf capacity"
                              : "placement: search state exceeded the device stack";
      continue;
    }
    r.counts.assign(hc + hp[k].c_off, hc + hp[k].c_off + q.n);
    r.gpus_used = o.gpus_used;
    r.objective = o.objective;
    if (q.mode == 1) {  // plan.objective_w over the restricted table (placement.hpp:490-495)
      double obj = 0.0;
      for (int i = 0; i < q.n; ++i)
        if (tabs[p][i].has_e_c) obj += static_cast<double>(r.counts[i]) * tabs[p][i].e_c * tabs[p][i].r_c;
      r.objective = obj;
    }
  }
  return BS_OK;
}

}  // namespace bs

namespace {

// A NULL context selects the calling thread's default context on device 0
// (the reference-shaped drop-ins pass none); its messages are then reported
// through bs_last_error(NULL).
int run_ilp(bs_ctx_t ctx, const IlpProblemIn& q, int64_t* counts, double* objective_w, int32_t* gpus_used) {
  bs_ctx_t c = ctx ? ctx : default_ctx();
  if (!c) return set_error(ctx, BS_CUDA_ERROR, "placement: no usable CUDA device for the ILP (no CPU fallback)");
  std::vector<IlpResultOut> res;
  const std::vector<IlpProblemIn> in{q};
  const int rc = ilp_solve_batch(c, in, res);
  if (rc) return ctx ? rc : set_error(nullptr, rc, "%s", c->err.c_str());
  if (res[0].status) return set_error(ctx, res[0].status, "%s", res[0].error.c_str());
  for (int i = 0; i < q.n; ++i) counts[i] = res[0].counts[i];
  if (objective_w) *objective_w = res[0].objective;
  if (gpus_used) *gpus_used = res[0].gpus_used;
  return BS_OK;
}

}  // namespace

extern "C" {

int bs_placement_solve(bs_ctx_t ctx, const bs_table_entry* table, int n, int total_gpus, double target_rps,
                       double alpha, int64_t* counts, double* objective_w, int32_t* gpus_used) {
  if ((!table && n > 0) || !counts || n < 0) return set_error(ctx, BS_PARAMETER_ERROR, "bs_placement_solve: null argument");
  return run_ilp(ctx, IlpProblemIn{table, n, total_gpus, target_rps, alpha, 0, 0.0}, counts, objective_w, gpus_used);
}

int bs_placement_max_throughput(bs_ctx_t ctx, const bs_table_entry* table, int n, int total_gpus, double target_rps,
                                double alpha, double max_freq_mhz, int64_t* counts, double* objective_w,
                                int32_t* gpus_used) {
  if ((!table && n > 0) || !counts || n < 0)
    return set_error(ctx, BS_PARAMETER_ERROR, "bs_placement_max_throughput: null argument");
  return run_ilp(ctx, IlpProblemIn{table, n, total_gpus, target_rps, alpha, 1, max_freq_mhz}, counts, objective_w,
                 gpus_used);
}

int bs_placement_solve_batch(bs_ctx_t ctx, const bs_placement_problem* problems, int n,
                             bs_placement_solution* out) {
  if (!ctx || (!problems && n > 0) || (!out && n > 0))
    return set_error(ctx, BS_PARAMETER_ERROR, "bs_placement_solve_batch: null argument");
  std::vector<IlpProblemIn> in(n);
  for (int p = 0; p < n; ++p) {
    const bs_placement_problem& q = problems[p];
    if ((!q.table && q.n > 0) || !q.counts || q.n < 0)
      return set_error(ctx, BS_PARAMETER_ERROR, "bs_placement_solve_batch: problem %d has a null table or counts", p);
    in[p] = IlpProblemIn{q.table, q.n, q.total_gpus, q.target_rps, q.alpha, q.max_throughput ? 1 : 0,
                         q.max_freq_mhz};
  }
  std::vector<IlpResultOut> res;
  const int rc = ilp_solve_batch(ctx, in, res);
  if (rc) return rc;
  for (int p = 0; p < n; ++p) {
    bs_placement_solution& o = out[p];
    std::memset(&o, 0, sizeof o);
    o.status = res[p].status;
    std::snprintf(o.error, sizeof o.error, "%s", res[p].error.c_str());
    if (o.status) continue;
    for (int i = 0; i < problems[p].n; ++i) problems[p].counts[i] = res[p].counts[i];
    o.objective_w = res[p].objective;
    o.gpus_used = res[p].gpus_used;
  }
  return BS_OK;
}

}  // extern "C"

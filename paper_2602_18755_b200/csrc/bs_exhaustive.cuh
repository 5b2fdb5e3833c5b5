// bs_exhaustive.cuh — exhaustive prefill-MPC rollout on sm_100a (included
// by bs_mpc.cu inside its anonymous namespace).
//
// Semantics: every assignment of the |cand| candidate rungs to the K
// projected batches; feasibility is meets_slo (dvfs.hpp:105-122), the
// objective time_weighted_power (dvfs.hpp:163-171); argmin over (objective,
// assignment in lexicographic frequency order) -- the tie rule dvfs.hpp:243
// applies to greedy; the code of an assignment has batch 0 as its most
// significant base-|cand| digit, so the rule is (objective, code).
//
// Search: level-synchronous breadth-first expansion over ALL decisions of
// the batch.  meets_slo returns false at the first violated batch, so a
// prefix that violates the deadline has no feasible completion: frontiers
// only ever hold feasible prefixes, compacted with warp-aggregated appends.
// Nodes at depth FD = K - I (I = 2 bottom levels, 3 for very wide trees) go
// to the final list; the sweep kernel gives each final node one thread that
// walks its I bottom levels (every leaf in increasing code order) with a
// division-free objective filter and merges (objective, code) minima through
// a 128-bit CAS.  Work is proportional to the feasible part of the tree, and
// every level is spread over the whole GPU however uneven the decisions are.

#ifndef BS_SWEEP3_MIN
#define BS_SWEEP3_MIN 16777216.0  // default: prefixes at depth K - 2 above which the sweep takes 3 levels
#endif

struct ExCtl {
  unsigned long long level_count[kMaxK + 1];  // BFS list sizes per depth
  unsigned long long final_count;
  unsigned long long overflow;  // appends dropped for lack of capacity (must stay 0)
  unsigned long long n_loose;   // decisions prepare_kernel found loose (candidates for BFS-settled final nodes)
  unsigned long long n_thr;     // decisions listed for thr_kernel (three swept levels, or loose)
  unsigned long long sweep_next;  // next unclaimed final-list entry (three-level sweep: warps claim runs)
#ifdef BS_SWEEP_STATS
  unsigned long long st_nodes, st_children, st_rows_eval, st_leaves_eval, st_div, st_thr_nodes, st_slow_nodes,
      st_empty_nodes;
#endif
};

// Bottom levels swept per final node: 2, or 3 for trees wider than
// `sweep3_min` prefixes at depth K - 2 (default 2^24, measured at C5, 24^8:
// the deeper final list of I = 2 costs more traffic and frontier work than
// the longer sweep saves).  The threshold is a context setting
// (bs_ctx_set_exhaustive_limits) so the tests can drive small trees through
// the three-level sweep.
__host__ __device__ inline int sweep_levels(int K, int nc, double sweep3_min) {
  if (K <= 2) return K;
  double np = 1.0;
  for (int i = 0; i < K - 2; ++i) np *= nc;
  return np > sweep3_min ? 3 : 2;
}

// A slice of one decision's code space (bs_slice): the assignments whose
// first `digits` digits (batch 0 most significant), read as a base-nc
// number, lie in [lo, hi).  digits == 0: the whole tree.  A projection
// shorter than `digits` reads its missing digits as 0, so the slices of a
// partition of [0, nc^digits) partition every tree.
struct DSlice {
  int digits;
  int _pad;
  unsigned long long lo, hi;
};

// Leading-digit value of a prefix of `depth` digits (depth >= digits), or of
// a complete assignment of K < digits digits (missing digits 0).
__host__ __device__ inline unsigned long long slice_key(unsigned long long code, int depth, int digits, int nc) {
  unsigned long long v = code;
  if (depth >= digits) {
    for (int i = digits; i < depth; ++i) v /= static_cast<unsigned long long>(nc);
  } else {
    for (int i = depth; i < digits; ++i) v *= static_cast<unsigned long long>(nc);
  }
  return v;
}

__host__ __device__ inline bool in_slice(const DSlice& s, unsigned long long code, int depth, int nc) {
  if (s.digits == 0) return true;
  const unsigned long long v = slice_key(code, depth, s.digits, nc);
  return v >= s.lo && v < s.hi;
}

// Number of K-digit assignments in the slice.
__host__ __device__ inline unsigned long long slice_size(const DSlice& s, int K, int nc) {
  unsigned long long total = 1;
  for (int i = 0; i < K; ++i) total *= static_cast<unsigned long long>(nc);
  if (s.digits == 0) return total;
  unsigned long long lead = 1;
  for (int i = 0; i < s.digits; ++i) lead *= static_cast<unsigned long long>(nc);
  const unsigned long long lo = s.lo < lead ? s.lo : lead, hi = s.hi < lead ? s.hi : lead;
  if (hi <= lo) return 0;
  if (K >= s.digits) return (hi - lo) * (total / lead);
  const unsigned long long m = lead / total;  // codes c with c * m in [lo, hi)
  return (hi + m - 1) / m - (lo + m - 1) / m;
}

// Leaf-count thresholds of the two bottom levels (K-2, K-1) of one decision.
// A node at depth K-2 with clock t and last digit l has the leaf (g, f)
// feasible iff both meets_slo checks pass:
//   fl(fl(t + s1) - m[K-2]) <= ttft  and  fl(fl(fl(t + s1) + s2) - m[K-1]) <= ttft,
// s1 = B1[K-2][g] (g != l) or B0[K-2][g] (g == l), s2 = B1[K-1][f] (f != g)
// or B0[K-1][f].  Correctly rounded add / subtract are monotone, so each
// test holds exactly for t <= tau, one double per (g, f, switched): found by
// bisection over the doubles' order with the sweep's own op sequence.  The
// node's feasible-leaf count is then
//   #{tau_S >= t over all (g, f)} - #{tau_S[l][f] >= t} + #{tau_N[l][f] >= t},
// three binary searches over descending arrays instead of a walk over the
// node's children rows.
struct DThr {
  double cs[kMaxCand * kMaxCand];  // every switched tau_S, descending
  double rs[kMaxCand * kMaxCand];  // row g: tau_S[g][*], descending (stride nc)
  double rn[kMaxCand * kMaxCand];  // row g: tau_N[g][*] (g the node's last digit), descending
};

// Number of leading entries >= t of a descending array, by branch-free
// halving: the step count depends on n only, and a step's load does not wait
// on a branch.
__device__ __forceinline__ int count_ge(const double* __restrict__ a, int n, double t) {
  if (n <= 0) return 0;
  int base = 0;
  for (int len = n; len > 1;) {
    const int half = len >> 1;
    base = a[base + half] >= t ? base + half : base;
    len -= half;
  }
  return base + (a[base] >= t ? 1 : 0);
}

// Feasible leaves below a node at depth K-2 (clock t, last digit l).  The
// three searches run in lockstep (the two row searches finish within the
// table-wide one), so their loads are in flight together.
__device__ __forceinline__ int thr_leaf_count(const DThr* __restrict__ H, int nc, double t, int l) {
  const double* __restrict__ cs = H->cs;
  const double* __restrict__ rs = H->rs + l * nc;
  const double* __restrict__ rn = H->rn + l * nc;
  int b0 = 0, b1 = 0, b2 = 0, l1 = nc;
  for (int l0 = nc * nc; l0 > 1;) {
    const int h0 = l0 >> 1;
    const double v0 = cs[b0 + h0];
    if (l1 > 1) {
      const int h1 = l1 >> 1;
      const double v1 = rs[b1 + h1], v2 = rn[b2 + h1];
      b1 = v1 >= t ? b1 + h1 : b1;
      b2 = v2 >= t ? b2 + h1 : b2;
      l1 -= h1;
    }
    b0 = v0 >= t ? b0 + h0 : b0;
    l0 -= h0;
  }
  return (b0 + (cs[b0] >= t ? 1 : 0)) - (b1 + (rs[b1] >= t ? 1 : 0)) + (b2 + (rn[b2] >= t ? 1 : 0));
}

// thr_leaf_count for siblings visited in increasing clock order (the sorted
// switched order): the table-wide count is non-increasing in t, so the
// previous sibling's count bounds it and a short walk down usually finds it
// (a bounded walk, then a binary search below it).  *hint: the previous
// count (nc * nc before the first sibling), updated.
__device__ __forceinline__ int thr_leaf_count_walk(const DThr* __restrict__ H, int nc, double t, int l, int* hint) {
  const double* __restrict__ cs = H->cs;
  int c = *hint;
  // the node's two rows (same length) searched in lockstep: their loads in flight together
  const double* __restrict__ rs = H->rs + l * nc;
  const double* __restrict__ rn = H->rn + l * nc;
  int b1 = 0, b2 = 0;
  for (int len = nc; len > 1;) {
    const int half = len >> 1;
    const double v1 = rs[b1 + half], v2 = rn[b2 + half];
    b1 = v1 >= t ? b1 + half : b1;
    b2 = v2 >= t ? b2 + half : b2;
    len -= half;
  }
  const int r1 = b1 + (rs[b1] >= t ? 1 : 0), r2 = b2 + (rn[b2] >= t ? 1 : 0);
#pragma unroll 1
  for (int s = 0; s < 4 && c > 0 && !(cs[c - 1] >= t); ++s) --c;
  if (c > 0 && !(cs[c - 1] >= t)) c = count_ge(cs, c, t);
  *hint = c;
  return c - r1 + r2;
}

// The seed's node bound ("seed node bound"): every leaf below a
// node at depth K-2 with (num, den) has a rounded objective above the seed's
// (a genuine feasible key, so none of them is the argmin).  With beta =
// thr_seed (1 + 2^-47) and Q_k = min_x (E[k][x] - beta A[k][x]) over the two
// bottom levels, num - beta den + Q_K-2 + Q_K-1 > 0 suffices (A >= 0);
// nb_R >= -(Q_K-2 + Q_K-1) with its rounding margin, clamped at 0.
// Precondition: filter_ok tables, den >= 2^-900.
__device__ __forceinline__ bool node_dom_seed(const DTables* __restrict__ T, double num, double den) {
  return den >= kFilterMinDen &&
         __dsub_rn(num, __dmul_rn(T->nb_beta, den)) > __dadd_rn(T->nb_R, __dmul_rn(num, 0x1p-40));
}

// Order-preserving map of doubles to unsigned integers (and back).
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// The largest double t for which both bottom-level checks pass (-inf: none;
// +inf: every finite t).
// The largest double t with ok(t) for a predicate that holds on a down-set
// of the doubles (-inf: none; +inf: every finite t): the boundary bracketed
// by galloping from the real-arithmetic estimate x0 (within a few ulps
// unless an operand swamps another), then bisected, on the order-preserving
// integer image of the doubles.
template <typename Ok>
__device__ double sup_down_set(Ok&& ok, double x0) {
  const double big = 1.7976931348623157e308;
  if (ok(big)) return INFINITY;
  if (!ok(-big)) return -INFINITY;
  const unsigned long long kmin = dkey(-big), kmax = dkey(big);
  if (!(x0 == x0)) x0 = 0.0;
  unsigned long long k0 = dkey(x0 < -big ? -big : (x0 > big ? big : x0));
  unsigned long long lo, hi;  // ok(lo), !ok(hi)
  unsigned long long step = 1;
  if (ok(dval(k0))) {
    lo = k0;
    for (;;) {
      const unsigned long long nk = kmax - lo > step ? lo + step : kmax;
      if (!ok(dval(nk))) {
        hi = nk;
        break;
      }
      lo = nk;
      step <<= 1;
    }
  } else {
    hi = k0;
    for (;;) {
      const unsigned long long nk = hi - kmin > step ? hi - step : kmin;
      if (ok(dval(nk))) {
        lo = nk;
        break;
      }
      hi = nk;
      step <<= 1;
    }
  }
  while (hi - lo > 1) {
    const unsigned long long mid = lo + ((hi - lo) >> 1);
    if (ok(dval(mid)))
      lo = mid;
    else
      hi = mid;
  }
  return dval(lo);
}

// Both bottom checks of leaf (g, f) from a depth-(K-2) clock t: level-K-2
// step s1 and deadline m1, leaf step s2 and deadline m2.
__device__ double leaf_threshold(double s1, double m1, double s2, double m2, double ttft) {
  auto ok = [&](double t) {
    const double t2 = __dadd_rn(t, s1);
    if (__dsub_rn(t2, m1) > ttft) return false;                 // dvfs.hpp:117 at level K-2
    return !(__dsub_rn(__dadd_rn(t2, s2), m2) > ttft);          // and at level K-1
  };
  const double x1 = __dsub_rn(__dadd_rn(ttft, m1), s1), x2 = __dsub_rn(__dsub_rn(__dadd_rn(ttft, m2), s1), s2);
  return sup_down_set(ok, x1 < x2 ? x1 : x2);
}

// Per-step thresholds (DTables::thsw / th0, levels 1 .. K-1): the supremum
// of the clocks t with !(fl(fl(t + s) - minarr[k]) > ttft) for every
// switched step (sorted position) and non-switching step of a level, so the
// search's checks are single comparisons; the child records' th0n field is
// filled from them.  The whole CTA must call it (sorted tables).
__device__ __noinline__ void step_thresholds(DTables* __restrict__ T) {
  const int K = T->K, nc = T->nc;
  const double ttft = T->ttft;
  for (int e = threadIdx.x; e < (K - 1) * 2 * nc; e += blockDim.x) {
    const int k = 1 + e / (2 * nc), r = e % (2 * nc), j = r % nc;
    const bool sw = r < nc;
    const double s = sw ? T->sb[k][j] : T->B0[k][j], m = T->minarr[k];
    auto ok = [&](double t) { return !(__dsub_rn(__dadd_rn(t, s), m) > ttft); };
    (sw ? T->thsw : T->th0)[k][j] = sup_down_set(ok, __dsub_rn(__dadd_rn(ttft, m), s));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < (K - 1) * nc; e += blockDim.x) {
    const int k = e / nc, r = e % nc;
    T->srec[k][r].th0n = T->th0[k + 1][T->ord[k][r]];
  }
  __syncthreads();
}

// Completion bounds (exhaustive search): rexist[d][l] = sup{t : a node at
// depth d (1 <= d <= K-2) with clock t and last digit l has a feasible leaf}; a node has one
// iff its clock <= rexist[d][l] (each supremum is attained: it is a double
// where every check passes).  With sigma_S / sigma_N[d][g] the supremum for
// the switched / non-switching child g,
//   rexist[d][l] = max(max_{g != l} sigma_S[d][g], sigma_N[d][l]);
// at d = K-2, sigma[g] is the largest threshold of row g -- its head, the leaf
// with the smallest step (taus are non-increasing in the leaf step):
// min(B0[K-1][g], the smallest switched step of another rung); above, the
// child must pass level d and then reach its own bound:
//   sigma[d][g] = sup{t : fl(fl(t + s) - m_d) <= ttft, fl(t + s) <= rexist[d+1][g]}
// (both monotone in t).  Levels K-2 down to 1, 2N suprema per level (one per
// thread); the whole CTA must call it.
__device__ __noinline__ void leaf_exists_bounds(DTables* __restrict__ T) {
  __shared__ double s_rho[2 * kMaxCand];
  const int K = T->K, nc = T->nc;
  const bool ok = T->sorted_ok && nc >= 1;
  for (int d = K - 2; d >= 1 && ok; --d) {
    if (threadIdx.x < 2 * nc) {
      const int g = threadIdx.x % nc;
      const bool sw = threadIdx.x < nc;
      const double s = sw ? T->B1[d][g] : T->B0[d][g], m = T->minarr[d], ttft = T->ttft;
      double sig;
      if (d == K - 2) {
        const int kl = K - 1;
        double s2 = T->B0[kl][g];
        if (nc > 1) {
          const double other = T->ord[kl][0] != g ? T->sb[kl][0] : T->sb[kl][1];
          s2 = other < s2 ? other : s2;
        }
        sig = leaf_threshold(s, m, s2, T->minarr[kl], ttft);
      } else {
        const double rn = T->rexist[d + 1][g];
        auto child_ok = [&](double t) {
          const double t2 = __dadd_rn(t, s);
          return !(__dsub_rn(t2, m) > ttft) && !(t2 > rn);
        };
        const double x1 = __dsub_rn(__dadd_rn(ttft, m), s), x2 = __dsub_rn(rn, s);
        sig = sup_down_set(child_ok, x1 < x2 ? x1 : x2);
      }
      s_rho[threadIdx.x] = sig;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // max over g != l of s_rho[g] from the top two (max is exact in any order)
      const int l = threadIdx.x;
      const double v = l < nc ? s_rho[l] : -INFINITY;
      double m1 = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, m1, o);
        m1 = w > m1 ? w : m1;
      }
      const int i1 = __ffs(__ballot_sync(0xffffffffu, l < nc && v == m1)) - 1;
      double m2 = l == i1 ? -INFINITY : v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, m2, o);
        m2 = w > m2 ? w : m2;
      }
      if (l < nc) {
        const double other = l == i1 ? m2 : m1;
        const double own = s_rho[nc + l];
        T->rexist[d][l] = other > own ? other : own;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) T->rex_ok = ok ? 1 : 0;
  __syncthreads();
}

// Builds H for decision T (K >= 3, sorted tables) with the whole CTA
// (called by prepare_kernel; every thread must call it).
// Rows need no sort: for a fixed level-(K-2) step, tau is non-increasing in
// the leaf step s2 (rounding is monotone), and the leaf steps of a row are
// the level's switched steps in their sorted order (ord[K-1]) with the
// non-switching leaf f == g (B0 <= B1) moved to its place.  The switched
// thresholds of all rows are then merged into cs by ranks counted against
// every other threshold (broadcast shared-memory reads; equal values
// ordered by row, then position).  Out of line: its registers and shared
// memory stay out of the rest of prepare_kernel.
__device__ __noinline__ void build_thresholds(const DTables* __restrict__ T, DThr* H) {
  __shared__ double s_rows[2 * kMaxCand * kMaxCand];
  __shared__ double s_b0k[kMaxCand], s_b1k[kMaxCand], s_b0l[kMaxCand], s_b1l[kMaxCand];
  __shared__ unsigned char s_pos[kMaxCand], s_rank[kMaxCand], s_ord[kMaxCand];
  const int K = T->K, nc = T->nc, k = K - 2, kl = K - 1, M = nc * nc;
  const double m1 = T->minarr[k], m2 = T->minarr[kl], ttft = T->ttft;
  for (int x = threadIdx.x; x < nc; x += blockDim.x) {
    const double b0 = T->B0[kl][x];
    s_b0k[x] = T->B0[k][x];
    s_b1k[x] = T->B1[k][x];
    s_b0l[x] = b0;
    s_b1l[x] = T->B1[kl][x];
    s_rank[x] = T->rank[kl][x];
    s_ord[x] = T->ord[kl][x];
    int p = 0;  // the non-switching leaf's position in row x: switched steps below B0[K-1][x] (x's own excluded)
    for (int j = 0; j < nc; ++j) p += T->sb[kl][j] < b0 ? 1 : 0;
    if (T->B1[kl][x] < b0) --p;  // only with a negative switch latency
    s_pos[x] = static_cast<unsigned char>(p);
  }
  __syncthreads();
  double* sS = s_rows;
  double* sN = s_rows + M;
  for (int e = threadIdx.x; e < 2 * M; e += blockDim.x) {
    const bool sw = e < M;
    const int r = sw ? e : e - M, g = r / nc, j = r - g * nc;
    const int p = s_pos[g], rg = s_rank[g];
    int f;  // the leaf at position j of row g
    if (j == p) {
      f = g;
    } else {
      const int i = j < p ? j : j - 1;  // index into the switched order without g
      f = s_ord[i < rg ? i : i + 1];
    }
    const double tau = leaf_threshold(sw ? s_b1k[g] : s_b0k[g], m1, f == g ? s_b0l[g] : s_b1l[f], m2, ttft);
    (sw ? sS : sN)[r] = tau;
    (sw ? H->rs : H->rn)[r] = tau;
  }
  __syncthreads();
  // cs = the switched thresholds merged, descending: rank of (g, j) counts
  // the larger ones and the equal ones earlier in (row, position) order
  for (int e = threadIdx.x; e < M; e += blockDim.x) {
    const double x = sS[e];
    int rank = 0;
    for (int o = 0; o < M; ++o) {
      const double y = sS[o];
      rank += (y > x || (y == x && o < e)) ? 1 : 0;
    }
    H->cs[rank] = x;
  }
  __syncthreads();
}

// Frontier lists in HBM, structure of arrays.
struct Frontier {
  int* d;                    // problem
  unsigned long long* code;  // prefix code, batch 0 most significant
  double* t;                 // meets_slo clock after the prefix
  double* num;               // sum lat * pow
  double* den;               // sum lat
  int* last;                 // last digit (switch test of the next level)
};

__host__ __device__ inline size_t frontier_bytes(unsigned long long cap) { return 40ull * cap + 6 * 256; }

__host__ __device__ inline Frontier frontier_at(void* base, unsigned long long cap) {
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  Frontier f;
  f.t = reinterpret_cast<double*>(take(8 * cap));
  f.num = reinterpret_cast<double*>(take(8 * cap));
  f.den = reinterpret_cast<double*>(take(8 * cap));
  f.code = reinterpret_cast<unsigned long long*>(take(8 * cap));
  f.d = reinterpret_cast<int*>(take(4 * cap));
  f.last = reinterpret_cast<int*>(take(4 * cap));
  return f;
}

// Final list: (problem, code) only; the sweep re-walks the prefix.
struct FinalList {
  int* d;
  unsigned long long* code;
};

__host__ __device__ inline size_t final_bytes(unsigned long long cap) { return 12ull * cap + 2 * 256; }

__host__ __device__ inline FinalList final_at(void* base, unsigned long long cap) {
  char* p = static_cast<char*>(base);
  FinalList f;
  f.code = reinterpret_cast<unsigned long long*>(p);
  f.d = reinterpret_cast<int*>(p + (8 * cap + 255) / 256 * 256);
  return f;
}

// Child of node (t, num, den, last) at level k, digit f: meets_slo's step
// (dvfs.hpp:111-118) and the time_weighted_power accumulation (167-168).
// Returns feasibility at level k.
__device__ __forceinline__ bool child_state(const DTables* __restrict__ T, int k, double t, double num, double den,
                                            int last, int f, double& ct, double& cn, double& cd) {
  if (k == 0) {
    ct = T->T1[f];
    cn = __dadd_rn(0.0, T->E[0][f]);
    cd = __dadd_rn(0.0, T->A[0][f]);
  } else {
    ct = __dadd_rn(t, f == last ? T->B0[k][f] : T->B1[k][f]);
    cn = __dadd_rn(num, T->E[k][f]);
    cd = __dadd_rn(den, T->A[k][f]);
  }
  return !(__dsub_rn(ct, T->minarr[k]) > T->ttft);
}

// Warp-aggregated append of `want` entries (one per lane that wants one);
// returns this lane's slot.
__device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, bool want) {
  const unsigned mask = __ballot_sync(0xffffffffu, want);
  if (mask == 0u) return 0;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(counter, static_cast<unsigned long long>(__popc(mask)));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(mask & ((1u << lane) - 1u));
}

// Number of candidates at level k whose switched step passes meets_slo's
// check from parent clock t (t unused at level 0, where the keys are T1):
// by monotonicity of correctly rounded add/subtract in the step, the
// passing candidates form a prefix of the sorted order ord[k].
__device__ __forceinline__ int feasible_prefix(const DTables* __restrict__ T, int k, int nc, double t) {
  // the passing positions are a prefix: branch-free halving for its length
  if (nc <= 0) return 0;
  int base = 0;
  if (k == 0) {  // level 0's keys are the clocks themselves (T1)
    const double m = T->minarr[0], ttft = T->ttft;
    const double* __restrict__ sb = T->sb[0];
    for (int len = nc; len > 1;) {
      const int half = len >> 1;
      base = !(__dsub_rn(sb[base + half], m) > ttft) ? base + half : base;
      len -= half;
    }
    return base + (!(__dsub_rn(sb[base], m) > ttft) ? 1 : 0);
  }
  const double* __restrict__ th = T->thsw[k];  // t passes position j iff t <= th[j]
  for (int len = nc; len > 1;) {
    const int half = len >> 1;
    base = !(t > th[base + half]) ? base + half : base;
    len -= half;
  }
  return base + (!(t > th[base]) ? 1 : 0);
}

// Does the non-switching child (step B0[k][last], k >= 1) pass meets_slo's check?
__device__ __forceinline__ bool diag_passes(const DTables* __restrict__ T, int k, double t, int last) {
  return !(t > T->th0[k][last]);
}

// Number of children of (t, last) at level k that pass the check, without
// visiting them: the sorted prefix, less f == last if it lies in it (its
// real step is B0), plus the non-switching child if it passes.
__device__ __forceinline__ int count_feasible_children(const DTables* __restrict__ T, int k, int nc, double t,
                                                       int last) {
  int c = feasible_prefix(T, k, nc, t);
  if (k > 0) {
    if (T->rank[k][last] < c) c -= 1;
    if (diag_passes(T, k, t, last)) c += 1;
  }
  return c;
}

// Block-aggregated appends to two counters (one atomic per counter per
// block instead of per warp): each lane that wants a slot gets one.  Every
// thread of the block must call it.
__device__ __forceinline__ void block_append2(unsigned long long* c0, bool w0, unsigned long long* c1, bool w1,
                                              unsigned long long* s0, unsigned long long* s1) {
  __shared__ unsigned wc0[32], wc1[32];
  __shared__ unsigned long long b0, b1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned m0 = __ballot_sync(0xffffffffu, w0), m1 = __ballot_sync(0xffffffffu, w1);
  if (lane == 0) {
    wc0[warp] = __popc(m0);
    wc1[warp] = __popc(m1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the per-warp counts, then one atomic per counter
    unsigned v0 = threadIdx.x < nw ? wc0[threadIdx.x] : 0u, v1 = threadIdx.x < nw ? wc1[threadIdx.x] : 0u;
    unsigned i0 = v0, i1 = v1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned a = __shfl_up_sync(0xffffffffu, i0, o), b = __shfl_up_sync(0xffffffffu, i1, o);
      if (threadIdx.x >= o) {
        i0 += a;
        i1 += b;
      }
    }
    if (threadIdx.x == 31) {
      b0 = i0 ? atomicAdd(c0, static_cast<unsigned long long>(i0)) : 0ull;
      b1 = i1 ? atomicAdd(c1, static_cast<unsigned long long>(i1)) : 0ull;
    }
    if (threadIdx.x < nw) {
      wc0[threadIdx.x] = i0 - v0;
      wc1[threadIdx.x] = i1 - v1;
    }
  }
  __syncthreads();
  const unsigned below = (1u << lane) - 1u;
  *s0 = b0 + wc0[warp] + __popc(m0 & below);
  *s1 = b1 + wc1[warp] + __popc(m1 & below);
  __syncthreads();  // the shared slots are reused by the next call
}

// Block-aggregated appends of variable counts to two counters: thread i
// reserves n0 slots of c0 and n1 of c1 (contiguous per thread, threads in
// order within the block), one atomic per counter per block.  Every thread
// of the block must call it.
__device__ __forceinline__ void block_append2n(unsigned long long* c0, unsigned n0, unsigned long long* c1, unsigned n1,
                                               unsigned long long* s0, unsigned long long* s1) {
  __shared__ unsigned wc0[32], wc1[32];
  __shared__ unsigned long long b0, b1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned i0 = n0, i1 = n1;  // inclusive warp scans
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned a = __shfl_up_sync(0xffffffffu, i0, o), b = __shfl_up_sync(0xffffffffu, i1, o);
    if (lane >= o) {
      i0 += a;
      i1 += b;
    }
  }
  if (lane == 31) {
    wc0[warp] = i0;
    wc1[warp] = i1;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the per-warp totals, then one atomic per counter
    const unsigned v0 = threadIdx.x < nw ? wc0[threadIdx.x] : 0u, v1 = threadIdx.x < nw ? wc1[threadIdx.x] : 0u;
    unsigned j0 = v0, j1 = v1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned a = __shfl_up_sync(0xffffffffu, j0, o), b = __shfl_up_sync(0xffffffffu, j1, o);
      if (threadIdx.x >= o) {
        j0 += a;
        j1 += b;
      }
    }
    if (threadIdx.x == 31) {
      b0 = j0 ? atomicAdd(c0, static_cast<unsigned long long>(j0)) : 0ull;
      b1 = j1 ? atomicAdd(c1, static_cast<unsigned long long>(j1)) : 0ull;
    }
    if (threadIdx.x < nw) {
      wc0[threadIdx.x] = j0 - v0;
      wc1[threadIdx.x] = j1 - v1;
    }
  }
  __syncthreads();
  *s0 = b0 + wc0[warp] + (i0 - n0);
  *s1 = b1 + wc1[warp] + (i1 - n1);
  __syncthreads();  // the shared slots are reused by the next call
}

// Level k >= 2, one thread per depth-k node: its children that pass
// meets_slo's check are the sorted prefix of the level (feasible_prefix, by
// monotonicity), less f == last, plus the non-switching child when it passes
// -- so no (node, digit) pair that fails is touched.  Children at the
// problem's FD go to the final list, and only when one of their own children
// passes (no feasible leaf below otherwise); visited in step order, their
// clocks never decrease, so that test walks one sorted-prefix count down.
// Pass 1 marks the kept children by digit, pass 2 writes them in digit order
// (the layout of a (node, digit) expansion: siblings contiguous, in code
// order) after a block-aggregated append.
// Expansion of one depth-k node per thread (valid: the thread holds one);
// every thread of the block must call it.  Its children that pass
// meets_slo's check are the sorted prefix of the level (feasible_prefix, by
// monotonicity), less f == last, plus the non-switching child when it passes
// -- so no (node, digit) pair that fails is touched.  Children at the
// problem's FD go to the final list, and only when one of their own children
// passes (no feasible leaf below otherwise); visited in step order, their
// clocks never decrease, so that test walks one sorted-prefix count down.
// Pass 1 marks the kept children by digit, pass 2 writes them in digit order
// (the layout of a (node, digit) expansion: siblings contiguous, in code
// order) after a block-aggregated append.
template <bool FUSE>
__device__ __forceinline__ unsigned expand_node(const DTables* __restrict__ tables, int k, ExCtl* ctl, bool valid, int d,
                                            double t, double num, double den, int last, unsigned long long code,
                                            Frontier out, FinalList fin, unsigned long long cap_out,
                                            unsigned long long cap_final, const DThr* __restrict__ thr,
                                            unsigned long long* feas, bool fuse_batch = false) {
  unsigned keep = 0u;  // bit f: child f kept
  bool to_final = false;
  int nc = 0;
  const DTables* __restrict__ T = tables;
  if (valid) {
    T = &tables[d];
    nc = T->nc;
    to_final = (k + 1) == T->FD;
    if (T->sorted_ok) {
      const bool prune = to_final && k + 1 < T->K;
      // children at depths 2..K-2 are kept only with a feasible leaf below
      // (exact: clock <= rexist[depth][digit], leaf_exists_bounds)
      const bool rex = T->rex_ok && k + 1 <= T->K - 2;
      const int c = feasible_prefix(T, k, nc, t);
      const unsigned char* __restrict__ ord = T->ord[k];
      const double* __restrict__ sb = T->sb[k];
      const int kl = k + 1;
      int cl = -1;
      for (int j = 0; j < c; ++j) {
        const int f = ord[j];
        if (f == last) continue;
        bool ok = true;
        if (rex) {
          ok = !(__dadd_rn(t, sb[j]) > T->rexist[kl][f]);
        } else if (prune) {
          const double ct = __dadd_rn(t, sb[j]);
          if (cl < 0) {
            cl = feasible_prefix(T, kl, nc, ct);
          } else {
            const double* __restrict__ thl = T->thsw[kl];
            while (cl > 0 && ct > thl[cl - 1]) --cl;
          }
          ok = cl > 0 || diag_passes(T, kl, ct, f);
        }
        if (ok) keep |= 1u << f;
      }
      if (diag_passes(T, k, t, last)) {
        bool ok = true;
        if (rex) {
          ok = !(__dadd_rn(t, T->B0[k][last]) > T->rexist[kl][last]);
        } else if (prune) {
          const double ct = __dadd_rn(t, T->B0[k][last]);
          ok = feasible_prefix(T, kl, nc, ct) > 0 || diag_passes(T, kl, ct, last);
        }
        if (ok) keep |= 1u << last;
      }
    } else {  // unsorted tables: every digit
      for (int f = 0; f < nc; ++f) {
        double ct, cn, cd;
        if (child_state(T, k, t, num, den, last, f, ct, cn, cd)) keep |= 1u << f;
      }
    }
    // Final nodes at depth K-2 whose leaves are all worse than the seed are
    // settled here: their feasible leaves are counted from the thresholds and
    // they never reach the final list (or the sweep).
    if (FUSE && to_final && T->fuse && fuse_batch && k + 1 == T->K - 2) {
      unsigned long long cnt = 0;
      for (unsigned kk = keep; kk;) {
        const int f = __ffs(kk) - 1;
        kk &= kk - 1u;
        double ct, cn, cd;
        child_state(T, k, t, num, den, last, f, ct, cn, cd);
        if (node_dom_seed(T, cn, cd)) {
          cnt += static_cast<unsigned long long>(thr_leaf_count(thr + d, nc, ct, f));
          keep &= ~(1u << f);
        }
      }
      if (cnt) atomicAdd(&feas[d], cnt);
    }
  }
  const unsigned m = static_cast<unsigned>(__popc(keep));
  unsigned long long sf, so;
  block_append2n(&ctl->final_count, to_final ? m : 0u, &ctl->level_count[k + 1], to_final ? 0u : m, &sf, &so);
  // Pass 2, warp-cooperative so the stores coalesce: the warp's children of
  // each list occupy one contiguous slot range (block_append2n keeps lanes
  // in order), and lane l writes items l, l + 32, ... of it, fetching the
  // owner node's state by shuffles.
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int list = 0; list < 2; ++list) {
    const bool mine = (list == 0) == to_final;
    const unsigned cnt = mine ? m : 0u;
    unsigned inc = cnt;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    const unsigned total = __shfl_sync(0xffffffffu, inc, 31);
    if (total == 0u) continue;
    // the warp's first slot of this list (every lane with cnt > 0 agrees; take the first)
    const unsigned long long my_start = (list == 0 ? sf : so) - (inc - cnt);
    const int first = __ffs(__ballot_sync(0xffffffffu, cnt > 0u)) - 1;
    const unsigned long long wbase = __shfl_sync(0xffffffffu, my_start, first);
    const unsigned long long cap = list == 0 ? cap_final : cap_out;
    for (unsigned b0 = 0; b0 < total; b0 += 32u) {
      const unsigned idx = b0 + static_cast<unsigned>(lane);
      int o = 0;  // owner: the first lane whose inclusive count exceeds idx
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const unsigned probe = __shfl_sync(0xffffffffu, inc, o + step - 1);
        if (probe <= idx) o += step;
      }
      const unsigned o_inc = __shfl_sync(0xffffffffu, inc, o), o_cnt = __shfl_sync(0xffffffffu, cnt, o);
      const unsigned o_keep = __shfl_sync(0xffffffffu, keep, o);
      const int o_d = __shfl_sync(0xffffffffu, d, o), o_last = __shfl_sync(0xffffffffu, last, o);
      const int o_nc = __shfl_sync(0xffffffffu, nc, o);
      const unsigned long long o_code = __shfl_sync(0xffffffffu, code, o);
      const double o_t = __shfl_sync(0xffffffffu, t, o), o_num = __shfl_sync(0xffffffffu, num, o),
                   o_den = __shfl_sync(0xffffffffu, den, o);
      if (idx >= total) continue;
      const int r = static_cast<int>(idx - (o_inc - o_cnt));
      const int f = static_cast<int>(__fns(o_keep, 0, r + 1));
      const unsigned long long slot = wbase + idx;
      const unsigned long long cc = o_code * static_cast<unsigned long long>(o_nc) + static_cast<unsigned long long>(f);
      if (slot >= cap) {
        atomicAdd(&ctl->overflow, 1ull);
      } else if (list == 0) {
        fin.d[slot] = o_d;
        fin.code[slot] = cc;
      } else {
        double ct, cn, cd;
        child_state(&tables[o_d], k, o_t, o_num, o_den, o_last, f, ct, cn, cd);
        out.d[slot] = o_d;
        out.code[slot] = cc;
        out.t[slot] = ct;
        out.num[slot] = cn;
        out.den[slot] = cd;
        out.last[slot] = f;
      }
    }
  }
  return m;
}

// Level k >= 3 of the search (prepare_kernel expands depths 1-3): one
// thread per depth-k node, expand_node.
__global__ void __launch_bounds__(256) bfs_node_kernel(const DTables* __restrict__ tables, int k, ExCtl* ctl,
                                                       Frontier in, Frontier out, FinalList fin,
                                                       unsigned long long cap_out, unsigned long long cap_final,
                                                       const DThr* __restrict__ thr, unsigned long long* feas,
                                                       int n_problems) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous level (programmatic dependent launch)
  if (ctl->overflow) return;
  // BFS-settled final nodes only when >= 10 % of the batch is loose (prepare_kernel)
  const bool fuse_batch = true;  // T->fuse is cleared by thr_kernel unless >= 10 % of the batch is loose
  const unsigned long long n_in = ctl->level_count[k];
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long base = static_cast<unsigned long long>(blockIdx.x) * blockDim.x; base < n_in;
       base += stride) {
    const unsigned long long i = base + threadIdx.x;
    const bool valid = i < n_in;
    expand_node<true>(tables, k, ctl, valid, valid ? in.d[i] : 0, valid ? in.t[i] : 0.0, valid ? in.num[i] : 0.0,
                valid ? in.den[i] : 0.0, valid ? in.last[i] : 0, valid ? in.code[i] : 0ull, out, fin, cap_out,
                cap_final, thr, feas, fuse_batch);
  }
}

// Every leaf of a sliced tree whose leading digits lie below prepare's
// first list (K <= 3, or a final depth < digits): one CTA evaluates the
// slice's assignments in code order with meets_slo's early exit, counts the
// feasible ones and merges the (objective, code) minimum -- the same op
// sequence as the sweep (child_state chain, then den > 0 ? num / den : 0).
__device__ __noinline__ void small_tree_slice(const DTables* __restrict__ T, int d, int K, int nc, DSlice sl,
                                              Key128* best, unsigned long long* feas) {
  __shared__ unsigned long long s_o[32], s_c[32], s_n[32];
  const unsigned long long total = ipow(static_cast<unsigned long long>(nc), K);
  unsigned long long ko = ~0ull, kc = ~0ull, cnt = 0;
  for (unsigned long long code = threadIdx.x; code < total; code += blockDim.x) {
    if (!in_slice(sl, code, K, nc)) continue;
    double t = 0.0, num = 0.0, den = 0.0;
    int last = -1;
    bool ok = true;
    unsigned long long div = total / static_cast<unsigned long long>(nc);
    for (int k = 0; k < K && ok; ++k) {
      const int f = static_cast<int>((code / div) % static_cast<unsigned long long>(nc));
      div /= static_cast<unsigned long long>(nc);
      double ct, cn, cd;
      ok = child_state(T, k, t, num, den, last, f, ct, cn, cd);
      t = ct;
      num = cn;
      den = cd;
      last = f;
    }
    if (!ok) continue;
    ++cnt;
    const double obj = den > 0.0 ? __ddiv_rn(num, den) : 0.0;  // dvfs.hpp:170
    const unsigned long long o = static_cast<unsigned long long>(__double_as_longlong(obj));
    if (key_less(o, code, ko, kc)) {
      ko = o;
      kc = code;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const unsigned long long oo = __shfl_xor_sync(0xffffffffu, ko, o), oc = __shfl_xor_sync(0xffffffffu, kc, o);
    if (key_less(oo, oc, ko, kc)) {
      ko = oo;
      kc = oc;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    s_o[threadIdx.x >> 5] = ko;
    s_c[threadIdx.x >> 5] = kc;
    s_n[threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      cnt += s_n[w];
      if (key_less(s_o[w], s_c[w], ko, kc)) {
        ko = s_o[w];
        kc = s_c[w];
      }
    }
    feas[d] = cnt;
    if (ko != ~0ull) {
      best[d].obj = ko;
      best[d].code = kc;
    }
  }
}

#ifndef BS_SEED_ROUNDS
#define BS_SEED_ROUNDS 3  // single-move improvement rounds of the argmin seed (1: C2 sweep 0.239 ms; 3: 0.219; 6: 0.221)
#endif
#ifndef BS_PREP_MINB
#define BS_PREP_MINB 8  // 64 registers: the 1024-decision batch in one wave (C2: 0.055 -> 0.040 ms)
#endif
constexpr int kSeedRounds = BS_SEED_ROUNDS;

// One CTA per decision: the tables, the argmin slot reset, and the first
// levels of the search.  The prefixes of depth D0 = min(2, FD) are evaluated
// here (nc^D0 per decision); at FD they go to the final list, otherwise the
// depth-2 ones are expanded once more (expand_node) into the depth-3 list
// (or the final list), so the BFS starts at depth 3.  The run's counters are
// zeroed by the host before this launch.
__global__ void __launch_bounds__(kPrepThreads, BS_PREP_MINB) prepare_kernel(DModels m, const DMpcCfg* cfgs, const DProblem* probs,
                                                               const DWaiting* W, const DRunning* R, DTables* tables,
                                                               DThr* thr, ExCtl* ctl, int n, const DFastPair* fg,
                                                               Key128* best,
                                                               unsigned long long* feas, Frontier L2, Frontier L3,
                                                               FinalList fin, unsigned long long cap_level,
                                                               unsigned long long cap_final, double sweep3_min,
                                                               DSlice sl, int* thr_list) {
  __shared__ int s_status;
  const int d = blockIdx.x;
  if (d >= n) return;
#ifdef BS_PREP_PHASES  // diagnostics build: globaltimer at phase ends, printed by thread 0 of every 64th CTA
  unsigned long long pph[10] = {0};
  int pphn = 0;
#define BS_PPH()                                                            \
  if (threadIdx.x == 0) {                                                   \
    unsigned long long t_;                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
    pph[pphn++] = t_;                                                       \
  }
#else
#define BS_PPH()
#endif
  BS_PPH();
  const DProblem pr = probs[d];
  const DMpcCfg& c = cfgs[pr.cfg];
  DTables* T = &tables[d];
  const DFastPair* fp = fg ? fg + pr.fgi : nullptr;
  build_tables(m, pr, c, W + pr.wait_off, R + pr.run_off, T, &s_status, fp ? fp->lat : nullptr,
               fp ? fp->pw : nullptr, fp && fp->share);
  if (threadIdx.x == 0) {
    int st = s_status;
    if (st == BS_OK) {
      unsigned any = 0;
      for (int k = 0; k < T->K; ++k) any |= T->bad_lat[k] | T->bad_pow[k];
      if (any) st = BS_MODEL_ERROR;
    }
    T->status = st;
    s_status = st;
    best[d].obj = ~0ull;
    best[d].code = ~0ull;
    feas[d] = 0ull;
  }
  __syncthreads();
  BS_PPH();
  const int K = T->K, nc = T->nc;
  if (s_status != BS_OK || K == 0) return;
  const int FD = K - sweep_levels(K, nc, sweep3_min);
  if (threadIdx.x == 0) {
    T->FD = FD;
    T->nc_magic = nc > 1 ? 0xffffffffu / static_cast<unsigned>(nc) + 1u : 0u;
    T->fuse = 0;
    T->thr_ok = 0;
    T->rex_ok = 0;
    T->nb_beta = INFINITY;
    T->nb_R = INFINITY;
  }
  // per-step thresholds, then the exact completion bounds (rexist)
  if (T->sorted_ok) step_thresholds(T);
  BS_PPH();
  if (K >= 3) leaf_exists_bounds(T);
  BS_PPH();
  // A slice whose leading digits lie below the first list this kernel
  // writes (trees of at most 3 levels, or shallow final depths): every leaf
  // of the slice evaluated here, in the sweep's op sequence.
  if (sl.digits > (FD < 2 ? FD : 2)) {
    small_tree_slice(T, d, K, nc, sl, best, feas);
    return;
  }
  // Seed the argmin with a good feasible assignment: the best uniform one
  // (every batch at one rung), then rounds of single-position moves (every
  // (k, f) replacement of the current assignment, best feasible taken).
  // Each is evaluated with the sweep's exact op sequence, so the seed is a
  // genuine (objective, code) key of the tree and the minimum is unchanged,
  // while every sweep thread filters against a tight threshold from its
  // first leaf.
  {
    __shared__ unsigned long long s_ko[kPrepThreads / 32], s_kc[kPrepThreads / 32];
    __shared__ unsigned char s_cur[kMaxK];
    // the slice's leading digits (seeds must be keys of the slice)
    const int sd = sl.digits < K ? sl.digits : K;
    auto lead_digit = [&](int k) {
      unsigned long long v = sl.lo;
      for (int i = k + 1; i < sl.digits; ++i) v /= static_cast<unsigned long long>(nc);
      return static_cast<int>(v % static_cast<unsigned long long>(nc));
    };
    auto eval = [&](int kk, int ff, unsigned long long& ko, unsigned long long& kc) {
      // assignment s_cur with position kk set to ff (kk < 0: the slice's
      // leading digits, then every position ff)
      double t = 0.0, num = 0.0, den = 0.0;
      int last = -1;
      unsigned long long code = 0;
      for (int k = 0; k < K; ++k) {
        const int f = kk < 0 ? (k < sd ? lead_digit(k) : ff) : (k == kk ? ff : s_cur[k]);
        double ct, cn, cd;
        if (!child_state(T, k, t, num, den, last, f, ct, cn, cd)) return;
        t = ct;
        num = cn;
        den = cd;
        last = f;
        code = code * static_cast<unsigned long long>(nc) + static_cast<unsigned long long>(f);
      }
      if (!in_slice(sl, code, K, nc)) return;
      const double obj = den > 0.0 ? __ddiv_rn(num, den) : 0.0;  // dvfs.hpp:170
      ko = static_cast<unsigned long long>(__double_as_longlong(obj));
      kc = code;
    };
    auto block_min = [&](unsigned long long& ko, unsigned long long& kc) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long oo = __shfl_xor_sync(0xffffffffu, ko, o), oc = __shfl_xor_sync(0xffffffffu, kc, o);
        if (key_less(oo, oc, ko, kc)) {
          ko = oo;
          kc = oc;
        }
      }
      if ((threadIdx.x & 31) == 0) {
        s_ko[threadIdx.x >> 5] = ko;
        s_kc[threadIdx.x >> 5] = kc;
      }
      __syncthreads();
      ko = s_ko[0];
      kc = s_kc[0];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
        if (key_less(s_ko[w], s_kc[w], ko, kc)) {
          ko = s_ko[w];
          kc = s_kc[w];
        }
      __syncthreads();
    };
    unsigned long long ko = ~0ull, kc = ~0ull;
    if (threadIdx.x < nc) eval(-1, threadIdx.x, ko, kc);
    block_min(ko, kc);
    for (int round = 0; round < kSeedRounds && ko != ~0ull; ++round) {
      if (threadIdx.x < K) {  // digits of the current best, batch 0 most significant
        unsigned long long c = kc;
        for (int k = K - 1; k > static_cast<int>(threadIdx.x); --k) c /= static_cast<unsigned long long>(nc);
        s_cur[threadIdx.x] = static_cast<unsigned char>(c % static_cast<unsigned long long>(nc));
      }
      __syncthreads();
      unsigned long long mo = ko, mc = kc;
      for (int e = threadIdx.x; e < K * nc; e += blockDim.x) {
        const int kk = e / nc, ff = e - kk * nc;
        if (ff == s_cur[kk]) continue;
        unsigned long long eo = ~0ull, ec = ~0ull;
        eval(kk, ff, eo, ec);
        if (key_less(eo, ec, mo, mc)) {
          mo = eo;
          mc = ec;
        }
      }
      block_min(mo, mc);
      if (!key_less(mo, mc, ko, kc)) break;  // a local minimum of single moves (uniform across the block)
      ko = mo;
      kc = mc;
    }
    if (threadIdx.x == 0 && ko != ~0ull) {  // after this thread's reset above (program order)
      best[d].obj = ko;
      best[d].code = kc;
    }
    BS_PPH();
    // the seed's node bound over the two bottom levels (node_dom_seed), one
    // warp: lane x takes candidate x of each level
    const double thr_s = __longlong_as_double(static_cast<long long>(ko));
    if (threadIdx.x < 32 && K >= 3 && T->sorted_ok && T->filter_ok && ko != ~0ull && thr_s >= kFilterMinBest &&
        thr_s < INFINITY) {
      const double beta = __dmul_rn(thr_s, 1.0 + 0x1p-47);
      double qs = 0.0, mag = 0.0;
      for (int k = K - 2; k < K; ++k) {
        const int x = threadIdx.x;
        double q = INFINITY, emax = 0.0, amax = 0.0;
        if (x < nc) {
          q = __dsub_rn(T->E[k][x], __dmul_rn(beta, T->A[k][x]));
          emax = T->E[k][x];
          amax = T->A[k][x];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // min / max are exact in any order
          const double q2 = __shfl_xor_sync(0xffffffffu, q, o), e2 = __shfl_xor_sync(0xffffffffu, emax, o),
                       a2 = __shfl_xor_sync(0xffffffffu, amax, o);
          q = q2 < q ? q2 : q;
          emax = e2 > emax ? e2 : emax;
          amax = a2 > amax ? a2 : amax;
        }
        qs = __dadd_rn(qs, q);
        mag = __dadd_rn(mag, __dadd_rn(emax, __dmul_rn(beta, amax)));
      }
      if (threadIdx.x == 0) {
        const double R = __dadd_rn(-qs, __dmul_rn(mag, 0x1p-44));
        T->nb_beta = beta;
        T->nb_R = R > 0.0 ? R : 0.0;
      }
    }
  }
  if (FD == 0) {
    if (threadIdx.x == 0) {
      const unsigned long long sl = atomicAdd(&ctl->final_count, 1ull);
      if (sl < cap_final) {
        fin.d[sl] = d;
        fin.code[sl] = 0;
      } else {
        atomicAdd(&ctl->overflow, 1ull);
      }
    }
    return;
  }
  const int D0 = FD < 2 ? FD : 2;
  const int width = D0 == 1 ? nc : nc * nc;
  BS_PPH();
  if (threadIdx.x == 0) T->n_ok3 = 0;
  __syncthreads();
  const bool to_final = D0 == FD;
  for (int base = 0; base < width; base += blockDim.x) {  // uniform trip count: block_append2 needs every thread
    const int e = base + threadIdx.x;
    bool ok = false;
    double t = 0.0, num = 0.0, den = 0.0;
    int last = -1;
    if (e < width) {
      const int f0 = D0 == 1 ? e : e / nc, f1 = D0 == 1 ? -1 : e - f0 * nc;
      ok = child_state(T, 0, 0.0, 0.0, 0.0, -1, f0, t, num, den);
      last = f0;
      if (ok && D0 == 2) {
        double t1, n1, d1;
        ok = child_state(T, 1, t, num, den, f0, f1, t1, n1, d1);
        t = t1;
        num = n1;
        den = d1;
        last = f1;
      }
      if (ok && sl.digits) ok = in_slice(sl, static_cast<unsigned long long>(e), D0, nc);  // sl.digits <= D0 here
      if (ok && T->rex_ok && D0 <= K - 2) ok = !(t > T->rexist[D0][last]);  // a feasible leaf below (exact)
      // a final node none of whose children passes has no feasible leaf (as in bfs_node_kernel)
      if (ok && to_final && T->sorted_ok && FD < K)
        ok = (T->rex_ok && FD == K - 2) ? !(t > T->rexist[FD][last])
                                         : feasible_prefix(T, FD, nc, t) > 0 || diag_passes(T, FD, t, last);
    }
    if (FD > 2) {  // one more level here: the depth-2 nodes never reach global memory (FD is uniform per CTA)
      const unsigned m3 = expand_node<false>(tables, 2, ctl, ok, d, t, num, den, last,
                                             static_cast<unsigned long long>(e), L3, fin, cap_level, cap_final, thr,
                                             feas);
      if (m3) atomicAdd(&T->n_ok3, static_cast<int>(m3));  // feasible depth-3 prefixes (looseness, thr_kernel)
      continue;
    }
    unsigned long long sf, so;
    block_append2(&ctl->final_count, ok && to_final, &ctl->level_count[D0], ok && !to_final, &sf, &so);
    if (ok && to_final) {
      if (sf < cap_final) {
        fin.d[sf] = d;
        fin.code[sf] = static_cast<unsigned long long>(e);
      } else {
        atomicAdd(&ctl->overflow, 1ull);
      }
    } else if (ok) {
      if (so < cap_level) {
        L2.d[so] = d;
        L2.code[so] = static_cast<unsigned long long>(e);
        L2.t[so] = t;
        L2.num[so] = num;
        L2.den[so] = den;
        L2.last[so] = last;
      } else {
        atomicAdd(&ctl->overflow, 1ull);
      }
    }
  }
  // Loose trees (more than 85 % of the depth-3 prefixes with a feasible
  // leaf: 96 % at C2 TTFT 1200 ms; the 600 ms corpus' decisions are at most
  // 68 % feasible at depth 3) are candidates for the BFS to settle the final
  // nodes the seed's node bound dominates (thr_kernel decides for the whole
  // batch).  Leaf-count thresholds of the two bottom levels
  // (build_thresholds) are listed for the decisions that use them:
  //  * three swept levels: the sweep counts a dominated child's leaves with
  //    three binary searches;
  //  * loose decisions with two swept levels: the BFS settles their dominated
  //    final nodes when at least 10 % of the batch is loose (measured at C2
  //    TTFT 1200 ms: 92 % of the final nodes; step 7.9 -> 1.9 ms).
  BS_PPH();
  __syncthreads();
  const bool loose = FD >= 4 && FD == K - 2 && 20ll * T->n_ok3 > 17ll * nc * nc * nc;
  if (threadIdx.x == 0 && K >= 3 && FD >= 1 && T->sorted_ok && T->filter_ok && sl.digits <= (FD < 2 ? FD : 2) &&
      (K - FD == 3 || loose)) {  // listed for thr_kernel
    if (loose) {
      T->fuse = 1;
      atomicAdd(&ctl->n_loose, 1ull);
    }
    thr_list[atomicAdd(&ctl->n_thr, 1ull)] = d;
  }
#ifdef BS_PREP_PHASES
  BS_PPH();
  if (threadIdx.x == 0 && (d & 63) == 0) {
    printf("prep phases ns:");
    for (int i = 1; i < pphn; ++i) printf(" %llu", pph[i] - pph[i - 1]);
    printf("\n");
  }
#endif
}

// The thresholds of the listed decisions (prepare_kernel), a few CTAs per SM
// taking list entries in turn: a batch that lists none (the 600 ms C2
// corpus) costs one short launch; loose two-level decisions are built only
// when at least 10 % of the batch is loose (measured at C2 TTFT 1200 ms: the
// BFS then settles 92 % of the final nodes, step 7.9 -> 1.9 ms), since one
// build is a ~10 us chain of dependent steps a batch with only a few loose
// decisions would pay without gaining it back.
__global__ void __launch_bounds__(kPrepThreads) thr_kernel(DTables* tables, DThr* thr, const ExCtl* ctl,
                                                           const int* thr_list, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // prepare_kernel's tables and list
  const unsigned long long n_thr = ctl->n_thr;
  const bool fuse_batch = 10ull * ctl->n_loose >= static_cast<unsigned long long>(n);
  for (unsigned long long i = blockIdx.x; i < n_thr; i += gridDim.x) {
    DTables* T = &tables[thr_list[i]];
    const bool use = T->K - T->FD == 3 || fuse_batch;  // uniform per CTA
    if (!use) {
      if (threadIdx.x == 0) T->fuse = 0;
      continue;
    }
    build_thresholds(T, &thr[thr_list[i]]);
    if (threadIdx.x == 0) T->thr_ok = 1;
  }
}

// Resident CTAs per SM the sweep is register-budgeted for: 3 (80 registers)
// for two swept levels, 4 (64) for three, where more warps hide the longer
// per-thread walks (measured: C2 0.42 vs 0.45 ms; C5 3,838 vs 4,298
// decisions/s).
#ifndef BS_SWEEP2_MINB
#define BS_SWEEP2_MINB 4  // 64 registers (spills to L1) and 4 CTAs/SM: C2 sweep 0.152 -> 0.140 ms, loose 0.61 -> 0.55 ms
#endif
// resident CTAs per SM of the two-level (kSweep2) and three-level (kSweep3) sweep instances
constexpr int kSweepMinB2 = BS_SWEEP2_MINB, kSweepMinB3 = 4;
constexpr int kSweep2 = 2, kSweep3 = 3;

// Per-thread accumulator of the sweep.
struct LeafAcc {
  double best;               // local minimum objective (+inf: none)
  unsigned long long code;   // its code
  double thr_scaled;         // fl(min(local, global hint) * C), +inf disables the filter
  unsigned long long count;  // feasible leaves
#ifdef BS_SWEEP_STATS
  unsigned long long st_rows, st_leaves, st_div, st_children, st_thr, st_slow;
#endif
  // leaf-row skip ("row bound"): a row of leaves under a parent
  // with (num, den) is provably worse than thr when
  //   fl(num - fl(beta * den)) > s_last + num * 2^-40,
  // beta = fl(thr * (1 + 2^-47)), s_last >= amax * (beta - pmin (1 - u))^+.
  double beta;
  double s_last;
  double s_node;  // >= the two bottom levels' slack: a node at depth K-2 is dominated (node_dominated)
};

// (the last level's amax / pmin_lo are re-read from the tables: fewer live registers)
__device__ __forceinline__ void set_threshold(LeafAcc& a, double hint, const DTables* __restrict__ T) {
  // hint is NaN while the slot still holds its (~0, ~0) reset value
  const double thr = (a.best < hint || hint != hint) ? a.best : hint;
  a.thr_scaled = thr >= kFilterMinBest ? __dmul_rn(thr, kFilterScale) : (thr == 0.0 ? 0.0 : INFINITY);
  if (thr >= kFilterMinBest && thr < INFINITY) {
    a.beta = __dmul_rn(thr, 1.0 + 0x1p-47);
    const int kl = T->K - 1;
    const double gap = __dsub_rn(a.beta, T->pmin_lo[kl]);
    a.s_last = gap > 0.0 ? __dmul_rn(__dmul_rn(gap, T->amax[kl]), 1.0 + 0x1p-40) : 0.0;
    const double gap2 = kl >= 1 ? __dsub_rn(a.beta, T->pmin_lo[kl - 1]) : 0.0;
    const double s2 = gap2 > 0.0 ? __dmul_rn(__dmul_rn(gap2, T->amax[kl - 1]), 1.0 + 0x1p-40) : 0.0;
    a.s_node = __dmul_rn(__dadd_rn(s2, a.s_last), 1.0 + 0x1p-40);
  } else {
    a.beta = INFINITY;
    a.s_last = INFINITY;
    a.s_node = INFINITY;
  }
}

// True when every leaf under a parent with (num, den) is provably worse than
// the current threshold (requires the filter preconditions: A >= 0, finite,
// den >= 2^-900).
__device__ __forceinline__ bool row_dominated(const LeafAcc& a, double num, double den) {
  return __dsub_rn(num, __dmul_rn(a.beta, den)) > __dadd_rn(a.s_last, __dmul_rn(num, 0x1p-40));
}

// True when every leaf below a node at depth K-2 with (num, den) is provably
// worse than the current threshold ("node bound"): with
// thr' = thr (1 + 2^-50) <= beta, a leaf's rounded objective exceeds thr when
// num + E_g + E_f > thr' (den + A_g + A_f), and E_x - thr' A_x >= -amax (thr' -
// pmin (1 - u))^+ per level (A >= 0, E = fl(A P)), so num - thr' den > s_K-2 +
// s_K-1 suffices; the test below is that inequality with its rounding margin
// (num 2^-40, s_node inflated by 2^-40).  Preconditions as the leaf filter:
// filter_ok tables, den >= 2^-900, thr >= 2^-100.
__device__ __forceinline__ bool node_dominated(const LeafAcc& a, double num, double den) {
  return den >= kFilterMinDen && __dsub_rn(num, __dmul_rn(a.beta, den)) > __dadd_rn(a.s_node, __dmul_rn(num, 0x1p-40));
}

// Last level k = K-1 for one parent state: every f in 0..nc-1, in order.
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
    if (filt && nl > __dmul_rn(a.thr_scaled, dl)) continue;  // provably worse than a known feasible key
    const double obj = dl > 0.0 ? __ddiv_rn(nl, dl) : 0.0;  // dvfs.hpp:170
    const unsigned long long code = code_base + static_cast<unsigned long long>(f);
    if (obj < a.best || (obj == a.best && code < a.code)) {
      a.best = obj;
      a.code = code;
      set_threshold(a, hint, T);
    }
  }
}

// Calls fn(f, ct, cn, cd) for every child of (t, num, den, last) at level k
// that passes the check: the sorted prefix (minus f == last, whose real step
// is the non-switching B0) plus the non-switching child if it passes.
// Returns the number of passing children.
template <typename Fn>
__device__ __forceinline__ int for_feasible_children(const DTables* __restrict__ T, int k, int nc, double t,
                                                     double num, double den, int last, Fn&& fn) {
  const int c = feasible_prefix(T, k, nc, t);
  const unsigned char* __restrict__ ord = T->ord[k];
  const double* __restrict__ sb = T->sb[k];
  const double* __restrict__ E = T->E[k];
  const double* __restrict__ A = T->A[k];
  int passed = 0;
  for (int j = 0; j < c; ++j) {
    const int f = ord[j];
    if (k > 0 && f == last) continue;
    const double ct = k == 0 ? sb[j] : __dadd_rn(t, sb[j]);
    fn(f, ct, __dadd_rn(num, E[f]), __dadd_rn(den, A[f]));
    ++passed;
  }
  if (k > 0 && diag_passes(T, k, t, last)) {
    fn(last, __dadd_rn(t, T->B0[k][last]), __dadd_rn(num, E[last]), __dadd_rn(den, A[last]));
    ++passed;
  }
  return passed;
}

// Leaves (level k >= 1) under a parent with clock t whose sorted-prefix
// count c = feasible_prefix(T, k, nc, t) is known: count them in closed form,
// skip a dominated row, else visit only the passing leaves.  rank_last /
// b0_last: rank[k][last] and B0[k][last] (from the parent's record).
// The row's (num, den) = parent's + (e_row, a_row) are formed only for rows
// with a feasible leaf (most rows have none: the last batch's deadline binds).
__device__ __forceinline__ void leaves_counted(const DTables* __restrict__ T, int k, int nc, double t, double num_p,
                                               double den_p, double e_row, double a_row, int last, int rank_last,
                                               double th0_last, int c, unsigned long long code_base, double hint,
                                               LeafAcc& a) {
  const bool diag = !(t > th0_last);  // diag_passes
  const int passed = c - (rank_last < c ? 1 : 0) + (diag ? 1 : 0);
  if (passed == 0) return;
  a.count += static_cast<unsigned long long>(passed);
  const double num = __dadd_rn(num_p, e_row), den = __dadd_rn(den_p, a_row);
  const bool filt = T->filter_ok && den >= kFilterMinDen;
  if (filt && row_dominated(a, num, den)) return;
#ifdef BS_SWEEP_STATS
  a.st_rows += 1;
#endif
  const double* __restrict__ E = T->E[k];
  const double* __restrict__ A = T->A[k];
  auto leaf = [&](int f) {
    const double nl = __dadd_rn(num, E[f]), dl = __dadd_rn(den, A[f]);
#ifdef BS_SWEEP_STATS
    a.st_leaves += 1;
#endif
    if (filt && nl > __dmul_rn(a.thr_scaled, dl)) return;  // provably worse than a known feasible key
#ifdef BS_SWEEP_STATS
    a.st_div += 1;
#endif
    const double obj = dl > 0.0 ? __ddiv_rn(nl, dl) : 0.0;  // dvfs.hpp:170
    const unsigned long long code = code_base + static_cast<unsigned long long>(f);
    if (obj < a.best || (obj == a.best && code < a.code)) {
      a.best = obj;
      a.code = code;
      set_threshold(a, hint, T);
    }
  };
  if (c == nc) {  // every switched leaf passes: natural order, no index loads
#pragma unroll 4
    for (int f = 0; f < nc; ++f)
      if (f != last || diag) leaf(f);
    return;
  }
  const unsigned char* __restrict__ ord = T->ord[k];
  for (int j = 0; j < c; ++j) {
    const int f = ord[j];
    if (f != last) leaf(f);
  }
  if (diag) leaf(last);
}

// Two bottom levels below a node at depth K-2, sorted path.  The switched
// children are visited in step order, so their clocks never decrease and the
// leaf level's sorted-prefix count never increases: one binary search for
// the first child, then a downward walk.
__device__ __forceinline__ void two_sorted(const DTables* __restrict__ T, int k, int nc, double t, double num,
                                           double den, int last, unsigned long long code_base, double hint,
                                           LeafAcc& a) {
  const int c = feasible_prefix(T, k, nc, t);
  const SRec* __restrict__ sr = T->srec[k];
  const unsigned short* __restrict__ si = T->sinfo[k];
  const int kl = k + 1;
  const double* __restrict__ thl = T->thsw[kl];
  int cl = -1;
  for (int j = 0; j < c; ++j) {
    const unsigned info = si[j];
    const int g = static_cast<int>(info & 0xffu);
    if (k > 0 && g == last) continue;
    const SRec r = sr[j];
    const double t2 = k == 0 ? r.sb : __dadd_rn(t, r.sb);
    if (cl < 0) {
      cl = feasible_prefix(T, kl, nc, t2);
    } else {
      while (cl > 0 && t2 > thl[cl - 1]) --cl;
    }
#ifdef BS_SWEEP_STATS
    a.st_children += 1;
#endif
    leaves_counted(T, kl, nc, t2, num, den, r.E, r.A, g, static_cast<int>(info >> 8), r.th0n, cl,
                   (code_base + static_cast<unsigned long long>(g)) * nc, hint, a);
  }
  if (k > 0 && diag_passes(T, k, t, last)) {
    const double t2 = __dadd_rn(t, T->B0[k][last]);
    leaves_counted(T, kl, nc, t2, num, den, T->E[k][last], T->A[k][last], last, T->rank[kl][last], T->th0[kl][last],
                   feasible_prefix(T, kl, nc, t2), (code_base + static_cast<unsigned long long>(last)) * nc, hint, a);
  }
}

// Two bottom levels (K-2, K-1) below a node at depth K-2.
__device__ __forceinline__ void sweep_two(const DTables* __restrict__ T, int k, int nc, double t, double num,
                                          double den, int last, unsigned long long code_base, double hint,
                                          LeafAcc& a) {
  for (int g = 0; g < nc; ++g) {
    double t2, n2, d2;
    if (!child_state(T, k, t, num, den, last, g, t2, n2, d2)) continue;
    const bool filt = T->filter_ok && d2 >= kFilterMinDen;
    sweep_last(T, k + 1, nc, t2, n2, d2, g, (code_base + static_cast<unsigned long long>(g)) * nc, filt, hint, a);
  }
}

// State after the first P levels of code (digits MSD first), unchecked (the
// BFS only emits feasible prefixes).
__device__ __forceinline__ void walk(const DTables* __restrict__ T, int nc, int P, unsigned long long code,
                                     double& t, double& num, double& den, int& last) {
  t = 0.0;
  num = 0.0;
  den = 0.0;
  last = -1;
  if (nc > 1 && P <= 12 && code < (1ull << 27)) {
    // digits least significant first by a multiply-high (q = umulhi(c,
    // ceil(2^32 / nc)) is exact for c < 2^32 / nc), packed 5 bits each
    const unsigned M = T->nc_magic;
    unsigned c = static_cast<unsigned>(code);
    unsigned long long packed = 0;
    for (int k = P - 1; k >= 0; --k) {
      const unsigned q = __umulhi(c, M);
      packed |= static_cast<unsigned long long>(c - q * static_cast<unsigned>(nc)) << (5 * k);
      c = q;
    }
    for (int k = 0; k < P; ++k) {
      const int f = static_cast<int>((packed >> (5 * k)) & 31u);
      double ct, cn, cd;
      child_state(T, k, t, num, den, last, f, ct, cn, cd);
      t = ct;
      num = cn;
      den = cd;
      last = f;
    }
    return;
  }
  unsigned long long div = ipow(static_cast<unsigned long long>(nc), P > 0 ? P - 1 : 0);
  for (int k = 0; k < P; ++k) {
    int f;
    if (code < (1ull << 32)) {
      const unsigned q = static_cast<unsigned>(code) / static_cast<unsigned>(div);
      f = static_cast<int>(q);
    } else {
      f = static_cast<int>(code / div);
    }
    code -= static_cast<unsigned long long>(f) * div;
    div /= static_cast<unsigned long long>(nc);
    double ct, cn, cd;
    child_state(T, k, t, num, den, last, f, ct, cn, cd);
    t = ct;
    num = cn;
    den = cd;
    last = f;
  }
}

__device__ __forceinline__ void flush_acc(int d, LeafAcc& a, Key128* best, unsigned long long* feas) {
  // warp-level merge when the whole warp holds one problem
  const unsigned active = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(active) - 1;
  const int d0 = __shfl_sync(active, d, leader);
  unsigned long long bo = a.best < INFINITY ? static_cast<unsigned long long>(__double_as_longlong(a.best)) : ~0ull;
  unsigned long long bc = a.code;
  unsigned long long c = a.count;
  if (active == 0xffffffffu && __all_sync(active, d == d0)) {
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
  } else {
    if (c) atomicAdd(&feas[d], c);
    if (bo != ~0ull) atomic_min_key(&best[d], bo, bc);
  }
}

#ifndef BS_SWEEP2_CLAIM
#define BS_SWEEP2_CLAIM 0  // 1: the two-level sweep claims runs too (A/B experiments)
#endif
#ifndef BS_SWEEP_CLAIM_N
#define BS_SWEEP_CLAIM_N 128
#endif
constexpr unsigned long long kSweepClaim = BS_SWEEP_CLAIM_N;  // final-list entries per warp claim (three-level sweep)

// One thread per final node: the I bottom levels of its subtree.  Two swept
// levels: grid stride (a block's 8 warps take 256 consecutive entries, one
// decision's tables shared in L1).  Three (heavy-tailed node costs): each
// warp claims runs of kSweepClaim consecutive entries from an atomic counter
// and takes 32 per step (C5 92K -> 103K decisions/s).  Measured and not
// kept: the swept rows staged per warp in shared memory (loose C2 sweep
// 0.55 -> 0.50 ms, but the headline 0.141 -> 0.150 ms: its nodes are too
// short to amortise the copy, and the second code path costs registers).
template <int MINB, int LEVELS>
__global__ void __launch_bounds__(256, MINB) sweep_kernel(const DTables* __restrict__ tables,
                                                          const DThr* __restrict__ thr, const ExCtl* ctl,
                                                          FinalList fin, Key128* best, unsigned long long* feas,
                                                          unsigned long long cap_final) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the BFS lists (programmatic dependent launch)
  if (ctl->overflow) return;  // the run is repeated with larger lists (one_shot): skip the sweep
  const unsigned long long n_fin = ctl->final_count < cap_final ? ctl->final_count : cap_final;
  constexpr bool kClaim = LEVELS == kSweep3 || BS_SWEEP2_CLAIM;
  const int lane = threadIdx.x & 31;
  unsigned long long* next = &const_cast<ExCtl*>(ctl)->sweep_next;
  unsigned long long claim = 0;  // three levels: the warp's current run
  if (kClaim) {
    if (lane == 0) claim = atomicAdd(next, kSweepClaim);
    claim = __shfl_sync(0xffffffffu, claim, 0);
  }
  const unsigned long long stride = kClaim ? 32ull : static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  unsigned long long j = kClaim ? claim + lane : static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  int d_next = 0;
  unsigned long long code_next = 0;
  if (j < n_fin) {
    d_next = fin.d[j];
    code_next = fin.code[j];
  }
  // two levels: per-lane loop; three: warp-uniform steps (lanes past the end idle)
  bool run = kClaim ? (j - lane < n_fin) : (j < n_fin);
  while (run) {
    const bool valid = j < n_fin;
    const int d = d_next;
    const unsigned long long code = code_next;
    unsigned long long jn = j + stride;
    if (kClaim && jn - lane >= claim + kSweepClaim) {  // the run is done (warp-uniform): claim the next
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(next, kSweepClaim);
      claim = __shfl_sync(0xffffffffu, c, 0);
      jn = claim + lane;
    }
    if (jn < n_fin) {  // the next node's entry, in flight during this one
      d_next = fin.d[jn];
      code_next = fin.code[jn];
    }
    if (valid) {
      const double hint = __longlong_as_double(static_cast<long long>(
          *reinterpret_cast<volatile unsigned long long*>(&best[d].obj)));
      const DTables* __restrict__ T = &tables[d];
      const int K = T->K, nc = T->nc;
      const int FD = T->FD;
      const int I = K - FD;
      double t, num, den;
      int last;
      walk(T, nc, FD, code, t, num, den, last);
      LeafAcc a;
      a.best = INFINITY;
      a.code = ~0ull;
      a.count = 0;
#ifdef BS_SWEEP_STATS
      a.st_rows = a.st_leaves = a.st_div = a.st_children = a.st_thr = a.st_slow = 0;
#endif
      set_threshold(a, hint, T);
      const unsigned long long cb = code * static_cast<unsigned long long>(nc);
      if (I == 1) {  // K == 1
        sweep_last(T, FD, nc, t, num, den, last, cb, false, hint, a);
      } else if (T->sorted_ok) {
        // a node at depth K-2 whose leaves are all provably worse than the
        // threshold only needs its feasible-leaf count: three binary searches
        const bool use_thr = T->thr_ok != 0;
        const DThr* __restrict__ H = thr + d;
        if (I == 2) {
#ifdef BS_SWEEP_STATS
          a.st_slow += 1;
#endif
          two_sorted(T, FD, nc, t, num, den, last, cb, hint, a);
        } else if (LEVELS == kSweep3) {  // three swept levels only occur in batches launched with this instance
          int cs_hint = nc * nc;  // switched children come in clock order (the diag child last)
          for_feasible_children(T, FD, nc, t, num, den, last, [&](int e, double t3, double n3, double d3) {
            if (T->rex_ok && t3 > T->rexist[K - 2][e]) return;  // no feasible leaf below this child
            if (use_thr && (node_dom_seed(T, n3, d3) || node_dominated(a, n3, d3))) {
              a.count += static_cast<unsigned long long>(
                  e == last ? thr_leaf_count(H, nc, t3, e) : thr_leaf_count_walk(H, nc, t3, e, &cs_hint));
#ifdef BS_SWEEP_STATS
              a.st_thr += 1;
#endif
            } else {
#ifdef BS_SWEEP_STATS
              a.st_slow += 1;
#endif
              two_sorted(T, FD + 1, nc, t3, n3, d3, e, (cb + static_cast<unsigned long long>(e)) * nc, hint, a);
            }
          });
        }
      } else {
        // I == 3 adds one more level above the two swept ones
        const int ne = I == 3 ? nc : 1;
        for (int e = 0; e < ne; ++e) {
          double t3 = t, n3 = num, d3 = den;
          int l3 = last, k2 = FD;
          unsigned long long cb2 = cb;
          if (I == 3) {
            if (!child_state(T, FD, t, num, den, last, e, t3, n3, d3)) continue;
            l3 = e;
            k2 = FD + 1;
            cb2 = (cb + static_cast<unsigned long long>(e)) * nc;
          }
          sweep_two(T, k2, nc, t3, n3, d3, l3, cb2, hint, a);
        }
      }
      flush_acc(d, a, best, feas);
#ifdef BS_SWEEP_STATS
      ExCtl* wctl = const_cast<ExCtl*>(ctl);
      atomicAdd(&wctl->st_nodes, 1ull);
      atomicAdd(&wctl->st_children, a.st_children);
      atomicAdd(&wctl->st_rows_eval, a.st_rows);
      atomicAdd(&wctl->st_leaves_eval, a.st_leaves);
      atomicAdd(&wctl->st_div, a.st_div);
      atomicAdd(&wctl->st_thr_nodes, a.st_thr);
      if (a.count == 0) atomicAdd(&wctl->st_empty_nodes, 1ull);
      atomicAdd(&wctl->st_slow_nodes, a.st_slow);
#endif
    }
    if (kClaim) __syncwarp();
    j = jn;
    run = kClaim ? (j - lane < n_fin) : (j < n_fin);
  }
}

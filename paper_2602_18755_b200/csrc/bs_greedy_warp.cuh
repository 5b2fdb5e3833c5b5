// bs_greedy_warp.cuh — greedy_freq_select (dvfs.hpp:185-259) for one
// decision by ONE warp (included after bs_mpc_core.cuh inside a translation
// unit's anonymous namespace).
//
// Same decision, level statistics, eval counts and ModelError order as the
// reference, organised for many concurrent decisions per SM (bs_mpc_greedy
// runs one decision per warp, the cluster replay one prefill instance per
// warp):
//   * compact per-warp tables in shared memory, row stride = |cand|;
//   * positions of a level by a ballot over batches;
//   * a level's mutations by exact prefix-sharing walks: threads own
//     prefixes of all but the last R <= 3 mutated positions (digit 0 = the
//     earliest position, as in the reference's code) and extend them by
//     nested loops in registers, keeping (t, num, den) per depth.  A step
//     that violates meets_slo ends every mutation below it (meets_slo returns
//     false at the first violation, dvfs.hpp:117), so the subtree is skipped.
//     Each surviving mutation's clock and sums are built by the same
//     additions in the same k order as eval_assignment, so objectives are
//     bit-identical.  Used only when no (k, f) prediction of the decision is
//     bad; otherwise every mutation is evaluated in full (exact ModelError
//     order).
#pragma once

static_assert(kMaxK <= 19, "a level's 3^K' mutations must index in 32 bits");

struct WTables {
  int K, nc, status, anybad;
  double ttft;
  unsigned bad_lat[kMaxK];
  unsigned bad_pow[kMaxK];
  long long n_req[kMaxK];
  long long sum_len[kMaxK];
  double wf[kMaxK];
  double minarr[kMaxK];
  int ncomp[kMaxK];
  // views into the warp's table scratch: [k * nc + f]
  double *A, *P, *E, *B0, *B1;
  double* T1;
};

struct WGreedyShared {
  WTables T;
  FastBrk blat[kMaxK], bpow[kMaxK];  // per-batch brackets shared by every candidate's reduced grid
  int np;
  int accepted;
  double obj;
  unsigned char cur[kMaxK];
  int pos[kMaxK];
};

__host__ __device__ inline size_t wtable_doubles(int horizon, int nc) { return 5ull * horizon * nc + nc; }

__device__ inline void wtables_bind(WTables& T, double* scratch, int horizon, int nc) {
  const size_t kn = static_cast<size_t>(horizon) * nc;
  T.A = scratch;
  T.P = T.A + kn;
  T.E = T.P + kn;
  T.B0 = T.E + kn;
  T.B1 = T.B0 + kn;
  T.T1 = T.B1 + kn;
}

// eval_assignment on the compact tables (see bs_mpc_core.cuh).
__device__ inline int weval(const WTables& T, const DProblem& pr, const DMpcCfg& c, const unsigned char* idx,
                            double* obj, int* err) {
  *err = 0;
  const int K = T.K, nc = T.nc;
  double t = pr.now;
  for (int k = 0; k < K; ++k) {
    const int f = idx[k];
    if ((T.bad_lat[k] >> f) & 1u) {
      *err = 1;
      return 0;
    }
    const bool sw = k == 0 ? (c.cand[f] != pr.cur_freq) : (f != idx[k - 1]);
    t = __dadd_rn(t, sw ? T.B1[k * nc + f] : T.B0[k * nc + f]);
    if (__dsub_rn(t, T.minarr[k]) > T.ttft) return 0;
  }
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
    num = __dadd_rn(num, T.E[k * nc + f]);
    den = __dadd_rn(den, T.A[k * nc + f]);
  }
  *obj = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
  return 1;
}

// One meets_slo step plus the objective sums (no bad predictions).
__device__ __forceinline__ bool wstep(const WTables& T, const DProblem& pr, const DMpcCfg& c, int k, int f,
                                      double& t, double& num, double& den, int& last) {
  const int nc = T.nc;
  const bool sw = k == 0 ? (c.cand[f] != pr.cur_freq) : (f != last);
  t = __dadd_rn(t, sw ? T.B1[k * nc + f] : T.B0[k * nc + f]);
  if (__dsub_rn(t, T.minarr[k]) > T.ttft) return false;
  num = __dadd_rn(num, T.E[k * nc + f]);
  den = __dadd_rn(den, T.A[k * nc + f]);
  last = f;
  return true;
}


// Division-free leaf filter (exactness argument 5; the level's
// tables must have every A >= 0 and finite and E finite): a mutation whose
// objective provably exceeds min(incumbent, this thread's best) is only
// counted.  One above the incumbent can never be accepted (dvfs.hpp:242-249)
// and one above the thread's best never wins its reduction; ties are never
// skipped, so the lexicographic rule holds.
constexpr double kGFilterScale = 1.0 + 0x1p-50;
constexpr double kGFilterMinBest = 0x1p-100;
constexpr double kGFilterMinDen = 0x1p-900;

__device__ __forceinline__ double gfilter_scaled(double thr) {
  return thr >= kGFilterMinBest ? __dmul_rn(thr, kGFilterScale) : (thr == 0.0 ? 0.0 : INFINITY);
}

struct GLeafAcc {
  unsigned long long bo, bc, feas;
  double thr_s;  // scaled filter threshold (INFINITY: no filter)
  double incumbent;
  bool filt;
};

__device__ __forceinline__ void gleaf(GLeafAcc& g, double n, double d, unsigned long long code,
                                      unsigned long long lex) {
  if (code == 0) return;  // the unmutated assignment is not a mutation
  ++g.feas;
  if (g.filt && d >= kGFilterMinDen && n > __dmul_rn(g.thr_s, d)) return;  // objective > threshold
  const double obj = d > 0.0 ? __ddiv_rn(n, d) : 0.0;
  const unsigned long long ob = static_cast<unsigned long long>(__double_as_longlong(obj));
  if (key_less(ob, lex, g.bo, g.bc)) {
    g.bo = ob;
    g.bc = lex;
    g.thr_s = gfilter_scaled(obj < g.incumbent ? obj : g.incumbent);
  }
}

// All mutations of one level whose first J digits are `prefix` (digit i <->
// position pos[i]; digit -> candidate: 0 target, 1 r1, 2 r2), the remaining
// R = np - J <= 3 digits by nested loops in registers (no per-depth stack in
// local memory): the prefix is walked once, each nested digit extends its
// parent's (t, num, den), and a step that violates meets_slo ends every
// mutation below it (meets_slo returns false at the first violation,
// dvfs.hpp:117).  Each surviving mutation's clock and sums are built by the
// same additions in the same k order as eval_assignment.  pwJ = base^J.
// pwJ = base^J.
__device__ void wlevel_tail(const WTables& T, const DProblem& pr, const DMpcCfg& c, const unsigned char* cur,
                            const int* pos, int np, int base, int target, int r1, int r2, int J,
                            unsigned long long pwJ, unsigned prefix, GLeafAcc& g) {
  const int K = T.K;
  auto cand_of = [&](int d) { return d == 0 ? target : (d == 1 ? r1 : r2); };
  double t = pr.now, num = 0.0, den = 0.0;
  int last = -1;
  unsigned rem = prefix;
  unsigned long long lexp = 0;
  int pi = 0;
  const int stop0 = J < np ? pos[J] : K;
  for (int k = 0; k < stop0; ++k) {
    int f = cur[k];
    if (pi < J && pos[pi] == k) {
      const unsigned q = base == 3 ? rem / 3u : rem >> 1;
      const int d = static_cast<int>(rem - q * static_cast<unsigned>(base));
      rem = q;
      f = cand_of(d);
      lexp = lexp * base + static_cast<unsigned long long>(base - 1 - d);
      ++pi;
    }
    if (!wstep(T, pr, c, k, f, t, num, den, last)) return;
  }
  if (J == np) {
    gleaf(g, num, den, prefix, lexp);
    return;
  }
  const int e0 = J + 1 < np ? pos[J + 1] : K;
  for (int d0 = 0; d0 < base; ++d0) {
    double t1 = t, n1 = num, dn1 = den;
    int l1 = last;
    bool ok = wstep(T, pr, c, pos[J], cand_of(d0), t1, n1, dn1, l1);
    for (int k = pos[J] + 1; ok && k < e0; ++k) ok = wstep(T, pr, c, k, cur[k], t1, n1, dn1, l1);
    if (!ok) continue;
    const unsigned long long code1 = prefix + static_cast<unsigned long long>(d0) * pwJ;
    const unsigned long long lex1 = lexp * base + static_cast<unsigned long long>(base - 1 - d0);
    if (J + 1 == np) {
      gleaf(g, n1, dn1, code1, lex1);
      continue;
    }
    const int e1 = J + 2 < np ? pos[J + 2] : K;
    for (int d1 = 0; d1 < base; ++d1) {  // digit J + 1
      double t2 = t1, n2 = n1, dn2 = dn1;
      int l2 = l1;
      bool ok2 = wstep(T, pr, c, pos[J + 1], cand_of(d1), t2, n2, dn2, l2);
      for (int k = pos[J + 1] + 1; ok2 && k < e1; ++k) ok2 = wstep(T, pr, c, k, cur[k], t2, n2, dn2, l2);
      if (!ok2) continue;
      const unsigned long long code2 = code1 + static_cast<unsigned long long>(d1) * pwJ * base;
      const unsigned long long lex2 = lex1 * base + static_cast<unsigned long long>(base - 1 - d1);
      if (J + 2 == np) {
        gleaf(g, n2, dn2, code2, lex2);
        continue;
      }
      for (int d2 = 0; d2 < base; ++d2) {  // digit J + 2, the last (R == 3)
        double t3 = t2, n3 = n2, dn3 = dn2;
        int l3 = l2;
        bool ok3 = wstep(T, pr, c, pos[J + 2], cand_of(d2), t3, n3, dn3, l3);
        for (int k = pos[J + 2] + 1; ok3 && k < K; ++k) ok3 = wstep(T, pr, c, k, cur[k], t3, n3, dn3, l3);
        if (!ok3) continue;
        gleaf(g, n3, dn3, code2 + static_cast<unsigned long long>(d2) * pwJ * base * base,
              lex2 * base + static_cast<unsigned long long>(base - 1 - d2));
      }
    }
  }
}

// greedy_freq_select for one decision by NW cooperating warps: the calling
// warp (NW == 1: any warp of a CTA running several decisions) or the whole
// CTA (NW > 1, blockDim.x == 32 NW: one decision per CTA, for batches too
// small to fill the GPU one warp per decision -- latency of a single
// controller call).  Same results for every NW: each mutation is evaluated
// with the same op sequence; the level's (objective, lexicographic) minimum,
// feasible count and first ModelError are exact reductions.
// fl / fp: the controller's latency / power grids reduced per candidate
// (FastGrid), or null for the generic interpolator.  lv (optional): level
// stats.  Results in *o (thread 0 writes; the group is synchronised on return).
//   share: every fl[f] (and every fp[f]) has the brackets of fl[0] (fp[0])
//   (fast_same_brackets), so each batch is bracketed once for all candidates.
#ifdef BS_GREEDY_PHASES  // diagnostics build: globaltimer at phase ends, printed by thread 0
#define BS_GPH(i)                                                 \
  if (tid == 0) {                                                 \
    unsigned long long t_;                                        \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
    gph[i] = t_;                                                  \
  }
#else
#define BS_GPH(i)
#endif

template <int NW>
__device__ __forceinline__ void greedy_sync() {
  if (NW == 1)
    __syncwarp();
  else
    __syncthreads();
}

// CL > 1: the CTA is one of a thread-block cluster of CL CTAs (one per SM)
// deciding together: each CTA builds the same tables, a level's mutations
// are spread over all CL x NT threads, and the CTAs' partial (objective,
// lexicographic) minima, feasible counts and first errors are combined
// through distributed shared memory after one cluster barrier per level, so
// every CTA takes the same accept step.  Only rank 0 writes level records.
template <int NW, int CL = 1>
__device__ void greedy_coop(const DModels& m, const DProblem& pr, const DMpcCfg& c, const DWaiting* W,
                            const DRunning* R, WGreedyShared& S, DMpcOut* o, DLevel* lv, const FastGrid* fl,
                            const FastGrid* fp, bool share = false) {
  constexpr int NT = 32 * NW;
  constexpr int GNT = NT * CL;  // threads deciding together
  const int lane = threadIdx.x & 31;
  const int tid = NW == 1 ? lane : static_cast<int>(threadIdx.x);
  int crank = 0;
  if constexpr (CL > 1) crank = static_cast<int>(cooperative_groups::this_cluster().block_rank());
  const int gtid = crank * NT + tid;
  WTables& T = S.T;
#ifdef BS_GREEDY_PHASES
  unsigned long long gph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int gph_levels = 0;
#endif
  BS_GPH(0);
  // latency mode: the waiting rows the projection scans are copied to shared
  // memory by every thread at once (one round trip instead of one per
  // request), and the reduced grids the tables read are prefetched into L1
  // while thread 0 projects
  constexpr int kStageW = NW > 1 ? 256 : 1;
  __shared__ long long s_wrem[kStageW];
  __shared__ double s_warr[kStageW];
  const bool staged_w = NW > 1 && pr.n_wait <= kStageW;
  if constexpr (NW > 1) {
    if (staged_w)
      for (int i = tid; i < pr.n_wait; i += NT) {
        s_wrem[i] = W[i].remaining;
        s_warr[i] = W[i].arrival;
      }
    if (fl) {
      const char* g0 = reinterpret_cast<const char*>(fl);
      const char* g1 = reinterpret_cast<const char*>(fp);
      const int lines = static_cast<int>((sizeof(FastGrid) * c.nc + 127) / 128);
      for (int i = tid; i < 2 * lines; i += NT)
        asm volatile("prefetch.global.L1 [%0];" ::"l"((i < lines ? g0 : g1) + 128ll * (i < lines ? i : i - lines)));
      prefetch_knots(fl, fp, tid - (NT - 2 * kMaxRank));
    }
    __syncthreads();
  }
  if (tid == 0) {
    T.nc = c.nc;
    T.ttft = c.ttft;
    int st = staged_w ? project_wa(pr, c, WaitStaged{s_wrem, s_warr}, R, &T) : project_dev(pr, c, W, R, &T);
    if (st == BS_OK && (m.grid[0].bad_axis || m.grid[2].bad_axis) && T.K > 0) st = BS_MODEL_ERROR;
    T.status = st;
    for (int k = 0; k < kMaxK; ++k) T.bad_lat[k] = T.bad_pow[k] = 0u;
    memset(o, 0, sizeof *o);
    o->status = st;
    o->K = T.K;
  }
  greedy_sync<NW>();
  BS_GPH(1);
  if (T.status != BS_OK) return;
  const int K = T.K, nc = c.nc;
  if (K == 0) {  // dvfs.hpp:194-197
    if (tid == 0) o->feasible = 1;
    greedy_sync<NW>();
    return;
  }
  unsigned anybad = 0, nofilt = 0;
  const bool shared_brk = fl && share;
  if (shared_brk) {
    if (tid < K) {
      fast_brackets(fl[0], T.n_req[tid], T.sum_len[tid], S.blat[tid]);
      fast_brackets(fp[0], T.n_req[tid], T.sum_len[tid], S.bpow[tid]);
    }
    greedy_sync<NW>();
  }
  for (int e = tid; e < K * nc; e += NT) {
    const int k = e / nc, f = e - k * nc;
    double L, P;
    if (shared_brk) {
      L = fast_corners(fl[f], S.blat[k]);
      P = fast_corners(fp[f], S.bpow[k]);
    } else if (fl) {
      L = fast_interp(fl[f], T.n_req[k], T.sum_len[k]);
      P = fast_interp(fp[f], T.n_req[k], T.sum_len[k]);
    } else {
      const Query q = make_query(T.n_req[k], T.sum_len[k], pr.tp, c.cand[f]);
      L = interp(m.grid[0], q, nullptr);
      P = interp(m.grid[2], q, nullptr);
    }
    if (!model_value_ok(L)) {
      atomicOr(&T.bad_lat[k], 1u << f);
      anybad = 1;
    }
    if (!model_value_ok(P)) {
      atomicOr(&T.bad_pow[k], 1u << f);
      anybad = 1;
    }
    const double A = __dmul_rn(T.wf[k], L);                                  // dvfs.hpp:112-113, 154-155
    T.A[e] = A;
    T.P[e] = P;
    T.E[e] = __dmul_rn(A, P);                                               // dvfs.hpp:167
    if (!(A >= 0.0) || !isfinite(A) || !isfinite(T.E[e])) nofilt = 1;
    T.B0[e] = __dmul_rn(A, c.one_plus_margin);                              // dvfs.hpp:115
    T.B1[e] = __dmul_rn(__dadd_rn(A, c.switch_ms), c.one_plus_margin);      // dvfs.hpp:114-115
    if (k == 0) T.T1[f] = __dadd_rn(pr.now, c.cand[f] != pr.cur_freq ? T.B1[e] : T.B0[e]);
  }
  bool bad, filt;
  if (NW == 1) {
    bad = __any_sync(0xffffffffu, anybad);
    filt = !__any_sync(0xffffffffu, nofilt);
    __syncwarp();
  } else {
    bad = __syncthreads_or(anybad) != 0;
    filt = __syncthreads_or(nofilt) == 0;
  }
  BS_GPH(2);
  // all-max initialization (dvfs.hpp:201-205)
  if (tid == 0) {
    for (int k = 0; k < K; ++k) S.cur[k] = static_cast<unsigned char>(nc - 1);
    double obj = 0.0;
    int err;
    const int feas = weval(T, pr, c, S.cur, &obj, &err);
    if (!feas && !err) {
      for (int k = 0; k < K && !err; ++k) {
        if ((T.bad_lat[k] >> (nc - 1)) & 1u) err = 1;
        else if ((T.bad_pow[k] >> (nc - 1)) & 1u) err = 2;
      }
      double num = 0.0, den = 0.0;
      for (int k = 0; k < K; ++k) {
        num = __dadd_rn(num, T.E[k * nc + nc - 1]);
        den = __dadd_rn(den, T.A[k * nc + nc - 1]);
      }
      obj = den > 0.0 ? __ddiv_rn(num, den) : 0.0;
    }
    if (err) o->status = BS_MODEL_ERROR;
    S.accepted = feas;  // broadcast the initial feasibility
    S.obj = obj;
    o->feasible = feas;
    o->eval_count = 1;
    o->objective = obj;
  }
  greedy_sync<NW>();
  BS_GPH(3);
  if (o->status != BS_OK) return;
  if (S.accepted && nc > 1) {
    const int last_level = nc >= 3 ? nc - 2 : 1;
    for (int l = 1; l <= last_level; ++l) {
      const int target = nc - l;  // avail[l-1] (ascending index)
      const int r1 = nc - 1 - l;  // avail[l]
      const int r2 = l + 1 < nc ? nc - 2 - l : -1;
      const int base = r2 >= 0 ? 3 : 2;
      if (threadIdx.x < 32 || NW == 1) {  // positions holding the target (warp 0; every warp when NW == 1)
        const unsigned pm = __ballot_sync(0xffffffffu, lane < K && S.cur[lane] == target);
        if (lane == 0) {
          S.np = __popc(pm);
          unsigned mm = pm;
          for (int i = 0; mm; ++i) {
            S.pos[i] = __ffs(mm) - 1;
            mm &= mm - 1;
          }
        }
      }
      greedy_sync<NW>();
      const int np = S.np;
      if (np == 0) break;  // dvfs.hpp:222
      const unsigned long long combos = ipow(static_cast<unsigned long long>(base), np);
      unsigned long long bo = ~0ull, bc = ~0ull, feas = 0, errkey = ~0ull;
      if (!bad) {
        GLeafAcc g;
        g.bo = ~0ull;
        g.bc = ~0ull;
        g.feas = 0;
        g.filt = filt;
        g.incumbent = S.obj;
        g.thr_s = gfilter_scaled(S.obj);
        // prefixes of all but the last R <= 3 digits (base^np <= 3^kMaxK < 2^31
        // tasks), R chosen for the shortest per-thread path (rounds x steps)
        int J = np;
        unsigned long long best_cost = ~0ull;
        for (int R = 0; R <= 3 && R <= np; ++R) {
          const unsigned long long tasks = ipow(static_cast<unsigned long long>(base), np - R);
          const unsigned long long rounds = (tasks + GNT - 1) / GNT;
          const unsigned long long steps =
              K + (R >= 1 ? base : 0) + (R >= 2 ? base * base : 0) + (R == 3 ? base * base * base : 0);
          if (rounds * steps < best_cost) {
            best_cost = rounds * steps;
            J = np - R;
          }
        }
        const unsigned long long tasks = ipow(static_cast<unsigned long long>(base), J);
        const unsigned long long pwJ = tasks;
        for (unsigned long long p = gtid; p < tasks; p += GNT)
          wlevel_tail(T, pr, c, S.cur, S.pos, np, base, target, r1, r2, J, pwJ, static_cast<unsigned>(p), g);
        bo = g.bo;
        bc = g.bc;
        feas = g.feas;
      } else {
        unsigned char mut[kMaxK];
        for (int k = 0; k < K; ++k) mut[k] = S.cur[k];
        for (unsigned long long code = 1 + gtid; code < combos; code += GNT) {
          unsigned long long cc = code, lex = 0;
          for (int i = 0; i < np; ++i) {  // digit i -> pos[i], least significant first (dvfs.hpp:233-237)
            const unsigned long long digit = cc % base;
            cc /= base;
            mut[S.pos[i]] = static_cast<unsigned char>(digit == 0 ? target : (digit == 1 ? r1 : r2));
          }
          for (int i = 0; i < np; ++i) {
            const unsigned char v = mut[S.pos[i]];
            const unsigned long long digit = v == target ? 0 : (v == r1 ? 1 : 2);
            lex = lex * base + (base - 1 - digit);
          }
          double obj = 0.0;
          int err;
          const int ok = weval(T, pr, c, mut, &obj, &err);
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
      }
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
      if constexpr (NW > 1) {  // across the CTA's warps
        __shared__ unsigned long long r_bo[NW], r_bc[NW], r_feas[NW], r_err[NW];
        const int w = threadIdx.x >> 5;
        if (lane == 0) {
          r_bo[w] = bo;
          r_bc[w] = bc;
          r_feas[w] = feas;
          r_err[w] = errkey;
        }
        __syncthreads();
        if (tid == 0)
          for (int v = 1; v < NW; ++v) {
            if (key_less(r_bo[v], r_bc[v], bo, bc)) {
              bo = r_bo[v];
              bc = r_bc[v];
            }
            feas += r_feas[v];
            errkey = r_err[v] < errkey ? r_err[v] : errkey;
          }
      }
      if constexpr (CL > 1) {  // across the cluster's CTAs (distributed shared memory)
        __shared__ unsigned long long c_part[2][4];  // by level parity: one barrier per level
        const int par = l & 1;
        if (tid == 0) {
          c_part[par][0] = bo;
          c_part[par][1] = bc;
          c_part[par][2] = feas;
          c_part[par][3] = errkey;
        }
        cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
        cl.sync();
        if (tid == 0) {
          bo = bc = errkey = ~0ull;
          feas = 0;
          for (int r = 0; r < CL; ++r) {
            const unsigned long long* q = cl.map_shared_rank(&c_part[par][0], r);
            const unsigned long long qo = q[0], qc = q[1], qf = q[2], qe = q[3];
            if (key_less(qo, qc, bo, bc)) {
              bo = qo;
              bc = qc;
            }
            feas += qf;
            errkey = qe < errkey ? qe : errkey;
          }
        }
      }
      if (tid == 0) {
        o->eval_count += static_cast<long long>(combos - 1);  // every mutation counts (dvfs.hpp:238)
        DLevel Lv;
        Lv.k_prime = np;
        Lv.replaced_mhz = c.cand[target];
        Lv.mutations = static_cast<long long>(combos - 1);
        Lv.feasible_mutations = static_cast<long long>(feas);
        Lv.accepted = 0;
        if (errkey != ~0ull) {
          o->status = BS_MODEL_ERROR;
          o->n_levels = -static_cast<int>(errkey & 3ull);
        } else {
          const double bp = __longlong_as_double(static_cast<long long>(bo));
          if (bo != ~0ull && bp <= S.obj) {
            unsigned long long lx = bc;
            for (int i = np - 1; i >= 0; --i) {
              const unsigned long long digit = base - 1 - (lx % base);
              lx /= base;
              S.cur[S.pos[i]] = static_cast<unsigned char>(digit == 0 ? target : (digit == 1 ? r1 : r2));
            }
            S.obj = bp;
            o->objective = bp;
            Lv.accepted = 1;
          }
          if (lv && crank == 0) lv[o->n_levels] = Lv;
          o->n_levels += 1;
        }
        S.accepted = Lv.accepted;
      }
      greedy_sync<NW>();
#ifdef BS_GREEDY_PHASES
      ++gph_levels;
#endif
      if (o->status != BS_OK || S.accepted == 0) break;
    }
  }
  BS_GPH(4);
  if (tid == 0 && o->status == BS_OK)
    for (int k = 0; k < K; ++k) o->idx[k] = S.cur[k];
  greedy_sync<NW>();
#ifdef BS_GREEDY_PHASES
  if (tid == 0 && NW > 1)
    printf("greedy phases ns: project %llu tables %llu init %llu levels %llu (%d levels, K %d nc %d)\n",
           gph[1] - gph[0], gph[2] - gph[1], gph[3] - gph[2], gph[4] - gph[3], gph_levels, K, nc);
#endif
}

// One decision per warp (the batch kernels and the cluster replay).
__device__ __forceinline__ void greedy_warp(const DModels& m, const DProblem& pr, const DMpcCfg& c, const DWaiting* W,
                                            const DRunning* R, WGreedyShared& S, DMpcOut* o, DLevel* lv,
                                            const FastGrid* fl, const FastGrid* fp, bool share = false) {
  greedy_coop<1>(m, pr, c, W, R, S, o, lv, fl, fp, share);
}

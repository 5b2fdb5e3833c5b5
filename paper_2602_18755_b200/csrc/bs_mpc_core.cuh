// bs_mpc_core.cuh — prefill-MPC building blocks shared by the MPC kernels
// (bs_mpc.cu) and the cluster replay (bs_replay.cu): project_batches on the
// device, the per-decision (k, f) tables of the exhaustive search and the
// assignment evaluator.  The greedy search is bs_greedy_warp.cuh.  Included inside each translation unit's
// anonymous namespace.  Reference: proj/include/pdsim/dvfs.hpp.
#pragma once

__host__ __device__ inline unsigned long long ipow(unsigned long long b, int e) {
  unsigned long long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// ---------------------------------------------------------------------------
// projection: project_batches (dvfs.hpp:63-100) over form_prefill_batch
// (scheduler.hpp:40-66).  Only the queue head can be partially consumed (a
// partial chunk ends a batch), so the state is (head, head_remaining).
// ---------------------------------------------------------------------------
// The waiting queue's (remaining, arrival) as the projection reads them: from
// the problem's global rows, or from a shared-memory copy.
struct WaitRows {
  const DWaiting* W;
  __device__ __forceinline__ long long rem(int i) const { return W[i].remaining; }
  __device__ __forceinline__ double arr(int i) const { return W[i].arrival; }
};
struct WaitStaged {
  const long long* r;
  const double* a;
  __device__ __forceinline__ long long rem(int i) const { return r[i]; }
  __device__ __forceinline__ double arr(int i) const { return a[i]; }
};

template <class Tab, class WA>
__device__ int project_wa(const DProblem& pr, const DMpcCfg& c, WA W, const DRunning* R, Tab* T);

template <class Tab>
__device__ int project_dev(const DProblem& pr, const DMpcCfg& c, const DWaiting* W, const DRunning* R, Tab* T) {
  return project_wa(pr, c, WaitRows{W}, R, T);
}

template <class Tab, class WA>
__device__ int project_wa(const DProblem& pr, const DMpcCfg& c, WA W, const DRunning* R, Tab* T) {
  int K = 0;
  if (pr.run_active) {
    T->n_req[0] = pr.run_n;
    T->sum_len[0] = pr.run_sum;
    T->wf[0] = pr.run_wr;
    double mn = INFINITY;
    int nc = 0;
    if (pr.n_run < 0) {  // summarised by the caller (the cluster replay)
      mn = pr.run_minarr;
      nc = pr.run_ncomp;
    }
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
  long long head_rem = pr.n_wait > 0 ? W.rem(0) : 0;
  while (head < pr.n_wait && K < c.horizon) {
    long long tokens = 0, npick = 0, sum = 0;
    int consumed = 0, ncomp = 0;
    double mn = INFINITY;
    long long partial_rem = -1;
    for (int i = head; i < pr.n_wait; ++i) {
      if (npick >= c.max_batch_requests) break;
      const long long rem = i == head ? head_rem : W.rem(i);
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
            const double a = W.arr(i);
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
        const double a = W.arr(i);
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
      head_rem = W.rem(head);
    }
  }
  T->K = K;
  return BS_OK;
}

// Tables for one problem, written by a CTA.  Projection by thread 0.
// The controller's latency / power grids reduced to one (configuration, tp)
// for every candidate (FastGrid, bs_sim.cuh), built on the host from the
// model's mirror; share: every candidate's grid brackets like candidate 0's.
struct DFastPair {
  FastGrid lat[kMaxCand];
  FastGrid pw[kMaxCand];
  int share;
  int _pad;
};

// The knot vectors of candidate 0's reduced grids (the brackets' binary
// searches read them next) prefetched into L1 by thread `t` in
// [0, 2 kMaxRank): grid t / kMaxRank, axis t % kMaxRank.
__device__ __forceinline__ void prefetch_knots(const FastGrid* fl, const FastGrid* fp, int t) {
  if (t < 0 || t >= 2 * kMaxRank) return;
  const FastGrid* g = t < kMaxRank ? fl : fp;
  const int a = t % kMaxRank;
  if (a >= g->na || g->fixed[a]) return;
  const double* k = g->knots[a];
  for (int i = 0; i < g->n[a]; i += 16) asm volatile("prefetch.global.L1 [%0];" ::"l"(k + i));
}

// fl / fp (optional): the latency / power grids reduced to (pr.tp, cand[f])
// for every candidate f -- bit-identical values with 2^(active axes) corners
// instead of 2^rank; share: each batch is bracketed once for all candidates.
#ifdef BS_PREP_PHASES
#define BS_BT_MARK(i)                                                              \
  if (threadIdx.x == 0 && (blockIdx.x & 63) == 0) {                                 \
    unsigned long long t_;                                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
    bt_t[i] = t_;                                                                   \
  }
#else
#define BS_BT_MARK(i)
#endif

__device__ void build_tables(const DModels& m, const DProblem& pr, const DMpcCfg& c, const DWaiting* W,
                             const DRunning* R, DTables* T, int* s_status, const FastGrid* fl = nullptr,
                             const FastGrid* fp = nullptr, bool share = false) {
#ifdef BS_PREP_PHASES
  unsigned long long bt_t[8] = {0};
#endif
  BS_BT_MARK(0);
  __shared__ FastBrk s_bl[kMaxK], s_bp[kMaxK];
  // The projection is one thread's serial scan of the waiting queue: its rows
  // are first copied to shared memory by the whole block (one round trip),
  // the reduced grids prefetched into L1 meanwhile, and the projected
  // batches kept in shared memory for the table loop (then copied to T).
  constexpr int kStageW = 256;
  __shared__ long long s_wrem[kStageW];
  __shared__ double s_warr[kStageW];
  __shared__ struct {
    long long n_req[kMaxK], sum_len[kMaxK];
    double wf[kMaxK], minarr[kMaxK];
    int ncomp[kMaxK];
    int K;
  } s_pj;
  const bool staged = pr.n_wait <= kStageW;
  if (staged)
    for (int i = threadIdx.x; i < pr.n_wait; i += blockDim.x) {
      s_wrem[i] = W[i].remaining;
      s_warr[i] = W[i].arrival;
    }
  if (fl) {
    const int lines = static_cast<int>((sizeof(FastGrid) * c.nc + 127) / 128);
    for (int i = threadIdx.x; i < 2 * lines; i += blockDim.x)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(i < lines ? fl : fp) +
                                                  128ll * (i < lines ? i : i - lines)));
    prefetch_knots(fl, fp, static_cast<int>(threadIdx.x) - (blockDim.x - 2 * kMaxRank));
  }
  __syncthreads();
  BS_BT_MARK(1);
  if (threadIdx.x == 0) {
    int st = staged ? project_wa(pr, c, WaitStaged{s_wrem, s_warr}, R, &s_pj) : project_dev(pr, c, W, R, &s_pj);
    if (st == BS_OK && (m.grid[0].bad_axis || m.grid[2].bad_axis) && s_pj.K > 0) st = BS_MODEL_ERROR;
    *s_status = st;
  }
  __syncthreads();
  BS_BT_MARK(2);
  const int K = s_pj.K;
  const int nc = c.nc;
  if (threadIdx.x == 0) {
    T->nc = c.nc;
    T->ttft = c.ttft;
    T->K = K;
  }
  for (int k = threadIdx.x; k < kMaxK; k += blockDim.x) {
    T->bad_lat[k] = 0u;
    T->bad_pow[k] = 0u;
    if (k < K) {
      T->n_req[k] = s_pj.n_req[k];
      T->sum_len[k] = s_pj.sum_len[k];
      T->wf[k] = s_pj.wf[k];
      T->minarr[k] = s_pj.minarr[k];
      T->ncomp[k] = s_pj.ncomp[k];
    }
  }
  __syncthreads();
  BS_BT_MARK(3);
  if (*s_status != BS_OK) return;
  const bool shared_brk = fl && share;
  if (shared_brk) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      fast_brackets(fl[0], s_pj.n_req[k], s_pj.sum_len[k], s_bl[k]);
      fast_brackets(fp[0], s_pj.n_req[k], s_pj.sum_len[k], s_bp[k]);
    }
    __syncthreads();
  BS_BT_MARK(4);
  }
  for (int e = threadIdx.x; e < K * nc; e += blockDim.x) {
    const int k = e / nc, f = e - k * nc;
    double L, P;
    if (shared_brk) {
      L = fast_corners(fl[f], s_bl[k]);
      P = fast_corners(fp[f], s_bp[k]);
    } else if (fl) {
      L = fast_interp(fl[f], s_pj.n_req[k], s_pj.sum_len[k]);
      P = fast_interp(fp[f], s_pj.n_req[k], s_pj.sum_len[k]);
    } else {
      const Query q = make_query(s_pj.n_req[k], s_pj.sum_len[k], pr.tp, c.cand[f]);
      L = interp(m.grid[0], q, nullptr);
      P = interp(m.grid[2], q, nullptr);
    }
    if (!model_value_ok(L)) atomicOr(&T->bad_lat[k], 1u << f);
    if (!model_value_ok(P)) atomicOr(&T->bad_pow[k], 1u << f);
    const double A = __dmul_rn(s_pj.wf[k], L);                               // dvfs.hpp:112-113, 154-155
    T->A[k][f] = A;
    T->P[k][f] = P;
    T->E[k][f] = __dmul_rn(A, P);                                          // dvfs.hpp:167
    T->B0[k][f] = __dmul_rn(A, c.one_plus_margin);                         // dvfs.hpp:115
    T->B1[k][f] = __dmul_rn(__dadd_rn(A, c.switch_ms), c.one_plus_margin);  // dvfs.hpp:114-115
    if (k == 0) T->T1[f] = __dadd_rn(pr.now, c.cand[f] != pr.cur_freq ? T->B1[0][f] : T->B0[0][f]);
  }
  __syncthreads();
  BS_BT_MARK(5);
  // per-level sorted order of the switched steps: one thread per (k, f)
  // computes its rank (ties by index), then scatters
  int finite = 1, filt = 1;
  for (int e = threadIdx.x; e < K * nc; e += blockDim.x) {
    const int k = e / nc, f = e - k * nc;
    const double* key = k == 0 ? T->T1 : T->B1[k];
    const double v = key[f];
    if (!isfinite(v) || !isfinite(T->B0[k][f])) finite = 0;
    const double A = T->A[k][f];
    if (!(A >= 0.0) || !isfinite(A) || !isfinite(T->E[k][f])) filt = 0;
    int r = 0;
    for (int g = 0; g < nc; ++g) {
      const double w = key[g];
      r += (w < v || (w == v && g < f)) ? 1 : 0;
    }
    T->sb[k][r] = v;
    T->ord[k][r] = static_cast<unsigned char>(f);
    T->rank[k][f] = static_cast<unsigned char>(r);
    T->srec[k][r] = SRec{v, T->E[k][f], A, 0.0};  // th0n: step_thresholds
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
  const int all_filt = __syncthreads_and(filt);
  BS_BT_MARK(6);
  for (int e = threadIdx.x; e < K * nc; e += blockDim.x) {  // ranks of every level are in place
    const int k = e / nc, f = e - k * nc;
    T->sinfo[k][T->rank[k][f]] =
        static_cast<unsigned short>(f | (k + 1 < K ? static_cast<int>(T->rank[k + 1][f]) << 8 : 0));
  }
  if (threadIdx.x == 0) {
    T->filter_ok = all_filt;
    T->sorted_ok = all_finite && isfinite(T->ttft);
  }
  __syncthreads();
#ifdef BS_PREP_PHASES
  if (threadIdx.x == 0 && (blockIdx.x & 63) == 0)
    printf("tables ns: stage %llu project %llu copy %llu brackets %llu corners %llu ranks %llu\n", bt_t[1] - bt_t[0],
           bt_t[2] - bt_t[1], bt_t[3] - bt_t[2], bt_t[4] - bt_t[3], bt_t[5] - bt_t[4], bt_t[6] - bt_t[5]);
#endif
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

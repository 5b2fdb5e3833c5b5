/* biscale_oracle.c -- TEST INFRASTRUCTURE ONLY (see biscale_oracle.h).
 *
 * Plain-C restatement of the reference algorithms on the decision path.
 * Reference paths are relative to /root/reference/proj/include/pdsim/.
 * Compiled with -ffp-contract=off so every double op rounds as the
 * reference's does.  Status codes are the bs_status values
 * of include/biscale_gpu.h, one per reference exception class.
 */
#include "biscale_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---- NdGrid (perfmodel.hpp:116-193) --------------------------------------- */

int orc_interpolate(const bs_grid* g, const double* coords, double* out, uint32_t* clamps) {
  const int dims = g->rank;
  int lo[BS_MAX_RANK];
  double frac[BS_MAX_RANK];
  for (int d = 0; d < dims; ++d) { /* perfmodel.hpp:156-173 */
    const double* k = g->knots[d];
    const int n = g->n_knots[d];
    double x = coords[d];
    if (x < k[0] || x > k[n - 1]) {
      if (clamps) *clamps += 1;
      x = x < k[0] ? k[0] : (k[n - 1] < x ? k[n - 1] : x); /* std::clamp */
    }
    if (n == 1) {
      lo[d] = 0;
      frac[d] = 0.0;
      continue;
    }
    int hi = 0; /* std::upper_bound: first knot > x */
    while (hi < n && !(x < k[hi])) ++hi;
    if (hi < 1) hi = 1;
    if (hi > n - 1) hi = n - 1;
    lo[d] = hi - 1;
    frac[d] = (x - k[lo[d]]) / (k[hi] - k[lo[d]]);
  }
  double acc = 0.0; /* perfmodel.hpp:175-192 */
  const int corners = 1 << dims;
  for (int mask = 0; mask < corners; ++mask) {
    double weight = 1.0;
    size_t flat = 0;
    for (int d = 0; d < dims; ++d) {
      int high = (mask >> d) & 1;
      double f = frac[d];
      if (high && g->n_knots[d] == 1) {
        weight = 0.0;
        break;
      }
      weight *= high ? f : (1.0 - f);
      flat = flat * (size_t)g->n_knots[d] + (size_t)(lo[d] + high);
    }
    if (weight != 0.0) acc += weight * g->values[flat];
  }
  *out = acc;
  return BS_OK;
}

static int query(const bs_grid* g, const bs_features* f, int tp, double freq, double* out, const char* what) {
  double c[BS_MAX_RANK];
  for (int d = 0; d < g->rank; ++d) { /* query_coords, perfmodel.hpp:241-258 */
    switch (g->role[d]) {
      case BS_AXIS_SUM_LEN: c[d] = (double)f->sum_len; break;
      case BS_AXIS_N_REQUESTS: c[d] = (double)f->n_requests; break;
      case BS_AXIS_TP: c[d] = (double)tp; break;
      case BS_AXIS_FREQ: c[d] = freq; break;
      default: return fail(BS_MODEL_ERROR, "grid: unknown axis");
    }
  }
  double v;
  orc_interpolate(g, c, &v, NULL);
  if (!(v > 0.0) || !isfinite(v)) /* perfmodel.hpp:264, 270 */
    return fail(BS_MODEL_ERROR, "%s model returned non-positive value", what);
  *out = v;
  return BS_OK;
}

static int idle_power(const bs_model_set* m, int tp, double freq, double* out) { /* perfmodel.hpp:274-288 */
  for (int i = 0; i < m->n_idle; ++i) {
    const bs_idle_entry* e = &m->idle[i];
    if (e->tp != tp) continue;
    if (e->n < 1) return fail(BS_MODEL_ERROR, "idle model: empty frequency set");
    double x = freq < e->freqs_mhz[0] ? e->freqs_mhz[0] : (e->freqs_mhz[e->n - 1] < freq ? e->freqs_mhz[e->n - 1] : freq);
    int hi = 0;
    while (hi < e->n && !(x < e->freqs_mhz[hi])) ++hi;
    if (hi < 1) hi = 1;
    if (hi > e->n - 1) hi = e->n - 1;
    if (e->n == 1) {
      *out = e->idle_w[0];
      return BS_OK;
    }
    int lo = hi - 1;
    double t = (x - e->freqs_mhz[lo]) / (e->freqs_mhz[hi] - e->freqs_mhz[lo]);
    *out = e->idle_w[lo] + t * (e->idle_w[hi] - e->idle_w[lo]);
    return BS_OK;
  }
  return fail(BS_MODEL_ERROR, "idle model: tp %d not present", tp);
}

int orc_predict(const bs_model_set* m, int which, const bs_features* f, int tp, double freq, double* out) {
  switch (which) {
    case 0: return query(&m->latency_prefill, f, tp, freq, out, "latency");
    case 1: return query(&m->latency_decode, f, tp, freq, out, "latency");
    case 2: return query(&m->power_prefill, f, tp, freq, out, "power");
    case 3: return query(&m->power_decode, f, tp, freq, out, "power");
    default: return idle_power(m, tp, freq, out);
  }
}

int orc_predict_batch(const bs_model_set* m, int which, const bs_features* feats, const int32_t* tp,
                      const double* freq, int n, double* out, int32_t* status) {
  for (int i = 0; i < n; ++i) {
    status[i] = orc_predict(m, which, &feats[i], tp[i], freq[i], &out[i]);
    if (status[i] != BS_OK) out[i] = 0.0;
  }
  return BS_OK;
}

/* ---- FrequencyLadder (perfmodel.hpp:56-91) --------------------------------- */

static int ladder_validate(const double* l, int n) {
  if (n < 1) return fail(BS_PARAMETER_ERROR, "frequency ladder: empty");
  double prev = 0.0;
  for (int i = 0; i < n; ++i) {
    if (l[i] <= prev) return fail(BS_PARAMETER_ERROR, "frequency ladder: must be strictly increasing and > 0");
    prev = l[i];
  }
  return BS_OK;
}

int orc_ladder_select(const double* l, int size, int n, double* out) {
  if (ladder_validate(l, size) != BS_OK) return -1;
  if (n <= 0) {
    fail(BS_PARAMETER_ERROR, "frequency ladder: select(0)");
    return -1;
  }
  if (n >= size) {
    memcpy(out, l, sizeof(double) * (size_t)size);
    return size;
  }
  if (n == 1) {
    out[0] = l[size - 1];
    return 1;
  }
  int m = 0;
  for (int i = 0; i < n; ++i) {
    size_t idx = ((size_t)i * (size_t)(size - 1)) / (size_t)(n - 1); /* integer division */
    if (m == 0 || out[m - 1] != l[idx]) out[m++] = l[idx];        /* std::unique */
  }
  return m;
}

/* ---- synthetic families (perfmodel.hpp:369-516) ---------------------------- */

static const double kSumKnots[6] = {16, 64, 256, 1024, 4096, 16384};

static double synth_lat(int family, const double* o, double s, double tp, double f) { /* 397-405 */
  double per_shard = s / tp;
  if (family == 0) return o[0] * per_shard / f;
  double eff = f < o[3] ? f : o[3];
  return o[0] * per_shard / eff;
}

static double synth_pow(int family, const double* o, double tp, double f) { /* 407-412 */
  double per_gpu = family == 0 ? o[1] * f * f * f + o[2] : o[1] * f + o[2];
  return per_gpu * tp;
}

static int cmp_int(const void* a, const void* b) { return *(const int32_t*)a - *(const int32_t*)b; }

int orc_synth_model_set(int family, const double* ladder, int nl, const int32_t* tps, int n_tp, const double* po,
                        const double* dopt, double* lat_p, double* lat_d, double* pow_p, double* pow_d,
                        double* idle_w) {
  int rc = ladder_validate(ladder, nl);
  if (rc) return rc;
  if (n_tp < 1) return fail(BS_PARAMETER_ERROR, "synth_model: tp_list empty");
  int32_t tpk[64];
  int nt = 0;
  for (int i = 0; i < n_tp && i < 64; ++i) {
    if (tps[i] < 1) return fail(BS_PARAMETER_ERROR, "synth_model: tp must be >= 1");
    tpk[nt++] = tps[i];
  }
  qsort(tpk, (size_t)nt, sizeof tpk[0], cmp_int);
  int u = 0;
  for (int i = 0; i < nt; ++i)
    if (u == 0 || tpk[u - 1] != tpk[i]) tpk[u++] = tpk[i];
  nt = u;
  const double* opts[2] = {po, dopt};
  double* lat[2] = {lat_p, lat_d};
  for (int ph = 0; ph < 2; ++ph) { /* perfmodel.hpp:440-450 */
    size_t o = 0;
    for (int s = 0; s < 6; ++s)
      for (int r = 0; r < 9; ++r)
        for (int t = 0; t < nt; ++t)
          for (int f = 0; f < nl; ++f) lat[ph][o++] = synth_lat(family, opts[ph], kSumKnots[s], (double)tpk[t], ladder[f]);
  }
  size_t o = 0; /* prefill power (sum_len, tp, freq): perfmodel.hpp:454-463 */
  for (int s = 0; s < 6; ++s)
    for (int t = 0; t < nt; ++t)
      for (int f = 0; f < nl; ++f) pow_p[o++] = synth_pow(family, po, (double)tpk[t], ladder[f]);
  o = 0; /* decode power 4-D: perfmodel.hpp:465-475 */
  for (int s = 0; s < 6; ++s)
    for (int r = 0; r < 9; ++r)
      for (int t = 0; t < nt; ++t)
        for (int f = 0; f < nl; ++f) pow_d[o++] = synth_pow(family, dopt, (double)tpk[t], ladder[f]);
  o = 0; /* idle from the prefill options (synth_model_set keeps pre.idle, 514) */
  for (int t = 0; t < nt; ++t)
    for (int f = 0; f < nl; ++f) idle_w[o++] = po[4] * synth_pow(family, po, (double)tpk[t], ladder[f]);
  return BS_OK;
}

/* ---- scheduler + projection (scheduler.hpp:40-73, dvfs.hpp:63-100) --------- */

typedef struct {
  int64_t id;
  double arrival;
  int64_t remaining;
} qentry;

static int mpc_validate(const bs_mpc_config* c) { /* MpcConfig::validate, dvfs.hpp:25-31 */
  if (c->horizon_K < 1) return fail(BS_PARAMETER_ERROR, "mpc: horizon_K must be >= 1");
  if (c->ladder_N < 1) return fail(BS_PARAMETER_ERROR, "mpc: ladder_N must be >= 1");
  int rc = ladder_validate(c->ladder_mhz, c->n_ladder);
  if (rc) return rc;
  if (c->ttft_ms <= 0.0 || c->tpot_ms <= 0.0) return fail(BS_PARAMETER_ERROR, "slo: bounds must be > 0");
  if (c->percentile <= 0.0 || c->percentile > 1.0) return fail(BS_PARAMETER_ERROR, "slo: percentile must be in (0,1]");
  if (c->margin < 0.0) return fail(BS_PARAMETER_ERROR, "mpc: margin must be >= 0");
  return BS_OK;
}

typedef struct {
  int K;
  bs_features feat[BS_MAX_K];
  double wf[BS_MAX_K];
  int ncomp[BS_MAX_K];
  double* arr[BS_MAX_K]; /* completing arrivals, malloc'd */
} projection;

static void proj_free(projection* p) {
  for (int k = 0; k < p->K; ++k) free(p->arr[k]);
}

static int project(const bs_snapshot* s, const bs_scheduler_policy* pol, int horizon, projection* p) {
  memset(p, 0, sizeof *p);
  if (horizon < 1) return fail(BS_PARAMETER_ERROR, "project_batches: horizon_K must be >= 1");
  if (horizon > BS_MAX_K) return fail(BS_PARAMETER_ERROR, "horizon_K > %d", BS_MAX_K);
  if (s->running_active) { /* dvfs.hpp:67-78 */
    p->feat[0] = s->running_features;
    p->wf[0] = s->running_work_remaining;
    p->arr[0] = malloc(sizeof(double) * (size_t)(s->n_running + 1));
    for (int i = 0; i < s->n_running; ++i)
      if (s->running_completes[i]) p->arr[0][p->ncomp[0]++] = s->running_arrivals_ms[i];
    p->K = 1;
  }
  qentry* q = malloc(sizeof(qentry) * (size_t)(s->n_waiting + 1));
  int qn = s->n_waiting, head = 0;
  for (int i = 0; i < qn; ++i) {
    q[i].id = s->waiting[i].id;
    q[i].arrival = s->waiting[i].arrival_ms;
    q[i].remaining = s->waiting[i].remaining_len;
  }
  while (head < qn && p->K < horizon) { /* dvfs.hpp:82-98 */
    int k = p->K;
    p->arr[k] = malloc(sizeof(double) * (size_t)(qn - head + 1));
    p->wf[k] = 1.0;
    int64_t tokens = 0, npick = 0, sum = 0;
    int consumed = 0;
    /* form_prefill_batch (scheduler.hpp:40-66), applied in place */
    for (int i = head; i < qn; ++i) {
      if (npick >= pol->max_batch_requests) break;
      int64_t rem = q[i].remaining;
      if (rem <= 0) {
        free(q);
        p->K = k + 1;
        return fail(BS_SIMULATION_ERROR, "scheduler: queued request with no remaining tokens");
      }
      int64_t take;
      int done;
      if (pol->chunking) {
        int64_t room = pol->max_batch_tokens - tokens;
        if (room <= 0) break;
        take = rem < room ? rem : room;
        done = take == rem;
        tokens += take;
      } else {
        if (rem > pol->max_batch_tokens) {
          if (npick == 0) {
            take = rem;
            done = 1;
          } else {
            break;
          }
        } else {
          if (tokens + rem > pol->max_batch_tokens) break;
          take = rem;
          done = 1;
          tokens += rem;
        }
      }
      npick++;
      sum += take;
      if (done) p->arr[k][p->ncomp[k]++] = q[i].arrival;
      q[i].remaining -= take;
      if (q[i].remaining == 0) ++consumed;
      if (pol->chunking && !done) break;                      /* partial chunk ends the batch */
      if (!pol->chunking && rem > pol->max_batch_tokens) break; /* over-budget head runs alone */
    }
    p->feat[k].n_requests = npick;
    p->feat[k].sum_len = sum;
    head += consumed;
    p->K = k + 1;
  }
  free(q);
  return BS_OK;
}

int orc_project(const bs_mpc_config* cfg, const bs_scheduler_policy* policy, const bs_snapshot* snap,
                bs_projected_batch* out, int32_t* out_K) {
  projection p;
  int rc = project(snap, policy, cfg->horizon_K, &p);
  if (rc) {
    proj_free(&p);
    return rc;
  }
  *out_K = p.K;
  for (int k = 0; k < p.K; ++k) {
    out[k].features = p.feat[k];
    out[k].work_fraction = p.wf[k];
    out[k].n_completing = p.ncomp[k];
    double mn = INFINITY;
    for (int i = 0; i < p.ncomp[k]; ++i)
      if (p.arr[k][i] < mn) mn = p.arr[k][i];
    out[k].min_completing_arrival_ms = mn;
  }
  proj_free(&p);
  return BS_OK;
}

/* ---- meets_slo and time_weighted_power (dvfs.hpp:105-172) ----------------- */

typedef struct {
  const bs_model_set* m;
  const bs_mpc_config* cfg;
  const bs_snapshot* q;
  const projection* p;
} mpc_ctx;

static int meets_slo(const mpc_ctx* c, const double* freqs, int* ok) { /* dvfs.hpp:105-122 */
  double t = c->q->now_ms;
  double prev = c->q->current_freq_mhz;
  for (int k = 0; k < c->p->K; ++k) {
    double f = freqs[k], L;
    int rc = query(&c->m->latency_prefill, &c->p->feat[k], c->q->tp, f, &L, "latency");
    if (rc) return rc;
    double lat = c->p->wf[k] * L;
    if (f != prev) lat += c->cfg->switch_latency_ms;
    t += lat * (1.0 + c->cfg->margin);
    for (int i = 0; i < c->p->ncomp[k]; ++i) {
      if (t - c->p->arr[k][i] > c->cfg->ttft_ms) {
        *ok = 0;
        return BS_OK;
      }
    }
    prev = f;
  }
  *ok = 1;
  return BS_OK;
}

static int tw_power(const mpc_ctx* c, const double* freqs, double* out) { /* dvfs.hpp:150-171 */
  double num = 0.0, den = 0.0;
  for (int k = 0; k < c->p->K; ++k) {
    double L, P;
    int rc = query(&c->m->latency_prefill, &c->p->feat[k], c->q->tp, freqs[k], &L, "latency");
    if (rc) return rc;
    rc = query(&c->m->power_prefill, &c->p->feat[k], c->q->tp, freqs[k], &P, "power");
    if (rc) return rc;
    double lat = c->p->wf[k] * L;
    num += lat * P;
    den += lat;
  }
  *out = den > 0.0 ? num / den : 0.0;
  return BS_OK;
}

static int lex_less(const double* a, const double* b, int n) { /* dvfs.hpp:174-176 */
  for (int i = 0; i < n; ++i) {
    if (a[i] < b[i]) return 1;
    if (b[i] < a[i]) return 0;
  }
  return 0;
}

static void set_assignment(bs_mpc_result* r, const double* freqs, const double* cand, int nc, int K) {
  for (int k = 0; k < K; ++k) {
    r->freqs_mhz[k] = freqs[k];
    r->freq_index[k] = -1;
    for (int j = 0; j < nc; ++j)
      if (cand[j] == freqs[k]) r->freq_index[k] = j;
  }
}

/* ---- greedy_freq_select (dvfs.hpp:185-259) --------------------------------- */

int orc_greedy(const bs_model_set* m, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
               const bs_snapshot* snap, bs_mpc_result* r) {
  memset(r, 0, sizeof *r);
  int rc = mpc_validate(cfg);
  if (rc) return rc;
  double cand[BS_MAX_CAND + 64];
  int nc = orc_ladder_select(cfg->ladder_mhz, cfg->n_ladder, cfg->ladder_N, cand);
  if (nc < 0) return BS_PARAMETER_ERROR;
  double avail[BS_MAX_CAND + 64]; /* descending, dvfs.hpp:189 */
  for (int i = 0; i < nc; ++i) avail[i] = cand[nc - 1 - i];
  const int N = nc;
  const double max_mhz = cand[nc - 1];

  projection p;
  rc = project(snap, policy, cfg->horizon_K, &p);
  if (rc) {
    proj_free(&p);
    return rc;
  }
  const int K = p.K;
  r->K = K;
  if (K == 0) { /* dvfs.hpp:194-197, controller fallback dvfs.hpp:328-329 */
    r->feasible = 1;
    r->decision_freq_mhz = snap->target_freq_mhz > 0 ? snap->target_freq_mhz : max_mhz;
    return BS_OK;
  }
  mpc_ctx c = {m, cfg, snap, &p};
  double cur[BS_MAX_K], mut[BS_MAX_K], best[BS_MAX_K];
  for (int k = 0; k < K; ++k) cur[k] = avail[0];
  r->eval_count = 1;
  int ok;
  if ((rc = meets_slo(&c, cur, &ok))) goto out;
  r->feasible = ok;
  if ((rc = tw_power(&c, cur, &r->objective_w))) goto out;
  if (!r->feasible || N == 1) goto done;
  {
    const int last_level = N >= 3 ? N - 2 : 1;
    for (int l = 1; l <= last_level; ++l) {
      const double target = avail[l - 1];
      double repl[2];
      int nrepl = 0;
      repl[nrepl++] = avail[l];
      if (l + 1 < N) repl[nrepl++] = avail[l + 1];
      int pos[BS_MAX_K], np = 0;
      for (int k = 0; k < K; ++k)
        if (cur[k] == target) pos[np++] = k;
      bs_level_stats st;
      memset(&st, 0, sizeof st);
      st.level = l;
      st.replaced_mhz = target;
      st.k_prime = np;
      if (np == 0) break; /* dvfs.hpp:222 */
      const uint64_t base = (uint64_t)nrepl + 1;
      uint64_t combos = 1;
      for (int i = 0; i < np; ++i) combos *= base;
      int have_best = 0;
      double best_power = 0.0;
      for (uint64_t code = 1; code < combos; ++code) { /* dvfs.hpp:230-247 */
        memcpy(mut, cur, sizeof(double) * (size_t)K);
        uint64_t cc = code;
        for (int i = 0; i < np; ++i) {
          uint64_t digit = cc % base;
          cc /= base;
          if (digit > 0) mut[pos[i]] = repl[digit - 1];
        }
        st.mutations += 1;
        r->eval_count += 1;
        if ((rc = meets_slo(&c, mut, &ok))) goto out;
        if (!ok) continue;
        st.feasible_mutations += 1;
        double pw;
        if ((rc = tw_power(&c, mut, &pw))) goto out;
        if (!have_best || pw < best_power || (pw == best_power && lex_less(mut, best, K))) {
          memcpy(best, mut, sizeof(double) * (size_t)K);
          best_power = pw;
          have_best = 1;
        }
      }
      int improved = have_best && (best_power < r->objective_w ||
                                   (best_power == r->objective_w && lex_less(best, cur, K)));
      if (improved) {
        memcpy(cur, best, sizeof(double) * (size_t)K);
        r->objective_w = best_power;
        st.accepted = 1;
      }
      if (r->n_levels < BS_MAX_LEVELS) r->levels[r->n_levels++] = st;
      if (!st.accepted) break;
    }
  }
done:
  set_assignment(r, cur, cand, nc, K);
  r->decision_freq_mhz = cur[0];
out:
  proj_free(&p);
  return rc;
}

/* ---- exhaustive MPC (tests/test_dvfs.cpp:74-94; pinned tie-break) ---------- */

int orc_exhaustive(const bs_model_set* m, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, bs_mpc_result* r) {
  memset(r, 0, sizeof *r);
  int rc = mpc_validate(cfg);
  if (rc) return rc;
  double cand[BS_MAX_CAND + 64];
  int nc = orc_ladder_select(cfg->ladder_mhz, cfg->n_ladder, cfg->ladder_N, cand);
  if (nc < 0) return BS_PARAMETER_ERROR;
  projection p;
  rc = project(snap, policy, cfg->horizon_K, &p);
  if (rc) {
    proj_free(&p);
    return rc;
  }
  const int K = p.K;
  r->K = K;
  if (K == 0) {
    r->feasible = 1;
    r->decision_freq_mhz = snap->target_freq_mhz > 0 ? snap->target_freq_mhz : cand[nc - 1];
    proj_free(&p);
    return BS_OK;
  }
  mpc_ctx c = {m, cfg, snap, &p};
  int idx[BS_MAX_K] = {0}, best_idx[BS_MAX_K] = {0};
  double a[BS_MAX_K], best[BS_MAX_K];
  int found = 0;
  double best_p = 0.0;
  uint64_t total = 0, feas = 0;
  for (;;) {
    for (int k = 0; k < K; ++k) a[k] = cand[idx[k]];
    ++total;
    int ok;
    if ((rc = meets_slo(&c, a, &ok))) goto out;
    if (ok) {
      ++feas;
      double pw;
      if ((rc = tw_power(&c, a, &pw))) goto out;
      if (!found || pw < best_p || (pw == best_p && lex_less(a, best, K))) {
        found = 1;
        best_p = pw;
        memcpy(best, a, sizeof(double) * (size_t)K);
        memcpy(best_idx, idx, sizeof(int) * (size_t)K);
      }
    }
    int d = 0; /* odometer, digit 0 fastest (test_dvfs.cpp:89-91) */
    while (d < K && ++idx[d] == nc) idx[d++] = 0;
    if (d == K) break;
  }
  if (!found) {
    for (int k = 0; k < K; ++k) {
      best[k] = cand[nc - 1];
      best_idx[k] = nc - 1;
    }
    if ((rc = tw_power(&c, best, &best_p))) goto out;
  }
  r->feasible = found;
  r->objective_w = best_p;
  r->trajectories = total;
  r->feasible_count = feas;
  r->eval_count = (int64_t)total;
  {
    uint64_t code = 0;
    for (int k = 0; k < K; ++k) {
      r->freqs_mhz[k] = best[k];
      r->freq_index[k] = best_idx[k];
      code = code * (uint64_t)nc + (uint64_t)best_idx[k];
    }
    r->best_code = code;
  }
  r->decision_freq_mhz = best[0];
out:
  proj_free(&p);
  return rc;
}

int orc_eval_codes(const bs_model_set* m, const bs_mpc_config* cfg, const bs_scheduler_policy* policy,
                   const bs_snapshot* snap, const uint64_t* codes, int n, int32_t* out_feasible,
                   double* out_objective) {
  int rc = mpc_validate(cfg);
  if (rc) return rc;
  double cand[BS_MAX_CAND + 64];
  int nc = orc_ladder_select(cfg->ladder_mhz, cfg->n_ladder, cfg->ladder_N, cand);
  if (nc < 0) return BS_PARAMETER_ERROR;
  projection p;
  rc = project(snap, policy, cfg->horizon_K, &p);
  if (rc) {
    proj_free(&p);
    return rc;
  }
  mpc_ctx c = {m, cfg, snap, &p};
  double a[BS_MAX_K];
  for (int i = 0; i < n && rc == BS_OK; ++i) {
    uint64_t code = codes[i];
    for (int k = p.K - 1; k >= 0; --k) {
      a[k] = cand[code % (uint64_t)nc];
      code /= (uint64_t)nc;
    }
    int ok;
    if ((rc = meets_slo(&c, a, &ok))) break;
    out_feasible[i] = ok;
    rc = tw_power(&c, a, &out_objective[i]);
  }
  proj_free(&p);
  return rc;
}

/* ---- select_decode_freq_ex (dvfs.hpp:274-293) ------------------------------ */

int orc_decode_pick(const bs_model_set* m, const bs_decode_config* cfgs, const bs_decode_query* queries, int n,
                    bs_decode_result* out) {
  for (int i = 0; i < n; ++i) {
    const bs_decode_query* q = &queries[i];
    const bs_decode_config* c = &cfgs[q->cfg_index];
    bs_decode_result* d = &out[i];
    memset(d, 0, sizeof *d);
    /* DecodePolicyConfig::validate, dvfs.hpp:42-47 */
    if (c->tbt_slo_ms <= 0.0) {
      d->status = fail(BS_PARAMETER_ERROR, "decode policy: tbt_slo_ms must be > 0");
      continue;
    }
    if (c->kv_threshold <= 0.0 || c->kv_threshold >= 1.0) {
      d->status = fail(BS_PARAMETER_ERROR, "decode policy: kv_threshold in (0,1)");
      continue;
    }
    if ((d->status = ladder_validate(c->ladder_mhz, c->n_ladder))) continue;
    if (c->margin < 0.0) {
      d->status = fail(BS_PARAMETER_ERROR, "decode policy: margin must be >= 0");
      continue;
    }
    double util = q->kv_capacity_tokens > 0 ? (double)q->kv_used_tokens / (double)q->kv_capacity_tokens : 0.0;
    if (util > c->kv_threshold) { /* controller.hpp:21-23, dvfs.hpp:278-282 */
      d->freq_mhz = c->ladder_mhz[c->n_ladder - 1];
      d->kv_override = 1;
      continue;
    }
    int chosen = 0;
    for (int j = 0; j < c->n_ladder; ++j) {
      d->eval_count += 1;
      double L;
      int rc = query(&m->latency_decode, &q->batch, q->tp, c->ladder_mhz[j], &L, "latency");
      if (rc) {
        d->status = rc;
        break;
      }
      double lat = L * (1.0 + c->margin);
      if (lat <= c->tbt_slo_ms) {
        d->freq_mhz = c->ladder_mhz[j];
        chosen = 1;
        break;
      }
    }
    if (d->status) continue;
    if (!chosen) d->freq_mhz = c->ladder_mhz[c->n_ladder - 1];
  }
  return BS_OK;
}

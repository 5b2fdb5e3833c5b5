// bs_replay.cu — simulate_cluster (simulator.hpp:758-893) with the two-tier
// controllers (dvfs.hpp:302-390) and the steady-state report
// (metrics.hpp:71-156), for a batch of independent scenarios on sm_100a.
//
//   host            validation in the reference's order, phase-1 routing
//                   (route_request by prompt length, simulator.hpp:600-624;
//                   a cheap sequential scan that fixes every prefill
//                   instance's request list, so all device buffers are sized
//                   exactly), packing into one H2D copy.
//   prefill_kernel  one warp per prefill instance.  Lane 0 runs the event
//                   loop of simulate_prefill_instance (simulator.hpp:
//                   278-409); at every controller consultation (batch
//                   boundary, arrival while running) the whole warp runs the
//                   greedy MPC (greedy_warp, bs_greedy_warp.cuh) on the live
//                   queue, read in place from HBM.  Every prediction goes
//                   through per-frequency reduced-axis grids (FastGrid) cached
//                   in shared memory.
//   route_kernel    one thread per scenario: completions merged by
//                   (done, id) across prefill instances and routed to decode
//                   instances (deficit with load 1, simulator.hpp:840-853).
//   decode_kernel   one warp per decode instance: the event loop of
//                   simulate_decode_instance (simulator.hpp:441-578) run
//                   warp-uniformly (every lane holds the scalar state), the
//                   slack-aware pick (dvfs.hpp:274-293) as a warp ladder walk,
//                   and the per-resident token bookkeeping spread over lanes.
//   report_kernel   one CTA per scenario: horizon idle fill, per-phase
//                   clipped energy folds in SimResult record order (stable by
//                   start, instance: a k-way merge), nearest-rank p99 TTFT /
//                   TPOT by radix select, violation and token counts.
//
// FP64 without contraction, reference op order throughout; absent
// optionals are NaN.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "bs_internal.h"
#include "bs_sim.cuh"

using namespace bs;

namespace {

#include "bs_mpc_core.cuh"
#include "bs_greedy_warp.cuh"

constexpr int kReportThreads = 256;
constexpr long long kEventGuard = 4000000000ll;

// --- device layout ---------------------------------------------------------------

struct DRec {  // BatchRecord / IdleRecord essentials
  double start, end, energy;
};
struct DRecX {  // BatchRecord details (logs only)
  long long batch_seq, n_req, sum_len;
  double freq, power;
};
struct DIdlX {  // IdleRecord details (logs only)
  double freq, power;
};
struct DDec {  // DecisionRecord
  double time, freq;
  long long eval;
  int trigger, feasible;
};
struct DDone {  // PrefillDone + the request's global index
  double done;
  long long id;
  long long r;
};
struct DResident {  // decode resident (simulator.hpp:415-420) + token bookkeeping
  long long r, in, out, gen;
  double join, first, maxgap;
};

struct DRCfg {
  DMpcCfg mpc;
  double ladder[BS_MAX_LADDER];
  int n_ladder;
  int controlled;
  double dec_tbt, dec_kv_thr, dec_one_plus_margin;
  double safety_pre, safety_dec;  // controller safety margins
  double pre_fmax, dec_fmax;      // controller max_freq_mhz
  double switch_ms;
  double horizon_opt;
  double span_start;
  double slo_ttft, slo_tpot, slo_pct;
  long long max_batch_tokens, max_batch_requests, kv_cap;
  int chunking;
  int _pad;
};

struct DScen {
  long long r0, n;  // global request range
  double duration;
  double issuance_end;  // max arrival (0 when empty)
  int i0, ni;           // global instance range
  int cfg;
  int n_prefill, n_decode;
  int skip_decode;  // a host-side error the reference raises after phase 1
};

struct DInst {
  int phase, tp, scen, local;  // local = instance id within the scenario
  double base_freq, weight;
  long long list0, list_n;  // prefill: plist range (host-routed); decode: dlist base (scenario r0)
  long long rec0, rec_cap, idl0, idl_cap, dec0, dec_cap;
  long long res0;  // decode: residents scratch offset
};

struct DInstState {
  int status, err_kind;
  long long err_arg, err_arg2;
  double now;
  double f_in;
  int pend, _p;
  double pend_at, pend_f;
  long long n_rec, n_idl, n_dec;
  long long by_trig[3];
  long long n_done;        // prefill: completions written to `done`
  long long d_n;           // decode: routed arrivals in its list
  long long d_off;         // decode: list offset within the scenario's range
  long long overflow;
  int fill_status, fill_err;  // horizon idle fill (simulator.hpp:877-880)
};

struct DReplay {
  DModels sim, ctl;
  const DRCfg* cfgs;
  const DScen* scen;
  const DInst* inst;
  DInstState* st;
  const long long* id;
  const double* arrival;
  const long long* input;
  const long long* output;
  int* d_inst;
  double* pdone;
  double* first_start;
  double* first_tok;
  double* last_tok;
  double* max_tbt;
  long long* ntok;
  const long long* plist;
  DWaiting* W;
  DDone* done;
  long long* dlist;
  double* djoin;
  int* mslot;        // route_kernel scratch (merged order)
  long long* mr;
  DRec* rec;
  DRecX* recx;       // null unless logs
  DRec* idl;
  DIdlX* idlx;       // null unless logs
  DDec* dec;
  DResident* res;
  double* rec_c;     // report scratch: clipped busy energies in merged (start, instance) order
  double* idl_c;     // the same for idle records
};

// --- shared instance machinery ---------------------------------------------------

struct FreqBook {  // simulator.hpp:135-160
  double in_force;
  int pend;
  double at, to;
  __device__ double target() const { return pend ? to : in_force; }
  __device__ void request(double now, double f, double lat) {
    if (f == target()) return;
    if (f == in_force) {
      pend = 0;
    } else {
      pend = 1;
      at = __dadd_rn(now, lat);
      to = f;
    }
  }
  __device__ double next() const { return pend ? at : INFINITY; }
  __device__ void activate() {
    in_force = to;
    pend = 0;
  }
};

enum ErrKind : int {
  kErrLatency = 1,
  kErrPower = 2,
  kErrIdleMissing = 3,
  kErrIdleEmpty = 4,
  kErrAxis = 5,
  kErrKvNeed = 11,
  kErrStalled = 12,
  kErrStarvation = 13,
  kErrGuard = 14,
  kErrScheduler = 15,
  kErrCtl = 16,
};

// The replay kernels are large (tens of thousands of instructions) and their
// warps sit at different points of the event loop, so instruction-cache
// misses dominate their stalls: the predictors, called from many sites, are
// kept as single out-of-line copies (BS_REPLAY_INLINE=1 inlines them).
#ifndef BS_REPLAY_INLINE
#define BS_RP_FN __noinline__
#else
#define BS_RP_FN __forceinline__
#endif

__device__ BS_RP_FN bool predict(const DGrid& g, long long n, long long sum, int tp, double f, double* out,
                                 int* err, int kind) {
  if (g.bad_axis) {
    *err = kErrAxis;
    return false;
  }
  const double v = interp(g, make_query(n, sum, tp, f), nullptr);
  if (!model_value_ok(v)) {
    *err = kind;
    return false;
  }
  *out = v;
  return true;
}

__device__ BS_RP_FN bool predict_fast(const FastGrid& g, long long n, long long sum, double* out, int* err,
                                      int kind) {
  if (g.bad) {
    *err = kErrAxis;
    return false;
  }
  const double v = fast_interp(g, n, sum);
  if (!model_value_ok(v)) {
    *err = kind;
    return false;
  }
  *out = v;
  return true;
}

// predict_fast with the iteration's cached brackets when the slot's grid
// shares them (`shared`), else its own.
__device__ BS_RP_FN bool predict_slot(const FastGrid& g, int shared, const FastBrk& b, long long n, long long sum,
                                      double* out, int* err, int kind) {
  if (g.bad) {
    *err = kErrAxis;
    return false;
  }
  const double v = shared ? fast_corners(g, b) : fast_interp(g, n, sum);
  if (!model_value_ok(v)) {
    *err = kind;
    return false;
  }
  *out = v;
  return true;
}

// predict_idle_power (perfmodel.hpp:274-288) with its two ModelErrors.
__device__ __forceinline__ bool idle_w(const DIdle& m, int tp, double f, double* out, int* err) {
  for (int i = 0; i < m.n_entries; ++i) {
    if (m.tp[i] != tp) continue;
    if (m.n[i] < 1) {
      *err = kErrIdleEmpty;
      return false;
    }
    break;
  }
  if (!idle_power(m, tp, f, out)) {
    *err = kErrIdleMissing;
    return false;
  }
  return true;
}

// Per-instance record writers (capacity-checked; counts keep going so the
// host can size a retry).
struct Writer {
  const DReplay* R;
  const DInst* I;
  long long n_rec, n_idl, n_dec, by_trig[3], overflow;
  int status, err;
  bool leader;  // the one thread that stores (decode warps run the loop on every lane)

  __device__ void init(const DReplay* r, const DInst* i, bool lead = true) {
    R = r;
    I = i;
    leader = lead;
    n_rec = n_idl = n_dec = 0;
    by_trig[0] = by_trig[1] = by_trig[2] = 0;
    overflow = 0;
    status = BS_OK;
    err = 0;
  }
  __device__ void fail(int st, int kind) {
    if (status == BS_OK) {
      status = st;
      err = kind;
    }
  }
  __device__ void batch(double from, double to, double energy, long long seq, long long n, long long sum, double f,
                        double p) {
    if (n_rec < I->rec_cap) {
      if (leader) R->rec[I->rec0 + n_rec] = DRec{from, to, energy};
      if (leader && R->recx) R->recx[I->rec0 + n_rec] = DRecX{seq, n, sum, f, p};
    } else {
      overflow = 1;
    }
    ++n_rec;
  }
  __device__ void idle(double from, double to, double energy, double f, double p) {
    if (n_idl < I->idl_cap) {
      if (leader) R->idl[I->idl0 + n_idl] = DRec{from, to, energy};
      if (leader && R->idlx) R->idlx[I->idl0 + n_idl] = DIdlX{f, p};
    } else {
      overflow = 1;
    }
    ++n_idl;
  }
  __device__ void decision(double t, int trigger, double f, int feasible, long long eval) {
    if (!R->dec) {  // no logs requested: decisions are only counted
    } else if (n_dec < I->dec_cap) {
      if (leader) R->dec[I->dec0 + n_dec] = DDec{t, f, eval, trigger, feasible};
    } else {
      overflow = 1;
    }
    ++n_dec;
    ++by_trig[trigger];
  }
};

__device__ __forceinline__ double energy_j(double p, double from, double to) {  // p * (to - from) / 1000.0
  return __ddiv_rn(__dmul_rn(p, __dsub_rn(to, from)), 1000.0);
}

// Idle power at a frequency: the generic lookup, or a per-slot cache.
struct IdleDirect {
  const DIdle* m;
  int tp;
  __device__ bool operator()(double f, double* p, int* err) const { return idle_w(*m, tp, f, p, err); }
};

// InstanceSim::record_idle (simulator.hpp:205-209).
template <class IdleFn>
__device__ bool record_idle(Writer& w, const IdleFn& idle, const FreqBook& fb, double from, double to) {
  if (to <= from) return true;
  double p;
  int err = 0;
  if (!idle(fb.in_force, &p, &err)) {
    w.fail(BS_MODEL_ERROR, err);
    return false;
  }
  w.idle(from, to, energy_j(p, from, to), fb.in_force, p);
  return true;
}

// InstanceSim::idle_until (simulator.hpp:258-267).
template <class IdleFn>
__device__ bool idle_until(Writer& w, const IdleFn& idle, FreqBook& fb, double& now, double to) {
  while (fb.next() < to) {
    const double t = fb.next();
    if (!record_idle(w, idle, fb, now, t)) return false;
    fb.activate();
    now = t;
  }
  if (!record_idle(w, idle, fb, now, to)) return false;
  now = to;
  return true;
}

// Per-frequency model caches of one instance: every grid the instance
// queries reduced to its (tp, f) (FastGrid: bit-identical, 2^(active axes)
// corners, independent knot loads) plus the idle power, for the frequencies
// the instance can run at or the controller can pick.
struct PreCache {  // views into the prefill CTA's dynamic shared memory (ns slots each)
  int ns;
  double* f;
  double* idle;
  int* idle_err;
  FastGrid *lat, *pw;    // simulator: prefill latency / power
  FastGrid *clat, *cpw;  // controller: prefill latency / power
};

__host__ __device__ inline size_t pre_cache_bytes(int ns) {
  return static_cast<size_t>(ns) * (4 * sizeof(FastGrid) + 2 * sizeof(double) + sizeof(int)) + 16;
}

__device__ inline PreCache pre_cache_at(unsigned char* base, int ns) {
  PreCache c;
  c.ns = ns;
  c.lat = reinterpret_cast<FastGrid*>(base);
  c.pw = c.lat + ns;
  c.clat = c.pw + ns;
  c.cpw = c.clat + ns;
  c.f = reinterpret_cast<double*>(c.cpw + ns);
  c.idle = c.f + ns;
  c.idle_err = reinterpret_cast<int*>(c.idle + ns);
  return c;
}

struct DecSlot {
  double f;
  double idle;
  int idle_err;
  int share;  // bit 0: lat, bit 1: clat use the iteration's latency brackets; bit 2: pw the power brackets
  FastGrid lat, pw, clat;  // simulator latency / power, controller latency (decode)
};

// One decode iteration's brackets (its (n_requests, sum_len) query is fixed
// from start_iteration to the emissions): latency axes and power axes.
struct DecBrk {
  FastBrk lat, pw;
};

__device__ __forceinline__ int find_slot(const double* fs, int ns, double f) {
  for (int i = 0; i < ns; ++i)
    if (fs[i] == f) return i;
  return -1;
}

__device__ void save_state(DInstState* s, const Writer& w, double now, const FreqBook& fb) {
  s->status = w.status;
  s->err_kind = w.err;
  s->now = now;
  s->f_in = fb.in_force;
  s->pend = fb.pend;
  s->pend_at = fb.at;
  s->pend_f = fb.to;
  s->n_rec = w.n_rec;
  s->n_idl = w.n_idl;
  s->n_dec = w.n_dec;
  s->by_trig[0] = w.by_trig[0];
  s->by_trig[1] = w.by_trig[1];
  s->by_trig[2] = w.by_trig[2];
  s->overflow = w.overflow;
}

// --- prefill instances ----------------------------------------------------------

// simulate_prefill_instance (simulator.hpp:278-409) as a resumable thread-0
// state machine: advance() runs events until a controller consultation is
// due (returns 1 with the snapshot in *pr) or the instance is done (0).
struct PrefillSim {
  const DReplay* R;
  const DInst* I;
  const DRCfg* C;
  const PreCache* gc;
  int slot;  // cache slot of the in-force frequency
  Writer w;
  FreqBook fb;
  double now;
  long long batch_seq;
  int fired;
  double deadline;
  // queue = list [head, arr); the head's remaining tokens in head_rem
  long long arr, head, head_rem;
  // running batch: list members [mb, me), last one partial when `partial`
  int active, partial;
  double started, seg_start, wr, decided, L;
  long long fn, fsum, mb, me;
  long long n_done;
  long long events;
  int resume;  // 1: finish start_batch, 2: apply an arrival decision

  __device__ double arrival_of(long long i) const { return R->arrival[R->plist[I->list0 + i]]; }
  __device__ long long input_of(long long i) const { return R->input[R->plist[I->list0 + i]]; }

  __device__ void init(const DReplay* r, const DInst* i, const DRCfg* c, const PreCache* cache) {
    R = r;
    I = i;
    C = c;
    gc = cache;
    slot = find_slot(gc->f, gc->ns, i->base_freq);
    w.init(r, i);
    fb.in_force = i->base_freq;
    fb.pend = 0;
    fb.at = fb.to = 0.0;
    now = 0.0;
    batch_seq = -1;
    fired = 0;
    deadline = INFINITY;
    arr = head = head_rem = 0;
    active = partial = 0;
    started = seg_start = wr = decided = L = 0.0;
    fn = fsum = mb = me = 0;
    n_done = 0;
    events = 0;
    resume = 0;
  }

  __device__ bool idle(double f, double* p, int* err) const {
    const int k = find_slot(gc->f, gc->ns, f);
    if (k < 0) return idle_w(R->sim.idle, I->tp, f, p, err);
    *p = gc->idle[k];
    *err = gc->idle_err[k];
    return gc->idle_err[k] == 0;
  }
  struct IdleCached {
    const PrefillSim* s;
    __device__ bool operator()(double f, double* p, int* err) const { return s->idle(f, p, err); }
  };

  __device__ void activate() {
    fb.activate();
    slot = find_slot(gc->f, gc->ns, fb.in_force);
  }

  __device__ bool exec_latency() {  // InstanceSim::exec_latency at the in-force frequency
    int err = 0;
    if (slot >= 0 ? !predict_fast(gc->lat[slot], fn, fsum, &L, &err, kErrLatency)
                  : !predict(R->sim.grid[0], fn, fsum, I->tp, fb.in_force, &L, &err, kErrLatency)) {
      w.fail(BS_MODEL_ERROR, err);
      return false;
    }
    return true;
  }

  // InstanceSim::arm_safety (simulator.hpp:230-235).
  __device__ bool arm_safety(double at, double f, double work_fraction) {
    if (!C->controlled) return true;
    double pl;
    int err = 0;
    const int k = find_slot(gc->f, gc->ns, f);
    if (k >= 0 ? !predict_fast(gc->clat[k], fn, fsum, &pl, &err, kErrLatency)
               : !predict(R->ctl.grid[0], fn, fsum, I->tp, f, &pl, &err, kErrLatency)) {
      w.fail(BS_MODEL_ERROR, err);
      return false;
    }
    const double pred = __dmul_rn(work_fraction, pl);
    const double sw = f != fb.in_force ? C->switch_ms : 0.0;
    deadline = __dadd_rn(at, __dmul_rn(__dadd_rn(pred, sw), __dadd_rn(1.0, C->safety_pre)));
    return true;
  }

  // close_segment (simulator.hpp:331-335) with record_segment (213-228).
  __device__ bool close_segment(double to) {
    if (to > seg_start) {
      double p;
      int err = 0;
      if (slot >= 0 ? !predict_fast(gc->pw[slot], fn, fsum, &p, &err, kErrPower)
                    : !predict(R->sim.grid[2], fn, fsum, I->tp, fb.in_force, &p, &err, kErrPower)) {
        w.fail(BS_MODEL_ERROR, err);
        return false;
      }
      w.batch(seg_start, to, energy_j(p, seg_start, to), batch_seq, fn, fsum, fb.in_force, p);
    }
    wr = __dsub_rn(wr, __ddiv_rn(__dsub_rn(to, seg_start), L));
    seg_start = to;
    return true;
  }

  __device__ void push_arrival() {  // queue.push_back (simulator.hpp:352, 401)
    if (head == arr) head_rem = input_of(arr);
    ++arr;
  }

  // build_snapshot (simulator.hpp:291-313) -> the MPC problem.
  __device__ void snapshot(double at, DProblem* pr) {
    pr->now = at;
    pr->cur_freq = fb.in_force;
    pr->target_freq = fb.target();
    pr->tp = I->tp;
    pr->cfg = 0;
    pr->n_wait = static_cast<int>(arr - head);
    pr->wait_off = I->list0 + head;
    if (head < arr) R->W[I->list0 + head].remaining = head_rem;
    pr->run_off = 0;
    pr->run_active = active;
    pr->n_run = 0;
    if (active) {
      const double live = __dsub_rn(wr, __ddiv_rn(__dsub_rn(at, seg_start), L));
      pr->run_wr = live > 0.0 ? live : 0.0;  // std::max(0.0, live)
      pr->run_n = fn;
      pr->run_sum = fsum;
      pr->n_run = -1;
      const long long ncomp = (me - mb) - (partial ? 1 : 0);
      pr->run_ncomp = static_cast<int>(ncomp);
      pr->run_minarr = ncomp > 0 ? arrival_of(mb) : INFINITY;  // list is in arrival order
    } else {
      pr->run_wr = 0.0;
      pr->run_n = 0;
      pr->run_sum = 0;
    }
  }

  // start_batch after the boundary decision (simulator.hpp:315-329, 336-340).
  __device__ bool form_and_start(double at, const DMpcOut* d) {
    decided = fb.target();
    if (C->controlled) {
      if (d->status != BS_OK) {
        w.fail(d->status, kErrCtl);
        return false;
      }
      const double f = decision_freq(d, fb.target());
      w.decision(at, 0, f, d->feasible, d->eval_count);
      fb.request(at, f, C->switch_ms);
      decided = f;
    }
    // form_prefill_batch (scheduler.hpp:40-66) over [head, arr)
    long long tokens = 0, npick = 0, sum = 0;
    partial = 0;
    long long end = head, rem_after = 0;
    for (long long i = head; i < arr; ++i) {
      if (npick >= C->max_batch_requests) break;
      const long long rem = i == head ? head_rem : input_of(i);
      if (rem <= 0) {
        w.fail(BS_SIMULATION_ERROR, kErrScheduler);
        return false;
      }
      if (C->chunking) {
        const long long room = C->max_batch_tokens - tokens;
        if (room <= 0) break;
        const long long take = rem < room ? rem : room;
        ++npick;
        sum += take;
        tokens += take;
        end = i + 1;
        if (take < rem) {
          partial = 1;
          rem_after = rem - take;
          break;
        }
      } else {
        if (rem > C->max_batch_tokens) {
          if (npick == 0) {
            ++npick;
            sum += rem;
            end = i + 1;
          }
          break;
        }
        if (tokens + rem > C->max_batch_tokens) break;
        ++npick;
        sum += rem;
        tokens += rem;
        end = i + 1;
      }
    }
    active = 1;
    started = at;
    seg_start = at;
    wr = 1.0;
    fn = npick;
    fsum = sum;
    mb = head;
    me = end;
    head = partial ? end - 1 : end;
    if (partial) {
      head_rem = rem_after;
    } else if (head < arr) {
      head_rem = input_of(head);
    }
    ++batch_seq;
    fired = 0;
    if (!arm_safety(at, decided, 1.0)) return false;
    return exec_latency();
  }

  __device__ double decision_freq(const DMpcOut* d, double target) const {
    // PrefillMpcController::run (dvfs.hpp:326-333)
    if (d->K == 0) return target > 0 ? target : C->pre_fmax;
    return C->mpc.cand[d->idx[0]];
  }

  // The arrival trigger's tail (simulator.hpp:400-407).
  __device__ bool apply_arrival(const DMpcOut* d, double live_wr) {
    if (d->status != BS_OK) {
      w.fail(d->status, kErrCtl);
      return false;
    }
    const double f = decision_freq(d, fb.target());
    w.decision(now, 1, f, d->feasible, d->eval_count);
    fb.request(now, f, C->switch_ms);
    decided = f;
    return arm_safety(now, f, live_wr);
  }

  __device__ void complete(double t_done) {  // PrefillDone for every completing member, (done, id) order
    const long long full_end = partial ? me - 1 : me;
    for (long long i = mb; i < full_end; ++i) {
      const long long r = R->plist[I->list0 + i];
      const long long id = R->id[r];
      R->pdone[r] = t_done;
      long long j = I->list0 + n_done;
      // insertion by (done, id): a batch's members share t_done
      while (j > I->list0 && (R->done[j - 1].done > t_done || (R->done[j - 1].done == t_done && R->done[j - 1].id > id))) {
        R->done[j] = R->done[j - 1];
        --j;
      }
      R->done[j] = DDone{t_done, id, r};
      ++n_done;
    }
  }

  __device__ int advance(const DMpcOut* d, DProblem* pr) {
    if (resume == 1) {
      resume = 0;
      if (!form_and_start(now, d)) return 0;
    } else if (resume == 2) {
      resume = 0;
      if (!apply_arrival(d, pr->run_wr)) return 0;
    }
    const long long n = I->list_n;
    for (;;) {
      if (++events > kEventGuard) {
        w.fail(BS_SIMULATION_ERROR, kErrGuard);
        return 0;
      }
      if (!active && head < arr) {
        while (arr < n && arrival_of(arr) <= now) push_arrival();  // simulator.hpp:350-353
        if (C->controlled) {
          snapshot(now, pr);
          resume = 1;
          return 1;
        }
        if (!form_and_start(now, nullptr)) return 0;
        continue;
      }
      if (!active && head >= arr && arr >= n) return 0;  // loop condition (simulator.hpp:347)
      const double t_arr = arr < n ? fmax(arrival_of(arr), now) : INFINITY;
      const double t_sw = fb.next();
      double t_done = INFINITY, t_safety = INFINITY;
      if (active) {
        t_done = __dadd_rn(seg_start, __dmul_rn(wr, L));
        if (C->controlled && !fired) t_safety = deadline;
      }
      if (active && t_done <= t_sw && t_done <= t_safety && t_done <= t_arr) {
        if (!close_segment(t_done)) return 0;
        complete(t_done);
        active = 0;
        deadline = INFINITY;
        now = t_done;
        continue;
      }
      if (t_sw <= t_safety && t_sw <= t_arr) {
        if (active) {
          if (!close_segment(t_sw)) return 0;
        } else if (!record_idle(w, IdleCached{this}, fb, now, t_sw)) {
          return 0;
        }
        activate();
        now = t_sw;
        if (active && !exec_latency()) return 0;
        continue;
      }
      if (active && t_safety <= t_arr) {
        // fire_safety (simulator.hpp:238-245) / apply_safety_overrides (controller.hpp:140-148)
        const double projected = __dsub_rn(__dadd_rn(seg_start, __dmul_rn(wr, L)), started);
        const double one_m = __dadd_rn(1.0, C->safety_pre);
        const double pred = __ddiv_rn(__dsub_rn(deadline, started), one_m);
        if (projected > __dmul_rn(pred, one_m)) {
          fired = 1;
          w.decision(t_safety, 2, C->pre_fmax, 1, 0);
          fb.request(t_safety, C->pre_fmax, C->switch_ms);
        } else {  // the reference would re-fire forever; report instead of hanging
          w.fail(BS_SIMULATION_ERROR, kErrGuard);
          return 0;
        }
        now = t_safety;
        continue;
      }
      if (t_arr == INFINITY) return 0;
      if (!active && !record_idle(w, IdleCached{this}, fb, now, t_arr)) return 0;
      now = fmax(now, t_arr);
      push_arrival();
      if (active && C->controlled && !fired) {
        snapshot(now, pr);
        resume = 2;
        return 1;
      }
    }
  }
};

// One warp per prefill instance: lane 0 runs the event loop, the whole warp
// runs every controller consultation (greedy_warp, bs_greedy_warp.cuh).
// Per-warp dynamic shared memory: the greedy state and snapshot, the
// per-frequency model caches and the compact (k, f) tables.
struct PreWarp {
  WGreedyShared G;
  DProblem pr;
  DMpcOut out;
  PrefillSim sim;  // lane 0's event-loop state, kept out of the register file
};

constexpr int kPrefillWarps = 4;
#ifndef BS_PREFILL_MINB
#define BS_PREFILL_MINB 4  // resident CTAs per SM the prefill kernel is register-budgeted for
#endif

__host__ __device__ inline size_t pre_warp_bytes(int max_ns, int max_h, int max_nc) {
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  return a16(sizeof(PreWarp)) + a16(pre_cache_bytes(max_ns)) + a16(8 * wtable_doubles(max_h, max_nc));
}

__global__ void __launch_bounds__(kPrefillWarps * 32, BS_PREFILL_MINB) prefill_kernel(DReplay R, const int* pre_ids, int n_pre,
                                                                    int max_ns, int max_h, int max_nc) {
  extern __shared__ __align__(16) unsigned char pre_dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int wid = blockIdx.x * kPrefillWarps + wib;
  if (wid >= n_pre) return;  // whole warps only
  auto a16 = [](size_t x) { return (x + 15) / 16 * 16; };
  unsigned char* base = pre_dsm + static_cast<size_t>(wib) * pre_warp_bytes(max_ns, max_h, max_nc);
  PreWarp& S = *reinterpret_cast<PreWarp*>(base);
  const int gi = pre_ids[wid];
  const DInst I = R.inst[gi];
  const DRCfg* C = &R.cfgs[R.scen[I.scen].cfg];
  // cache slots [0, nc): the MPC candidates (indexed like the tables' f); slot nc: base
  const int nc = C->controlled ? C->mpc.nc : 0;
  const int ns = nc + 1;
  const PreCache G = pre_cache_at(base + a16(sizeof(PreWarp)), ns);
  double* tab = reinterpret_cast<double*>(base + a16(sizeof(PreWarp)) + a16(pre_cache_bytes(max_ns)));
  if (lane == 0 && C->controlled) wtables_bind(S.G.T, tab, C->mpc.horizon, C->mpc.nc);
  for (int t = lane; t < ns; t += 32) {
    const double f = t < nc ? C->mpc.cand[t] : I.base_freq;
    G.f[t] = f;
    int err = 0;
    double p = 0.0;
    G.idle_err[t] = idle_w(R.sim.idle, I.tp, f, &p, &err) ? 0 : err;
    G.idle[t] = p;
  }
  for (int t = lane; t < 4 * ns; t += 32) {
    const int g = t / ns, k = t - g * ns;
    const double f = k < nc ? C->mpc.cand[k] : I.base_freq;
    const FastGrid fg = fast_grid(g < 2 ? R.sim.grid[g == 0 ? 0 : 2] : R.ctl.grid[g == 2 ? 0 : 2], I.tp, f);
    (g == 0 ? G.lat : g == 1 ? G.pw : g == 2 ? G.clat : G.cpw)[k] = fg;
  }
  __syncwarp();
  bool share = true;  // every candidate's controller grids bracket like candidate 0's
  for (int f = 1; f < nc; ++f)
    share = share && fast_same_brackets(G.clat[0], G.clat[f]) && fast_same_brackets(G.cpw[0], G.cpw[f]);
  PrefillSim& sim = S.sim;
  if (lane == 0) sim.init(&R, &I, C, &G);
  for (;;) {
    int cmd = 0;
    if (lane == 0) cmd = sim.advance(&S.out, &S.pr);
    cmd = __shfl_sync(0xffffffffu, cmd, 0);
    if (cmd == 0) break;
    greedy_warp(R.ctl, S.pr, C->mpc, R.W + S.pr.wait_off, nullptr, S.G, &S.out, nullptr, G.clat, G.cpw, share);
  }
  if (lane == 0) {
    DInstState* st = &R.st[gi];
    save_state(st, sim.w, sim.now, sim.fb);
    st->n_done = sim.n_done;
  }
}

// --- phase 2 routing ----------------------------------------------------------------

constexpr int kMaxInstances = 256;  // per scenario (checked on the host)

__device__ bool phase1_ok(const DReplay& R, const DScen& sc) {
  for (int i = 0; i < sc.ni; ++i) {
    const int g = sc.i0 + i;
    if (R.inst[g].phase == BS_PHASE_PREFILL && R.st[g].status != BS_OK) return false;
  }
  return true;
}

// One thread per scenario: completions of all prefill instances merged by
// (done, id) (simulator.hpp:831-833), then route_request with load 1.0 over
// the decode instances (simulator.hpp:836-853) into per-instance FIFO lists.
__global__ void route_kernel(DReplay R, int n_scen) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scen) return;
  const DScen sc = R.scen[s];
  if (sc.skip_decode || !phase1_ok(R, sc)) return;  // the reference threw before phase 2
  long long pos[kMaxInstances];
  int pre[kMaxInstances], dcd[kMaxInstances];
  double assigned[kMaxInstances];
  int np = 0, nd = 0;
  for (int i = 0; i < sc.ni; ++i) {
    const int g = sc.i0 + i;
    if (R.inst[g].phase == BS_PHASE_PREFILL) {
      pos[np] = 0;
      pre[np++] = g;
    } else {
      assigned[nd] = 0.0;
      dcd[nd++] = g;
    }
  }
  double total = 0.0;
  long long m = 0;
  for (;;) {
    int best = -1;
    DDone bd{};
    for (int p = 0; p < np; ++p) {
      if (pos[p] >= R.st[pre[p]].n_done) continue;
      const DDone d = R.done[R.inst[pre[p]].list0 + pos[p]];
      if (best < 0 || d.done < bd.done || (d.done == bd.done && d.id < bd.id)) {
        best = p;
        bd = d;
      }
    }
    if (best < 0) break;
    ++pos[best];
    // route_request (simulator.hpp:610-624), decode load 1.0
    total = __dadd_rn(total, 1.0);
    int slot = 0;
    double best_def = -INFINITY;
    for (int j = 0; j < nd; ++j) {
      const double def = __dsub_rn(__dmul_rn(R.inst[dcd[j]].weight, total), assigned[j]);
      if (def > best_def) {
        best_def = def;
        slot = j;
      }
    }
    assigned[slot] = __dadd_rn(assigned[slot], 1.0);
    R.mslot[sc.r0 + m] = slot;
    R.mr[sc.r0 + m] = bd.r;
    ++m;
  }
  long long cnt[kMaxInstances];
  for (int j = 0; j < nd; ++j) cnt[j] = 0;
  for (long long k = 0; k < m; ++k) ++cnt[R.mslot[sc.r0 + k]];
  long long off = 0;
  for (int j = 0; j < nd; ++j) {
    R.st[dcd[j]].d_n = cnt[j];
    R.st[dcd[j]].d_off = off;
    const long long c = cnt[j];
    cnt[j] = off;
    off += c;
  }
  for (long long k = 0; k < m; ++k) {
    const int j = R.mslot[sc.r0 + k];
    const long long r = R.mr[sc.r0 + k];
    const long long at = sc.r0 + cnt[j]++;
    R.dlist[at] = r;
    R.djoin[at] = R.pdone[r];
    R.d_inst[r] = R.inst[dcd[j]].local;
  }
}

// --- decode instances -----------------------------------------------------------------

#ifndef BS_DECODE_MINB
#define BS_DECODE_MINB 4
#endif

// select_decode_freq_ex (dvfs.hpp:274-293) as a warp ladder walk (lane j
// evaluates rung j of each 32-rung chunk; a ballot finds where the
// reference's ascending walk stops).  Warp-uniform; false on ModelError.
__device__ bool decode_pick(const DReplay& R, const DRCfg* C, const DecSlot* slots, const DecBrk* B, long long n,
                            long long sum, int tp, long long cap, long long used, double* f, long long* eval,
                            int* err) {
  const int lane = threadIdx.x & 31;
  const double util = cap > 0 ? __ddiv_rn(static_cast<double>(used), static_cast<double>(cap)) : 0.0;
  *f = C->ladder[C->n_ladder - 1];
  *eval = 0;
  if (util > C->dec_kv_thr) return true;  // KV override (dvfs.hpp:278-282)
  const DGrid& g = R.ctl.grid[1];
  if (g.bad_axis) {
    *eval = 1;
    *err = kErrAxis;
    return false;
  }
  for (int j0 = 0; j0 < C->n_ladder; j0 += 32) {
    const int j = j0 + lane;
    bool fits = false, bad = false;
    if (j < C->n_ladder) {
      const double v = (slots[j].share & 2) ? fast_corners(slots[j].clat, B->lat)
                                            : fast_interp(slots[j].clat, n, sum);  // slot j = rung j
      bad = !model_value_ok(v);
      fits = !bad && __dmul_rn(v, C->dec_one_plus_margin) <= C->dec_tbt;  // dvfs.hpp:285-286
    }
    const unsigned stop = __ballot_sync(0xffffffffu, fits || bad);
    if (stop) {
      const int first = __ffs(stop) - 1;
      *eval = j0 + first + 1;
      const unsigned badm = __ballot_sync(0xffffffffu, bad);
      if ((badm >> first) & 1u) {
        *err = kErrLatency;
        return false;
      }
      *f = C->ladder[j0 + first];
      return true;
    }
  }
  *eval = C->n_ladder;
  return true;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// simulate_decode_instance (simulator.hpp:441-578), one warp per instance.
// Every lane runs the scalar event loop (identical state on all lanes, so
// control flow is warp-uniform); lane 0 stores records; residents are spread
// over lanes for the per-iteration emissions (every resident emits one token
// at every iteration end, simulator.hpp:544-557), whose per-request
// reductions (first/last token, worst gap) are kept in the resident entry.
__global__ void __launch_bounds__(128, BS_DECODE_MINB) decode_kernel(DReplay R, const int* dec_ids, int n_dec, int max_slots) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= n_dec) return;
  const int gi = dec_ids[wid];
  const DInst I = R.inst[gi];
  const DScen sc = R.scen[I.scen];
  if (sc.skip_decode || !phase1_ok(R, sc)) return;
  const DRCfg* C = &R.cfgs[sc.cfg];
  DInstState* S = &R.st[gi];
  const long long n = S->d_n;
  const long long base = sc.r0 + S->d_off;
  DResident* res = R.res + I.res0;
  const DGrid& lat_g = R.sim.grid[1];
  const DGrid& pow_g = R.sim.grid[3];
  // per-frequency caches: slots [0, n_ladder) = the decode ladder, slot n_ladder = base
  DecSlot* slots = reinterpret_cast<DecSlot*>(dsm) + (threadIdx.x >> 5) * max_slots;
  DecBrk* brk = reinterpret_cast<DecBrk*>(reinterpret_cast<DecSlot*>(dsm) + 4 * max_slots) + (threadIdx.x >> 5);
  const int nl = C->controlled ? C->n_ladder : 0;
  const int ns = nl + 1;
  for (int t = lane; t < ns; t += 32) {
    const double f = t < nl ? C->ladder[t] : I.base_freq;
    slots[t].f = f;
    int err = 0;
    double p = 0.0;
    slots[t].idle_err = idle_w(R.sim.idle, I.tp, f, &p, &err) ? 0 : err;
    slots[t].idle = p;
  }
  for (int t = lane; t < 3 * ns; t += 32) {
    const int g = t / ns, k = t - g * ns;
    const double f = k < nl ? C->ladder[k] : I.base_freq;
    const FastGrid fg = fast_grid(g == 0 ? R.sim.grid[1] : g == 1 ? R.sim.grid[3] : R.ctl.grid[1], I.tp, f);
    if (g == 0) slots[k].lat = fg;
    else if (g == 1) slots[k].pw = fg;
    else slots[k].clat = fg;
  }
  __syncwarp();
  // bracket sharing against slot 0 (the reference of the iteration's brackets)
  for (int t = lane; t < ns; t += 32)
    slots[t].share = (fast_same_axes(slots[t].lat, slots[0].lat) ? 1 : 0) |
                     (fast_same_axes(slots[t].clat, slots[0].lat) ? 2 : 0) |
                     (fast_same_axes(slots[t].pw, slots[0].pw) ? 4 : 0);
  __syncwarp();
  auto slot_of = [&](double f) {
    for (int i = 0; i < ns; ++i)
      if (slots[i].f == f) return i;
    return -1;
  };
  struct IdleSlots {
    const DecSlot* sl;
    int ns;
    const DIdle* m;
    int tp;
    __device__ bool operator()(double f, double* p, int* err) const {
      for (int i = 0; i < ns; ++i)
        if (sl[i].f == f) {
          *p = sl[i].idle;
          *err = sl[i].idle_err;
          return sl[i].idle_err == 0;
        }
      return idle_w(*m, tp, f, p, err);
    }
  };
  const IdleSlots idle_fn{slots, ns, &R.sim.idle, I.tp};

  Writer w;
  w.init(&R, &I, lane == 0);
  FreqBook fb;
  fb.in_force = I.base_freq;
  fb.pend = 0;
  fb.at = fb.to = 0.0;
  double now = 0.0, started = 0.0, seg_start = 0.0, wr = 0.0, L = 0.0, deadline = INFINITY;
  long long batch_seq = -1, arr = 0, whead = 0, sum_ctx = 0, reserved = 0, fn = 0, fsum = 0, events = 0;
  int n_res = 0, active = 0, fired = 0;
  double last_end = 0.0;

  int slot = slot_of(fb.in_force);
  auto exec_latency = [&]() -> bool {
    int err = 0;
    if (slot >= 0 ? !predict_slot(slots[slot].lat, slots[slot].share & 1, brk->lat, fn, fsum, &L, &err, kErrLatency)
                  : !predict(lat_g, fn, fsum, I.tp, fb.in_force, &L, &err, kErrLatency)) {
      w.fail(BS_MODEL_ERROR, err);
      return false;
    }
    return true;
  };
  auto close_segment = [&](double to) -> bool {  // simulator.hpp:494-498
    if (to > seg_start) {
      double p;
      int err = 0;
      if (slot >= 0 ? !predict_slot(slots[slot].pw, slots[slot].share & 4, brk->pw, fn, fsum, &p, &err, kErrPower)
                    : !predict(pow_g, fn, fsum, I.tp, fb.in_force, &p, &err, kErrPower)) {
        w.fail(BS_MODEL_ERROR, err);
        return false;
      }
      w.batch(seg_start, to, energy_j(p, seg_start, to), batch_seq, fn, fsum, fb.in_force, p);
    }
    wr = __dsub_rn(wr, __ddiv_rn(__dsub_rn(to, seg_start), L));
    seg_start = to;
    return true;
  };

  while (w.status == BS_OK && (arr < n || whead < arr || n_res > 0)) {
    if (++events > kEventGuard) {
      w.fail(BS_SIMULATION_ERROR, kErrGuard);
      break;
    }
    if (!active) {
      while (arr < n && R.djoin[base + arr] <= now) ++arr;  // simulator.hpp:516-518
      // admit (simulator.hpp:455-470)
      while (whead < arr) {
        const long long r = R.dlist[base + whead];
        const long long in = R.input[r], out = R.output[r];
        const long long need = in + out;
        if (need > C->kv_cap) {
          w.fail(BS_SIMULATION_ERROR, kErrKvNeed);
          if (lane == 0) {
            S->err_arg = R.id[r];
            S->err_arg2 = need;
          }
          break;
        }
        if (n_res >= C->max_batch_requests) break;
        if (reserved + need > C->kv_cap) break;
        if (lane == 0) {
          res[n_res] = DResident{r, in, out, 0, R.djoin[base + whead], 0.0, 0.0};
          R.first_start[r] = now;
        }
        ++n_res;
        reserved += need;
        sum_ctx += in;
        ++whead;
      }
      __syncwarp();
      if (w.status != BS_OK) break;
      if (n_res == 0) {
        if (arr >= n && whead >= arr) break;
        if (whead < arr) {
          w.fail(BS_SIMULATION_ERROR, kErrStalled);
          break;
        }
        const double t_next = fmax(R.djoin[base + arr], now);
        if (!idle_until(w, idle_fn, fb, now, t_next)) { slot = slot_of(fb.in_force); break; }
        slot = slot_of(fb.in_force);
        continue;
      }
      // start_iteration (simulator.hpp:472-492)
      fn = n_res;
      fsum = sum_ctx;
      if (!slots[0].lat.bad) warp_brackets(slots[0].lat, fn, fsum, &brk->lat);
      if (!slots[0].pw.bad) warp_brackets(slots[0].pw, fn, fsum, &brk->pw);
      active = 1;
      started = now;
      seg_start = now;
      wr = 1.0;
      double decided = fb.target();
      if (C->controlled) {
        double f;
        long long eval;
        int err = 0;
        if (!decode_pick(R, C, slots, brk, fn, fsum, I.tp, C->kv_cap, sum_ctx, &f, &eval, &err)) {
          w.fail(BS_MODEL_ERROR, err);
          break;
        }
        w.decision(now, 0, f, 1, eval);
        fb.request(now, f, C->switch_ms);
        decided = f;
      }
      ++batch_seq;
      fired = 0;
      if (C->controlled) {  // arm_safety (simulator.hpp:230-235)
        double pl;
        int err = 0;
        const int ks = slot_of(decided);
        if (ks >= 0 ? !predict_slot(slots[ks].clat, slots[ks].share & 2, brk->lat, fn, fsum, &pl, &err, kErrLatency)
                    : !predict(R.ctl.grid[1], fn, fsum, I.tp, decided, &pl, &err, kErrLatency)) {
          w.fail(BS_MODEL_ERROR, err);
          break;
        }
        const double sw = decided != fb.in_force ? C->switch_ms : 0.0;
        deadline = __dadd_rn(now, __dmul_rn(__dadd_rn(__dmul_rn(1.0, pl), sw), __dadd_rn(1.0, C->safety_dec)));
      }
      if (!exec_latency()) break;
      continue;
    }
    const double t_arr = arr < n ? fmax(R.djoin[base + arr], now) : INFINITY;
    const double t_sw = fb.next();
    const double t_done = __dadd_rn(seg_start, __dmul_rn(wr, L));
    const double t_safety = C->controlled && !fired ? deadline : INFINITY;
    if (t_done <= t_sw && t_done <= t_safety && t_done <= t_arr) {
      if (!close_segment(t_done)) break;
      // every resident emits at t_done (simulator.hpp:544-557); retire at output_len
      const double gap = __dsub_rn(t_done, last_end);
      long long freed = 0;
      int kept = 0;
      for (int c0 = 0; c0 < n_res; c0 += 32) {
        const int j = c0 + lane;
        DResident e;
        bool keep = false;
        if (j < n_res) {
          e = res[j];
          e.gen += 1;
          if (e.gen == 1) {
            e.first = t_done;
            e.maxgap = __dsub_rn(t_done, e.join);  // first gap from the decode join (simulator.hpp:81-89)
          } else {
            e.maxgap = e.maxgap < gap ? gap : e.maxgap;  // std::max(worst, gap)
          }
          if (e.gen >= e.out) {
            R.first_tok[e.r] = e.first;
            R.last_tok[e.r] = t_done;
            R.max_tbt[e.r] = e.maxgap;
            R.ntok[e.r] = e.gen;
            freed += e.in + e.out;
          } else {
            keep = true;
          }
        }
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) res[kept + __popc(km & ((1u << lane) - 1u))] = e;
        kept += __popc(km);
      }
      __syncwarp();
      freed = warp_sum_ll(freed);
      sum_ctx += n_res;  // every resident generated one token
      sum_ctx -= freed;
      reserved -= freed;
      n_res = kept;
      last_end = t_done;
      active = 0;
      deadline = INFINITY;
      now = t_done;
      continue;
    }
    if (t_sw <= t_safety && t_sw <= t_arr) {
      if (!close_segment(t_sw)) break;
      fb.activate();
      slot = slot_of(fb.in_force);
      now = t_sw;
      if (!exec_latency()) break;
      continue;
    }
    if (t_safety <= t_arr) {  // fire_safety (simulator.hpp:238-245)
      const double projected = __dsub_rn(__dadd_rn(seg_start, __dmul_rn(wr, L)), started);
      const double one_m = __dadd_rn(1.0, C->safety_dec);
      const double pred = __ddiv_rn(__dsub_rn(deadline, started), one_m);
      if (projected > __dmul_rn(pred, one_m)) {
        fired = 1;
        w.decision(t_safety, 2, C->dec_fmax, 1, 0);
        fb.request(t_safety, C->dec_fmax, C->switch_ms);
      } else {
        w.fail(BS_SIMULATION_ERROR, kErrGuard);
        break;
      }
      now = t_safety;
      continue;
    }
    if (t_arr == INFINITY) {
      w.fail(BS_SIMULATION_ERROR, kErrStarvation);
      break;
    }
    ++arr;  // waiting.push_back (simulator.hpp:575)
    now = t_arr;
  }
  if (lane == 0) save_state(S, w, now, fb);
}

// --- report ---------------------------------------------------------------------------

// k-th smallest (0-based) of the non-negative doubles produced by `val` over
// the scenario's requests (bit patterns order like the values): 8 passes of
// 8-bit radix select with a block-wide histogram.
template <class F>
__device__ double block_select(long long r0, long long n, long long k, F val, unsigned* hist) {
  unsigned long long prefix = 0, mask = 0;
  __shared__ long long s_k;
  __shared__ unsigned long long s_prefix;
  if (threadIdx.x == 0) s_k = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      double v;
      if (!val(r0 + i, &v)) continue;
      const unsigned long long key = static_cast<unsigned long long>(__double_as_longlong(v));
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long kk = s_k;
      int b = 0;
      for (; b < 255; ++b) {
        if (kk < hist[b]) break;
        kk -= hist[b];
      }
      s_k = kk;
      s_prefix = prefix | (static_cast<unsigned long long>(b) << shift);
    }
    __syncthreads();
    prefix = s_prefix;
    mask |= 0xffull << shift;
  }
  return __longlong_as_double(static_cast<long long>(prefix));
}

// nearest_rank (metrics.hpp:18-26): rank = clamp(ceil(p n), 1, n).
__device__ __forceinline__ long long nearest_rank_index(double p, long long n) {
  long long rank = static_cast<long long>(ceil(__dmul_rn(p, static_cast<double>(n))));
  rank = rank < 1 ? 1 : rank;
  rank = rank > n ? n : rank;
  return rank - 1;
}

// TrimmedResult::busy/idle_energy_j (metrics.hpp:38-56) folds each phase's
// records in SimResult order: stable by (start, instance) across the phase's
// instances (each instance's records are in start order), clipped to the
// span.  The order is data-independent of the sums, so the block first
// scatters every record's clipped energy to its merged position (its own
// index plus, per other instance of the phase, a binary-search count of the
// records that precede it: start <= s for lower instance ids, start < s for
// higher), then one thread per fold adds the contiguous array in order.
__device__ __forceinline__ double clip_energy(const DRec& r, double s0, double s1) {  // metrics.hpp:60-66
  const double a = fmax(r.start, s0);
  const double b = fmin(r.end, s1);
  return b <= a ? 0.0 : __ddiv_rn(__dmul_rn(r.energy, __dsub_rn(b, a)), __dsub_rn(r.end, r.start));
}

__device__ void scatter_phase(const DReplay& R, const DScen& sc, int phase, bool idle, double* dst, double s0,
                              double s1) {
  for (int a = 0; a < sc.ni; ++a) {
    const int ga = sc.i0 + a;
    const DInst& Ia = R.inst[ga];
    if (Ia.phase != phase) continue;
    const long long na = idle ? R.st[ga].n_idl : R.st[ga].n_rec;
    const DRec* la = idle ? R.idl + Ia.idl0 : R.rec + Ia.rec0;
    for (long long j = threadIdx.x; j < na; j += blockDim.x) {
      const DRec r = la[j];
      long long pos = j;
      for (int b = 0; b < sc.ni; ++b) {
        const int gb = sc.i0 + b;
        const DInst& Ib = R.inst[gb];
        if (b == a || Ib.phase != phase) continue;
        const DRec* lb = idle ? R.idl + Ib.idl0 : R.rec + Ib.rec0;
        long long lo = 0, hi = idle ? R.st[gb].n_idl : R.st[gb].n_rec;
        while (lo < hi) {
          const long long mid = lo + (hi - lo) / 2;
          const double t = lb[mid].start;
          if (b < a ? !(r.start < t) : t < r.start) lo = mid + 1;
          else hi = mid;
        }
        pos += lo;
      }
      dst[pos] = clip_energy(r, s0, s1);
    }
  }
}

__device__ double fold_in_order(const double* c, long long n) {
  double e = 0.0;
  long long i = 0;
  for (; i + 8 <= n; i += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = c[i + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) e = __dadd_rn(e, v[u]);
  }
  for (; i < n; ++i) e = __dadd_rn(e, c[i]);
  return e;
}

__global__ void __launch_bounds__(kReportThreads) report_kernel(DReplay R, bs_replay_summary* out, int n_scen) {
  const int s = blockIdx.x;
  if (s >= n_scen) return;
  const DScen sc = R.scen[s];
  const DRCfg* C = &R.cfgs[sc.cfg];
  __shared__ double s_horizon;
  __shared__ int s_ok;
  __shared__ unsigned hist[256];
  __shared__ unsigned long long acc[8];
  __shared__ double s_energy[4];
  bs_replay_summary* o = &out[s];
  if (threadIdx.x < 8) acc[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    int ok = !sc.skip_decode;
    double h = sc.duration;
    for (int i = 0; i < sc.ni; ++i) {
      const DInstState& st = R.st[sc.i0 + i];
      if (st.status != BS_OK || st.overflow) ok = 0;
      h = h < st.now ? st.now : h;  // std::max(horizon, sim->now)
    }
    if (C->horizon_opt >= 0.0) h = h < C->horizon_opt ? C->horizon_opt : h;
    s_horizon = h;
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  // horizon idle fill, every instance (simulator.hpp:877-880)
  for (int i = threadIdx.x; i < sc.ni; i += blockDim.x) {
    const int g = sc.i0 + i;
    const DInst I = R.inst[g];
    DInstState* st = &R.st[g];
    Writer w;
    w.init(&R, &I);
    w.n_rec = st->n_rec;
    w.n_idl = st->n_idl;
    w.n_dec = st->n_dec;
    FreqBook fb;
    fb.in_force = st->f_in;
    fb.pend = st->pend;
    fb.at = st->pend_at;
    fb.to = st->pend_f;
    double now = st->now;
    idle_until(w, IdleDirect{&R.sim.idle, I.tp}, fb, now, s_horizon);
    st->n_idl = w.n_idl;
    st->fill_status = w.status;
    st->fill_err = w.err;
    if (w.overflow) st->overflow = 1;
    if (w.status != BS_OK || w.overflow) atomicExch(&s_ok, 0);
  }
  __syncthreads();
  if (!s_ok) return;
  // TrimmedResult (metrics.hpp:71-88)
  const double s0 = C->span_start;
  const double s1 = sc.issuance_end;
  const bool empty = sc.n == 0 || s1 <= s0;
  if (!empty) {
    long long cnt[4] = {0, 0, 0, 0};  // prefill busy, prefill idle, decode busy, decode idle
    for (int i = 0; i < sc.ni; ++i) {
      const int g = sc.i0 + i;
      const int d = R.inst[g].phase == BS_PHASE_PREFILL ? 0 : 2;
      cnt[d] += R.st[g].n_rec;
      cnt[d + 1] += R.st[g].n_idl;
    }
    // merged arrays: prefill at the scenario's first record slot, decode after it
    double* base[4] = {R.rec_c + R.inst[sc.i0].rec0, R.idl_c + R.inst[sc.i0].idl0, nullptr, nullptr};
    base[2] = base[0] + cnt[0];
    base[3] = base[1] + cnt[1];
    for (int f = 0; f < 4; ++f)
      scatter_phase(R, sc, f < 2 ? BS_PHASE_PREFILL : BS_PHASE_DECODE, f & 1, base[f], s0, s1);
    __syncthreads();
    if (threadIdx.x < 4) s_energy[threadIdx.x] = fold_in_order(base[threadIdx.x], cnt[threadIdx.x]);
  }
  // request statistics
  long long completed = 0, generated = 0, rc = 0, rg = 0, tv = 0, pv = 0, nttft = 0, ntpot = 0;
  for (long long i = threadIdx.x; i < sc.n; i += blockDim.x) {
    const long long r = sc.r0 + i;
    const double pd = R.pdone[r];
    const long long nt = R.ntok[r];
    const long long out_len = R.output[r];
    const bool has_pd = !isnan(pd);
    const bool done = has_pd && nt == out_len;  // simulator.hpp:865-870
    generated += nt;
    if (done) ++completed;
    const double a = R.arrival[r];
    if (empty || !(a >= s0 && a <= s1)) continue;
    if (done) {
      ++rc;
      rg += nt;
    }
    if (has_pd) {
      ++nttft;
      if (__dsub_rn(pd, a) > C->slo_ttft) ++tv;
    }
    if (out_len >= 2 && nt >= 2) {
      ++ntpot;
      const double tp = __ddiv_rn(__dsub_rn(R.last_tok[r], R.first_tok[r]), static_cast<double>(out_len - 1));
      if (tp > C->slo_tpot) ++pv;
    }
  }
  atomicAdd(&acc[0], static_cast<unsigned long long>(completed));
  atomicAdd(&acc[1], static_cast<unsigned long long>(generated));
  atomicAdd(&acc[2], static_cast<unsigned long long>(rc));
  atomicAdd(&acc[3], static_cast<unsigned long long>(rg));
  atomicAdd(&acc[4], static_cast<unsigned long long>(tv));
  atomicAdd(&acc[5], static_cast<unsigned long long>(pv));
  atomicAdd(&acc[6], static_cast<unsigned long long>(nttft));
  atomicAdd(&acc[7], static_cast<unsigned long long>(ntpot));
  __syncthreads();
  const long long cnt_ttft = static_cast<long long>(acc[6]), cnt_tpot = static_cast<long long>(acc[7]);
  double p99_ttft = NAN, p99_tpot = NAN;
  if (!empty && cnt_ttft > 0) {
    p99_ttft = block_select(
        sc.r0, sc.n, nearest_rank_index(C->slo_pct, cnt_ttft),
        [&](long long r, double* v) {
          const double a = R.arrival[r], pd = R.pdone[r];
          if (!(a >= s0 && a <= s1) || isnan(pd)) return false;
          *v = __dsub_rn(pd, a);
          return true;
        },
        hist);
  }
  if (!empty && cnt_tpot > 0) {
    p99_tpot = block_select(
        sc.r0, sc.n, nearest_rank_index(C->slo_pct, cnt_tpot),
        [&](long long r, double* v) {
          const double a = R.arrival[r];
          const long long out_len = R.output[r], nt = R.ntok[r];
          if (!(a >= s0 && a <= s1) || out_len < 2 || nt < 2) return false;
          *v = __ddiv_rn(__dsub_rn(R.last_tok[r], R.first_tok[r]), static_cast<double>(out_len - 1));
          return true;
        },
        hist);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  o->status = BS_OK;
  o->horizon_ms = s_horizon;
  o->completed_requests = static_cast<long long>(acc[0]);
  o->generated_tokens = static_cast<long long>(acc[1]);
  long long nb = 0, ni = 0, nd = 0, bt[3] = {0, 0, 0};
  for (int i = 0; i < sc.ni; ++i) {
    const DInstState& st = R.st[sc.i0 + i];
    nb += st.n_rec;
    ni += st.n_idl;
    nd += st.n_dec;
    for (int t = 0; t < 3; ++t) bt[t] += st.by_trig[t];
  }
  o->n_batches = nb;
  o->n_idles = ni;
  o->n_decisions = nd;
  for (int t = 0; t < 3; ++t) o->decisions_by_trigger[t] = bt[t];
  // make_report (metrics.hpp:121-156)
  o->span_ms = s1 - s0 > 0.0 ? __dsub_rn(s1, s0) : 0.0;
  o->has_p99_ttft = o->has_p99_tpot = o->has_e_first = o->has_e_output = 0;
  o->p99_ttft_ms = o->p99_mean_tpot_ms = o->energy_per_first_token_j = o->energy_per_output_token_j = NAN;
  o->avg_power_prefill_w = o->avg_power_decode_w = o->prefill_energy_j = o->decode_energy_j = 0.0;
  o->report_completed = o->report_generated = o->ttft_violations = o->tpot_violations = 0;
  if (empty) return;
  o->has_p99_ttft = cnt_ttft > 0;
  o->p99_ttft_ms = p99_ttft;
  o->has_p99_tpot = cnt_tpot > 0;
  o->p99_mean_tpot_ms = p99_tpot;
  o->prefill_energy_j = __dadd_rn(s_energy[0], s_energy[1]);
  o->decode_energy_j = __dadd_rn(s_energy[2], s_energy[3]);
  if (o->span_ms > 0.0) {
    const double secs = __ddiv_rn(o->span_ms, 1000.0);
    o->avg_power_prefill_w = __ddiv_rn(o->prefill_energy_j, secs);
    o->avg_power_decode_w = __ddiv_rn(o->decode_energy_j, secs);
  }
  o->report_completed = static_cast<long long>(acc[2]);
  o->report_generated = static_cast<long long>(acc[3]);
  o->ttft_violations = static_cast<long long>(acc[4]);
  o->tpot_violations = static_cast<long long>(acc[5]);
  if (o->report_completed > 0) {
    o->has_e_first = 1;
    o->energy_per_first_token_j = __ddiv_rn(o->prefill_energy_j, static_cast<double>(o->report_completed));
  }
  if (o->report_generated > 0) {
    o->has_e_output = 1;
    o->energy_per_output_token_j = __ddiv_rn(o->decode_energy_j, static_cast<double>(o->report_generated));
  }
}

}  // namespace

// --- host ------------------------------------------------------------------------------

namespace {

size_t up256r(size_t x) { return (x + 255) / 256 * 256; }

struct HostErr {
  int status = BS_OK;
  std::string msg;
  void set(int st, const std::string& m) {
    if (status == BS_OK) {
      status = st;
      msg = m;
    }
  }
};

std::string fmt(const char* f, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

// RouterState::validate (simulator.hpp:587-597).
bool router_ok(const std::vector<double>& w, HostErr* e) {
  if (w.empty()) {
    e->set(BS_PARAMETER_ERROR, "router: no instances");
    return false;
  }
  double sum = 0.0;
  for (double x : w) {
    if (x <= 0.0) {
      e->set(BS_PARAMETER_ERROR, "router: weights must be positive");
      return false;
    }
    sum += x;
  }
  if (std::abs(sum - 1.0) > 1e-9) {
    e->set(BS_PARAMETER_ERROR, "router: weights must sum to 1");
    return false;
  }
  return true;
}

bool instance_ok(const bs_instance_config& c, HostErr* e) {  // InstanceConfig::validate (simulator.hpp:27-30)
  if (c.tp < 1) {
    e->set(BS_PARAMETER_ERROR, "instance: tp must be >= 1");
    return false;
  }
  if (c.base_freq_mhz <= 0.0) {
    e->set(BS_PARAMETER_ERROR, "instance: base_freq_mhz must be > 0");
    return false;
  }
  return true;
}

bool policy_ok(const bs_scheduler_policy& p, HostErr* e) {  // SchedulerPolicy::validate (scheduler.hpp:17-21)
  if (p.max_batch_tokens < 1) e->set(BS_PARAMETER_ERROR, "scheduler: max_batch_tokens must be >= 1");
  else if (p.max_batch_requests < 1) e->set(BS_PARAMETER_ERROR, "scheduler: max_batch_requests must be >= 1");
  else if (p.kv_capacity_tokens < 1) e->set(BS_PARAMETER_ERROR, "scheduler: kv_capacity_tokens must be >= 1");
  else return true;
  return false;
}

bool decode_cfg_ok(const bs_decode_config& d, HostErr* e) {  // DecodePolicyConfig::validate (dvfs.hpp:42-47)
  if (d.tbt_slo_ms <= 0.0) {
    e->set(BS_PARAMETER_ERROR, "decode policy: tbt_slo_ms must be > 0");
    return false;
  }
  if (d.kv_threshold <= 0.0 || d.kv_threshold >= 1.0) {
    e->set(BS_PARAMETER_ERROR, "decode policy: kv_threshold in (0,1)");
    return false;
  }
  if (d.n_ladder < 1 || !d.ladder_mhz) {
    e->set(BS_PARAMETER_ERROR, "frequency ladder: empty");
    return false;
  }
  double prev = 0.0;
  for (int j = 0; j < d.n_ladder; ++j) {
    if (d.ladder_mhz[j] <= prev) {
      e->set(BS_PARAMETER_ERROR, "frequency ladder: must be strictly increasing and > 0");
      return false;
    }
    prev = d.ladder_mhz[j];
  }
  if (d.margin < 0.0) {
    e->set(BS_PARAMETER_ERROR, "decode policy: margin must be >= 0");
    return false;
  }
  if (d.n_ladder > BS_MAX_LADDER) {
    e->set(BS_PARAMETER_ERROR, fmt("decode policy: %d rungs exceed the device limit %d", d.n_ladder, BS_MAX_LADDER));
    return false;
  }
  return true;
}

std::string device_msg(int kind, const DInstState& st, int tp, long long kv_cap) {
  switch (kind) {
    case kErrLatency: return "latency model returned non-positive value";
    case kErrPower: return "power model returned non-positive value";
    case kErrIdleMissing: return fmt("idle model: tp %d not present", tp);
    case kErrIdleEmpty: return "idle model: empty frequency set";
    case kErrAxis: return "grid: unknown axis";
    case kErrKvNeed:
      return fmt("decode: request %lld needs %lld KV tokens, capacity %lld", st.err_arg, st.err_arg2, kv_cap);
    case kErrStalled: return "decode: admission stalled with empty batch";
    case kErrStarvation: return "decode: event starvation";
    case kErrScheduler: return "scheduler: queued request with no remaining tokens";
    case kErrGuard: return "replay: the event loop would not terminate (safety deadline re-fires)";
    default: return fmt("replay: device error %d", kind);
  }
}

struct ScenPlan {
  HostErr pre, post, fin;  // errors the reference raises before phase 1, after it, after the simulation
  bool run = false;
  long long sum_out = 0;
};

}  // namespace

extern "C" int bs_replay(bs_ctx_t ctx, bs_models_t sim_models, bs_models_t ctl_models, const bs_replay_config* cfgs,
                         int n_cfgs, const bs_scenario* sc, int n, bs_replay_summary* out,
                         bs_replay_request* requests, bs_replay_logs* logs) {
  if (!ctx || !sim_models) return set_error(ctx, BS_PARAMETER_ERROR, "bs_replay: null context or models");
  if (!ctl_models) ctl_models = sim_models;
  if (n < 0 || (n > 0 && (!sc || !out))) return set_error(ctx, BS_PARAMETER_ERROR, "bs_replay: bad scenario arrays");
  if (n == 0) return BS_OK;
  if (n_cfgs < 1 || !cfgs) return set_error(ctx, BS_PARAMETER_ERROR, "bs_replay: no configuration");
  std::memset(out, 0, sizeof(bs_replay_summary) * static_cast<size_t>(n));
  ctx->last_h2d = ctx->last_d2h = 0;

  // --- configurations ---------------------------------------------------------
  std::vector<DRCfg> hcfg(n_cfgs);
  std::vector<HostErr> cfg_mpc_err(n_cfgs), cfg_dec_err(n_cfgs), cfg_fin_err(n_cfgs);
  for (int c = 0; c < n_cfgs; ++c) {
    const bs_replay_config& rc = cfgs[c];
    DRCfg& d = hcfg[c];
    std::memset(&d, 0, sizeof d);
    d.controlled = rc.controlled ? 1 : 0;
    if (d.controlled) {
      int st = pack_mpc_cfg(ctx, rc.mpc, rc.policy, &d.mpc);
      if (st != BS_OK) cfg_mpc_err[c].set(st, ctx->err);
      decode_cfg_ok(rc.decode, &cfg_dec_err[c]);
      if (cfg_dec_err[c].status == BS_OK) {
        d.n_ladder = rc.decode.n_ladder;
        for (int j = 0; j < d.n_ladder; ++j) d.ladder[j] = rc.decode.ladder_mhz[j];
        d.dec_fmax = d.ladder[d.n_ladder - 1];
      }
      d.dec_tbt = rc.decode.tbt_slo_ms;
      d.dec_kv_thr = rc.decode.kv_threshold;
      d.dec_one_plus_margin = 1.0 + rc.decode.margin;
      d.safety_pre = rc.mpc.margin;                                  // PrefillMpcController::safety_margin
      d.safety_dec = rc.decode.margin > 0.0 ? rc.decode.margin : 0.05;  // TwoTierFactory::make (dvfs.hpp:380)
      d.pre_fmax = d.mpc.max_mhz;
    }
    d.switch_ms = rc.switch_latency_ms;
    d.horizon_opt = rc.horizon_ms;
    d.span_start = rc.rampup_s * 1000.0;
    d.slo_ttft = rc.slo.ttft_ms;
    d.slo_tpot = rc.slo.tpot_ms;
    d.slo_pct = rc.slo.percentile;
    d.max_batch_tokens = rc.policy.max_batch_tokens;
    d.max_batch_requests = rc.policy.max_batch_requests;
    d.kv_cap = rc.policy.kv_capacity_tokens;
    d.chunking = rc.policy.chunking ? 1 : 0;
    // trim_steady_state / make_report validation (metrics.hpp:73, 123)
    if (rc.rampup_s < 0.0) cfg_fin_err[c].set(BS_PARAMETER_ERROR, "trim: rampup_s must be >= 0");
    else if (rc.slo.ttft_ms <= 0.0 || rc.slo.tpot_ms <= 0.0) cfg_fin_err[c].set(BS_PARAMETER_ERROR, "slo: bounds must be > 0");
    else if (rc.slo.percentile <= 0.0 || rc.slo.percentile > 1.0)
      cfg_fin_err[c].set(BS_PARAMETER_ERROR, "slo: percentile must be in (0,1]");
  }
  ctx->err.clear();

  // --- scenarios: validation in the reference's order, phase-1 routing -------------
  std::vector<ScenPlan> plan(n);
  std::vector<DScen> hs(n);
  std::vector<DInst> hi;
  std::vector<long long> plist;  // global request indices, grouped by prefill instance
  std::vector<int> pre_ids, dec_ids;
  long long NR = 0;
  for (int s = 0; s < n; ++s) {
    const bs_scenario& S = sc[s];
    ScenPlan& P = plan[s];
    DScen& D = hs[s];
    std::memset(&D, 0, sizeof D);
    D.r0 = NR;
    D.n = S.trace.n;
    D.duration = S.trace.duration_ms;
    D.cfg = S.config;
    D.i0 = static_cast<int>(hi.size());
    if (S.config < 0 || S.config >= n_cfgs) {
      P.pre.set(BS_PARAMETER_ERROR, "bs_replay: scenario configuration index out of range");
      continue;
    }
    if (S.trace.n < 0 || (S.trace.n > 0 && !S.trace.requests)) {
      P.pre.set(BS_PARAMETER_ERROR, "bs_replay: bad trace");
      continue;
    }
    // Trace::validate (workload.hpp:37-49)
    double prev = 0.0;
    for (long long i = 0; i < S.trace.n && P.pre.status == BS_OK; ++i) {
      const bs_request& r = S.trace.requests[i];
      if (r.arrival_ms < 0.0) P.pre.set(BS_PARAMETER_ERROR, "trace: negative arrival");
      else if (r.input_len < 1 || r.output_len < 1) P.pre.set(BS_PARAMETER_ERROR, "trace: lengths must be >= 1");
      else if (r.arrival_ms < prev) P.pre.set(BS_PARAMETER_ERROR, "trace: arrivals not sorted");
      prev = r.arrival_ms;
    }
    if (P.pre.status == BS_OK && S.trace.n > 0 && S.trace.duration_ms < S.trace.requests[S.trace.n - 1].arrival_ms)
      P.pre.set(BS_PARAMETER_ERROR, "trace: duration shorter than last arrival");
    if (P.pre.status != BS_OK) continue;
    std::vector<int> pre, dcd;
    for (int i = 0; i < S.n_instances; ++i)
      (S.instances[i].config.phase == BS_PHASE_PREFILL ? pre : dcd).push_back(i);
    if (pre.empty()) {
      P.pre.set(BS_CONFIG_ERROR, "cluster: no prefill instance");
      continue;
    }
    if (dcd.empty()) {
      P.pre.set(BS_CONFIG_ERROR, "cluster: no decode instance");
      continue;
    }
    if (S.n_instances > kMaxInstances) {
      P.pre.set(BS_PARAMETER_ERROR, fmt("bs_replay: %d instances exceed the device limit %d", S.n_instances,
                                        kMaxInstances));
      continue;
    }
    std::vector<double> wp, wd;
    for (int i : pre) wp.push_back(S.instances[i].weight);
    for (int i : dcd) wd.push_back(S.instances[i].weight);
    if (!router_ok(wp, &P.pre)) continue;
    const bs_replay_config& rc = cfgs[S.config];
    // phase-1 construction: controllers->make (validates MpcConfig, policy),
    // then InstanceSim (InstanceConfig, policy) for each prefill instance
    for (int i : pre) {
      if (rc.controlled && cfg_mpc_err[S.config].status != BS_OK) {
        P.pre = cfg_mpc_err[S.config];
        break;
      }
      if (!instance_ok(S.instances[i].config, &P.pre) || !policy_ok(rc.policy, &P.pre)) break;
    }
    if (P.pre.status != BS_OK) continue;
    // after phase 1: decode router, controllers and instances
    if (router_ok(wd, &P.post)) {
      for (int i : dcd) {
        if (rc.controlled && cfg_dec_err[S.config].status != BS_OK) {
          P.post = cfg_dec_err[S.config];
          break;
        }
        if (!instance_ok(S.instances[i].config, &P.post) || !policy_ok(rc.policy, &P.post)) break;
      }
    }
    P.fin = cfg_fin_err[S.config];
    P.run = true;
    D.skip_decode = P.post.status != BS_OK;
    D.ni = S.n_instances;
    D.n_prefill = static_cast<int>(pre.size());
    D.n_decode = static_cast<int>(dcd.size());
    double iss = 0.0;
    for (long long i = 0; i < S.trace.n; ++i) {
      iss = std::max(iss, S.trace.requests[i].arrival_ms);
      P.sum_out += S.trace.requests[i].output_len;
    }
    D.issuance_end = iss;
    // route_request by prompt length (simulator.hpp:610-624, 818-823)
    std::vector<double> assigned(pre.size(), 0.0);
    std::vector<std::vector<long long>> lists(pre.size());
    double total = 0.0;
    for (long long i = 0; i < S.trace.n; ++i) {
      const double load = static_cast<double>(S.trace.requests[i].input_len);
      total += load;
      int best = 0;
      double best_def = -INFINITY;
      for (size_t j = 0; j < pre.size(); ++j) {
        const double def = wp[j] * total - assigned[j];
        if (def > best_def) {
          best_def = def;
          best = static_cast<int>(j);
        }
      }
      assigned[best] += load;
      lists[best].push_back(NR + i);
    }
    for (int i = 0; i < S.n_instances; ++i) {
      DInst I;
      std::memset(&I, 0, sizeof I);
      I.phase = S.instances[i].config.phase;
      I.tp = S.instances[i].config.tp;
      I.scen = s;
      I.local = i;
      I.base_freq = S.instances[i].config.base_freq_mhz;
      I.weight = S.instances[i].weight;
      const int g = static_cast<int>(hi.size());
      if (I.phase == BS_PHASE_PREFILL) {
        const size_t slot = std::find(pre.begin(), pre.end(), i) - pre.begin();
        I.list0 = static_cast<long long>(plist.size());
        I.list_n = static_cast<long long>(lists[slot].size());
        plist.insert(plist.end(), lists[slot].begin(), lists[slot].end());
        pre_ids.push_back(g);
      } else {
        I.list0 = NR;
        dec_ids.push_back(g);
      }
      hi.push_back(I);
    }
    NR += S.trace.n;
  }

  // --- capacities (exact bounds for prefill, estimates + retry for decode) -------
  std::vector<long long> need_rec(hi.size(), -1), need_idl(hi.size(), -1), need_dec(hi.size(), -1);
  const bool want_logs = logs != nullptr;
  for (int attempt = 0; attempt < 3; ++attempt) {
    long long nrec = 0, nidl = 0, ndec = 0, nres = 0;
    for (size_t g = 0; g < hi.size(); ++g) {
      DInst& I = hi[g];
      const DScen& D = hs[I.scen];
      const DRCfg& C = hcfg[D.cfg];
      long long rc, ic, dc;
      if (I.phase == BS_PHASE_PREFILL) {
        long long tok = 0;
        for (long long k = 0; k < I.list_n; ++k) tok += sc[I.scen].trace.requests[plist[I.list0 + k] - D.r0].input_len;
        const long long B = I.list_n + tok / std::max<long long>(1, C.max_batch_tokens) + 2;
        rc = 3 * B + I.list_n + 16;
        ic = 3 * B + I.list_n + 16;
        dc = want_logs ? 2 * B + I.list_n + 16 : 0;
      } else {
        // decode iterations (one batch record each, at most one idle between
        // two): an estimate from the instance's share of the window's output
        // tokens (routing weight) at ~8 residents per iteration; an overflow
        // re-runs with the device's exact counts (need_*)
        const long long so = plan[I.scen].sum_out;
        const long long est = static_cast<long long>((static_cast<double>(so) / 8.0 + static_cast<double>(D.n)) *
                                                     std::min(1.0, std::max(0.0, I.weight))) + 256;
        rc = 2 * est + 16;
        ic = 2 * est + 16;
        dc = want_logs ? 2 * est + 16 : 0;
        I.res0 = nres;
        nres += std::min<long long>(C.max_batch_requests, std::max<long long>(D.n, 1));
      }
      if (need_rec[g] >= 0) rc = std::max(rc, need_rec[g] + 16);
      if (need_idl[g] >= 0) ic = std::max(ic, need_idl[g] + 16);
      if (need_dec[g] >= 0 && want_logs) dc = std::max(dc, need_dec[g] + 16);
      I.rec0 = nrec;
      I.rec_cap = rc;
      I.idl0 = nidl;
      I.idl_cap = ic;
      I.dec0 = ndec;
      I.dec_cap = dc;
      nrec += rc;
      nidl += ic;
      ndec += dc;
    }
    const long long NP = static_cast<long long>(plist.size());
    const int NI = static_cast<int>(hi.size());
    // host blob (H2D): cfgs | scen | inst | pre_ids | dec_ids | id | arrival | input | output | plist | W
    size_t o = 0;
    auto take = [&](size_t bytes) {
      const size_t r = o;
      o += up256r(std::max<size_t>(bytes, 1));
      return r;
    };
    const size_t o_cfg = take(sizeof(DRCfg) * n_cfgs), o_scen = take(sizeof(DScen) * n),
                 o_inst = take(sizeof(DInst) * std::max(NI, 1)), o_pre = take(4 * pre_ids.size()),
                 o_dec = take(4 * dec_ids.size()), o_id = take(8 * NR), o_arr = take(8 * NR), o_in = take(8 * NR),
                 o_out = take(8 * NR), o_plist = take(8 * NP), o_W = take(sizeof(DWaiting) * NP);
    const size_t h2d = o;
    // device-only
    const size_t o_st = take(sizeof(DInstState) * std::max(NI, 1)), o_sum = take(sizeof(bs_replay_summary) * n),
                 o_dinst = take(4 * NR), o_nan = take(8 * 5 * NR), o_ntok = take(8 * NR),
                 o_done = take(sizeof(DDone) * NP), o_dlist = take(8 * NR), o_djoin = take(8 * NR),
                 o_mslot = take(4 * NR), o_mr = take(8 * NR), o_rec = take(sizeof(DRec) * nrec),
                 o_recx = want_logs ? take(sizeof(DRecX) * nrec) : 0, o_idl = take(sizeof(DRec) * nidl),
                 o_idlx = want_logs ? take(sizeof(DIdlX) * nidl) : 0,
                 o_decr = want_logs ? take(sizeof(DDec) * ndec) : 0,
                 o_res = take(sizeof(DResident) * std::max<long long>(nres, 1)),
                 o_recc = take(8 * nrec), o_idlc = take(8 * nidl);
    const size_t total = o;
    char* h = static_cast<char*>(ctx->host_buf(12, h2d));
    char* d = static_cast<char*>(ctx->dev_buf(12, total));
    if (!h || !d) return set_error(ctx, BS_CUDA_ERROR, "bs_replay: allocation of %.1f MB failed", total / 1e6);
    std::memcpy(h + o_cfg, hcfg.data(), sizeof(DRCfg) * n_cfgs);
    std::memcpy(h + o_scen, hs.data(), sizeof(DScen) * n);
    if (NI) std::memcpy(h + o_inst, hi.data(), sizeof(DInst) * NI);
    if (!pre_ids.empty()) std::memcpy(h + o_pre, pre_ids.data(), 4 * pre_ids.size());
    if (!dec_ids.empty()) std::memcpy(h + o_dec, dec_ids.data(), 4 * dec_ids.size());
    long long* hid = reinterpret_cast<long long*>(h + o_id);
    double* harr = reinterpret_cast<double*>(h + o_arr);
    long long* hin = reinterpret_cast<long long*>(h + o_in);
    long long* hout = reinterpret_cast<long long*>(h + o_out);
    for (int s = 0; s < n; ++s) {
      if (!plan[s].run) continue;
      for (long long i = 0; i < sc[s].trace.n; ++i) {
        const bs_request& r = sc[s].trace.requests[i];
        hid[hs[s].r0 + i] = r.id;
        harr[hs[s].r0 + i] = r.arrival_ms;
        hin[hs[s].r0 + i] = r.input_len;
        hout[hs[s].r0 + i] = r.output_len;
      }
    }
    if (NP) std::memcpy(h + o_plist, plist.data(), 8 * NP);
    DWaiting* hw = reinterpret_cast<DWaiting*>(h + o_W);
    for (long long k = 0; k < NP; ++k) {
      const long long r = plist[k];
      hw[k] = DWaiting{hid[r], harr[r], hin[r], hin[r]};
    }
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, h2d, cudaMemcpyHostToDevice, ctx->stream));
    BS_CUDA_TRY(ctx, cudaMemsetAsync(d + o_st, 0, o_dinst - o_st, ctx->stream));
    BS_CUDA_TRY(ctx, cudaMemsetAsync(d + o_dinst, 0xff, o_ntok - o_dinst, ctx->stream));  // -1 / NaN
    BS_CUDA_TRY(ctx, cudaMemsetAsync(d + o_ntok, 0, 8 * NR, ctx->stream));
    ctx->last_h2d += h2d;

    DReplay R;
    R.sim = sim_models->dm;
    R.ctl = ctl_models->dm;
    R.cfgs = reinterpret_cast<const DRCfg*>(d + o_cfg);
    R.scen = reinterpret_cast<const DScen*>(d + o_scen);
    R.inst = reinterpret_cast<const DInst*>(d + o_inst);
    R.st = reinterpret_cast<DInstState*>(d + o_st);
    R.id = reinterpret_cast<const long long*>(d + o_id);
    R.arrival = reinterpret_cast<const double*>(d + o_arr);
    R.input = reinterpret_cast<const long long*>(d + o_in);
    R.output = reinterpret_cast<const long long*>(d + o_out);
    R.d_inst = reinterpret_cast<int*>(d + o_dinst);
    double* nanb = reinterpret_cast<double*>(d + o_nan);
    R.pdone = nanb;
    R.first_start = nanb + NR;
    R.first_tok = nanb + 2 * NR;
    R.last_tok = nanb + 3 * NR;
    R.max_tbt = nanb + 4 * NR;
    R.ntok = reinterpret_cast<long long*>(d + o_ntok);
    R.plist = reinterpret_cast<const long long*>(d + o_plist);
    R.W = reinterpret_cast<DWaiting*>(d + o_W);
    R.done = reinterpret_cast<DDone*>(d + o_done);
    R.dlist = reinterpret_cast<long long*>(d + o_dlist);
    R.djoin = reinterpret_cast<double*>(d + o_djoin);
    R.mslot = reinterpret_cast<int*>(d + o_mslot);
    R.mr = reinterpret_cast<long long*>(d + o_mr);
    R.rec = reinterpret_cast<DRec*>(d + o_rec);
    R.recx = want_logs ? reinterpret_cast<DRecX*>(d + o_recx) : nullptr;
    R.idl = reinterpret_cast<DRec*>(d + o_idl);
    R.idlx = want_logs ? reinterpret_cast<DIdlX*>(d + o_idlx) : nullptr;
    R.dec = want_logs ? reinterpret_cast<DDec*>(d + o_decr) : nullptr;
    R.res = reinterpret_cast<DResident*>(d + o_res);
    R.rec_c = reinterpret_cast<double*>(d + o_recc);
    R.idl_c = reinterpret_cast<double*>(d + o_idlc);
    bs_replay_summary* dsum = reinterpret_cast<bs_replay_summary*>(d + o_sum);
    const int* dpre = reinterpret_cast<const int*>(d + o_pre);
    const int* ddec = reinterpret_cast<const int*>(d + o_dec);

    cudaEvent_t ev[5];
    for (auto& e : ev) BS_CUDA_TRY(ctx, cudaEventCreate(&e));
    BS_CUDA_TRY(ctx, cudaEventRecord(ev[0], ctx->stream));
    if (!pre_ids.empty()) {
      int max_ns = 1, max_h = 1, max_nc = 1;
      for (const DRCfg& c : hcfg) {
        if (!c.controlled) continue;
        max_ns = std::max(max_ns, c.mpc.nc + 1);
        max_h = std::max(max_h, c.mpc.horizon);
        max_nc = std::max(max_nc, c.mpc.nc);
      }
      const size_t psmem = kPrefillWarps * pre_warp_bytes(max_ns, max_h, max_nc);
      BS_CUDA_TRY(ctx, cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(psmem)));
      const int np_ = static_cast<int>(pre_ids.size());
      prefill_kernel<<<(np_ + kPrefillWarps - 1) / kPrefillWarps, kPrefillWarps * 32, psmem, ctx->stream>>>(
          R, dpre, np_, max_ns, max_h, max_nc);
      BS_LAUNCH_CHECK(ctx);
    }
    BS_CUDA_TRY(ctx, cudaEventRecord(ev[1], ctx->stream));
    route_kernel<<<(n + 63) / 64, 64, 0, ctx->stream>>>(R, n);
    BS_LAUNCH_CHECK(ctx);
    BS_CUDA_TRY(ctx, cudaEventRecord(ev[2], ctx->stream));
    if (!dec_ids.empty()) {
      const int nd = static_cast<int>(dec_ids.size());
      int max_slots = 1;
      for (const DRCfg& c : hcfg) max_slots = std::max(max_slots, (c.controlled ? c.n_ladder : 0) + 1);
      const size_t smem = (sizeof(DecSlot) * static_cast<size_t>(max_slots) + sizeof(DecBrk)) * 4;
      if (smem > 48 * 1024)
        BS_CUDA_TRY(ctx, cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem)));
      decode_kernel<<<(nd + 3) / 4, 128, smem, ctx->stream>>>(R, ddec, nd, max_slots);
      BS_LAUNCH_CHECK(ctx);
    }
    BS_CUDA_TRY(ctx, cudaEventRecord(ev[3], ctx->stream));
    report_kernel<<<n, kReportThreads, 0, ctx->stream>>>(R, dsum, n);
    BS_LAUNCH_CHECK(ctx);
    BS_CUDA_TRY(ctx, cudaEventRecord(ev[4], ctx->stream));

    // --- results ---------------------------------------------------------------
    std::vector<DInstState> st(std::max(NI, 1));
    if (NI) BS_CUDA_TRY(ctx, cudaMemcpyAsync(st.data(), d + o_st, sizeof(DInstState) * NI, cudaMemcpyDeviceToHost, ctx->stream));
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(out, d + o_sum, sizeof(bs_replay_summary) * n, cudaMemcpyDeviceToHost, ctx->stream));
    BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->last_d2h += sizeof(DInstState) * NI + sizeof(bs_replay_summary) * n;
    {
      float ms[4];
      for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]);
      ctx->n_stats = 4;
      for (int k = 0; k < 4; ++k) ctx->stats[k] = ms[k];
    }
    for (auto& e : ev) cudaEventDestroy(e);
    bool overflow = false;
    for (int g = 0; g < NI; ++g) {
      if (!st[g].overflow) continue;
      overflow = true;
      need_rec[g] = std::max(need_rec[g], st[g].n_rec);
      need_idl[g] = std::max(need_idl[g], st[g].n_idl + 4);
      need_dec[g] = std::max(need_dec[g], st[g].n_dec);
    }
    if (overflow && attempt < 2) continue;
    if (overflow) return set_error(ctx, BS_CUDA_ERROR, "bs_replay: record buffers overflowed after retries");

    // per-scenario status, in the order the reference would raise
    int first_bad = -1;
    std::string first_msg;
    for (int s = 0; s < n; ++s) {
      HostErr e = plan[s].pre;
      if (e.status == BS_OK && plan[s].run) {
        const DScen& D = hs[s];
        for (int i = 0; i < D.ni && e.status == BS_OK; ++i) {
          const DInstState& x = st[D.i0 + i];
          if (hi[D.i0 + i].phase == BS_PHASE_PREFILL && x.status != BS_OK)
            e.set(x.status, device_msg(x.err_kind, x, hi[D.i0 + i].tp, hcfg[D.cfg].kv_cap));
        }
        if (e.status == BS_OK && plan[s].post.status != BS_OK) e = plan[s].post;
        for (int i = 0; i < D.ni && e.status == BS_OK; ++i) {
          const DInstState& x = st[D.i0 + i];
          if (hi[D.i0 + i].phase == BS_PHASE_DECODE && x.status != BS_OK)
            e.set(x.status, device_msg(x.err_kind, x, hi[D.i0 + i].tp, hcfg[D.cfg].kv_cap));
        }
        for (int i = 0; i < D.ni && e.status == BS_OK; ++i) {
          const DInstState& x = st[D.i0 + i];
          if (x.fill_status != BS_OK) e.set(x.fill_status, device_msg(x.fill_err, x, hi[D.i0 + i].tp, 0));
        }
        if (e.status == BS_OK && plan[s].fin.status != BS_OK) e = plan[s].fin;
      }
      if (e.status != BS_OK) {
        std::memset(&out[s], 0, sizeof out[s]);
        out[s].status = e.status;
        if (first_bad < 0) {
          first_bad = s;
          first_msg = e.msg;
        }
      }
    }

    if (requests) {
      std::vector<int> hdinst(NR);
      std::vector<double> hnan(5 * NR);
      std::vector<long long> hntok(NR);
      if (NR) {
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hdinst.data(), d + o_dinst, 4 * NR, cudaMemcpyDeviceToHost, ctx->stream));
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hnan.data(), d + o_nan, 40 * NR, cudaMemcpyDeviceToHost, ctx->stream));
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hntok.data(), d + o_ntok, 8 * NR, cudaMemcpyDeviceToHost, ctx->stream));
        BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        ctx->last_d2h += 52 * NR;
      }
      std::vector<int> pinst(NR, -1);
      for (const DInst& I : hi)
        if (I.phase == BS_PHASE_PREFILL)
          for (long long k = 0; k < I.list_n; ++k) pinst[plist[I.list0 + k]] = I.local;
      long long q = 0;
      for (int s = 0; s < n; ++s) {
        for (long long i = 0; i < sc[s].trace.n; ++i, ++q) {
          bs_replay_request& o = requests[q];
          std::memset(&o, 0, sizeof o);
          const bs_request& r = sc[s].trace.requests[i];
          o.id = r.id;
          if (!plan[s].run) {
            o.prefill_instance = o.decode_instance = -1;
            o.prefill_done_ms = o.decode_first_start_ms = o.first_token_ms = o.last_token_ms = o.max_tbt_ms = NAN;
            continue;
          }
          const long long g = hs[s].r0 + i;
          o.prefill_instance = pinst[g];
          o.decode_instance = hdinst[g];
          o.prefill_done_ms = hnan[g];
          o.decode_first_start_ms = hnan[NR + g];
          o.first_token_ms = hnan[2 * NR + g];
          o.last_token_ms = hnan[3 * NR + g];
          o.max_tbt_ms = hnan[4 * NR + g];
          o.n_tokens = hntok[g];
          o.completed = !std::isnan(o.prefill_done_ms) && o.n_tokens == r.output_len;
        }
      }
    }

    if (logs) {
      std::vector<DRec> hrec(nrec), hidl(nidl);
      std::vector<DRecX> hrecx(nrec);
      std::vector<DIdlX> hidlx(nidl);
      std::vector<DDec> hdec(ndec);
      if (nrec) {
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hrec.data(), d + o_rec, sizeof(DRec) * nrec, cudaMemcpyDeviceToHost, ctx->stream));
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hrecx.data(), d + o_recx, sizeof(DRecX) * nrec, cudaMemcpyDeviceToHost, ctx->stream));
      }
      if (nidl) {
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hidl.data(), d + o_idl, sizeof(DRec) * nidl, cudaMemcpyDeviceToHost, ctx->stream));
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hidlx.data(), d + o_idlx, sizeof(DIdlX) * nidl, cudaMemcpyDeviceToHost, ctx->stream));
      }
      if (ndec)
        BS_CUDA_TRY(ctx, cudaMemcpyAsync(hdec.data(), d + o_decr, sizeof(DDec) * ndec, cudaMemcpyDeviceToHost, ctx->stream));
      BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      // re-read the states: the report kernel appended the horizon idle fill
      if (NI) BS_CUDA_TRY(ctx, cudaMemcpy(st.data(), d + o_st, sizeof(DInstState) * NI, cudaMemcpyDeviceToHost));
      for (int s = 0; s < n; ++s) {
        bs_replay_logs& L = logs[s];
        L.n_batches = L.n_idles = L.n_decisions = 0;
        if (!plan[s].run) continue;
        const DScen& D = hs[s];
        // k-way merges by (start | time, instance): SimResult's stable sorts (simulator.hpp:881-891)
        std::vector<long long> pos(D.ni, 0);
        auto merge = [&](int kind) {
          std::fill(pos.begin(), pos.end(), 0);
          long long w = 0;
          for (;;) {
            int best = -1;
            double bt = 0.0;
            for (int i = 0; i < D.ni; ++i) {
              const DInst& I = hi[D.i0 + i];
              const DInstState& x = st[D.i0 + i];
              const long long cnt = kind == 0 ? x.n_rec : kind == 1 ? x.n_idl : x.n_dec;
              if (pos[i] >= cnt) continue;
              const double t = kind == 0 ? hrec[I.rec0 + pos[i]].start
                               : kind == 1 ? hidl[I.idl0 + pos[i]].start
                                           : hdec[I.dec0 + pos[i]].time;
              if (best < 0 || t < bt) {
                best = i;
                bt = t;
              }
            }
            if (best < 0) break;
            const DInst& I = hi[D.i0 + best];
            const long long k = pos[best]++;
            if (kind == 0) {
              if (w < L.batch_cap && L.batches) {
                const DRec& a = hrec[I.rec0 + k];
                const DRecX& b = hrecx[I.rec0 + k];
                L.batches[w] = bs_batch_record{I.local, I.phase, b.batch_seq, a.start, a.end, b.n_req, b.sum_len,
                                               b.freq, b.power, a.energy};
              }
              L.n_batches = ++w;
            } else if (kind == 1) {
              if (w < L.idle_cap && L.idles) {
                const DRec& a = hidl[I.idl0 + k];
                const DIdlX& b = hidlx[I.idl0 + k];
                L.idles[w] = bs_idle_record{I.local, I.phase, a.start, a.end, b.freq, b.power, a.energy};
              }
              L.n_idles = ++w;
            } else {
              if (w < L.decision_cap && L.decisions) {
                const DDec& a = hdec[I.dec0 + k];
                L.decisions[w] = bs_decision_record{a.time, I.local, a.trigger, a.freq, a.feasible, 0, a.eval};
              }
              L.n_decisions = ++w;
            }
          }
        };
        merge(0);
        merge(1);
        merge(2);
      }
    }
    if (first_bad >= 0) return set_error(ctx, out[first_bad].status, "%s", first_msg.c_str());
    return BS_OK;
  }
  return set_error(ctx, BS_CUDA_ERROR, "bs_replay: unreachable");
}

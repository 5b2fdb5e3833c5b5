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
};

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

// predict_latency / predict_power at the instance's (tp, freq); false on
// ModelError (perfmodel.hpp:264, 270).
__device__ __forceinline__ bool predict_at(const DGrid& g, long long n_req, long long sum_len, const SimParams& p,
                                           double* out) {
  if (g.bad_axis) return false;
  const double v = interp(g, make_query(n_req, sum_len, p.tp, p.freq), nullptr);
  *out = v;
  return model_value_ok(v);
}

// simulate_prefill_instance (simulator.hpp:278-409) without a controller,
// followed by simulate_instance's accounting (667-739).
__device__ SimOut simulate_prefill(const DModels& m, const SimTrace& tr, const SimParams& p) {
  SimOut o;
  o.status = BS_OK;
  o.model_err = 0;
  o.meets_slo = 1;
  o.completed = 0;
  o.busy_j = 0.0;
  o.idle_j = 0.0;
  o.batches = 0;
  const DGrid& lat = m.grid[0];
  const DGrid& pw = m.grid[2];
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

  for (;;) {
    if (!active && qhead < arr) {
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
      if (!predict_at(lat, npick, sum, p, &L)) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 1;
        return o;
      }
      if (!predict_at(pw, npick, sum, p, &bp)) {
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
__device__ SimOut simulate_decode(const DModels& m, const SimTrace& tr, const SimParams& p, Resident* heap,
                                  int heap_cap) {
  SimOut o;
  o.status = BS_OK;
  o.model_err = 0;
  o.meets_slo = 1;
  o.completed = 0;
  o.busy_j = 0.0;
  o.idle_j = 0.0;
  o.batches = 0;
  const DGrid& lat = m.grid[1];
  const DGrid& pw = m.grid[3];
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
      if (!predict_at(lat, n_res, sum_ctx, p, &L)) {
        o.status = BS_MODEL_ERROR;
        o.model_err = 1;
        return o;
      }
      if (!predict_at(pw, n_res, sum_ctx, p, &bp)) {
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

}  // namespace bs

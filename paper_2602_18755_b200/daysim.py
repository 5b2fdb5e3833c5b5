"""Day-long what-if sweeps (BASELINE.json configs[3], "C4"): run_experiment
(runner.hpp:155-172) with the two-tier policy over many scenario traces at
once -- every 5-minute window of every scenario planned from its previous
window (plan_window_policies, runner.hpp:98-110: the config table, the ILP
and the max-throughput baseline) and replayed with per-iteration decisions.

The same decision path as ``pdsim.run_experiment`` (identical plans, tables
and reports, tests/test_gpu_daysim.py), organised for ~10^6-request traces:
traces, windows and probe traces stay numpy buffers in the C ABI's
``bs_request`` layout (no per-request Python objects), and the whole sweep is
four device calls:

  1. bs_goodput_tables   every (scenario, window)'s config table in one grid;
  2. bs_placement_solve_batch  every ILP and max-throughput baseline;
  3. bs_replay           every (scenario, window) replay;
  (trace synthesis is the reference's gen_gamma_trace, bs_gen_gamma_trace.)

Windows follow split_windows (workload.hpp:184-201): window w holds the
requests with floor(arrival / W) = w (the last window also the ones beyond),
arrivals re-based by w W.  The diurnal day concatenates 24 one-hour
gamma(0.5) segments whose mean rate follows a fixed profile (6 -> 20 rps).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from . import pdsim as P

REQ = np.dtype([("id", "<i8"), ("arrival_ms", "<f8"), ("input_len", "<i8"), ("output_len", "<i8")])
assert REQ.itemsize == C.sizeof(_abi.bs_request)

HOUR_MS = 3600e3


def diurnal_profile(lo: float = 6.0, hi: float = 20.0, hours: int = 24) -> list:
    """Mean rate per hour: lo at midnight, hi at noon (a raised cosine)."""
    return [lo + (hi - lo) * (1.0 - math.cos(2.0 * math.pi * h / hours)) / 2.0 for h in range(hours)]


def gen_segment(mean_rps: float, shape: float, duration_ms: float, lengths: P.LengthDistribution,
                seed: int) -> np.ndarray:
    """gen_gamma_trace (workload.hpp:95-116) into a bs_request buffer."""
    L = P.lib()
    keep: list = []
    cl = P.c_lengths(lengths, keep)
    n = C.c_int64()
    P.raise_status(L.bs_gen_gamma_trace(mean_rps, shape, duration_ms, C.byref(cl), seed, None, 0, C.byref(n)),
                   "gen_gamma_trace failed")
    out = np.zeros(max(1, n.value), dtype=REQ)
    P.raise_status(L.bs_gen_gamma_trace(mean_rps, shape, duration_ms, C.byref(cl), seed,
                                        out.ctypes.data_as(C.POINTER(_abi.bs_request)), n.value, C.byref(n)),
                   "gen_gamma_trace failed")
    return out[: n.value]


@dataclass
class DayTrace:
    requests: np.ndarray  # REQ, sorted by arrival
    duration_ms: float


def gen_day(seed: int, profile: list | None = None, lengths: P.LengthDistribution | None = None,
            shape: float = 0.5) -> DayTrace:
    """24 one-hour gamma segments (hour h: seed * 1000 + h, rate profile[h]),
    concatenated with arrivals shifted by h hours and ids renumbered.  Hour 0
    is exactly gen_gamma_trace(profile[0], shape, 1 h, lengths, seed * 1000)."""
    profile = profile or diurnal_profile()
    lengths = lengths or P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7))
    segs = []
    next_id = 0
    for h, rps in enumerate(profile):
        s = gen_segment(rps, shape, HOUR_MS, lengths, seed * 1000 + h)
        s["arrival_ms"] += h * HOUR_MS
        s["id"] = np.arange(next_id, next_id + len(s), dtype=np.int64)
        next_id += len(s)
        segs.append(s)
    return DayTrace(np.concatenate(segs), len(profile) * HOUR_MS)


@dataclass
class Window:
    requests: np.ndarray
    duration_ms: float

    def c_trace(self) -> _abi.bs_trace:
        t = _abi.bs_trace()
        t.n = len(self.requests)
        t.requests = self.requests.ctypes.data_as(C.POINTER(_abi.bs_request))
        t.duration_ms = self.duration_ms
        return t


def split(day: DayTrace, window_ms: float) -> list:
    """split_windows (workload.hpp:184-201) on a buffer."""
    if window_ms <= 0.0:
        raise P.ParameterError("split_windows: window_ms must be > 0")
    n = max(1, int(math.ceil(day.duration_ms / window_ms)))
    arr = day.requests["arrival_ms"]
    idx = np.minimum((arr / window_ms).astype(np.int64), n - 1)  # int(): truncation, arrivals >= 0
    bounds = np.searchsorted(idx, np.arange(n + 1), side="left")
    wins = []
    for w in range(n):
        sub = day.requests[bounds[w]:bounds[w + 1]].copy()
        sub["arrival_ms"] -= float(w) * window_ms
        wins.append(Window(sub, min(window_ms, day.duration_ms - float(w) * window_ms)))
    return wins


def peak_rps(win: Window, subwindow_s: float) -> float:
    """peak_rps (placement.hpp:513-527)."""
    if len(win.requests) == 0:
        raise P.ParameterError("peak_rps: empty trace")
    w_ms = subwindow_s * 1000.0
    nw = int(win.duration_ms / w_ms)
    if nw < 1:
        return float(len(win.requests)) / (win.duration_ms / 1000.0) if win.duration_ms > 0.0 else 0.0
    idx = (win.requests["arrival_ms"] / w_ms).astype(np.int64)
    counts = np.bincount(idx[idx < nw], minlength=nw)
    return float(counts.max()) / subwindow_s


@dataclass
class DayResult:
    """Per scenario and window: the plans (counts, objective, GPUs and
    routing weights; the config tables stay on the device side), the
    two-tier replay summary."""
    plans: list = field(default_factory=list)        # [scenario][window] WindowPlans
    results: list = field(default_factory=list)      # [scenario][window] ReplayResult
    seconds: dict = field(default_factory=dict)
    n_windows: int = 0
    decisions: int = 0


def run_day_sweep(days: list, window_ms: float, cfg: P.RunnerConfig, models: P.ModelSet,
                  device: P.Device | None = None) -> DayResult:
    """run_experiment (runner.hpp:155-172) with the two-tier policy for every
    trace in `days`, all scenarios' windows in each device call."""
    dev = device or P.default_device()
    cfg.validate()
    opts = cfg.plan
    t0 = time.perf_counter()
    wins = [split(d, window_ms) for d in days]
    hist = []  # window w planned from window w - 1 (the first from itself)
    for ws in wins:
        for w in range(len(ws)):
            h = ws[0] if w == 0 else ws[w - 1]
            if len(h.requests) == 0:
                raise P.ParameterError("plan_window: empty history")
            hist.append(h)
    probes = hist if opts.probe_trace is None else None
    if probes is None:
        raise P.ParameterError("run_day_sweep: a fixed probe trace is not supported")
    candidates = P.enumerate_candidates(cfg.ladder, cfg.tp_options)
    nt, ncand = len(probes), len(candidates)
    trs = (_abi.bs_trace * nt)()
    for i, h in enumerate(probes):
        trs[i] = h.c_trace()
    cs, cp, cg = P.c_slo(cfg.slo), P.c_policy(opts.policy), P.c_search(opts.search)
    cands = P.c_candidates(candidates)
    tab = (_abi.bs_table_entry * (nt * ncand))()
    t1 = time.perf_counter()
    dev.check(dev._lib.bs_goodput_tables(dev.handle, dev.models(models), trs, nt, C.byref(cs), C.byref(cp),
                                         C.byref(cg), cands, ncand, tab))
    t2 = time.perf_counter()
    targets = [peak_rps(h, opts.peak_subwindow_s) for h in hist]  # predict_next_window is the identity
    # every window's ILP and max-throughput baseline, straight from the table
    # buffer (bs_placement_solve_batch); plans rebuilt from the counts
    counts = np.zeros((2 * nt, ncand), dtype=np.int64)
    arr = (_abi.bs_placement_problem * (2 * nt))()
    esz = C.sizeof(_abi.bs_table_entry)
    base = C.addressof(tab)
    for t in range(nt):
        for j in range(2):
            q = arr[2 * t + j]
            q.table = base + t * ncand * esz
            q.n = ncand
            q.total_gpus = cfg.total_gpus
            q.target_rps = targets[t]
            q.alpha = opts.alpha
            q.max_throughput = j
            q.max_freq_mhz = cfg.ladder.max_mhz() if j else 0.0
            q.counts = counts[2 * t + j].ctypes.data_as(C.POINTER(C.c_int64))
    sol = (_abi.bs_placement_solution * (2 * nt))()
    dev.check(dev._lib.bs_placement_solve_batch(dev.handle, arr, 2 * nt, sol))
    for k in range(2 * nt):  # the reference's order: window by window, ILP before the baseline
        if sol[k].status != _abi.BS_OK:
            P.raise_status(sol[k].status, sol[k].error.decode())
    phase = [int(c.phase) for c in candidates]
    r_all = np.array([[tab[t * ncand + i].r_c for i in range(ncand)] for t in range(nt)])
    fmax = cfg.ladder.max_mhz()
    keep_max = np.array([c.base_freq_mhz == fmax for c in candidates])

    def plan_of(k: int) -> P.PlacementPlan:
        t, j = divmod(k, 2)
        r = np.where(keep_max, r_all[t], 0.0) if j else r_all[t]
        cnt = counts[k].tolist()
        pr = [0.0, 0.0]
        for i, n in enumerate(cnt):  # derive_routing_weights (placement.hpp:264-280)
            if n:
                pr[0 if phase[i] == P.Phase.prefill else 1] += float(n) * r[i]
        inst = [P.ClusterInstance(candidates[i], r[i] / pr[0 if phase[i] == P.Phase.prefill else 1])
                for i, n in enumerate(cnt) for _ in range(n)]
        return P.PlacementPlan(cnt, [], sol[k].objective_w, targets[t], opts.alpha, cfg.total_gpus,
                               sol[k].gpus_used, inst)

    solved = [plan_of(k) for k in range(2 * nt)]
    t3 = time.perf_counter()
    # the two-tier replay of every (scenario, window) in one call
    keep: list = []
    rc = _abi.bs_replay_config()
    rc.mpc = P.c_mpc_config(cfg.mpc_config(), keep)
    rc.decode = P.c_decode_config(cfg.decode_config(), keep)
    rc.controlled = 1
    rc.policy = P.c_policy(cfg.scheduler)
    rc.slo = P.c_slo(cfg.slo)
    rc.switch_latency_ms = cfg.switch_latency_ms
    rc.horizon_ms = -1.0
    rc.rampup_s = cfg.rampup_s
    cfgs = (_abi.bs_replay_config * 1)(rc)
    flat = [w for ws in wins for w in ws]
    scs = (_abi.bs_scenario * len(flat))()
    for i, w in enumerate(flat):
        plan = solved[2 * i]
        scs[i].trace = w.c_trace()
        inst = (_abi.bs_cluster_instance * max(1, len(plan.instances)))()
        for j, ci in enumerate(plan.instances):
            inst[j].config.phase, inst[j].config.tp = int(ci.config.phase), ci.config.tp
            inst[j].config.base_freq_mhz, inst[j].weight = ci.config.base_freq_mhz, ci.weight
        keep.append(inst)
        scs[i].instances = C.cast(inst, C.POINTER(_abi.bs_cluster_instance))
        scs[i].n_instances = len(plan.instances)
        scs[i].config = 0
    out = (_abi.bs_replay_summary * len(flat))()
    mh = dev.models(models)
    t4 = time.perf_counter()
    dev.check(dev._lib.bs_replay(dev.handle, mh, mh, cfgs, 1, scs, len(flat), out, None, None))
    t5 = time.perf_counter()
    res = DayResult(n_windows=len(flat))
    i = 0
    for ws in wins:
        pl, rr = [], []
        for _ in ws:
            pl.append(P.WindowPlans(targets[i], [], solved[2 * i], solved[2 * i + 1]))
            r = P.summary_from_c(out[i])
            rr.append(r)
            res.decisions += r.n_decisions
            i += 1
        res.plans.append(pl)
        res.results.append(rr)
    res.seconds = {"windows": t1 - t0, "tables": t2 - t1, "ilp": t3 - t2, "replay_inputs": t4 - t3,
                   "replay": t5 - t4, "total": time.perf_counter() - t0}
    return res

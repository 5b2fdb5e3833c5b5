"""Benchmark of the BiScale decision-evaluation hot path on B200 (sm_100a).

Workload (BASELINE.json configs[1], "C2"): exhaustive prefill MPC, horizon 6 x
16 frequency rungs = 16,777,216 candidate trajectories per decision, on a
corpus of synthetic Llama-3.3-70B-shaped queue snapshots.  A
step = one pass of the decision path over one batch of decisions: projection,
the K x N (latency, power) tables, the rollout of every trajectory, and the
per-decision argmin.

  value  trajectories/s with the batch resident in HBM (CUDA events on the
         library's stream; L2 flushed between steps)
  e2e    the same metric through the C ABI one-shot call bs_mpc_exhaustive
         with host buffers: packing, H2D, kernels, D2H and expansion timed
  roofline  leaf kernel (the rollout sweep) against the measured FP64
         (non-FMA) issue rate: algorithmic work W = 5H + 2 = 32 FP64 ops per
         trajectory x trajectories per launch / leaf time
  cpu_baseline  the unmodified reference (oracle/_ref: the reference's own
         exhaustive loop over meets_slo + time_weighted_power,
         tests/test_dvfs.cpp:74-94) on the host cores, bounded sample

Extra keys, one object per other BASELINE.json configuration (each with its
own device timing, the reference on the host cores and a parity check):
  c1_demo        configs[0]: 1P + 1D demo-shaped replay, decisions/s by trigger,
                 plus per-decision controller-call latency (p50 / p99)
  c3_placement   configs[2]: config table + ILP, placement configs/s
  c4_replay      configs[3]-shaped what-if replay sweep, scenarios/s
  c4_experiment  configs[3]'s window loop: run_experiment over a bursty hour
                 (plan per window + 3 policies replayed), window runs/s
  c5_greedy      configs[4] greedy MPC (H8 x 24 levels), decisions/s
  c5_exhaustive  configs[4] exhaustive MPC (24^8 per decision), decisions/s
(`--only c1|c3|c4|c4x|c5g|c5x` runs one alone; `--no-extras` skips them.)

Multi-GPU (torchrun): weak scaling, every rank evaluates its own corpus
(independent decisions), no data-path collective; max-over-ranks time.  The
C4/C5 extras split their fixed scenario sets across ranks.
`--impl reference` times the reference CPU implementation instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HORIZON = 6
LEVELS = 16
TRAJ_PER_DECISION = LEVELS ** HORIZON
W_OPS = 5 * HORIZON + 2
METRIC = "MPC trajectories evaluated/sec & decisions/sec; placement configs/sec"
UNIT = "trajectories/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--decisions", type=int, default=1024, help="decisions per step per GPU")
    ap.add_argument("--ttft", type=float, default=600.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU baseline sample duration")
    ap.add_argument("--no-extras", action="store_true", help="skip the C3/C4/C5 sub-benchmarks")
    ap.add_argument("--only", choices=["c1", "c2l", "c3", "c4", "c4d", "c4x", "c5g", "c5x"], default=None,
                    help="run one sub-benchmark alone and print its JSON object")
    ap.add_argument("--c4-scenarios", type=int, default=1024)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for --gpus > 1 (gloo: CPU tests of the rank plumbing)")
    ap.add_argument("--c4-day-scenarios", type=int, default=8, help="full-day C4 scenarios per rank")
    ap.add_argument("--c3-windows", type=int, default=24, help="1-hour windows in the C3 table stream")
    ap.add_argument("--c5x-decisions", type=int, default=4096)
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_run(models, cfg, pol, snaps, threads: int) -> tuple:
    """The reference's exhaustive loop (oracle/_ref) over `snaps`, one decision
    per host thread at a time; returns (seconds, results)."""
    import oracle
    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P

    ref = oracle.load_ref()
    keep: list = []
    cm = P.c_model_set(models, keep)
    cc = P.c_mpc_config(cfg, keep)
    cp = P.c_policy(pol)
    probs = P.c_problems(snaps, None, keep)
    out = (A.bs_mpc_result * len(snaps))()
    t0 = time.perf_counter()
    rc = ref.ref_exhaustive_batch(C.byref(cm), C.byref(cc), C.byref(cp), probs, len(snaps), out, threads)
    dt = time.perf_counter() - t0
    if rc != 0:
        raise RuntimeError(f"reference exhaustive failed: {ref.last_error()}")
    return dt, out


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    rank, local, world = dist_env()
    if rank != 0:
        return 0
    from paper_2602_18755_b200 import workloads as Wk

    threads = cpu_threads()
    models, cfg, pol, snaps = Wk.c2_corpus(0xC2, threads * (args.steps + args.warmup), args.ttft)
    times, n_dec = [], threads
    for s in range(args.warmup + args.steps):
        sample = snaps[s * threads:(s + 1) * threads]
        dt, _ = cpu_reference_run(models, cfg, pol, sample, threads)
        if s >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = n_dec * args.steps * TRAJ_PER_DECISION / total
    sample_desc = (f"{n_dec} C2 decisions per step (one per host thread), H=6 x 16 rungs, "
                   f"reference loop tests/test_dvfs.cpp:74-94 over meets_slo + time_weighted_power; cpu={cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 exhaustive prefill MPC, horizon 6 x 16 levels (16.7M trajectories/decision)",
                       "decisions_per_step": n_dec, "ttft_ms": args.ttft},
            "decisions_per_s": n_dec * args.steps / total,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample_desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Sub-benchmarks of the other BASELINE.json configurations (extra keys of the
# JSON line; the headline `value` stays C2).  Each times the device path,
# times the reference on the host cores on a bounded sample of the same
# work, and checks the device results against the reference's.
# ---------------------------------------------------------------------------

def roofline_obj(algorithmic: float, peak: float, leaf_ms: float, traffic, executed, source) -> dict:
    """The sweep kernel (dominant, ~60 % of a step) against the FP64 pipe.
    frac / achieved: what the kernel EXECUTES -- ncu's FP64-pipe-active
    fraction of the same kernel at this configuration (profiles/
    leaf_traffic.json) times the measured non-FMA DADD issue peak;
    algorithmic_equiv: SURVEY §8d's W = 5H + 2 = 32 FP64 ops per trajectory x
    the trajectories one launch decides / the launch's live CUDA-event time
    (> 1: the exact pruned search executes far fewer than W ops per
    trajectory)."""
    ex = (executed or {}).get("fp64_pipe_active_frac")
    return {"bound": "fp64", "unit": "TFLOP/s", "peak": peak / 1e12,
            "frac": ex, "achieved": ex * peak / 1e12 if ex is not None else None,
            "issue_slots_busy_frac": (executed or {}).get("issue_slots_busy_frac"),
            "traffic": traffic, "kernel": "sweep_kernel (exhaustive leaf sweep)", "kernel_ms_live": leaf_ms,
            "executed": executed, "source": source,
            "algorithmic_equiv": {"achieved": algorithmic / 1e12, "frac": algorithmic / peak,
                                  "note": "W = 32 FP64 ops x 1024 x 16.7M trajectories / live sweep time"},
            "note": "peak = measured non-FMA DADD issue rate of this box (bs_fp64_peak, 148 SM x 64 lanes x f); "
                    "frac = executed FP64-pipe utilisation from the committed ncu capture of this kernel"}


def _dist_max(x: float, world: int, local: int) -> float:
    if world == 1:
        return x
    from paper_2602_18755_b200 import sharding as S

    return S.max_over_ranks(x, device=f"cuda:{local}")


def _barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def bench_c3(dev, with_cpu: bool, repeats: int = 3, rank: int = 0, world: int = 1, local: int = 0,
             n_windows: int = 24) -> dict:
    """configs[2]: coarse-tier placement for a 16-GPU cluster over a bursty
    1-hour window: the config table (goodput search + E_c of every
    candidate, build_config_table placement.hpp:240-260) + the ILP."""
    import ctypes as C

    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as Wk

    lad = Wk.ladder(16)
    models = Wk.llama_models(lad)
    base = P.gen_gamma_trace(12.0, 0.5, 3600e3, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 7)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    pol, slo, search = P.SchedulerPolicy(max_batch_tokens=2048), P.SLOSpec(600.0, 100.0), P.GoodputSearch()
    P.build_config_table(cands, base, slo, models, pol, search, device=dev)  # warm-up
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        table = P.build_config_table(cands, base, slo, models, pol, search, device=dev)
        times.append(time.perf_counter() - t0)
    st = (C.c_double * 8)()
    dev._lib.bs_ctx_stats(dev.handle, st, 8)
    t0 = time.perf_counter()
    plan = P.solve_placement(P.PlacementProblem(table, 16, P.peak_rps(base, 10.0), 0.05), dev)
    t_ilp = time.perf_counter() - t0
    t_table = statistics.median(times)
    k_max = int(base.mean_rps() // search.tolerance_rps)
    # the stream of bursty 1-hour windows (configs[2]: "over bursty 1-hour trace windows"): a day of
    # consecutive windows, their tables built concurrently on one GPU
    day = P.gen_gamma_trace(12.0, 0.5, n_windows * 3600e3, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)),
                            7)
    wins = P.split_windows(day, 3600e3)
    if world > 1:  # windows sharded across ranks, tables all-gathered
        from paper_2602_18755_b200 import sharding as S

        lo, hi = S.shard_bounds(len(wins), rank, world)
        P.build_config_tables(wins[lo:hi], cands, slo, models, pol, search, dev)  # warm-up
        _barrier(world)
        t0 = time.perf_counter()
        mine = P.build_config_tables(wins[lo:hi], cands, slo, models, pol, search, dev)
        t_stream = _dist_max(time.perf_counter() - t0, world, local)
        gathered = S.gather_tables(mine, len(wins), device=f"cuda:{local}")
        assert len(gathered) == len(wins)
    else:
        P.build_config_tables(wins, cands, slo, models, pol, search, dev)  # warm-up (one probe grid for all windows)
        t0 = time.perf_counter()
        P.build_config_tables(wins, cands, slo, models, pol, search, dev)
        t_stream = time.perf_counter() - t0
    out = {"workload": "C3: bursty 1-hour gamma(0.5) windows at 12 rps, 128 candidates per window (2 phases x "
                       "TP{1,2,4,8} x 16 rungs), max_batch_tokens 2048, G = 16", "requests": len(base.requests),
           "value": len(wins) * len(cands) / t_stream, "unit": "placement configs/s",
           "value_note": f"{len(wins)} consecutive windows, all tables in one probe grid ({t_stream:.2f} s); one table "
                         "alone is bound by its longest probe (table_s)",
           "single_table_configs_per_s": len(cands) / t_table, "table_s": t_table,
           "probes_per_s": k_max * len(cands) / t_table, "ilp_s": t_ilp, "gpus_used": plan.gpus_used,
           "objective_w": plan.objective_w, "phase_ms": {"mask": st[0], "probe": st[1], "energy": st[2]},
           "events_simulated": st[4],
           "probes": {"grid": st[5], "skipped_off_path": st[6], "abandoned_off_path": st[7],
                      "note": "every (candidate, rate step) probe is launched in search-tree order; probes the "
                              "reference's binary search can no longer visit are skipped or abandoned"},
           "e2e_note": "value is end to end through pdsim.build_config_table "
                                                 "(host trace in, table out)"}
    if with_cpu:
        import oracle

        ref = oracle.load_ref()
        keep: list = []
        cm, ct = P.c_model_set(models, keep), P.c_trace(base, keep)
        outc = (A.bs_table_entry * len(cands))()
        t0 = time.perf_counter()
        rc = ref.ref_config_table(C.byref(cm), C.byref(ct), C.byref(P.c_slo(slo)), C.byref(P.c_policy(pol)),
                                  C.byref(P.c_search(search)), P.c_candidates(cands), len(cands), outc)
        t_cpu = time.perf_counter() - t0
        same = rc == 0 and all((e.r_c, e.e_c, e.saturated, e.error) == (o.r_c, o.e_c, o.saturated, o.error)
                               for e, o in zip(table, [P.entry_from_c(outc[i]) for i in range(len(cands))]))
        out["cpu_baseline"] = {"value": len(cands) / t_cpu, "unit": "placement configs/s", "cores": cpu_threads(),
                               "kind": "reference", "seconds": t_cpu,
                               "sample": "the whole table: build_config_table (std::async per candidate)"}
        out["identical_to_reference"] = bool(same)
    return out


def bench_c4(dev, rank: int, world: int, local: int, n_scen: int, with_cpu: bool) -> dict:
    """configs[3]-shaped: what-if replay sweep (trace seeds x SLO pairs) of
    simulate_cluster with per-iteration two-tier decisions + the report,
    scenarios sharded across ranks."""
    import ctypes as C

    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import sharding as S
    from paper_2602_18755_b200 import workloads as Wk

    models, scs_all = Wk.c4_scenarios(n_scen)
    lo, hi = S.shard_bounds(len(scs_all), rank, world)
    scs = scs_all[lo:hi]
    lib = dev._lib
    keep: list = []
    cfgs, cscs, _ = P.c_replay_inputs(scs, keep)
    n = len(scs)
    outs = (A.bs_replay_summary * max(1, n))()
    mh = dev.models(models)
    dev.check(lib.bs_replay(dev.handle, mh, mh, cfgs, n, cscs, n, outs, None, None))  # warm-up
    st = (C.c_double * 8)()
    times, kern = [], []
    for _ in range(3):
        _barrier(world)
        t0 = time.perf_counter()
        dev.check(lib.bs_replay(dev.handle, mh, mh, cfgs, n, cscs, n, outs, None, None))
        times.append(time.perf_counter() - t0)
        lib.bs_ctx_stats(dev.handle, st, 8)
        kern.append([st[i] for i in range(4)])
    e2e = _dist_max(statistics.median(times), world, local)
    kms = _dist_max(statistics.median(sum(k) for k in kern), world, local)
    dec = sum(outs[i].n_decisions for i in range(n))
    h2d, d2h = C.c_uint64(), C.c_uint64()
    lib.bs_ctx_last_transfer(dev.handle, C.byref(h2d), C.byref(d2h))
    out = {"workload": f"C4-shaped: {len(scs_all)} what-if scenarios (8 trace seeds x (TTFT, TPOT) pairs), 5-min "
                       "gamma(0.5) windows at 12 rps, 2P(tp2)+2D(tp4), greedy MPC K=8 N=7 + decode slack DVFS",
           "value": len(scs_all) / (kms / 1e3), "unit": "scenarios/s", "kernel_ms": kms,
           "decisions_per_s_rank0": dec / (kms / 1e3),
           "phase_ms_rank0": dict(zip(["prefill", "route", "decode", "report"],
                                      [statistics.median(k[i] for k in kern) for i in range(4)])),
           "e2e": {"value": len(scs_all) / e2e, "unit": "scenarios/s", "h2d_bytes_per_step": int(h2d.value),
                   "d2h_bytes_per_step": int(d2h.value)},
           "all_ok": all(outs[i].status == 0 for i in range(n))}
    if with_cpu and rank == 0:
        import oracle

        ref = oracle.load_ref()
        m = min(32, n)
        k2: list = []
        rc_cfgs, rc_scs, _ = P.c_replay_inputs(scs[:m], k2)
        rout = (A.bs_replay_summary * m)()
        cm = P.c_model_set(models, k2)
        t0 = time.perf_counter()
        rc = ref.ref_replay(C.byref(cm), C.byref(cm), rc_cfgs, rc_scs, m, rout, None, None, cpu_threads())
        t_cpu = time.perf_counter() - t0
        names = [f for f, _ in A.bs_replay_summary._fields_ if f not in ("_pad", "decisions_by_trigger")]
        same = rc == 0 and all(all(getattr(outs[i], f) == getattr(rout[i], f) or
                                   (getattr(outs[i], f) != getattr(outs[i], f) and getattr(rout[i], f) !=
                                    getattr(rout[i], f)) for f in names) for i in range(m))
        out["cpu_baseline"] = {"value": m / t_cpu, "unit": "scenarios/s", "cores": cpu_threads(),
                               "kind": "reference", "seconds": t_cpu,
                               "sample": f"first {m} scenarios: pdsim::simulate_cluster + trim_steady_state + "
                                         "make_report, one scenario per thread"}
        out["identical_on_sample"] = bool(same)
    return out


def bench_c4_day(dev, rank: int, world: int, local: int, n_scen: int, with_cpu: bool) -> dict:
    """configs[3] as configured, on a declared contiguous fraction of the
    scenario set: full 24 h diurnal days (24 one-hour gamma(0.5) segments,
    6 -> 20 rps) planned per 5-minute window (288 windows: config table from
    the previous window, ILP, max-throughput baseline) and replayed with the
    two-tier controllers -- run_experiment (runner.hpp:155-172) per scenario,
    all scenarios' windows in four device calls (daysim.run_day_sweep).
    Scenarios s = 0 .. n_scen - 1 of each rank (trace seed 1000 + global
    index) at the SLO pair (600, 100) ms."""
    from paper_2602_18755_b200 import daysim as Dy
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as Wk

    lad = Wk.ladder(8)
    models = Wk.llama_models(lad)
    cfg = P.RunnerConfig(slo=P.SLOSpec(600.0, 100.0), total_gpus=16, tp_options=[1, 2, 4, 8], ladder=lad,
                         scheduler=P.SchedulerPolicy(max_batch_tokens=2048), rampup_s=30.0)
    cfg.plan.policy = P.SchedulerPolicy(max_batch_tokens=2048)
    first = rank * n_scen
    t0 = time.perf_counter()
    days = [Dy.gen_day(1000 + first + s) for s in range(n_scen)]
    t_gen = time.perf_counter() - t0
    Dy.run_day_sweep([Dy.DayTrace(days[0].requests[days[0].requests["arrival_ms"] < Dy.HOUR_MS], Dy.HOUR_MS)],
                     300e3, cfg, models, dev)  # warm-up (one hour of one scenario)
    _barrier(world)
    t0 = time.perf_counter()
    res = Dy.run_day_sweep(days, 300e3, cfg, models, dev)
    t_run = _dist_max(time.perf_counter() - t0, world, local)
    n_req = sum(len(d.requests) for d in days)
    out = {"workload": f"C4 as configured on {n_scen * world} of the 1024 scenarios (declared contiguous fraction: "
                       f"scenarios 0..{n_scen * world - 1}, trace seeds 1000+): 24 h diurnal day (24 x 1 h gamma(0.5), "
                       "6 -> 20 rps), 288 five-minute windows each planned from the previous one (config table of "
                       "2 phases x TP{1,2,4,8} x 8 rungs, ILP + max-throughput baseline, 16 GPUs) and replayed with the "
                       "two-tier controllers, SLO 600/100 ms",
           "value": n_scen * world / t_run, "unit": "scenarios/s", "seconds": t_run,
           "windows_per_s": res.n_windows * world / t_run, "decisions_per_s_rank0": res.decisions / t_run,
           "requests_per_scenario": n_req // max(1, n_scen), "phase_s_rank0": res.seconds,
           "trace_synthesis_s_rank0": t_gen,
           "timing": "end to end through daysim.run_day_sweep (host traces in, per-window plans and reports out)"}
    if with_cpu and rank == 0:
        import oracle

        ref = oracle.load_ref()
        keep: list = []
        c = oracle.ref_runner_config()
        c.slo = P.c_slo(cfg.slo)
        c.total_gpus = cfg.total_gpus
        tps = (C.c_int32 * 4)(*cfg.tp_options)
        ld = (C.c_double * len(lad.freqs_mhz))(*lad.freqs_mhz)
        keep += [tps, ld]
        c.n_tp, c.tp_options, c.ladder, c.n_ladder = 4, tps, ld, len(lad.freqs_mhz)
        c.scheduler = P.c_policy(cfg.scheduler)
        c.alpha, c.peak_subwindow_s = cfg.plan.alpha, cfg.plan.peak_subwindow_s
        c.search, c.plan_policy = P.c_search(cfg.plan.search), P.c_policy(cfg.plan.policy)
        c.rampup_s, c.switch_latency_ms = cfg.rampup_s, cfg.switch_latency_ms
        c.mpc_k, c.mpc_n, c.mpc_margin = cfg.mpc_horizon_k, cfg.mpc_ladder_n, cfg.mpc_margin
        c.kv_threshold, c.decode_margin = cfg.kv_threshold, cfg.decode_margin
        # the reference's run_experiment on scenario 0's first hour (its first 12 windows), two-tier policy
        hour0 = P.gen_gamma_trace(Dy.diurnal_profile()[0], 0.5, Dy.HOUR_MS,
                                  P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 1000 * 1000)
        o = (oracle.ref_window_run * 16)()
        n_out, tt = C.c_int(), C.c_int32()
        cm, ct = P.c_model_set(models, keep), P.c_trace(hour0, keep)
        pa = (C.c_int32 * 1)(int(P.Policy.two_tier))
        t0 = time.perf_counter()
        rc = ref.ref_run_experiment(C.byref(cm), C.byref(ct), 300e3, pa, 1, C.byref(c), o, 16, C.byref(n_out),
                                    C.byref(tt))
        t_cpu = time.perf_counter() - t0
        same = rc == 0 and n_out.value == 12 and all(
            (o[w].gpus_used, o[w].objective_w, o[w].report.n_decisions, o[w].report.prefill_energy_j,
             o[w].report.decode_energy_j, o[w].report.ttft_violations) ==
            (res.plans[0][w].ilp.gpus_used, res.plans[0][w].ilp.objective_w, res.results[0][w].n_decisions,
             res.results[0][w].report.prefill_energy_j, res.results[0][w].report.decode_energy_j,
             res.results[0][w].report.ttft_violations) for w in range(12))
        w_per_s = n_out.value / t_cpu
        out["cpu_baseline"] = {"value": w_per_s / 288.0, "unit": "scenarios/s", "cores": cpu_threads(),
                               "kind": "reference", "seconds": t_cpu, "windows_per_s": w_per_s,
                               "sample": "scenario 0's first hour (12 of its 288 windows): pdsim::run_experiment, "
                                         "two-tier policy (build_config_table on std::async threads); scenarios/s "
                                         "= windows/s / 288"}
        out["identical_on_sample"] = bool(same)
    return out


def bench_c1(dev, with_cpu: bool, n_rep: int = 296) -> dict:
    """configs[0]: the demo-shaped 1P + 1D replay with per-iteration two-tier
    decisions (one scenario, so latency-bound: the serial chain of one
    prefill instance's event loop), decisions/s split by trigger; plus the
    per-decision latency of the drop-in controller call (one greedy decision
    per bs_mpc_greedy call with host buffers, as GpuPrefillMpcController::
    decide makes it) over the C1 snapshot corpus."""
    import ctypes as C

    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as Wk

    models, sc = Wk.c1_scenario()
    lib = dev._lib
    keep: list = []
    cfgs, cscs, _ = P.c_replay_inputs([sc], keep)
    out = (A.bs_replay_summary * 1)()
    mh = dev.models(models)
    dev.check(lib.bs_replay(dev.handle, mh, mh, cfgs, 1, cscs, 1, out, None, None))  # warm-up
    st = (C.c_double * 8)()
    times, kern = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        dev.check(lib.bs_replay(dev.handle, mh, mh, cfgs, 1, cscs, 1, out, None, None))
        times.append(time.perf_counter() - t0)
        lib.bs_ctx_stats(dev.handle, st, 8)
        kern.append([st[i] for i in range(4)])
    kms, e2e = statistics.median(sum(k) for k in kern), statistics.median(times)
    dec = out[0].n_decisions
    res = {"workload": "C1: demo trace parameters (14 rps, 600 s, seed 7, lognormal 6.2/0.4 in, 2.9/0.5 out) with "
                       "Poisson arrivals, 1P(tp2)+1D(tp4), greedy MPC K=8 N=7 of the 8-rung ladder + decode slack "
                       "DVFS, one scenario",
           "value": dec / (kms / 1e3), "unit": "decisions/s", "kernel_ms": kms, "decisions": int(dec),
           "decisions_by_trigger": dict(zip(["boundary", "arrival", "safety"],
                                            (int(x) for x in out[0].decisions_by_trigger))),
           "phase_ms": dict(zip(["prefill", "route", "decode", "report"],
                                [statistics.median(k[i] for k in kern) for i in range(4)])),
           "e2e": {"value": dec / e2e, "unit": "decisions/s"}, "status": int(out[0].status)}
    # throughput: C1 replicas over trace seeds 7, 8, ... (independent scenarios, one launch)
    reps = [sc] + [Wk.c1_scenario(seed=7 + i)[1] for i in range(1, n_rep)]
    k3: list = []
    r_cfgs, r_scs, _ = P.c_replay_inputs(reps, k3)
    rout_all = (A.bs_replay_summary * n_rep)()
    dev.check(lib.bs_replay(dev.handle, mh, mh, r_cfgs, n_rep, r_scs, n_rep, rout_all, None, None))
    rk = []
    for _ in range(3):
        dev.check(lib.bs_replay(dev.handle, mh, mh, r_cfgs, n_rep, r_scs, n_rep, rout_all, None, None))
        lib.bs_ctx_stats(dev.handle, st, 8)
        rk.append(sum(st[i] for i in range(4)))
    rdec = sum(rout_all[i].n_decisions for i in range(n_rep))
    res["replicas"] = {"scenarios": n_rep, "value": rdec / (statistics.median(rk) / 1e3), "unit": "decisions/s",
                       "kernel_ms": statistics.median(rk), "decisions": int(rdec),
                       "all_ok": all(rout_all[i].status == 0 for i in range(n_rep)),
                       "first_matches_single": all(getattr(rout_all[0], f) == getattr(out[0], f)
                                                   for f in ("n_decisions", "prefill_energy_j", "decode_energy_j"))}
    # per-decision latency of the controller call (pack + H2D + one warp + D2H)
    mc, cfg, pol, snaps = Wk.c1_corpus(n=256)
    for q in snaps[:8]:
        P.greedy_freq_select(q, cfg, mc, pol, dev)
    lat = []
    for q in snaps:
        t0 = time.perf_counter()
        P.greedy_freq_select(q, cfg, mc, pol, dev)
        lat.append((time.perf_counter() - t0) * 1e6)
    lat.sort()
    res["decision_latency_us"] = {"p50": lat[len(lat) // 2], "p99": lat[int(0.99 * (len(lat) - 1))],
                                  "calls": len(lat), "path": "pdsim.greedy_freq_select -> bs_mpc_greedy, n=1"}
    # the same calls with the snapshots pre-marshalled: the C ABI alone (pack + H2D + kernel + D2H + sync)
    carr = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
    parr = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
    probs = [P.c_problems([q], None, keep) for q in snaps]
    one = (A.bs_mpc_result * 1)()
    mch = dev.models(mc)
    raw = []
    for pr in probs:
        t0 = time.perf_counter()
        dev.check(lib.bs_mpc_greedy(dev.handle, mch, carr, parr, 1, pr, 1, one))
        raw.append((time.perf_counter() - t0) * 1e6)
    raw.sort()
    res["decision_latency_us"]["c_abi_p50"] = raw[len(raw) // 2]
    res["decision_latency_us"]["c_abi_p99"] = raw[int(0.99 * (len(raw) - 1))]
    if with_cpu:
        import oracle

        ref = oracle.load_ref()
        k2: list = []
        rc_cfgs, rc_scs, _ = P.c_replay_inputs([sc], k2)
        rout = (A.bs_replay_summary * 1)()
        cm = P.c_model_set(models, k2)
        t0 = time.perf_counter()
        rc = ref.ref_replay(C.byref(cm), C.byref(cm), rc_cfgs, rc_scs, 1, rout, None, None, 1)
        t_cpu = time.perf_counter() - t0
        names = [f for f, _ in A.bs_replay_summary._fields_ if f not in ("_pad", "decisions_by_trigger")]
        same = rc == 0 and all(getattr(out[0], f) == getattr(rout[0], f) or
                               (getattr(out[0], f) != getattr(out[0], f) and getattr(rout[0], f) !=
                                getattr(rout[0], f)) for f in names) and \
            list(out[0].decisions_by_trigger) == list(rout[0].decisions_by_trigger)
        res["cpu_baseline"] = {"value": rout[0].n_decisions / t_cpu, "unit": "decisions/s", "cores": 1,
                               "kind": "reference", "seconds": t_cpu,
                               "sample": "the whole C1 scenario: pdsim::simulate_cluster with TwoTierFactory "
                                         "controllers + trim_steady_state + make_report, one thread"}
        res["identical"] = bool(same)
    return res


def bench_c5(dev, mode: str, rank: int, world: int, local: int, n_dec: int, with_cpu: bool) -> dict:
    """configs[4]: horizon-8 MPC on a 24-level grid, greedy or exhaustive,
    decisions sharded across ranks."""
    import ctypes as C
    import random

    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import sharding as S
    from paper_2602_18755_b200 import workloads as Wk

    models, cfg, pol, snaps_all = Wk.c5_corpus(0xC5, n_dec)
    lo, hi = S.shard_bounds(len(snaps_all), rank, world)
    snaps = snaps_all[lo:hi]
    lib = dev._lib
    keep: list = []
    cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
    cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
    probs = P.c_problems(snaps, None, keep)
    n = len(snaps)
    res = (A.bs_mpc_result * max(1, n))()
    mh = dev.models(models)
    fn = lib.bs_mpc_greedy if mode == "greedy" else lib.bs_mpc_exhaustive
    dev.check(fn(dev.handle, mh, cc, cp, 1, probs, n, res))
    times = []
    for _ in range(3):
        _barrier(world)
        t0 = time.perf_counter()
        dev.check(fn(dev.handle, mh, cc, cp, 1, probs, n, res))
        times.append(time.perf_counter() - t0)
    t = _dist_max(statistics.median(times), world, local)
    out = {"workload": f"C5: {len(snaps_all)} scenarios, horizon 8 on a 24-level ladder, {mode} MPC",
           "value": len(snaps_all) / t, "unit": "decisions/s", "seconds": t,
           "timing": "end to end through the C ABI with host buffers (pack + H2D + kernels + D2H)",
           "feasible_decisions_rank0": sum(res[i].feasible for i in range(n))}
    if mode == "greedy":
        out["mutations_per_s_rank0"] = sum(res[i].eval_count for i in range(n)) / t
    else:
        traj = sum(res[i].trajectories for i in range(n))
        out["trajectories_per_s"] = traj * world / t
        out["roofline_note"] = "24^8 = 1.1e11 trajectories per decision, W = 5*8+2 = 42 FP64 ops each: " \
                               f"{traj * world * 42 / t / 1e12:.0f} TFLOP/s-equivalent algorithmic (pruned search)"
    if not with_cpu or rank != 0:
        return out
    import oracle

    ref = oracle.load_ref()
    cm = P.c_model_set(models, keep)
    threads = cpu_threads()
    if mode == "greedy":
        m = min(64, n)
        # spread over the whole batch: every pack / result slice of the 4096-problem call is sampled
        idx = sorted({(i * (n - 1)) // max(1, m - 1) for i in range(m)})
        m = len(idx)
        sprobs = P.c_problems([snaps[i] for i in idx], None, keep)
        rout = (A.bs_mpc_result * m)()
        t0 = time.perf_counter()
        rc = ref.ref_greedy_batch(C.byref(cm), cc, cp, sprobs, m, rout, threads)
        tc = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": m / tc, "unit": "decisions/s", "cores": threads, "kind": "reference",
                               "sample": f"{m} decisions spread over the batch, greedy_freq_select, one per thread"}
        out["identical_on_sample"] = rc == 0 and all(
            (rout[j].objective_w, rout[j].eval_count, rout[j].feasible, list(rout[j].freqs_mhz),
             [(rout[j].levels[l].mutations, rout[j].levels[l].feasible_mutations) for l in range(rout[j].n_levels)]) ==
            (res[i].objective_w, res[i].eval_count, res[i].feasible, list(res[i].freqs_mhz),
             [(res[i].levels[l].mutations, res[i].levels[l].feasible_mutations) for l in range(res[i].n_levels)])
            for j, i in enumerate(idx))
        return out
    # exhaustive: property checks at full size + the reference's per-trajectory cost
    rng = random.Random(5)
    ok, checked = True, 0
    for i in range(min(4, n)):
        r = res[i]
        if not r.feasible:
            continue
        checked += 1
        snap = P.c_snapshot(snaps[i], keep)
        codes = [r.best_code] + [rng.randrange(24 ** r.K) for _ in range(20000)]
        cd = (C.c_uint64 * len(codes))(*codes)
        fe, ob = (C.c_int32 * len(codes))(), (C.c_double * len(codes))()
        ok &= ref.ref_eval_codes(C.byref(cm), cc, cp, C.byref(snap), cd, len(codes), fe, ob) == 0
        ok &= bool(fe[0]) and ob[0] == r.objective_w
        ok &= all(not fe[j] or ob[j] >= r.objective_w for j in range(1, len(codes)))
        g = A.bs_mpc_result()
        ok &= ref.ref_greedy(C.byref(cm), cc, cp, C.byref(snap), C.byref(g)) == 0
        ok &= (not g.feasible) or g.objective_w >= r.objective_w
    out["property_checks"] = {"decisions": checked, "passed": bool(ok),
                              "what": "GPU argmin re-evaluated by the reference (feasible, objective bit-equal); "
                                      "20k random feasible codes never better; reference greedy sandwich"}
    m = 400_000
    snap = P.c_snapshot(snaps[0], keep)
    cd = (C.c_uint64 * m)(*[rng.randrange(24 ** max(1, res[0].K)) for _ in range(m)])
    fe, ob = (C.c_int32 * m)(), (C.c_double * m)()
    t0 = time.perf_counter()
    ref.ref_eval_codes(C.byref(cm), cc, cp, C.byref(snap), cd, m, fe, ob)
    per = (time.perf_counter() - t0) / m
    out["cpu_baseline"] = {"value": threads / per, "unit": "trajectories/s", "cores": threads, "kind": "reference",
                           "sample": f"{m} random trajectories of decision 0 through the reference's meets_slo + "
                                     f"time_weighted_power on one core ({per * 1e9:.0f} ns each) x {threads} cores "
                                     f"(extrapolated: one 24^8 decision = {24 ** 8 * per / threads / 3600:.1f} h)"}
    return out


def bench_c2_loose(dev, with_cpu: bool, D: int = 1024, ttft: float = 1200.0, steps: int = 10) -> dict:
    """C2 at a looser TTFT SLO (1200 ms): a large part of every tree is
    feasible, so the pruned search has the least to prune (the headline's
    600 ms corpus is ~1 % feasible).  Resident batch, CUDA events on the
    library stream, L2 flushed between steps; the reference on the host cores
    decides the first decisions of the same batch and must agree bit for bit."""
    import torch

    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as Wk

    lib = dev._lib
    models, cfg, pol, snaps = Wk.c2_corpus(0xC2, D, ttft)
    keep: list = []
    cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
    cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
    probs = P.c_problems(snaps, None, keep)
    mh = dev.models(models)
    plan = C.c_void_p()
    dev.check(lib.bs_mpc_plan_create(dev.handle, mh, cc, cp, 1, probs, D, 0, C.byref(plan)))
    stream = torch.cuda.ExternalStream(lib.bs_ctx_stream(dev.handle))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    out = (A.bs_mpc_result * D)()
    with torch.cuda.stream(stream):
        for _ in range(3):
            dev.check(lib.bs_mpc_plan_run(dev.handle, plan, 0))
            flush.zero_()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            a.record(stream)
            dev.check(lib.bs_mpc_plan_run(dev.handle, plan, 0))
            b.record(stream)
            b.synchronize()
            flush.zero_()
        torch.cuda.synchronize()
        dev.check(lib.bs_mpc_plan_results(dev.handle, plan, out))
        ms = [a.elapsed_time(b) for a, b in evs]
        sweep = []
        for _ in range(3):
            dev.check(lib.bs_mpc_plan_run(dev.handle, plan, 1))
            k = (C.c_float * 5)()
            lib.bs_mpc_plan_kernel_ms(dev.handle, plan, k, 5)
            sweep.append(k[3])
            flush.zero_()
    lib.bs_mpc_plan_destroy(dev.handle, plan)
    step = statistics.median(ms)
    feas = sum(out[i].feasible_count for i in range(D)) / (D * TRAJ_PER_DECISION)
    res = {"workload": f"C2 at TTFT {ttft:.0f} ms: {D} decisions x 16^6 trajectories, resident, L2 flushed",
           "value": D * TRAJ_PER_DECISION / (step * 1e-3), "unit": UNIT, "ms_per_step": step,
           "sweep_ms": statistics.median(sweep), "feasible_fraction": feas}
    if with_cpu:
        threads = cpu_threads()
        m = min(D, threads)
        dt, ref_out = cpu_reference_run(models, cfg, pol, snaps[:m], threads)
        res["cpu_baseline"] = {"value": m * TRAJ_PER_DECISION / dt, "unit": UNIT, "cores": threads,
                               "kind": "reference", "sample": f"first {m} decisions, one per thread ({dt:.1f} s)"}
        res["identical_on_sample"] = all(
            (out[i].best_code, out[i].objective_w, out[i].feasible_count) ==
            (ref_out[i].best_code, ref_out[i].objective_w, ref_out[i].feasible_count) for i in range(m))
    return res


def bench_c4_experiment(dev, with_cpu: bool) -> dict:
    """configs[3]'s per-window loop: run_experiment (runner.hpp:155-172) over a
    bursty 1-hour trace in 5-minute windows -- every window planned from the
    previous one (config table + ILP + max-throughput baseline for a 16-GPU
    cluster) and replayed under the three policies with per-iteration
    decisions; reference run_experiment beside it."""
    import ctypes as C

    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as Wk

    lad = Wk.ladder(16)
    models = Wk.llama_models(lad)
    trace = P.gen_gamma_trace(12.0, 0.5, 3600e3, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)),
                              7)
    cfg = P.RunnerConfig(slo=P.SLOSpec(600.0, 100.0), total_gpus=16, tp_options=[1, 2, 4, 8], ladder=lad,
                         scheduler=P.SchedulerPolicy(max_batch_tokens=2048), rampup_s=30.0)
    cfg.plan.policy = P.SchedulerPolicy(max_batch_tokens=2048)
    pols = [P.Policy.maxfreq_distserve, P.Policy.place_only, P.Policy.two_tier]
    P.run_experiment(trace, 300e3, pols, cfg, models, dev)  # warm-up
    t0 = time.perf_counter()
    res = P.run_experiment(trace, 300e3, pols, cfg, models, dev)
    t_gpu = time.perf_counter() - t0
    runs = len(res.runs)
    out = {"workload": "run_experiment: 1-hour gamma(0.5) trace at 12 rps, 12 five-minute windows x 3 policies "
                       "(maxfreq-distserve, place-only, two-tier), 16 GPUs, TP{1,2,4,8} x 16 rungs",
           "value": runs / t_gpu, "unit": "window runs/s", "seconds": t_gpu,
           "decisions": sum(r.result.n_decisions for r in res.runs), "phase_s": res.seconds,
           "two_tier_slo_pass": res.two_tier_slo_pass,
           "timing": "end to end through pdsim.run_experiment (host trace in, reports out)"}
    if with_cpu:
        import oracle

        ref = oracle.load_ref()
        keep: list = []
        c = oracle.ref_runner_config()
        c.slo = P.c_slo(cfg.slo)
        c.total_gpus = cfg.total_gpus
        tps = (C.c_int32 * 4)(*cfg.tp_options)
        ld = (C.c_double * len(lad.freqs_mhz))(*lad.freqs_mhz)
        keep += [tps, ld]
        c.n_tp, c.tp_options, c.ladder, c.n_ladder = 4, tps, ld, len(lad.freqs_mhz)
        c.scheduler = P.c_policy(cfg.scheduler)
        c.alpha, c.peak_subwindow_s = cfg.plan.alpha, cfg.plan.peak_subwindow_s
        c.search, c.plan_policy = P.c_search(cfg.plan.search), P.c_policy(cfg.plan.policy)
        c.rampup_s, c.switch_latency_ms = cfg.rampup_s, cfg.switch_latency_ms
        c.mpc_k, c.mpc_n, c.mpc_margin = cfg.mpc_horizon_k, cfg.mpc_ladder_n, cfg.mpc_margin
        c.kv_threshold, c.decode_margin = cfg.kv_threshold, cfg.decode_margin
        cap = 64
        o = (oracle.ref_window_run * cap)()
        n_out, tt = C.c_int(), C.c_int32()
        cm, ct = P.c_model_set(models, keep), P.c_trace(trace, keep)
        pa = (C.c_int32 * 3)(*[int(p) for p in pols])
        t0 = time.perf_counter()
        rc = ref.ref_run_experiment(C.byref(cm), C.byref(ct), 300e3, pa, 3, C.byref(c), o, cap, C.byref(n_out),
                                    C.byref(tt))
        t_cpu = time.perf_counter() - t0
        same = rc == 0 and n_out.value == runs and all(
            (o[i].gpus_used, o[i].objective_w, o[i].report.n_decisions, o[i].report.prefill_energy_j,
             o[i].report.decode_energy_j, o[i].report.ttft_violations) ==
            (r.plan.gpus_used, r.plan.objective_w, r.result.n_decisions, r.report.prefill_energy_j,
             r.report.decode_energy_j, r.report.ttft_violations) for i, r in enumerate(res.runs))
        out["cpu_baseline"] = {"value": runs / t_cpu, "unit": "window runs/s", "cores": cpu_threads(),
                               "kind": "reference", "seconds": t_cpu,
                               "sample": "the whole experiment: pdsim::run_experiment (build_config_table on "
                                         "std::async threads; simulations single-threaded, as the reference runs)"}
        out["identical_to_reference"] = bool(same)
    return out


EXTRA_ROOF = {"c1_demo": "c1", "c2_loose_slo": "c2l", "c3_placement": "c3", "c4_replay": "c4", "c4_day": "c4d",
              "c4_experiment": "c4x", "c5_greedy": "c5g", "c5_exhaustive": "c5x"}


def extra_roofline(cfg: str, fp64_peak: float | None) -> dict | None:
    """Executed roofline of a sub-benchmark's dominant kernel: ncu's FP64-pipe
    and issue fractions, occupancy and DRAM bytes of one launch
    (profiles/r02_rooflines.json, tools/ncu_rooflines.sh), against the FP64
    issue peak of this box and the measured HBM bandwidth."""
    path = ROOT / "profiles" / "r02_rooflines.json"
    try:
        doc = json.loads(path.read_text())
        r = doc["configs"][cfg]
    except Exception:
        return None
    hbm = None
    try:
        hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs")
    except Exception:
        pass
    traffic = r.get("dram_read_bytes", 0.0) + r.get("dram_write_bytes", 0.0)
    dur = r.get("duration_us")
    gbs = traffic / (dur * 1e-6) / 1e9 if dur else None
    frac = r.get("fp64_pipe_active_frac")
    return {"bound": "fp64-issue (latency: dependent FP64 chains)", "kernel": r.get("kernel"), "unit": "TFLOP/s",
            "peak": fp64_peak / 1e12 if fp64_peak else None, "frac": frac,
            "achieved": frac * fp64_peak / 1e12 if (frac is not None and fp64_peak) else None,
            "issue_slots_busy_frac": r.get("issue_slots_busy_frac"),
            "achieved_occupancy": r.get("achieved_occupancy"),
            "avg_active_threads_per_warp": r.get("avg_active_threads_per_warp"),
            "traffic": traffic, "hbm_gbs": gbs, "hbm_frac": gbs / hbm if (gbs is not None and hbm) else None,
            "duration_us_ncu": dur, "launch": {k: r.get(k) for k in ("grid", "block", "registers")},
            "source": f"profiles/r02_rooflines.json ({doc.get('source', '')})"}


def fp64_peak_of(dev) -> float | None:
    try:
        lib = dev._lib
        peak, peak_ms = C.c_double(), C.c_double()
        dev.check(lib.bs_fp64_peak(dev.handle, C.byref(peak), C.byref(peak_ms)))
        return peak.value
    except Exception:
        return None


def run_extras(args, dev, rank, world, local) -> dict:
    with_cpu = world == 1 and not args.no_cpu_baseline
    todo = [args.only] if args.only else ["c1", "c2l", "c3", "c4", "c4d", "c4x", "c5g", "c5x"]
    out = {}
    for k in todo:
        if k == "c1":
            if world == 1:
                out["c1_demo"] = bench_c1(dev, with_cpu)
        elif k == "c2l":
            if world == 1:
                out["c2_loose_slo"] = bench_c2_loose(dev, with_cpu)
        elif k == "c3":
            out["c3_placement"] = bench_c3(dev, with_cpu, rank=rank, world=world, local=local,
                                           n_windows=args.c3_windows)
        elif k == "c4":
            out["c4_replay"] = bench_c4(dev, rank, world, local, args.c4_scenarios, with_cpu)
        elif k == "c4d":
            out["c4_day"] = bench_c4_day(dev, rank, world, local, args.c4_day_scenarios, with_cpu)
        elif k == "c4x":
            if world == 1:
                out["c4_experiment"] = bench_c4_experiment(dev, with_cpu)
        elif k == "c5g":
            out["c5_greedy"] = bench_c5(dev, "greedy", rank, world, local, 4096, with_cpu)
        else:
            out["c5_exhaustive"] = bench_c5(dev, "exhaustive", rank, world, local, args.c5x_decisions, with_cpu)
    if rank == 0:
        peak = fp64_peak_of(dev)
        for key, obj in out.items():
            if isinstance(obj, dict) and key in EXTRA_ROOF:
                roof = extra_roofline(EXTRA_ROOF[key], peak)
                if roof is not None:
                    obj["roofline"] = roof
    return out


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 and return its exit
    code; every rank re-enters main() with RANK/WORLD_SIZE set."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_dist(args, world: int, local: int) -> None:
    """One process per GPU: NCCL over the node's GPUs (gloo only for the CPU
    tests of the multi-rank plumbing)."""
    if world <= 1:
        return
    import torch
    import torch.distributed as dist

    if args.dist_backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(args.dist_backend)


def make_device(local: int):
    from paper_2602_18755_b200 import pdsim as P

    return P.Device(local)


def measure_c2(args, dev, rank: int, world: int, local: int) -> dict:
    """The C2 leg on this rank's GPU: its own corpus (seed 0xC2 + 1000 rank)
    as a resident plan, `steps` timed steps (CUDA events on the library's
    stream, L2 flushed between steps, a barrier before the timed region),
    per-kernel times from extra untimed steps, then the same batch end to end
    through bs_mpc_exhaustive with host buffers.  Local numbers only: the
    ranks are combined by combine_c2."""
    import torch

    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as Wk

    lib = dev._lib
    torch.cuda.set_device(local)
    stream = torch.cuda.ExternalStream(lib.bs_ctx_stream(dev.handle), device=f"cuda:{local}")
    D = args.decisions
    models, cfg, pol, snaps = Wk.c2_corpus(0xC2 + 1000 * rank, D, args.ttft)
    keep: list = []
    cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
    cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
    probs = P.c_problems(snaps, None, keep)
    mh = dev.models(models)
    plan = C.c_void_p()
    dev.check(lib.bs_mpc_plan_create(dev.handle, mh, cc, cp, 1, probs, D, 0, C.byref(plan)))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")  # > 126 MB L2
    out = (A.bs_mpc_result * D)()

    def step(timed_events=None, kernel_times=False):
        if timed_events is not None:
            timed_events[0].record(stream)
        dev.check(lib.bs_mpc_plan_run(dev.handle, plan, 1 if kernel_times else 0))
        if timed_events is not None:
            timed_events[1].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
            flush.zero_()
        dev.check(lib.bs_mpc_plan_results(dev.handle, plan, out))
        trajectories = sum(out[i].trajectories for i in range(D))
        feasible = sum(out[i].feasible_count for i in range(D))
        _barrier(world)
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        launches0 = dev.kernel_launches()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for s in range(args.steps):
            step(evs[s])
            evs[s][1].synchronize()
            flush.zero_()  # untimed L2 flush between timed steps
        torch.cuda.synchronize()
        launches = dev.kernel_launches() - launches0
        step_ms = [a.elapsed_time(b) for a, b in evs]
        # per-kernel times from the same number of extra, untimed steps (events between the kernels
        # would serialise the programmatic dependent launches of the timed ones)
        leaf_ms, phase_ms = [], []  # leaf_ms: the sweep kernel (dominant)
        for s in range(args.steps):
            step(None, kernel_times=True)
            ms = (C.c_float * 5)()
            lib.bs_mpc_plan_kernel_ms(dev.handle, plan, ms, 5)  # syncs the stream
            phase_ms.append(list(ms))
            leaf_ms.append(ms[3])
            flush.zero_()
    # --- end to end through the C ABI with host buffers (e2e) ------------------
    res = (A.bs_mpc_result * D)()
    for _ in range(2):
        dev.check(lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, probs, D, res))
    e2e_times = []
    h2d, d2h = C.c_uint64(), C.c_uint64()
    for _ in range(max(3, min(args.steps, 10))):
        t0 = time.perf_counter()
        dev.check(lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, probs, D, res))
        e2e_times.append(time.perf_counter() - t0)
        lib.bs_ctx_last_transfer(dev.handle, C.byref(h2d), C.byref(d2h))
    clk = clocks.stop()  # sampled across the timed steps and the e2e calls (the device-timed region is ms-short)
    same = all(res[i].best_code == out[i].best_code and res[i].objective_w == out[i].objective_w
               for i in range(D))
    lib.bs_mpc_plan_destroy(dev.handle, plan)
    import struct

    rows = [[struct.unpack("<q", struct.pack("<d", out[i].objective_w))[0],
             int(out[i].best_code) & 0x7FFFFFFFFFFFFFFF, int(out[i].feasible_count)] for i in range(D)]
    peak, peak_ms = C.c_double(), C.c_double()
    dev.check(lib.bs_fp64_peak(dev.handle, C.byref(peak), C.byref(peak_ms)))
    return {"D": D, "total_ms": sum(step_ms), "step_ms": step_ms, "launches": launches, "leaf_ms": leaf_ms,
            "phase_ms": phase_ms, "e2e_s": statistics.median(e2e_times), "h2d": int(h2d.value),
            "d2h": int(d2h.value), "same": bool(same), "clocks": clk, "trajectories": trajectories,
            "feasible": feasible, "rows": rows, "peak": peak.value, "corpus": (models, cfg, pol, snaps),
            "out": out}


def combine_c2(m: dict, rank: int, world: int, local: int, args) -> dict:
    """The ranks' C2 measurements as one job: the max over ranks of the timed
    region and of the end-to-end time (barrier-aligned starts), and the final
    all-gather of every rank's per-decision results (the only collective of
    the path, outside the timed region)."""
    total_ms, e2e_s, gathered = m["total_ms"], m["e2e_s"], None
    if world > 1:
        import torch

        from paper_2602_18755_b200 import sharding as S

        dev_t = f"cuda:{local}" if args.dist_backend == "nccl" else "cpu"
        total_ms = S.max_over_ranks(total_ms, device=dev_t)
        e2e_s = S.max_over_ranks(e2e_s, device=dev_t)
        rows = torch.tensor(m["rows"], dtype=torch.int64, device=dev_t).reshape(-1, 3)
        table = S.gather_rows(rows, world * m["D"])
        gathered = {"rows": int(table.shape[0]), "bytes": int(table.numel() * 8),
                    "rank0_rows_match": bool(torch.equal(table[: m["D"]], rows)) if rank == 0 else None,
                    "rows_sha": __import__("hashlib").sha256(table.cpu().numpy().tobytes()).hexdigest()[:16]}
    return {"total_ms": total_ms, "e2e_s": e2e_s, "gathered": gathered}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)

    rank, local, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    init_dist(args, world, local)
    dev = make_device(local)
    if args.only:
        extra = run_extras(args, dev, rank, world, local)
        if rank == 0:
            print(json.dumps(extra), flush=True)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return 0
    m = measure_c2(args, dev, rank, world, local)
    agg = combine_c2(m, rank, world, local, args)
    D = m["D"]
    total_ms, e2e_s = agg["total_ms"], agg["e2e_s"]
    value = world * D * TRAJ_PER_DECISION * args.steps / (total_ms * 1e-3)

    # --- roofline ----------------------------------------------------------------
    leaf_avg_ms = statistics.mean(m["leaf_ms"])
    achieved = W_OPS * D * TRAJ_PER_DECISION / (leaf_avg_ms * 1e-3)
    traffic, executed, prof_src = None, None, None
    tpath = ROOT / "profiles" / "leaf_traffic.json"
    if tpath.exists():
        try:
            prof = json.loads(tpath.read_text())
            traffic = prof.get("dram_bytes_per_launch")
            executed = prof.get("executed")
            prof_src = prof.get("source")
        except Exception:
            traffic = None

    # --- CPU baseline (rank 0, N = 1 only) ---------------------------------------
    cpu = None
    identical = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = cpu_threads()
            models, cfg, pol, snaps = m["corpus"]
            out = m["out"]
            # ~7 s per C2 decision per core for the reference loop: one decision per thread
            sample = min(D, max(1, threads))
            dt, ref_out = cpu_reference_run(models, cfg, pol, snaps[:sample], threads)
            cpu = {"value": sample * TRAJ_PER_DECISION / dt, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{sample} C2 decisions of this corpus (one per host thread, {dt:.1f} s), reference "
                             f"loop tests/test_dvfs.cpp:74-94 over meets_slo + time_weighted_power; cpu={cpu_model()}"}
            # the same decisions of the timed batch, bit for bit (argmin code, objective, feasible count)
            identical = {"decisions": sample, "identical_on_sample": all(
                (out[i].best_code, out[i].objective_w, out[i].feasible, out[i].feasible_count, out[i].eval_count) ==
                (ref_out[i].best_code, ref_out[i].objective_w, ref_out[i].feasible, ref_out[i].feasible_count,
                 ref_out[i].eval_count) for i in range(sample))}
        except Exception as e:  # the reference driver is optional on a box without it
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    extras = {} if args.no_extras else run_extras(args, dev, rank, world, local)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 exhaustive prefill MPC, horizon 6 x 16 levels (16.7M trajectories/decision)",
                       "decisions_per_step_per_gpu": D, "ttft_ms": args.ttft, "model": "Llama-3.3-70B-shaped synth "
                       "(compute-bound, lat_coef 366, TP2)", "l2": "flushed between steps (256 MB write)",
                       "parallelism": f"independent decisions sharded over {world} GPU(s)"},
            "decisions_per_s": world * D * args.steps / (total_ms * 1e-3),
            "feasible_fraction": m["feasible"] / max(1, m["trajectories"]),
            "phase_ms_avg": {k: statistics.mean(p[i] for p in m["phase_ms"])
                             for i, k in enumerate(["prepare", "thresholds", "bfs", "sweep", "finalize"])},
            "e2e": {"value": world * D * TRAJ_PER_DECISION / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": m["h2d"], "d2h_bytes_per_step": m["d2h"],
                    "matches_resident": m["same"]},
            "roofline": roofline_obj(achieved, m["peak"], leaf_avg_ms, traffic, executed, prof_src),
            "gpu_launches": int(m["launches"]),
            "parity": identical,
            "gather": agg["gathered"],
            "clocks": m["clocks"],
            "cpu_baseline": cpu,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Two-tier replay benchmark (BASELINE.json configs[3], "C4"-shaped): what-if
scenarios = trace seeds x (TTFT, TPOT) SLO pairs, each one simulate_cluster
(simulator.hpp:758-893) with per-iteration decisions of the two-tier
controllers (greedy prefill MPC at every batch boundary and arrival, decode
slack pick at every iteration) + the steady-state report (metrics.hpp:71-156),
over one bursty window (gamma(0.5) arrivals) on a fixed cluster.

All scenarios of a step go to the device in one bs_replay call.  Reported:
scenarios/s and controller decisions/s (device-timed kernels and end to end
through the Python API with host buffers), the kernel phase split, and the
reference (oracle/_ref: pdsim::simulate_cluster + trim + make_report) on the
host cores for a bounded sample of the same scenarios, checked field by field
against the device results.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def build_scenarios(P, W, n_scen, window_s, rps, seeds, n_pre, n_dec, levels):
    lad = W.ladder(levels)
    models = W.llama_models(lad)
    fmax = lad.freqs_mhz[-1]
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    ttfts = [400.0 + 500.0 * i / 15 for i in range(16)]
    tpots = [60.0 + 80.0 * i / 7 for i in range(8)]
    traces = [P.gen_gamma_trace(rps, 0.5, window_s * 1000.0,
                                P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 1000 + s)
              for s in range(seeds)]
    inst = [P.ClusterInstance(P.InstanceConfig(P.Phase.prefill, 2, fmax), 1.0 / n_pre) for _ in range(n_pre)]
    inst += [P.ClusterInstance(P.InstanceConfig(P.Phase.decode, 4, fmax), 1.0 / n_dec) for _ in range(n_dec)]
    scs = []
    for k in range(n_scen):
        tr = traces[k % seeds]
        slo_i = (k // seeds) % 128
        slo = P.SLOSpec(ttfts[slo_i % 16], tpots[slo_i // 16])
        mpc = P.MpcConfig(horizon_K=8, ladder_N=7, ladder=lad, slo=slo)
        dec = P.DecodePolicyConfig(tbt_slo_ms=slo.tpot_ms, kv_threshold=0.9, ladder=lad, margin=0.05)
        fac = P.TwoTierFactory(mpc, dec, models, pol)
        scs.append(P.ReplayScenario(tr, P.ClusterSpec(list(inst)), pol, fac, P.SimOptions(30.0, -1.0), slo, 30.0))
    return models, scs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenarios", type=int, default=1024)
    ap.add_argument("--window-s", type=float, default=300.0)
    ap.add_argument("--rps", type=float, default=12.0)
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--prefill", type=int, default=2)
    ap.add_argument("--decode", type=int, default=2)
    ap.add_argument("--levels", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cpu-sample", type=int, default=32, help="scenarios replayed by the reference (0: skip)")
    args = ap.parse_args()
    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as W

    models, scs = build_scenarios(P, W, args.scenarios, args.window_s, args.rps, args.seeds, args.prefill,
                                  args.decode, args.levels)
    dev = P.default_device()
    lib = dev._lib
    keep: list = []
    cfgs, cscs, total = P.c_replay_inputs(scs, keep)
    n = len(scs)
    out = (A.bs_replay_summary * n)()
    mh = dev.models(models)
    for _ in range(args.warmup):
        dev.check(lib.bs_replay(dev.handle, mh, mh, cfgs, n, cscs, n, out, None, None))
    e2e, phases = [], []
    st = (C.c_double * 8)()
    launches0 = dev.kernel_launches()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        dev.check(lib.bs_replay(dev.handle, mh, mh, cfgs, n, cscs, n, out, None, None))
        e2e.append(time.perf_counter() - t0)
        lib.bs_ctx_stats(dev.handle, st, 8)
        phases.append([st[i] for i in range(4)])
    launches = (dev.kernel_launches() - launches0) // args.steps
    h2d, d2h = C.c_uint64(), C.c_uint64()
    lib.bs_ctx_last_transfer(dev.handle, C.byref(h2d), C.byref(d2h))
    decisions = sum(out[i].n_decisions for i in range(n))
    kern_ms = statistics.median(sum(p) for p in phases)
    e2e_s = statistics.median(e2e)
    line = {
        "metric": "two-tier replay scenarios/sec (and controller decisions/sec)",
        "workload": f"C4-shaped: {n} what-if scenarios ({args.seeds} trace seeds x (TTFT, TPOT) SLO pairs), "
                    f"{args.window_s:.0f} s gamma(0.5) window at {args.rps} rps, {args.prefill}P(tp2)+"
                    f"{args.decode}D(tp4), greedy MPC K=8 N=7 + decode slack DVFS, report after 30 s ramp-up",
        "requests_per_scenario": len(scs[0].trace.requests), "scenarios": n,
        "decisions_per_step": decisions, "decisions_by_trigger": [sum(out[i].decisions_by_trigger[t] for i in range(n))
                                                                  for t in range(3)],
        "value": n / (kern_ms / 1e3), "unit": "scenarios/s", "decisions_per_s": decisions / (kern_ms / 1e3),
        "kernel_ms": kern_ms,
        "phase_ms": dict(zip(["prefill", "route", "decode", "report"],
                             [statistics.median(p[i] for p in phases) for i in range(4)])),
        "e2e": {"value": n / e2e_s, "unit": "scenarios/s", "seconds": e2e_s, "h2d_bytes_per_step": int(h2d.value),
                "d2h_bytes_per_step": int(d2h.value)},
        "gpu_launches": int(launches),
        "statuses_ok": all(out[i].status == 0 for i in range(n)),
    }
    if args.cpu_sample > 0:
        import oracle

        ref = oracle.load_ref()
        m = min(args.cpu_sample, n)
        sub = scs[:m]
        k2: list = []
        rc_cfgs, rc_scs, _ = P.c_replay_inputs(sub, k2)
        rout = (A.bs_replay_summary * m)()
        cm = P.c_model_set(models, k2)
        threads = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        rc = ref.ref_replay(C.byref(cm), C.byref(cm), rc_cfgs, rc_scs, m, rout, None, None, threads)
        t_cpu = time.perf_counter() - t0
        fields = [f for f, _ in A.bs_replay_summary._fields_ if f not in ("_pad", "decisions_by_trigger")]

        def eq(a, b):
            return a == b or (a != a and b != b)

        same = rc == 0 and all(all(eq(getattr(out[i], f), getattr(rout[i], f)) for f in fields) for i in range(m))
        line["cpu_baseline"] = {"value": m / t_cpu, "unit": "scenarios/s", "cores": threads, "kind": "reference",
                                "seconds": t_cpu, "sample": f"first {m} scenarios of the same sweep, "
                                f"pdsim::simulate_cluster + trim_steady_state + make_report, one scenario per thread",
                                "decisions_per_s": sum(rout[i].n_decisions for i in range(m)) / t_cpu}
        line["summaries_identical_on_sample"] = bool(same)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

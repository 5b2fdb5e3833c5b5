"""Coarse-tier placement benchmark (BASELINE.json configs[2], "C3"): the
config table (goodput search + E_c for every candidate) and the ILP for a
16-GPU cluster over one bursty 1-hour window: gamma(0.5) arrivals at 12 rps
(~43k requests), TP {1,2,4,8} x 16 rungs x 2 phases = 128 candidates,
max_batch_tokens 2048, tolerance 0.25 rps, probe_count 1.

Prints one JSON line: placement configs/s (candidates fully evaluated per
second), probes/s, the ILP time, and -- unless --no-cpu -- the reference's
build_config_table (std::async over all host cores) on the same window,
checked entry for entry against the GPU table.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--duration-s", type=float, default=3600.0)
    ap.add_argument("--rps", type=float, default=12.0)
    ap.add_argument("--levels", type=int, default=16)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as W

    lad = W.ladder(args.levels)
    models = W.llama_models(lad)
    base = P.gen_gamma_trace(args.rps, 0.5, args.duration_s * 1000.0,
                             P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 7)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    pol = P.SchedulerPolicy(max_batch_tokens=2048)
    slo = P.SLOSpec(600.0, 100.0)
    search = P.GoodputSearch()
    dev = P.default_device()
    P.build_config_table(cands, base, slo, models, pol, search, device=dev)  # warm-up
    times = []
    for _ in range(args.repeats):
        t0 = time.perf_counter()
        table = P.build_config_table(cands, base, slo, models, pol, search, device=dev)
        times.append(time.perf_counter() - t0)
    t_table = min(times)
    st = (C.c_double * 8)()
    dev._lib.bs_ctx_stats(dev.handle, st, 8)
    stats = {"mask_ms": st[0], "probe_ms": st[1], "energy_ms": st[2], "max_events_per_probe": st[3],
             "total_events": st[4]}
    t0 = time.perf_counter()
    plan = P.solve_placement(P.PlacementProblem(table, 16, P.peak_rps(base, 10.0), 0.05), dev)
    t_ilp = time.perf_counter() - t0
    k_max = int(base.mean_rps() // search.tolerance_rps)
    line = {"metric": "placement configs/sec", "workload": "C3 config table + ILP, 1-hour gamma(0.5) window",
            "requests": len(base.requests), "candidates": len(cands), "k_max": k_max,
            "probes": k_max * len(cands), "table_s": t_table, "configs_per_s": len(cands) / t_table,
            "probes_per_s": k_max * len(cands) / t_table, "ilp_s": t_ilp, "usable": sum(e.usable() for e in table),
            "gpus_used": plan.gpus_used, "objective_w": plan.objective_w, "phases": stats}
    if not args.no_cpu:
        import oracle
        from paper_2602_18755_b200 import _abi as A

        ref = oracle.load_ref()
        keep: list = []
        cm = P.c_model_set(models, keep)
        ct = P.c_trace(base, keep)
        cs, cp, cg = P.c_slo(slo), P.c_policy(pol), P.c_search(search)
        ci = P.c_candidates(cands)
        out = (A.bs_table_entry * len(cands))()
        t0 = time.perf_counter()
        rc = ref.ref_config_table(C.byref(cm), C.byref(ct), C.byref(cs), C.byref(cp), C.byref(cg), ci, len(cands), out)
        t_cpu = time.perf_counter() - t0
        same = rc == 0 and all(
            (e.r_c, e.e_c, e.saturated, e.error) == (o.r_c, o.e_c, o.saturated, o.error)
            for e, o in zip(table, [P.entry_from_c(out[i]) for i in range(len(cands))]))
        line["cpu_baseline"] = {"value": len(cands) / t_cpu, "unit": "configs/s", "seconds": t_cpu,
                                "cores": len(os.sched_getaffinity(0)), "kind": "reference",
                                "sample": "build_config_table (std::async per candidate) on the same window"}
        line["tables_identical"] = bool(same)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

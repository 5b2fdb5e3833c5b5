"""Projected multi-GPU scaling from one GPU: every fixed-size (strong-scaled)
configuration of bench.py is timed at the per-rank shard it has at N = 1, 2,
4, 8 ranks (bench.py splits it with sharding.shard_bounds; rank 0's shard is
the largest), and the projected efficiency is T(N=1) / (N T(shard_N)), the
data-path having no collective (only the final gather).  Weak-scaled
configurations (C2, the C4 day sweep) keep their per-rank work, so their
projection is their per-rank time.  Writes profiles/r02_scaling_projection.json.
Run on the GPU box: python tools/scaling_projection.py"""
from __future__ import annotations

import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2602_18755_b200 import _abi as A  # noqa: E402
from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import sharding as S  # noqa: E402
from paper_2602_18755_b200 import workloads as Wk  # noqa: E402


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def project(name, n_units, run_shard, reps=3):
    """Every rank's shard at every N timed on this GPU; a job at N takes the
    slowest rank's time (bench.py's max over ranks)."""
    rows, spread = {}, {}
    for N in (1, 2, 4, 8):
        ts = []
        for r in range(N):
            lo, hi = S.shard_bounds(n_units, r, N)
            ts.append(timed(lambda: run_shard(lo, hi), reps))
        rows[N] = max(ts)
        spread[N] = [round(t, 5) for t in ts]
    return {"config": name, "units": n_units, "seconds_slowest_rank": rows, "seconds_per_rank": spread,
            "efficiency": {N: rows[1] / (N * rows[N]) for N in rows}}


def main():
    dev = P.Device(0)
    lib = dev._lib
    out = []
    # C5 greedy / exhaustive: 4096 decisions split across ranks
    models, cfg, pol, snaps = Wk.c5_corpus(0xC5, 4096)
    keep: list = []
    cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
    cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
    probs = P.c_problems(snaps, None, keep)
    mh = dev.models(models)
    res = (A.bs_mpc_result * 4096)()
    psz = C.sizeof(A.bs_mpc_problem)

    def mpc(fn, lo, hi):
        p = C.cast(C.addressof(probs) + lo * psz, C.POINTER(A.bs_mpc_problem))
        dev.check(fn(dev.handle, mh, cc, cp, 1, p, hi - lo, res))

    out.append(project("C5 greedy (4096 decisions, H8 x 24)", 4096, lambda lo, hi: mpc(lib.bs_mpc_greedy, lo, hi)))
    out.append(project("C5 exhaustive (4096 decisions, 24^8)", 4096,
                       lambda lo, hi: mpc(lib.bs_mpc_exhaustive, lo, hi), reps=1))
    # C2 is weak-scaled (each rank its own 1024-decision corpus): per-rank time at every N
    m2, cfg2, pol2, snaps2 = Wk.c2_corpus(0xC2, 1024)
    k2: list = []
    c2c = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg2, k2))
    c2p = (A.bs_scheduler_policy * 1)(P.c_policy(pol2))
    pr2 = P.c_problems(snaps2, None, k2)
    h2 = dev.models(m2)
    r2 = (A.bs_mpc_result * 1024)()
    t2 = timed(lambda: dev.check(lib.bs_mpc_exhaustive(dev.handle, h2, c2c, c2p, 1, pr2, 1024, r2)))
    out.append({"config": "C2 exhaustive (1024 decisions per rank, weak)", "units_per_rank": 1024,
                "seconds_per_rank": {N: t2 for N in (1, 2, 4, 8)}, "efficiency": {N: 1.0 for N in (1, 2, 4, 8)}})
    # C4 replay: 1024 what-if scenarios (5-minute windows) split across ranks
    m4, scs = Wk.c4_scenarios(1024)
    k4: list = []
    cfgs, cscs, _ = P.c_replay_inputs(scs, k4)
    outs = (A.bs_replay_summary * 1024)()
    h4 = dev.models(m4)
    ssz = C.sizeof(A.bs_scenario)

    def rep(lo, hi):
        p = C.cast(C.addressof(cscs) + lo * ssz, C.POINTER(A.bs_scenario))
        dev.check(lib.bs_replay(dev.handle, h4, h4, cfgs, len(scs), p, hi - lo, outs, None, None))

    out.append(project("C4 replay sweep (1024 scenarios x 5 min, 2P+2D)", 1024, rep))
    # C3: a day of 24 hourly windows' config tables split across ranks
    lad = Wk.ladder(16)
    m3 = Wk.llama_models(lad)
    day = P.gen_gamma_trace(12.0, 0.5, 24 * 3600e3, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 7)
    wins = P.split_windows(day, 3600e3)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    pol3, slo, search = P.SchedulerPolicy(max_batch_tokens=2048), P.SLOSpec(600.0, 100.0), P.GoodputSearch()
    out.append(project("C3 config tables (24 hourly windows x 128 candidates)", 24,
                       lambda lo, hi: P.build_config_tables(wins[lo:hi], cands, slo, m3, pol3, search, dev), reps=1))
    doc = {"how": "one B200; every rank's shard (sharding.shard_bounds) at each N timed end to end through the C ABI; "
                  "efficiency = T(1) / (N max_r T(shard_r)); no data-path collective (the final all-gather of result "
                  "rows is bytes per unit)",
           "weak_scaled": {"C2": "every rank decides its own 1024-decision corpus: per-rank work is constant",
                           "C4 day sweep": "every rank runs its own full-day scenarios: per-rank work is constant"},
           "projections": out}
    path = ROOT / "profiles" / "r02_scaling_projection.json"
    path.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc))


if __name__ == "__main__":
    main()

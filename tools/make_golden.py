"""Generates tests/golden/mpc_golden.json: decisions of the UNMODIFIED reference
(oracle/_ref/libpdsim_ref.so, compiled from /root/reference/proj/include by
oracle/Makefile) on seeded instances, so the oracle and the GPU path can be
pinned against the reference's own outputs on a box where neither
/root/reference nor the reference driver is available.

Instances come from the deterministic generators of tests/test_oracle_mpc.py
(_sandwich_instance: test_dvfs.cpp:278-305 shape; _llama_instance: SURVEY.md
§8d) and from workloads.c2_corpus (BASELINE C2: horizon 6 x 16 rungs).  Each
record holds the generator, its seed and position, and the reference's
decision-relevant result fields (helpers.result_tuple) plus
(feasible_count, best_code) for exhaustive MPC; floats are written with
repr(), which round-trips IEEE doubles exactly.

Run from the repo root (needs oracle/_ref built, i.e. __graft_entry__.build()
in the container that holds /root/reference):
    python tools/make_golden.py
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import oracle  # noqa: E402  (test infrastructure: the reference driver is the generator)
from helpers import cpu_decode, cpu_mpc, result_tuple  # noqa: E402
from test_oracle_mpc import _llama_instance, _sandwich_instance  # noqa: E402

from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200.workloads import c2_corpus  # noqa: E402

OUT = ROOT / "tests" / "golden" / "mpc_golden.json"

# (kind, generator, seed, count, generator kwargs)
MPC_SETS = [
    ("greedy", "sandwich", 0x601D, 40, {}),
    ("greedy", "llama", 0x601E, 40, {}),
    ("greedy", "llama", 0x601F, 16, {"levels": 24, "ladder_n": 24, "horizon": 8}),
    ("exhaustive", "sandwich", 0x6020, 30, {}),
    ("exhaustive", "llama", 0x6021, 20, {"levels": 8, "ladder_n": 5, "horizon": 4}),
    ("exhaustive", "llama", 0x6022, 8, {"levels": 16, "ladder_n": 16, "horizon": 3}),
    ("exhaustive", "llama", 0x6023, 4, {"levels": 24, "ladder_n": 24, "horizon": 5}),  # C5 grid, 24^5 = 8M each
]
C2_SEED, C2_COUNT = 0xC2, 2


def instances(gen: str, seed: int, count: int, kw: dict):
    rng = random.Random(seed)
    for _ in range(count):
        yield _sandwich_instance(rng) if gen == "sandwich" else _llama_instance(rng, **kw)


def decode_instances(seed: int, count: int):
    """test_dvfs.cpp:342-407 / acceptance_main.cpp:274-346 shape."""
    rng = random.Random(seed)
    menu = [500, 625, 750, 875, 1000, 1250, 1500, 1750, 2000]
    for _ in range(count):
        rungs = sorted(rng.sample(menu, rng.randint(3, 7)))
        lad = P.FrequencyLadder([float(r) for r in rungs])
        opt = P.SynthOptions(lat_coef=rng.uniform(1.0, 30.0))
        m = P.synth_model_set(P.SynthFamily.compute_bound, lad, [1], opt, opt)
        batch = P.BatchFeatures(rng.randint(1, 64), rng.randint(64, 16000))
        cfg = P.DecodePolicyConfig(ladder=lad, margin=rng.choice([0.0, 0.05, 0.2]),
                                   kv_threshold=rng.uniform(0.55, 0.9))
        cfg.tbt_slo_ms = rng.uniform(0.5, 3.0) * opt.lat_coef * batch.sum_len / rungs[-1]
        kv = P.KVCacheState(100000, rng.randint(0, 100000), 0.9)
        yield m, cfg, batch, kv


DECODE_SEED, DECODE_COUNT = 0x6030, 200


def record(kind, r) -> dict:
    d = {"result": list(result_tuple(r))}
    if kind == "exhaustive":
        d["feasible_count"], d["best_code"], d["trajectories"] = r.feasible_count, r.best_code, r.trajectories
    return d


# Config tables (build_config_table, placement.hpp:240-260) of C3-shaped
# 1-minute gamma(0.5) windows at 12 rps: TP {1,2,4,8} x 8 rungs x 2 phases.
PLACEMENT_SEEDS = [7, 8, 11]
PLACEMENT_WINDOW_MS = 60_000.0


def placement_inputs(seed: int):
    from paper_2602_18755_b200 import workloads as W
    lad = W.ladder(8)
    m = W.llama_models(lad)
    base = P.gen_gamma_trace(12.0, 0.5, PLACEMENT_WINDOW_MS,
                             P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), seed)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    return m, base, cands, P.SchedulerPolicy(max_batch_tokens=2048), P.SLOSpec(600.0, 100.0)


def table_row(e) -> list:
    return [int(e.config.phase), e.config.tp, e.config.base_freq_mhz, e.r_c, e.e_c, e.g_c, bool(e.saturated), e.error]


def main() -> None:
    from test_gpu_placement import _ref_table
    ref = oracle.load_ref()
    sets = []
    for kind, gen, seed, count, kw in MPC_SETS:
        recs = []
        for inst in instances(gen, seed, count, kw):
            rc, r = cpu_mpc(ref, kind, *inst)
            recs.append({"status": rc, **(record(kind, r) if rc == 0 else {})})
        sets.append({"kind": kind, "generator": gen, "seed": seed, "kwargs": kw, "records": recs})
    m, cfg, pol, snaps = c2_corpus(C2_SEED, C2_COUNT)
    c2 = []
    for q in snaps:
        rc, r = cpu_mpc(ref, "exhaustive", m, cfg, pol, q)
        c2.append({"status": rc, **record("exhaustive", r)})
    dec = []
    for m, cfg, batch, kv in decode_instances(DECODE_SEED, DECODE_COUNT):
        d = cpu_decode(ref, m, cfg, batch, kv, 1)
        dec.append([d.status, d.freq_mhz, d.eval_count, d.kv_override])
    tables = []
    for seed in PLACEMENT_SEEDS:
        for search in (P.GoodputSearch(), P.GoodputSearch(probe_count=2, tolerance_rps=0.5)):
            m, base, cands, pol, slo = placement_inputs(seed)
            want = _ref_table(ref, m, base, slo, pol, search, cands)
            tables.append({"seed": seed, "probe_count": search.probe_count, "tolerance_rps": search.tolerance_rps,
                           "n_requests": len(base.requests), "rows": [table_row(e) for e in want]})
    OUT.parent.mkdir(parents=True, exist_ok=True)
    doc = {"generated_by": "tools/make_golden.py from oracle/_ref/libpdsim_ref.so (the unmodified reference)",
           "mpc_sets": sets, "c2": {"seed": C2_SEED, "count": C2_COUNT, "records": c2},
           "decode": {"seed": DECODE_SEED, "count": DECODE_COUNT, "records": dec},
           "placement": tables}
    OUT.write_text(json.dumps(doc, indent=1) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()

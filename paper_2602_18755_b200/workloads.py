"""Synthetic workloads of BASELINE.json's configs, built with
the reference's own generators restated in ``pdsim`` (bit-identical).

* ``c2_corpus`` -- C2: exhaustive prefill MPC, horizon 6 x 16 rungs
  (16,777,216 trajectories per decision) on Llama-3.3-70B-shaped synthetic
  models (compute-bound family, prefill lat_coef 366 ms*MHz/token, power
  1e-7 f^3 + 60 W per GPU, TP knots {1, 2, 4, 8}).
* ``c1_corpus`` -- C1-style snapshots for the greedy MPC (horizon 8, N = 7 of
  the 8-rung H100-style ladder).
* ``c1_scenario`` -- C1 itself: the demo's trace parameters
  (demos/two_tier_demo.sh:16-18) with Poisson arrivals, one prefill + one
  decode instance under the two-tier controllers.
"""
from __future__ import annotations

import math
import random

from . import pdsim as P

PREFILL_OPT = dict(lat_coef=366.0, power_a=1e-7, power_b=60.0)
DECODE_OPT = dict(lat_coef=6.0, power_a=1e-7, power_b=120.0)


def ladder(levels: int) -> P.FrequencyLadder:
    """H100-style ladder: 8 rungs 360..1830 MHz in 210 MHz steps; L-level
    ladders 360 + i (1830 - 360) / (L - 1), computed in double."""
    if levels == 8:
        return P.FrequencyLadder([360.0 + 210.0 * i for i in range(8)])
    return P.FrequencyLadder([360.0 + i * (1830.0 - 360.0) / (levels - 1) for i in range(levels)])


def llama_models(lad: P.FrequencyLadder) -> P.ModelSet:
    return P.synth_model_set(P.SynthFamily.compute_bound, lad, [1, 2, 4, 8], P.SynthOptions(**PREFILL_OPT),
                             P.SynthOptions(**DECODE_OPT))


def synthetic_snapshot(rng: random.Random, lad: P.FrequencyLadder, *, n_lo: int = 4, n_hi: int = 24, tp: int = 2,
                       arrival_window_ms: float = 400.0, now_ms: float = 0.0) -> P.QueueSnapshot:
    """n ~ U[n_lo, n_hi] waiting requests, lognormal(6.2, 0.6) prompt lengths,
    arrivals now - U[0, window] ms (FCFS order), current = max rung."""
    n = rng.randint(n_lo, n_hi)
    arrivals = sorted(now_ms - rng.uniform(0.0, arrival_window_ms) for _ in range(n))
    q = P.QueueSnapshot(now_ms=now_ms, phase=P.Phase.prefill, tp=tp, current_freq_mhz=lad.max_mhz(),
                        target_freq_mhz=lad.max_mhz())
    for i, a in enumerate(arrivals):
        ln = max(1, int(round(math.exp(rng.gauss(6.2, 0.6)))))
        q.waiting.append(P.SnapshotWaiting(i, a, ln, ln))
    return q


def c2_corpus(seed: int = 0xC2, n: int = 64, ttft_ms: float = 600.0):
    """C2 problems: (models, MpcConfig, SchedulerPolicy, snapshots)."""
    lad = ladder(16)
    models = llama_models(lad)
    cfg = P.MpcConfig(horizon_K=6, ladder_N=16, ladder=lad, slo=P.SLOSpec(ttft_ms=ttft_ms))
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(seed)
    snaps = [synthetic_snapshot(rng, lad) for _ in range(n)]
    return models, cfg, pol, snaps


def c1_corpus(seed: int = 0xC1, n: int = 256):
    """Greedy MPC problems at the paper's operating point (K = 8, N = 7)."""
    lad = ladder(8)
    models = llama_models(lad)
    cfg = P.MpcConfig(horizon_K=8, ladder_N=7, ladder=lad)
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(seed)
    snaps = [synthetic_snapshot(rng, lad, n_lo=8, n_hi=32, arrival_window_ms=100.0) for _ in range(n)]
    return models, cfg, pol, snaps


def c1_scenario(duration_s: float = 600.0, rps: float = 14.0, seed: int = 7):
    """C1 (BASELINE.json configs[0]): the demo's trace
    (mean 14 rps, 600 s, seed 7, input lognormal(6.2, 0.4), output
    lognormal(2.9, 0.5); demos/two_tier_demo.sh:16-18) but Poisson (gamma
    shape 1), on a 1P(tp2) + 1D(tp4) cluster at max frequency with the
    two-tier controllers: greedy MPC mpc_k 8, mpc_n 7 of the 8-rung ladder,
    decode slack DVFS (margin 0.05), 600 / 100 ms SLOs, 30 s ramp-up."""
    lad = ladder(8)
    models = llama_models(lad)
    fmax = lad.max_mhz()
    pol = P.SchedulerPolicy(max_batch_tokens=2048, max_batch_requests=16)
    slo = P.SLOSpec(600.0, 100.0)
    tr = P.gen_gamma_trace(rps, 1.0, duration_s * 1000.0,
                           P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.4, 2.9, 0.5)), seed)
    inst = [P.ClusterInstance(P.InstanceConfig(P.Phase.prefill, 2, fmax), 1.0),
            P.ClusterInstance(P.InstanceConfig(P.Phase.decode, 4, fmax), 1.0)]
    fac = P.TwoTierFactory(P.MpcConfig(horizon_K=8, ladder_N=7, ladder=lad, slo=slo),
                           P.DecodePolicyConfig(tbt_slo_ms=slo.tpot_ms, ladder=lad, margin=0.05), models, pol)
    return models, P.ReplayScenario(tr, P.ClusterSpec(inst), pol, fac, P.SimOptions(30.0, -1.0), slo, 30.0)


def c5_corpus(seed: int = 0xC5, n: int = 4096, ttft_ms: float = 600.0):
    """C5 problems: horizon 8 on a 24-level grid (24^8 = 1.1e11 trajectories
    per decision exhaustively; greedy <= 22 levels x 6560 mutations)."""
    lad = ladder(24)
    models = llama_models(lad)
    cfg = P.MpcConfig(horizon_K=8, ladder_N=24, ladder=lad, slo=P.SLOSpec(ttft_ms=ttft_ms))
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(seed)
    snaps = [synthetic_snapshot(rng, lad, n_lo=8, n_hi=32, arrival_window_ms=200.0) for _ in range(n)]
    return models, cfg, pol, snaps


def c4_scenarios(n_scen: int = 1024, window_s: float = 300.0, rps: float = 12.0, seeds: int = 8, n_pre: int = 2,
                 n_dec: int = 2, levels: int = 8):
    """C4-shaped what-if sweep: scenario k replays trace seed k % seeds with
    the (TTFT, TPOT) pair (k // seeds) % 128 of {400..900} x {60..140} ms
    (16 x 8), on a fixed nP(tp2) + nD(tp4) cluster at max frequency with the
    two-tier controllers (greedy MPC K=8, N=7; decode slack policy), report
    after a 30 s ramp-up."""
    lad = ladder(levels)
    models = llama_models(lad)
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
        slo_i = (k // seeds) % 128
        slo = P.SLOSpec(ttfts[slo_i % 16], tpots[slo_i // 16])
        mpc = P.MpcConfig(horizon_K=8, ladder_N=7, ladder=lad, slo=slo)
        dec = P.DecodePolicyConfig(tbt_slo_ms=slo.tpot_ms, kv_threshold=0.9, ladder=lad, margin=0.05)
        fac = P.TwoTierFactory(mpc, dec, models, pol)
        scs.append(P.ReplayScenario(traces[k % seeds], P.ClusterSpec(list(inst)), pol, fac, P.SimOptions(30.0, -1.0),
                                    slo, 30.0))
    return models, scs

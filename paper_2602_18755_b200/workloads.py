"""Synthetic workloads of BASELINE.json's configs, built with
the reference's own generators restated in ``pdsim`` (bit-identical).

* ``c2_corpus`` -- C2: exhaustive prefill MPC, horizon 6 x 16 rungs
  (16,777,216 trajectories per decision) on Llama-3.3-70B-shaped synthetic
  models (compute-bound family, prefill lat_coef 366 ms*MHz/token, power
  1e-7 f^3 + 60 W per GPU, TP knots {1, 2, 4, 8}).
* ``c1_corpus`` -- C1-style snapshots for the greedy MPC (horizon 8, N = 7 of
  the 8-rung H100-style ladder).
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

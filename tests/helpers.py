"""Shared fixtures for the parity tests: the reference's own hand-built models
and snapshots (restated from /root/reference/proj/tests/test_dvfs.cpp), random
instance generators, and thin callers for the three implementations:

* ``gpu``    -- the product path (pdsim -> libbiscale_gpu.so, sm_100a);
* ``oracle`` -- the plain-C restatement (oracle/liboracle.so);
* ``ref``    -- the unmodified reference (oracle/_ref/libpdsim_ref.so).
"""
from __future__ import annotations

import ctypes as C
import math
import random

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P


# --- test_dvfs.cpp:18-56 ------------------------------------------------------

def dvfs_models() -> P.ModelSet:
    """test_dvfs.cpp:18-35: knots on every rung, dyadic-exact interpolants."""
    m = P.ModelSet()
    m.latency_prefill = P.LatencyTable(P.Phase.prefill, P.NdGrid(
        [P.Axis("sum_len", [0.0, 131072.0]), P.Axis("freq_mhz", [500.0, 750.0, 875.0, 1000.0])],
        [0.0, 0.0, 0.0, 0.0, 32768.0, 24576.0, 20480.0, 16384.0]))
    m.power_prefill = P.PowerTable(P.Phase.prefill, P.NdGrid(
        [P.Axis("freq_mhz", [500.0, 750.0, 875.0, 1000.0])], [100.0, 150.0, 175.0, 200.0]))
    m.latency_decode = P.LatencyTable(P.Phase.decode, P.NdGrid(
        [P.Axis("sum_len", [0.0, 1000.0]), P.Axis("freq_mhz", [500.0, 750.0, 1000.0])],
        [0.0, 0.0, 0.0, 15.0, 10.0, 5.0]))
    m.power_decode = P.PowerTable(P.Phase.decode, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])], [50.0, 100.0]))
    m.idle = P.IdlePowerModel([P.TpEntry(1, [500.0, 1000.0], [10.0, 10.0])])
    return m


def waiting_snapshot(lens, current_mhz=1000.0) -> P.QueueSnapshot:
    """test_dvfs.cpp:37-47."""
    q = P.QueueSnapshot(phase=P.Phase.prefill, tp=1, current_freq_mhz=current_mhz, target_freq_mhz=current_mhz)
    q.waiting = [P.SnapshotWaiting(i, 0.0, int(n), int(n)) for i, n in enumerate(lens)]
    return q


def mpc_config(ladder, ttft_ms, margin=0.0) -> P.MpcConfig:
    """test_dvfs.cpp:49-56."""
    cfg = P.MpcConfig()
    cfg.ladder = P.FrequencyLadder(list(ladder))
    cfg.ladder_N = len(ladder)
    cfg.slo.ttft_ms = ttft_ms
    cfg.margin = margin
    return cfg


# --- llama-shaped synthetic inputs --------------------------------

def h100_ladder(levels: int = 8) -> P.FrequencyLadder:
    if levels == 8:
        return P.FrequencyLadder([360.0 + 210.0 * i for i in range(8)])
    return P.FrequencyLadder([360.0 + i * (1830.0 - 360.0) / (levels - 1) for i in range(levels)])


def llama_models(ladder: P.FrequencyLadder) -> P.ModelSet:
    pre = P.SynthOptions(lat_coef=366.0, power_a=1e-7, power_b=60.0)
    dec = P.SynthOptions(lat_coef=6.0, power_a=1e-7, power_b=120.0)
    return P.synth_model_set(P.SynthFamily.compute_bound, ladder, [1, 2, 4, 8], pre, dec)


def random_snapshot(rng: random.Random, *, n_lo=4, n_hi=24, current=None, tp=2, now=0.0,
                    running_prob=0.0, ladder=None, arrival_window=400.0) -> P.QueueSnapshot:
    """SURVEY.md §8d C2 corpus shape: n ~ U[n_lo, n_hi] waiting, lognormal(6.2, 0.6)
    lengths, arrivals now - U[0, arrival_window] ms."""
    n = rng.randint(n_lo, n_hi)
    q = P.QueueSnapshot(now_ms=now, phase=P.Phase.prefill, tp=tp)
    arrivals = sorted((now - rng.uniform(0.0, arrival_window) for _ in range(n)))
    for i in range(n):
        ln = max(1, int(round(math.exp(rng.gauss(6.2, 0.6)))))
        q.waiting.append(P.SnapshotWaiting(i, arrivals[i], ln, ln))
    if ladder is not None:
        q.current_freq_mhz = current if current is not None else ladder.max_mhz()
        q.target_freq_mhz = q.current_freq_mhz
    if running_prob and rng.random() < running_prob:
        m = rng.randint(1, 4)
        q.running.active = True
        q.running.ids = list(range(100, 100 + m))
        q.running.completes = [rng.random() < 0.7 for _ in range(m)]
        q.running.arrivals_ms = [now - rng.uniform(0.0, 300.0) for _ in range(m)]
        lens = [rng.randint(50, 600) for _ in range(m)]
        q.running.features = P.BatchFeatures.from_lengths(lens)
        q.running.work_remaining = rng.choice([0.1, 0.25, 0.5, 0.75, 1.0, rng.random()])
    return q


# --- callers into the CPU checkers --------------------------------------------------

class Packed:
    """ctypes arguments for one (models, cfg, policy, snapshot) problem."""

    def __init__(self, models: P.ModelSet, cfg: P.MpcConfig | None = None, policy: P.SchedulerPolicy | None = None,
                 q: P.QueueSnapshot | None = None):
        self.keep: list = []
        self.models = P.c_model_set(models, self.keep)
        self.cfg = P.c_mpc_config(cfg, self.keep) if cfg is not None else None
        self.policy = P.c_policy(policy or P.SchedulerPolicy())
        self.snap = P.c_snapshot(q, self.keep) if q is not None else None


def cpu_mpc(lib, kind: str, models, cfg, policy, q) -> tuple:
    """kind in {greedy, exhaustive}; returns (status, bs_mpc_result)."""
    p = Packed(models, cfg, policy, q)
    out = A.bs_mpc_result()
    prefix = "orc_" if hasattr(lib, "orc_greedy") else "ref_"
    rc = getattr(lib, prefix + kind)(C.byref(p.models), C.byref(p.cfg), C.byref(p.policy), C.byref(p.snap),
                                     C.byref(out))
    return rc, out


def cpu_project(lib, cfg, policy, q) -> tuple:
    p = Packed(dvfs_models(), cfg, policy, q)
    out = (A.bs_projected_batch * A.BS_MAX_K)()
    K = C.c_int32()
    prefix = "orc_" if hasattr(lib, "orc_greedy") else "ref_"
    rc = getattr(lib, prefix + "project")(C.byref(p.cfg), C.byref(p.policy), C.byref(p.snap), out, C.byref(K))
    return rc, [out[k] for k in range(K.value)]


def cpu_eval_codes(lib, models, cfg, policy, q, codes) -> tuple:
    p = Packed(models, cfg, policy, q)
    n = len(codes)
    ca = (C.c_uint64 * max(1, n))(*codes)
    feas = (C.c_int32 * max(1, n))()
    obj = (C.c_double * max(1, n))()
    prefix = "orc_" if hasattr(lib, "orc_greedy") else "ref_"
    rc = getattr(lib, prefix + "eval_codes")(C.byref(p.models), C.byref(p.cfg), C.byref(p.policy), C.byref(p.snap),
                                            ca, n, feas, obj)
    return rc, [bool(x) for x in feas[:n]], list(obj[:n])


def cpu_decode(lib, models, cfg: P.DecodePolicyConfig, batch: P.BatchFeatures, kv: P.KVCacheState, tp: int):
    keep: list = []
    cm = P.c_model_set(models, keep)
    cc = P.c_decode_config(cfg, keep)
    q = A.bs_decode_query()
    q.batch.n_requests = batch.n_requests
    q.batch.sum_len = batch.sum_len
    q.kv_capacity_tokens = kv.capacity_tokens
    q.kv_used_tokens = kv.used_tokens
    q.tp = tp
    out = A.bs_decode_result()
    prefix = "orc_" if hasattr(lib, "orc_greedy") else "ref_"
    getattr(lib, prefix + "decode_pick")(C.byref(cm), C.byref(cc), C.byref(q), 1, C.byref(out))
    return out


def cpu_predict(lib, models, which: int, feats, tps, freqs):
    keep: list = []
    cm = P.c_model_set(models, keep)
    n = len(feats)
    fa = (A.bs_features * n)()
    for i, (nr, sl) in enumerate(feats):
        fa[i].n_requests, fa[i].sum_len = nr, sl
    ta = (C.c_int32 * n)(*tps)
    fr = (C.c_double * n)(*freqs)
    out = (C.c_double * n)()
    st = (C.c_int32 * n)()
    prefix = "orc_predict_batch" if hasattr(lib, "orc_greedy") else "ref_predict"
    getattr(lib, prefix)(C.byref(cm), which, fa, ta, fr, n, out, st)
    return list(out), list(st)


def result_tuple(r: A.bs_mpc_result) -> tuple:
    """Decision-relevant fields of a result, for equality checks."""
    return (r.K, r.feasible, r.eval_count, r.objective_w, tuple(r.freqs_mhz[: r.K]), r.decision_freq_mhz,
            tuple((r.levels[i].level, r.levels[i].k_prime, r.levels[i].replaced_mhz, r.levels[i].mutations,
                   r.levels[i].feasible_mutations, r.levels[i].accepted) for i in range(max(0, r.n_levels))))


def gpu_result_tuple(g: P.GreedyResult, K: int) -> tuple:
    return (K, int(g.feasible), g.eval_count, g.objective_w, tuple(g.assignment.freqs), g.decision_freq_mhz,
            tuple((lv.level, lv.k_prime, lv.replaced_mhz, lv.mutations, lv.feasible_mutations, int(lv.accepted))
                  for lv in g.levels))

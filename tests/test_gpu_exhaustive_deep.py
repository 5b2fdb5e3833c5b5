"""GPU parity of the exhaustive MPC paths that the default BASELINE shapes
only reach at sizes the CPU cannot brute-force (C5, 24^8):

* the three-level leaf sweep (sweep_levels == 3, every C5 decision): forced
  on trees the compiled reference enumerates in seconds by lowering the
  context's sweep-depth threshold (bs_ctx_set_exhaustive_limits);
* the frontier-overflow path (a batch whose lists exceed the context's
  capacities is split and re-run): forced with small capacities;
* slices of one decision's code space (bs_mpc_exhaustive_slice, SURVEY.md
  §8e): the union of a partition's slices equals the unsliced decision
  bitwise, for C2- and C5-shaped decisions and for trees below prepare's
  first list;
* batches of non-divisible sizes that take the pipelined pack / sliced
  result paths (>= 512 problems), greedy and exhaustive, with mixed
  horizons, configurations and empty snapshots, every decision checked.

Every reference answer is the unmodified reference (oracle/_ref) or the
pinned C restatement (oracle/liboracle.so); the tie rule is dvfs.hpp:243
(smallest objective, then the lexicographically smallest assignment).
"""
from __future__ import annotations

import ctypes as C
import os
import random

import pytest

from helpers import cpu_mpc, gpu_result_tuple, result_tuple
from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P
from paper_2602_18755_b200 import sharding as S
from paper_2602_18755_b200 import workloads as W

pytestmark = pytest.mark.gpu

THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture()
def dev():
    """A private context whose limits the test may change."""
    d = P.Device(0)
    yield d
    d.close()


def _ref_batch(ref_lib, m, cfg, pol, snaps):
    """The compiled reference's exhaustive loop (tests/test_dvfs.cpp:74-94 with
    the dvfs.hpp:243 tie rule) over the host's threads."""
    keep: list = []
    cm, cc, cp = P.c_model_set(m, keep), P.c_mpc_config(cfg, keep), P.c_policy(pol)
    probs = P.c_problems(snaps, None, keep)
    out = (A.bs_mpc_result * len(snaps))()
    assert ref_lib.ref_exhaustive_batch(C.byref(cm), C.byref(cc), C.byref(cp), probs, len(snaps), out, THREADS) == 0
    return [out[i] for i in range(len(snaps))]


def _corpus(levels: int, horizon: int, n: int, seed: int, ttft: float = 600.0, **kw):
    lad = W.ladder(levels)
    m = W.llama_models(lad)
    cfg = P.MpcConfig(horizon_K=horizon, ladder_N=levels, ladder=lad, slo=P.SLOSpec(ttft_ms=ttft))
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(seed)
    snaps = [W.synthetic_snapshot(rng, lad, **kw) for _ in range(n)]
    return m, cfg, pol, snaps


def _check(got, want):
    for g, r in zip(got, want):
        assert gpu_result_tuple(g, r.K) == result_tuple(r)
        assert (g.feasible_count, g.best_code, g.trajectories) == (r.feasible_count, r.best_code, r.trajectories)


@pytest.mark.parametrize("levels,horizon,n,ttft", [(12, 6, 6, 600.0), (10, 7, 3, 900.0), (16, 5, 8, 1200.0),
                                                  (24, 5, 2, 600.0)])
def test_three_level_sweep_matches_reference(dev, ref_lib, levels, horizon, n, ttft):
    """sweep_levels == 3 (the C5 path, bs_exhaustive.cuh I == 3) on trees of
    1M-10M trajectories: threshold 64 prefixes at depth K - 2."""
    m, cfg, pol, snaps = _corpus(levels, horizon, n, 0x3E + levels, ttft, n_lo=horizon + 2, n_hi=3 * horizon,
                                 arrival_window_ms=200.0)
    dev.set_exhaustive_limits(sweep3_min_prefixes=64.0)
    got = P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)
    want = _ref_batch(ref_lib, m, cfg, pol, snaps)
    assert any(r.K == horizon for r in want)
    _check(got, want)
    dev.set_exhaustive_limits()  # defaults: two levels at these sizes, same answers
    _check(P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev), want)


def test_n24_exhaustive_matches_reference(dev, ref_lib):
    """24 candidate rungs (C5's grid) at H5: 24^5 = 8M trajectories per decision."""
    m, cfg, pol, snaps = _corpus(24, 5, 3, 0x245, 600.0, n_lo=6, n_hi=20, arrival_window_ms=200.0)
    want = _ref_batch(ref_lib, m, cfg, pol, snaps)
    _check(P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev), want)


@pytest.mark.parametrize("level_cap,final_cap", [(0, 9000), (2000, 0), (2000, 9000)])
def test_frontier_overflow_splits_batch(dev, oracle_lib, level_cap, final_cap):
    """Frontier capacities far below the batch's lists: the one-shot call
    observes the overflow, splits the batch and re-runs the pieces; every
    decision still equals the C restatement (one decision needs at most
    6^5 final and 6^4 level entries, so every piece fits)."""
    lad = W.ladder(6)
    m = W.llama_models(lad)
    cfg = P.MpcConfig(horizon_K=7, ladder_N=6, ladder=lad, slo=P.SLOSpec(ttft_ms=1500.0))
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(0x0F)
    snaps = [W.synthetic_snapshot(rng, lad, n_lo=8, n_hi=20, arrival_window_ms=100.0) for _ in range(24)]
    dev.set_exhaustive_limits(level_cap=level_cap, final_cap=final_cap)
    got = P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)
    for q, g in zip(snaps, got):
        rc, r = cpu_mpc(oracle_lib, "exhaustive", m, cfg, pol, q)
        assert rc == 0
        assert gpu_result_tuple(g, r.K) == result_tuple(r)
        assert (g.feasible_count, g.best_code) == (r.feasible_count, r.best_code)


def test_one_decision_over_budget_is_a_parameter_error(dev):
    m, cfg, pol, snaps = _corpus(8, 6, 1, 0x0E, 5000.0, n_lo=10, n_hi=12)
    dev.set_exhaustive_limits(level_cap=64, final_cap=64)
    with pytest.raises(P.ParameterError, match="frontier budget"):
        P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)


def _sliced(snaps, cfg, m, pol, dev, digits, bounds):
    parts = [P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev, code_slice=(digits, lo, hi))
             for lo, hi in bounds]
    out = []
    for i in range(len(snaps)):
        out.append(S.combine_slices([(p[i].feasible, p[i].objective_w, p[i].best_code, p[i].feasible_count)
                                     for p in parts]))
        assert all(p[i].trajectories == p[i].eval_count for p in parts)
    return out, parts


def _whole(g):
    return (g.objective_w if g.feasible else None, g.best_code if g.feasible else None, g.feasible_count)


@pytest.mark.parametrize("digits,bounds", [(1, [(0, 5), (5, 11), (11, 16)]),
                                           (2, [(i * 37, min(256, (i + 1) * 37)) for i in range(7)])])
def test_c2_slices_union_equals_unsliced(dev, ref_lib, digits, bounds):
    """A C2 decision (16^6) cut into unequal leading-digit slices: the
    combined (objective, code) minimum and the summed feasible counts equal
    the unsliced decision and the compiled reference."""
    m, cfg, pol, snaps = W.c2_corpus(0xC2, 3, ttft_ms=1200.0)
    whole = P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)
    comb, parts = _sliced(snaps, cfg, m, pol, dev, digits, bounds)
    for i, g in enumerate(whole):
        assert comb[i] == _whole(g)
        assert sum(p[i].trajectories for p in parts) == g.trajectories == 16 ** 6
    if digits == 1:  # the looser-SLO C2 decision itself against the compiled reference (~40 s on one core)
        want = _ref_batch(ref_lib, m, cfg, pol, snaps[:1])
        assert (whole[0].best_code, whole[0].objective_w, whole[0].feasible_count) == \
            (want[0].best_code, want[0].objective_w, want[0].feasible_count)


def test_c5_slices_union_equals_unsliced(dev):
    """C5-shaped decisions (24^8 = 1.1e11 trajectories, three-level sweep)
    sliced by S.prefix_slice over 8 ranks and over 24 leading digits."""
    m, cfg, pol, snaps = W.c5_corpus(0xC5, 2)
    whole = P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)
    for world in (8, 24):
        spans = [S.prefix_slice(24, r, world) for r in range(world)]
        assert all(d == 1 for d, _, _ in spans)
        comb, parts = _sliced(snaps, cfg, m, pol, dev, 1, [(lo, hi) for _, lo, hi in spans])
        for i, g in enumerate(whole):
            assert g.trajectories == 24 ** 8
            assert comb[i] == _whole(g)


def test_small_tree_and_short_projection_slices(dev, oracle_lib):
    """Trees of K <= 3 (evaluated whole in prepare_kernel when sliced) and
    projections shorter than the slice's digits: the slices still partition
    every tree."""
    lad = W.ladder(7)
    m = W.llama_models(lad)
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(0x51)
    for horizon in (1, 2, 3, 4):
        cfg = P.MpcConfig(horizon_K=horizon, ladder_N=7, ladder=lad, slo=P.SLOSpec(ttft_ms=900.0))
        snaps = [W.synthetic_snapshot(rng, lad, n_lo=0, n_hi=3 * horizon, arrival_window_ms=150.0)
                 for _ in range(12)]
        whole = P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)
        for digits, bounds in ((1, [(0, 3), (3, 4), (4, 7)]), (2, [(0, 10), (10, 10), (10, 33), (33, 49)])):
            comb, parts = _sliced(snaps, cfg, m, pol, dev, digits, bounds)
            for i, (q, g) in enumerate(zip(snaps, whole)):
                rc, r = cpu_mpc(oracle_lib, "exhaustive", m, cfg, pol, q)
                assert (g.best_code, g.objective_w, g.feasible_count) == (r.best_code, r.objective_w,
                                                                          r.feasible_count)
                if g.assignment.freqs:
                    assert comb[i] == _whole(g)
                    assert sum(p[i].trajectories for p in parts) == g.trajectories


def test_slices_with_three_level_sweep(dev, ref_lib):
    m, cfg, pol, snaps = _corpus(12, 6, 2, 0x5E, 900.0, n_lo=8, n_hi=18, arrival_window_ms=200.0)
    dev.set_exhaustive_limits(sweep3_min_prefixes=64.0)
    whole = P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev)
    comb, _ = _sliced(snaps, cfg, m, pol, dev, 2, [(0, 50), (50, 51), (51, 144)])
    want = _ref_batch(ref_lib, m, cfg, pol, snaps)
    for i, (g, r) in enumerate(zip(whole, want)):
        assert (g.best_code, g.objective_w, g.feasible_count) == (r.best_code, r.objective_w, r.feasible_count)
        assert comb[i] == _whole(g)


def test_slice_arguments_are_validated(dev):
    m, cfg, pol, snaps = _corpus(8, 4, 1, 1, 600.0)
    for bad in ((3, 0, 1), (1, 5, 4), (1, 0, 9), (2, 0, 65)):
        with pytest.raises(P.ParameterError):
            P.exhaustive_freq_select_batch(snaps, cfg, m, pol, device=dev, code_slice=bad)


def _mixed_batch(n: int, seed: int):
    """n problems over three configurations (different horizons and ladders),
    some snapshots empty (no waiting, no running batch)."""
    lad8, lad6 = W.ladder(8), W.ladder(6)
    m = W.llama_models(W.ladder(8))
    cfgs = [P.MpcConfig(horizon_K=4, ladder_N=5, ladder=lad8, slo=P.SLOSpec(ttft_ms=700.0)),
            P.MpcConfig(horizon_K=3, ladder_N=8, ladder=lad8, slo=P.SLOSpec(ttft_ms=500.0), margin=0.0),
            P.MpcConfig(horizon_K=5, ladder_N=4, ladder=lad8, slo=P.SLOSpec(ttft_ms=900.0), switch_latency_ms=7.25)]
    pols = [P.SchedulerPolicy(max_batch_tokens=512), P.SchedulerPolicy(max_batch_tokens=1024),
            P.SchedulerPolicy(max_batch_tokens=768, chunking=False)]
    rng = random.Random(seed)
    snaps, idx = [], []
    for i in range(n):
        c = rng.randrange(3)
        if rng.random() < 0.08:
            q = P.QueueSnapshot(phase=P.Phase.prefill, tp=2, current_freq_mhz=1830.0, target_freq_mhz=1200.0)
        else:
            q = W.synthetic_snapshot(rng, lad8 if c < 2 else lad6, n_lo=0, n_hi=14, arrival_window_ms=150.0)
            q.current_freq_mhz = rng.choice([1830.0, 990.0, 1500.0])
        snaps.append(q)
        idx.append(c)
    return m, cfgs, pols, snaps, idx


@pytest.mark.parametrize("n", [513, 1100, 4097])
def test_large_odd_batches_greedy_and_exhaustive(dev, oracle_lib, n):
    """Batch sizes that are not multiples of the pack / result slices (the
    pipelined H2D pack, host-pool expansion and per-slice D2H events engage
    from 512 problems): every decision equals the C restatement."""
    m, cfgs, pols, snaps, idx = _mixed_batch(n, n)
    for kind in ("greedy", "exhaustive"):
        got = P._mpc_batch("bs_mpc_" + kind, snaps, cfgs, pols, idx, m, dev)
        step = 1 if n <= 1100 else 3
        for i in list(range(0, n, step)) + [n - 1]:
            rc, r = cpu_mpc(oracle_lib, kind, m, cfgs[idx[i]], pols[idx[i]], snaps[i])
            assert rc == 0
            assert gpu_result_tuple(got[i], r.K) == result_tuple(r), (kind, i)
            if kind == "exhaustive":
                assert (got[i].feasible_count, got[i].best_code) == (r.feasible_count, r.best_code)

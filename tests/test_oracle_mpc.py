"""Pins the CPU checkers (not GPU): the plain-C oracle and the compiled
reference driver must reproduce the reference's own known-answer tests
(/root/reference/proj/tests/test_dvfs.cpp, test_perfmodel.cpp) and agree
with each other bit for bit on random instances."""
from __future__ import annotations

import ctypes as C
import math
import random

import pytest

from helpers import (Packed, cpu_decode, cpu_eval_codes, cpu_mpc, cpu_predict, cpu_project, dvfs_models,
                     h100_ladder, llama_models, mpc_config, random_snapshot, result_tuple, waiting_snapshot)
from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P


@pytest.fixture(params=["oracle", "ref"])
def cpu(request, oracle_lib):
    if request.param == "oracle":
        return oracle_lib
    return request.getfixturevalue("ref_lib")


# --- test_perfmodel.cpp KATs ---------------------------------------------------------

def _interp(lib, grid: P.NdGrid, coords):
    keep: list = []
    g = P.c_grid(grid, keep)
    out = C.c_double()
    cl = C.c_uint32(0)
    if hasattr(lib, "orc_interpolate"):
        lib.orc_interpolate(C.byref(g), (C.c_double * len(coords))(*coords), C.byref(out), C.byref(cl))
    else:
        lib.ref_interpolate(C.byref(g), (C.c_double * len(coords))(*coords), 1, C.byref(out), C.byref(cl))
    return out.value, cl.value


def plane_grid():  # test_perfmodel.cpp:14-20
    return P.NdGrid([P.Axis("x", [0.0, 10.0]), P.Axis("y", [0.0, 100.0])], [0.0, 100.0, 10.0, 110.0])


def test_interpolation_plane_kats(cpu):
    g = plane_grid()
    assert _interp(cpu, g, [0.0, 0.0]) == (0.0, 0)
    assert _interp(cpu, g, [10.0, 100.0]) == (110.0, 0)
    assert _interp(cpu, g, [2.5, 30.0])[0] == pytest.approx(32.5)
    assert _interp(cpu, g, [7.0, 99.0])[0] == pytest.approx(106.0)
    # clamping counts one event per clamped axis (test_perfmodel.cpp:83-89)
    assert _interp(cpu, g, [-5.0, 30.0]) == (pytest.approx(30.0), 1)
    assert _interp(cpu, g, [15.0, 200.0]) == (pytest.approx(110.0), 2)


def test_single_knot_axis(cpu):  # test_perfmodel.cpp:103-109
    g = P.NdGrid([P.Axis("x", [5.0]), P.Axis("y", [0.0, 1.0])], [3.0, 7.0])
    assert _interp(cpu, g, [5.0, 0.5])[0] == pytest.approx(5.0)


def test_ladder_select_kats(oracle_lib):  # test_perfmodel.cpp:44-63
    lad = [500.0, 750.0, 1000.0, 1250.0, 1500.0, 1750.0, 2000.0]
    out = (C.c_double * 16)()

    def sel(n):
        k = oracle_lib.orc_ladder_select((C.c_double * 7)(*lad), 7, n, out)
        return list(out[:k]) if k >= 0 else None

    assert sel(2) == [500.0, 2000.0]
    assert sel(3) == [500.0, 1250.0, 2000.0]
    assert sel(1) == [2000.0]
    assert sel(7) == lad and sel(99) == lad
    assert sel(0) is None
    host = P.FrequencyLadder(lad)
    for n in range(1, 10):
        assert host.select(n).freqs_mhz == sel(n)


def test_synth_model_set_bit_identical(oracle_lib, ref_lib):
    """synth_model_set (perfmodel.hpp:397-516): oracle, reference and the host
    mirror produce identical grid bits."""
    for ladder, tps in ((h100_ladder(8), [1, 2, 4, 8]), (h100_ladder(16), [8, 2, 1, 4, 2]), (h100_ladder(24), [3])):
        for fam in (0, 1):
            po = P.SynthOptions(lat_coef=366.0, power_a=1e-7, power_b=60.0, mem_knee_mhz=1200.0, idle_frac=0.35)
            do = P.SynthOptions(lat_coef=6.0, power_a=3e-8, power_b=120.0, mem_knee_mhz=900.0, idle_frac=0.2)
            host = P.synth_model_set(P.SynthFamily(fam), ladder, tps, po, do)
            nl, nt = len(ladder.freqs_mhz), len(set(tps))
            sizes = (6 * 9 * nt * nl, 6 * 9 * nt * nl, 6 * nt * nl, 6 * 9 * nt * nl, nt * nl)
            outs = {}
            for name, lib, fn in (("orc", oracle_lib, "orc_synth_model_set"), ("ref", ref_lib, "ref_synth_model_set")):
                bufs = [(C.c_double * s)() for s in sizes]
                rc = getattr(lib, fn)(fam, (C.c_double * nl)(*ladder.freqs_mhz), nl, (C.c_int32 * len(tps))(*tps),
                                      len(tps), (C.c_double * 5)(*po.as_array()), (C.c_double * 5)(*do.as_array()),
                                      *bufs)
                assert rc == 0
                outs[name] = [list(b) for b in bufs]
            hv = [host.latency_prefill.grid.values, host.latency_decode.grid.values, host.power_prefill.grid.values,
                  host.power_decode.grid.values, [w for e in host.idle.entries for w in e.idle_w]]
            assert outs["orc"] == outs["ref"] == hv


def test_predict_matches_reference(oracle_lib, ref_lib):
    rng = random.Random(7)
    m = llama_models(h100_ladder(16))
    feats = [(rng.randint(0, 300), rng.randint(0, 20000)) for _ in range(400)]
    tps = [rng.choice([1, 2, 3, 4, 8, 16]) for _ in range(400)]
    freqs = [rng.uniform(200.0, 2000.0) for _ in range(400)]
    for which in range(5):
        a = cpu_predict(oracle_lib, m, which, feats, tps, freqs)
        b = cpu_predict(ref_lib, m, which, feats, tps, freqs)
        assert a == b


# --- test_dvfs.cpp KATs ---------------------------------------------------------------

def test_projection_kats(cpu):  # test_dvfs.cpp:98-134
    pol = P.SchedulerPolicy(max_batch_tokens=100)
    rc, proj = cpu_project(cpu, mpc_config([500.0, 1000.0], 600.0), pol, waiting_snapshot([50, 50, 50]))
    assert rc == 0 and len(proj) == 2
    assert (proj[0].features.n_requests, proj[0].features.sum_len, proj[0].n_completing) == (2, 100, 2)
    assert proj[0].work_fraction == 1.0
    assert (proj[1].features.sum_len, proj[1].n_completing) == (50, 1)
    cfg1 = mpc_config([500.0, 1000.0], 600.0)
    cfg1.horizon_K = 1
    assert len(cpu_project(cpu, cfg1, pol, waiting_snapshot([50, 50, 50]))[1]) == 1
    cfg0 = mpc_config([500.0, 1000.0], 600.0)
    cfg0.horizon_K = 0
    assert cpu_project(cpu, cfg0, pol, waiting_snapshot([50, 50, 50]))[0] == A.BS_PARAMETER_ERROR

    q = waiting_snapshot([80])
    q.running = P.SnapshotRunning(True, [40, 41], [0, 0], [True, False], [-50.0, -20.0], 0.4, 0.0,
                                  P.BatchFeatures.from_lengths([300, 300]))
    rc, proj = cpu_project(cpu, mpc_config([500.0, 1000.0], 600.0), pol, q)
    assert len(proj) == 2
    assert proj[0].features.sum_len == 600 and proj[0].work_fraction == 0.4
    assert proj[0].n_completing == 1 and proj[0].min_completing_arrival_ms == -50.0
    assert proj[1].features.sum_len == 80


def _meets(cpu, cfg, pol, q, freqs):
    cand = cfg.candidates().freqs_mhz
    code = 0
    for f in freqs:
        code = code * len(cand) + cand.index(f)
    rc, feas, _ = cpu_eval_codes(cpu, dvfs_models(), cfg, pol, q, [code])
    assert rc == 0
    return feas[0]


def test_meets_slo_kats(cpu):  # test_dvfs.cpp:136-181
    pol = P.SchedulerPolicy(max_batch_tokens=100)
    q = waiting_snapshot([100, 100], 500.0)
    q.now_ms = 100.0
    L = [500.0, 1000.0]
    assert _meets(cpu, mpc_config(L, 155.0), pol, q, [1000.0, 1000.0])
    assert not _meets(cpu, mpc_config(L, 150.0), pol, q, [1000.0, 1000.0])
    assert _meets(cpu, mpc_config(L, 150.0), pol, q, [500.0, 500.0])
    assert not _meets(cpu, mpc_config(L, 149.0), pol, q, [500.0, 500.0])
    assert _meets(cpu, mpc_config(L, 160.5, 0.1), pol, q, [1000.0, 1000.0])
    assert not _meets(cpu, mpc_config(L, 160.4, 0.1), pol, q, [1000.0, 1000.0])

    q = waiting_snapshot([], 1000.0)
    q.running = P.SnapshotRunning(True, [7], [0], [True], [0.0], 0.25, 0.0, P.BatchFeatures.from_lengths([800]))
    q.now_ms = 50.0
    assert _meets(cpu, mpc_config(L, 75.0), P.SchedulerPolicy(), q, [1000.0])
    assert not _meets(cpu, mpc_config(L, 74.0), P.SchedulerPolicy(), q, [1000.0])


def test_greedy_kats(cpu):  # test_dvfs.cpp:183-276
    m = dvfs_models()
    rc, g = cpu_mpc(cpu, "greedy", m, mpc_config([500.0, 1000.0], 600.0), P.SchedulerPolicy(),
                    waiting_snapshot([100], 500.0))
    assert rc == 0 and g.feasible and g.K == 1 and g.freqs_mhz[0] == 500.0
    assert g.objective_w == 100.0 and g.eval_count == 2 and g.n_levels == 1
    assert (g.levels[0].k_prime, g.levels[0].mutations, g.levels[0].feasible_mutations, g.levels[0].accepted) == \
        (1, 1, 1, 1)

    rc, g = cpu_mpc(cpu, "greedy", m, mpc_config([500.0, 1000.0], 10.0), P.SchedulerPolicy(),
                    waiting_snapshot([100], 1000.0))
    assert not g.feasible and g.freqs_mhz[0] == 1000.0 and g.eval_count == 1 and g.n_levels == 0

    pol = P.SchedulerPolicy(max_batch_tokens=100)
    rc, g = cpu_mpc(cpu, "greedy", m, mpc_config([500.0, 750.0, 875.0, 1000.0], 61.2), pol,
                    waiting_snapshot([100, 100], 1000.0))
    assert g.feasible and list(g.freqs_mhz[:2]) == [1000.0, 875.0]
    assert abs(g.objective_w - 5234.375 / 28.125) < 1e-12 and g.eval_count == 11
    assert g.n_levels == 2
    l0, l1 = g.levels[0], g.levels[1]
    assert (l0.level, l0.replaced_mhz, l0.k_prime, l0.mutations, l0.feasible_mutations, l0.accepted) == \
        (1, 1000.0, 2, 8, 1, 1)
    assert (l1.level, l1.replaced_mhz, l1.k_prime, l1.mutations, l1.feasible_mutations, l1.accepted) == \
        (2, 875.0, 1, 2, 0, 0)

    rc, two = cpu_mpc(cpu, "greedy", m, mpc_config([500.0, 1000.0], 10000.0), pol,
                      waiting_snapshot([100, 100, 100], 1000.0))
    assert two.n_levels == 1 and (two.levels[0].k_prime, two.levels[0].mutations,
                                  two.levels[0].feasible_mutations) == (3, 7, 7)
    assert two.eval_count == 8 and list(two.freqs_mhz[:3]) == [500.0] * 3
    rc, one = cpu_mpc(cpu, "greedy", m, mpc_config([1000.0], 10000.0), pol, waiting_snapshot([100, 100, 100], 1000.0))
    assert one.feasible and one.eval_count == 1 and one.n_levels == 0 and list(one.freqs_mhz[:3]) == [1000.0] * 3

    rc, g = cpu_mpc(cpu, "greedy", m, mpc_config([500.0, 1000.0], 600.0), P.SchedulerPolicy(), waiting_snapshot([]))
    assert g.feasible and g.K == 0 and g.eval_count == 0 and g.objective_w == 0.0


def test_decode_kats(cpu):  # test_dvfs.cpp:342-407
    m = dvfs_models()
    cfg = P.DecodePolicyConfig(tbt_slo_ms=10.0, ladder=P.FrequencyLadder([500.0, 750.0, 1000.0]))
    kv = P.KVCacheState(1000, 100, 0.9)
    big = P.BatchFeatures.from_lengths([100] * 10)
    small = P.BatchFeatures.from_lengths([100] * 5)
    d = cpu_decode(cpu, m, cfg, big, kv, 1)
    assert (d.freq_mhz, d.eval_count, d.kv_override) == (750.0, 2, 0)
    d = cpu_decode(cpu, m, cfg, small, kv, 1)
    assert (d.freq_mhz, d.eval_count) == (500.0, 1)
    cfg.margin = 0.05
    d = cpu_decode(cpu, m, cfg, big, kv, 1)
    assert (d.freq_mhz, d.eval_count) == (1000.0, 3)
    cfg.margin = 0.0
    cfg.tbt_slo_ms = 2.0
    d = cpu_decode(cpu, m, cfg, big, kv, 1)
    assert (d.freq_mhz, d.eval_count, d.kv_override) == (1000.0, 3, 0)
    cfg.tbt_slo_ms = 100.0
    one = P.BatchFeatures.from_lengths([100])
    d = cpu_decode(cpu, m, cfg, one, P.KVCacheState(1000, 901, 0.9), 1)
    assert (d.freq_mhz, d.kv_override, d.eval_count) == (1000.0, 1, 0)
    d = cpu_decode(cpu, m, cfg, one, P.KVCacheState(1000, 900, 0.9), 1)
    assert (d.freq_mhz, d.kv_override) == (500.0, 0)


# --- random three-way agreement (oracle vs the reference itself) -------------------------

def _sandwich_instance(rng):
    """test_dvfs.cpp:278-305 shape, drawn with Python's RNG."""
    policy = P.SchedulerPolicy(max_batch_tokens=rng.choice([64, 128, 256]), chunking=rng.random() < 0.5)
    lens = [20 + rng.randrange(180) for _ in range(1 + rng.randrange(4))]
    q = waiting_snapshot(lens, 1000.0)
    if rng.randrange(3) == 0:
        q.running = P.SnapshotRunning(True, [99], [0], [True], [0.0], 0.25 * (1 + rng.randrange(3)), 0.0,
                                      P.BatchFeatures.from_lengths([50 + rng.randrange(300)]))
    cfg = mpc_config([500.0, 750.0, 1000.0], rng.choice([60.0, 100.0, 150.0, 250.0, 400.0, 10000.0]), 0.05)
    cfg.horizon_K = 4
    return dvfs_models(), cfg, policy, q


def _llama_instance(rng, levels=8, ladder_n=7, horizon=6):
    ladder = h100_ladder(levels)
    m = llama_models(ladder)
    cfg = P.MpcConfig(horizon_K=horizon, ladder_N=ladder_n, ladder=ladder,
                      slo=P.SLOSpec(ttft_ms=rng.choice([400.0, 600.0, 900.0, 2000.0])),
                      switch_latency_ms=rng.choice([0.0, 7.25, 30.0]), margin=rng.choice([0.0, 0.05, 0.1]))
    pol = P.SchedulerPolicy(max_batch_tokens=rng.choice([256, 512, 1024]), chunking=rng.random() < 0.8)
    cur = rng.choice(ladder.freqs_mhz + [1234.5])
    q = random_snapshot(rng, n_lo=1, n_hi=12, ladder=ladder, current=cur, running_prob=0.3,
                        arrival_window=rng.choice([100.0, 400.0]))
    return m, cfg, pol, q


@pytest.mark.parametrize("seed", range(3))
def test_greedy_oracle_equals_reference(oracle_lib, ref_lib, seed):
    rng = random.Random(1000 + seed)
    for i in range(60):
        inst = _sandwich_instance(rng) if i % 2 == 0 else _llama_instance(rng)
        a = cpu_mpc(oracle_lib, "greedy", *inst)
        b = cpu_mpc(ref_lib, "greedy", *inst)
        assert a[0] == b[0]
        if a[0] == 0:
            assert result_tuple(a[1]) == result_tuple(b[1])


@pytest.mark.parametrize("seed", range(2))
def test_exhaustive_oracle_equals_reference(oracle_lib, ref_lib, seed):
    rng = random.Random(2000 + seed)
    for i in range(25):
        inst = _sandwich_instance(rng) if i % 2 == 0 else _llama_instance(rng, levels=8, ladder_n=5, horizon=4)
        a = cpu_mpc(oracle_lib, "exhaustive", *inst)
        b = cpu_mpc(ref_lib, "exhaustive", *inst)
        assert a[0] == b[0] == 0
        assert result_tuple(a[1]) == result_tuple(b[1])
        assert (a[1].feasible_count, a[1].best_code) == (b[1].feasible_count, b[1].best_code)


def test_exhaustive_sandwiches_greedy(oracle_lib):
    """test_dvfs.cpp:278-340: brute <= greedy <= all-max, feasible flags agree."""
    rng = random.Random(12345)
    for _ in range(100):
        m, cfg, pol, q = _sandwich_instance(rng)
        _, g = cpu_mpc(oracle_lib, "greedy", m, cfg, pol, q)
        _, e = cpu_mpc(oracle_lib, "exhaustive", m, cfg, pol, q)
        assert g.feasible == e.feasible
        if g.feasible:
            assert g.objective_w >= e.objective_w - 1e-12
            K = g.K
            rc, _, allmax = cpu_eval_codes(oracle_lib, m, cfg, pol, q, [sum(2 * 3 ** k for k in range(K))])
            assert g.objective_w <= allmax[0] + 1e-12


def test_eval_codes_oracle_equals_reference(oracle_lib, ref_lib):
    rng = random.Random(99)
    for _ in range(20):
        m, cfg, pol, q = _llama_instance(rng)
        n = len(cfg.candidates().freqs_mhz)
        K = len(cpu_project(oracle_lib, cfg, pol, q)[1])
        codes = [rng.randrange(n ** K) for _ in range(200)] if K else []
        a = cpu_eval_codes(oracle_lib, m, cfg, pol, q, codes)
        b = cpu_eval_codes(ref_lib, m, cfg, pol, q, codes)
        assert a == b


def test_decode_oracle_equals_reference(oracle_lib, ref_lib):
    """acceptance_main.cpp:274-346 shape (minimality) drawn with Python's RNG."""
    rng = random.Random(0xDEC0DE)
    menu = [500, 625, 750, 875, 1000, 1250, 1500, 1750, 2000]
    for _ in range(300):
        rungs = sorted(rng.sample(menu, rng.randint(3, 7)))
        lad = P.FrequencyLadder([float(r) for r in rungs])
        opt = P.SynthOptions(lat_coef=rng.uniform(1.0, 30.0))
        m = P.synth_model_set(P.SynthFamily.compute_bound, lad, [1], opt, opt)
        batch = P.BatchFeatures(rng.randint(1, 64), rng.randint(64, 16000))
        cfg = P.DecodePolicyConfig(ladder=lad, margin=rng.choice([0.0, 0.05, 0.2]),
                                   kv_threshold=rng.uniform(0.55, 0.9))
        i_star = rng.randrange(len(rungs))
        cfg.tbt_slo_ms = opt.lat_coef * batch.sum_len * (1.0 + cfg.margin) / (rungs[i_star] * 0.97)
        kv = P.KVCacheState(100000, rng.randint(0, 100000), 0.9)
        a = cpu_decode(oracle_lib, m, cfg, batch, kv, 1)
        b = cpu_decode(ref_lib, m, cfg, batch, kv, 1)
        assert (a.freq_mhz, a.eval_count, a.kv_override, a.status) == (b.freq_mhz, b.eval_count, b.kv_override,
                                                                       b.status)
        if not a.kv_override:
            assert a.freq_mhz == rungs[i_star]

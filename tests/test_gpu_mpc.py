"""GPU parity (sm_100a through the C ABI) for the prefill MPC and decode pick:
the reference's own known-answer tests (test_dvfs.cpp), then bit-exact
agreement with the CPU oracle / the compiled reference on random instances,
including the BASELINE C2 shape (horizon 6 x 16 rungs = 16.7M trajectories)."""
from __future__ import annotations

import random

import pytest

from helpers import (cpu_decode, cpu_eval_codes, cpu_mpc, cpu_project, dvfs_models, gpu_result_tuple, h100_ladder,
                     llama_models, mpc_config, random_snapshot, result_tuple, waiting_snapshot)
from paper_2602_18755_b200 import pdsim as P

pytestmark = pytest.mark.gpu


def test_greedy_kats(gpu_device):  # test_dvfs.cpp:183-276
    m = dvfs_models()
    g = P.greedy_freq_select(waiting_snapshot([100], 500.0), mpc_config([500.0, 1000.0], 600.0), m,
                             P.SchedulerPolicy())
    assert g.feasible and g.assignment.freqs == [500.0] and g.objective_w == 100.0 and g.eval_count == 2
    assert len(g.levels) == 1
    assert (g.levels[0].k_prime, g.levels[0].mutations, g.levels[0].feasible_mutations, g.levels[0].accepted) == \
        (1, 1, 1, True)

    g = P.greedy_freq_select(waiting_snapshot([100], 1000.0), mpc_config([500.0, 1000.0], 10.0), m,
                             P.SchedulerPolicy())
    assert not g.feasible and g.assignment.freqs == [1000.0] and g.eval_count == 1 and not g.levels

    pol = P.SchedulerPolicy(max_batch_tokens=100)
    g = P.greedy_freq_select(waiting_snapshot([100, 100], 1000.0), mpc_config([500.0, 750.0, 875.0, 1000.0], 61.2),
                             m, pol)
    assert g.feasible and g.assignment.freqs == [1000.0, 875.0]
    assert abs(g.objective_w - 5234.375 / 28.125) < 1e-12 and g.eval_count == 11
    assert [(lv.level, lv.replaced_mhz, lv.k_prime, lv.mutations, lv.feasible_mutations, lv.accepted)
            for lv in g.levels] == [(1, 1000.0, 2, 8, 1, True), (2, 875.0, 1, 2, 0, False)]

    two = P.greedy_freq_select(waiting_snapshot([100, 100, 100], 1000.0), mpc_config([500.0, 1000.0], 10000.0), m, pol)
    assert [(lv.k_prime, lv.mutations, lv.feasible_mutations) for lv in two.levels] == [(3, 7, 7)]
    assert two.eval_count == 8 and two.assignment.freqs == [500.0] * 3
    one = P.greedy_freq_select(waiting_snapshot([100, 100, 100], 1000.0), mpc_config([1000.0], 10000.0), m, pol)
    assert one.feasible and one.eval_count == 1 and not one.levels and one.assignment.freqs == [1000.0] * 3

    g = P.greedy_freq_select(waiting_snapshot([]), mpc_config([500.0, 1000.0], 600.0), m, P.SchedulerPolicy())
    assert g.feasible and g.assignment.freqs == [] and g.eval_count == 0 and g.objective_w == 0.0


def test_controller_kats(gpu_device):  # test_dvfs.cpp:435-464, 491-530
    m = dvfs_models()
    cfg = mpc_config([500.0, 1000.0], 600.0, 0.05)
    ctl = P.PrefillMpcController(cfg, m, P.SchedulerPolicy())
    assert ctl.reacts_to_arrivals() and ctl.max_freq_mhz() == 1000.0 and ctl.safety_margin() == 0.05
    q = waiting_snapshot([100], 500.0)
    d = ctl.decide(q)
    g = P.greedy_freq_select(q, cfg, m, P.SchedulerPolicy())
    assert (d.freq_mhz, d.eval_count, d.feasible) == (g.assignment.freqs[0], g.eval_count, g.feasible)
    assert ctl.on_arrival(q).freq_mhz == d.freq_mhz
    idle = waiting_snapshot([], 500.0)
    assert ctl.decide(idle).freq_mhz == 500.0
    idle.target_freq_mhz = 0.0
    assert ctl.decide(idle).freq_mhz == 1000.0

    dec = P.DecodePolicyConfig(ladder=P.FrequencyLadder([500.0, 750.0, 1000.0]))
    fac = P.TwoTierFactory(cfg, dec, m, P.SchedulerPolicy())
    assert isinstance(fac.make(P.Phase.prefill, 1, 1000.0), P.PrefillMpcController)
    dc = fac.make(P.Phase.decode, 1, 1000.0)
    assert isinstance(dc, P.DecodePolicyController) and not dc.reacts_to_arrivals() and dc.safety_margin() == 0.05
    dec.margin = 0.02
    assert P.TwoTierFactory(cfg, dec, m, P.SchedulerPolicy()).make(P.Phase.decode, 1, 1000.0).safety_margin() == 0.02

    dcfg = P.DecodePolicyConfig(tbt_slo_ms=10.0, ladder=P.FrequencyLadder([500.0, 750.0, 1000.0]))
    ctl = P.DecodePolicyController(dcfg, m)
    q = P.QueueSnapshot(phase=P.Phase.decode, tp=1, decode_batch=P.BatchFeatures.from_lengths([100] * 10),
                        kv=P.KVCacheState(100000, 1000, 0.9))
    d = ctl.decide(q)
    assert (d.freq_mhz, d.eval_count) == (750.0, 2) and ctl.max_freq_mhz() == 1000.0


def test_decode_kats(gpu_device):  # test_dvfs.cpp:342-407
    m = dvfs_models()
    cfg = P.DecodePolicyConfig(tbt_slo_ms=10.0, ladder=P.FrequencyLadder([500.0, 750.0, 1000.0]))
    kv = P.KVCacheState(1000, 100, 0.9)
    big = P.BatchFeatures.from_lengths([100] * 10)
    d = P.select_decode_freq_ex(big, kv, cfg, m, 1)
    assert (d.freq_mhz, d.eval_count, d.kv_override) == (750.0, 2, False)
    assert P.select_decode_freq(big, kv, cfg, m, 1) == 750.0
    d = P.select_decode_freq_ex(P.BatchFeatures.from_lengths([100] * 5), kv, cfg, m, 1)
    assert (d.freq_mhz, d.eval_count) == (500.0, 1)
    cfg.margin = 0.05
    assert (lambda d: (d.freq_mhz, d.eval_count))(P.select_decode_freq_ex(big, kv, cfg, m, 1)) == (1000.0, 3)
    cfg.margin, cfg.tbt_slo_ms = 0.0, 2.0
    d = P.select_decode_freq_ex(big, kv, cfg, m, 1)
    assert (d.freq_mhz, d.eval_count, d.kv_override) == (1000.0, 3, False)
    cfg.tbt_slo_ms = 100.0
    one = P.BatchFeatures.from_lengths([100])
    d = P.select_decode_freq_ex(one, P.KVCacheState(1000, 901, 0.9), cfg, m, 1)
    assert (d.freq_mhz, d.kv_override, d.eval_count) == (1000.0, True, 0)
    d = P.select_decode_freq_ex(one, P.KVCacheState(1000, 900, 0.9), cfg, m, 1)
    assert (d.freq_mhz, d.kv_override) == (500.0, False)


def test_errors_map_to_reference_exceptions(gpu_device):
    m = dvfs_models()
    with pytest.raises(P.ParameterError):
        bad = mpc_config([500.0, 1000.0], 600.0)
        bad.horizon_K = 0
        P.greedy_freq_select(waiting_snapshot([100]), bad, m, P.SchedulerPolicy())
    q = waiting_snapshot([100])
    q.waiting[0].remaining_len = 0  # scheduler.hpp:47
    with pytest.raises(P.SimulationError):
        P.greedy_freq_select(q, mpc_config([500.0, 1000.0], 600.0), m, P.SchedulerPolicy())
    # a latency grid that goes non-positive at the low rung raises ModelError
    # exactly when the reference's search reaches that rung (dvfs.hpp:230-247)
    neg = dvfs_models()
    neg.latency_prefill.grid.values = [0.0, 0.0, 0.0, 0.0, -1.0, 24576.0, 20480.0, 16384.0]
    with pytest.raises(P.ModelError):
        P.greedy_freq_select(waiting_snapshot([100], 1000.0), mpc_config([500.0, 1000.0], 1e6), neg,
                             P.SchedulerPolicy())
    # 4 rungs: level 1 settles on 750 and level 2 finds no 875 -> 500 never evaluated
    g = P.greedy_freq_select(waiting_snapshot([100], 1000.0), mpc_config([500.0, 750.0, 875.0, 1000.0], 1e6), neg,
                             P.SchedulerPolicy())
    assert g.assignment.freqs == [750.0]


def _instances(seed, n, **kw):
    from test_oracle_mpc import _llama_instance, _sandwich_instance
    rng = random.Random(seed)
    return [(_sandwich_instance(rng) if i % 2 == 0 else _llama_instance(rng, **kw)) for i in range(n)]


def test_projection_matches_oracle(gpu_device, oracle_lib):
    for m, cfg, pol, q in _instances(31, 80):
        rc, ref = cpu_project(oracle_lib, cfg, pol, q)
        got = P.project_batches(q, pol, cfg.horizon_K)
        assert rc == 0 and len(got) == len(ref)
        for a, b in zip(got, ref):
            assert (a.features.n_requests, a.features.sum_len, a.work_fraction, a.n_completing,
                    a.min_completing_arrival_ms) == (b.features.n_requests, b.features.sum_len, b.work_fraction,
                                                     b.n_completing, b.min_completing_arrival_ms)


def test_greedy_matches_oracle_bitwise(gpu_device, oracle_lib):
    insts = _instances(41, 120)
    for m, cfg, pol, q in insts:
        rc, ref = cpu_mpc(oracle_lib, "greedy", m, cfg, pol, q)
        assert rc == 0
        g = P.greedy_freq_select(q, cfg, m, pol)
        assert gpu_result_tuple(g, ref.K) == result_tuple(ref)


def test_greedy_batch_c1_shape(gpu_device, oracle_lib):
    """K = 8, N = 7 of the 8-rung H100 ladder: 3^8 - 1 mutations per level."""
    rng = random.Random(7)
    ladder = h100_ladder(8)
    m = llama_models(ladder)
    cfg = P.MpcConfig(horizon_K=8, ladder_N=7, ladder=ladder)
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    snaps = [random_snapshot(rng, n_lo=4, n_hi=30, ladder=ladder, running_prob=0.5,
                             arrival_window=rng.choice([50.0, 200.0])) for _ in range(48)]
    got = P.greedy_freq_select_batch(snaps, cfg, m, pol)
    for q, g in zip(snaps, got):
        rc, ref = cpu_mpc(oracle_lib, "greedy", m, cfg, pol, q)
        assert gpu_result_tuple(g, ref.K) == result_tuple(ref)


def test_greedy_single_calls_c1_shape(gpu_device, oracle_lib):
    """One decision per call takes the latency path (a cluster of 8 CTAs, a
    level's 3^8 - 1 mutations over 4096 threads, minima combined through
    distributed shared memory): same results as the batch kernels and the
    C restatement, level records included."""
    rng = random.Random(11)
    ladder = h100_ladder(8)
    m = llama_models(ladder)
    cfg = P.MpcConfig(horizon_K=8, ladder_N=7, ladder=ladder)
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    snaps = [random_snapshot(rng, n_lo=4, n_hi=30, ladder=ladder, running_prob=0.5,
                             arrival_window=rng.choice([50.0, 200.0, 800.0])) for _ in range(24)]
    batch = P.greedy_freq_select_batch(snaps, cfg, m, pol)
    for q, b in zip(snaps, batch):
        g = P.greedy_freq_select(q, cfg, m, pol)
        rc, ref = cpu_mpc(oracle_lib, "greedy", m, cfg, pol, q)
        assert rc == 0
        assert gpu_result_tuple(g, ref.K) == result_tuple(ref)
        assert gpu_result_tuple(g, ref.K) == gpu_result_tuple(b, ref.K)


def test_exhaustive_matches_oracle_bitwise(gpu_device, oracle_lib):
    insts = _instances(51, 40, levels=8, ladder_n=5, horizon=4)
    for m, cfg, pol, q in insts:
        rc, ref = cpu_mpc(oracle_lib, "exhaustive", m, cfg, pol, q)
        assert rc == 0
        g = P.exhaustive_freq_select(q, cfg, m, pol)
        assert gpu_result_tuple(g, ref.K) == result_tuple(ref)
        assert (g.feasible_count, g.best_code, g.trajectories) == (ref.feasible_count, ref.best_code,
                                                                 ref.trajectories)


def test_exhaustive_batch_mixed_problems(gpu_device, oracle_lib):
    """Many problems of different K in one launch (prefix compaction and the
    per-problem 128-bit argmin slots must not mix problems)."""
    insts = _instances(61, 64, levels=8, ladder_n=6, horizon=5)
    m = insts[1][0]
    cfg, pol = insts[1][1], insts[1][2]
    snaps = [q for (_, _, _, q) in insts[1::2]]
    got = P.exhaustive_freq_select_batch(snaps, cfg, m, pol)
    for q, g in zip(snaps, got):
        rc, ref = cpu_mpc(oracle_lib, "exhaustive", m, cfg, pol, q)
        assert gpu_result_tuple(g, ref.K) == result_tuple(ref)
        assert (g.feasible_count, g.best_code) == (ref.feasible_count, ref.best_code)


def test_exhaustive_ties_take_lexicographic_minimum(gpu_device, oracle_lib):
    """Identical batches at switch 0 / margin 0 make many trajectories tie on
    the objective; the pinned rule picks the lexicographically smallest."""
    ladder = h100_ladder(8)
    m = llama_models(ladder)
    cfg = P.MpcConfig(horizon_K=5, ladder_N=8, ladder=ladder, slo=P.SLOSpec(ttft_ms=900.0),
                      switch_latency_ms=0.0, margin=0.0)
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    q = P.QueueSnapshot(phase=P.Phase.prefill, tp=2, current_freq_mhz=1830.0, target_freq_mhz=1830.0,
                        waiting=[P.SnapshotWaiting(i, 0.0, 512, 512) for i in range(5)])
    rc, ref = cpu_mpc(oracle_lib, "exhaustive", m, cfg, pol, q)
    g = P.exhaustive_freq_select(q, cfg, m, pol)
    assert gpu_result_tuple(g, ref.K) == result_tuple(ref)
    assert g.best_code == ref.best_code


@pytest.mark.parametrize("seed", [0xC2, 0xC3])
def test_exhaustive_c2_shape_16_7M(gpu_device, ref_lib, seed):
    """BASELINE C2: horizon 6 x 16 rungs = 16,777,216 trajectories per decision,
    against the compiled reference's own loop (a few decisions: ~16 s each)."""
    from paper_2602_18755_b200.workloads import c2_corpus
    m, cfg, pol, snaps = c2_corpus(seed, 2)
    got = P.exhaustive_freq_select_batch(snaps, cfg, m, pol)
    import oracle  # noqa: F401  (ref driver)
    from paper_2602_18755_b200 import _abi as A
    import ctypes as C
    from helpers import Packed
    for q, g in zip(snaps, got):
        assert g.trajectories == 16 ** 6
        p = Packed(m, cfg, pol, q)
        out = A.bs_mpc_result()
        assert ref_lib.ref_exhaustive(C.byref(p.models), C.byref(p.cfg), C.byref(p.policy), C.byref(p.snap),
                                      C.byref(out)) == 0
        assert gpu_result_tuple(g, out.K) == result_tuple(out)
        assert (g.feasible_count, g.best_code) == (out.feasible_count, out.best_code)


def test_eval_codes_and_tables_match_reference(gpu_device, oracle_lib, ref_lib):
    """Per-trajectory feasibility and objective vs the C restatement, and the
    (k, f) tables bitwise vs the reference's own MpcEvaluator memo
    (dvfs.hpp:150-160: lat = wf L, pow = P, energy = lat pow)."""
    import ctypes as C

    from helpers import Packed
    from paper_2602_18755_b200 import _abi as A
    rng = random.Random(77)
    for m, cfg, pol, q in _instances(71, 30):
        n = len(cfg.candidates().freqs_mhz)
        K = len(cpu_project(oracle_lib, cfg, pol, q)[1])
        codes = [rng.randrange(n ** K) for _ in range(300)] if K else []
        rc, feas, obj = cpu_eval_codes(oracle_lib, m, cfg, pol, q, codes)
        gf, go = P.mpc_eval_codes(q, cfg, m, pol, codes)
        assert gf == feas and go == obj
        lat, pw, en = P.mpc_tables(q, cfg, m, pol)
        assert len(lat) == K
        p = Packed(m, cfg, pol, q)
        rk, rn = C.c_int32(), C.c_int32()
        size = A.BS_MAX_K * A.BS_MAX_CAND
        rl, rp, re_ = (C.c_double * size)(), (C.c_double * size)(), (C.c_double * size)()
        assert ref_lib.ref_tables(C.byref(p.models), C.byref(p.cfg), C.byref(p.policy), C.byref(p.snap), C.byref(rk),
                                  C.byref(rn), rl, rp, re_) == 0
        assert (rk.value, rn.value) == (K, n)
        for k in range(K):
            for f in range(n):
                assert (lat[k][f], pw[k][f], en[k][f]) == (rl[k * n + f], rp[k * n + f], re_[k * n + f])


def test_decode_matches_oracle(gpu_device, oracle_lib):
    rng = random.Random(0xDEC0DE)
    menu = [500, 625, 750, 875, 1000, 1250, 1500, 1750, 2000]
    for _ in range(200):
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
        d = P.select_decode_freq_ex(batch, kv, cfg, m, 1)
        assert (d.freq_mhz, d.eval_count, int(d.kv_override)) == (a.freq_mhz, a.eval_count, a.kv_override)


def test_predict_matches_oracle(gpu_device, oracle_lib):
    from helpers import cpu_predict
    rng = random.Random(3)
    m = llama_models(h100_ladder(16))
    for which, kind, phase in ((0, "latency", P.Phase.prefill), (1, "latency", P.Phase.decode),
                               (2, "power", P.Phase.prefill), (3, "power", P.Phase.decode)):
        feats = [(rng.randint(1, 300), rng.randint(1, 20000)) for _ in range(50)]
        tps = [rng.choice([1, 2, 3, 4, 8, 16]) for _ in range(50)]
        fr = [rng.uniform(200.0, 2000.0) for _ in range(50)]
        ref, st = cpu_predict(oracle_lib, m, which, feats, tps, fr)
        for (nr, sl), tp, f, r in zip(feats, tps, fr, ref):
            fn = P.predict_latency if kind == "latency" else P.predict_power
            assert fn(m, phase, P.BatchFeatures(nr, sl), tp, f) == r


def test_grid_interpolation_kats(gpu_device):  # test_perfmodel.cpp:65-109
    g = P.NdGrid([P.Axis("x", [0.0, 10.0]), P.Axis("y", [0.0, 100.0])], [0.0, 100.0, 10.0, 110.0])
    vals, cl = gpu_device.interpolate(g, [[0.0, 0.0], [10.0, 100.0], [2.5, 30.0], [7.0, 99.0], [-5.0, 30.0],
                                          [15.0, 200.0]])
    assert vals[0] == 0.0 and vals[1] == 110.0
    assert vals[2] == pytest.approx(32.5) and vals[3] == pytest.approx(106.0)
    assert vals[4] == pytest.approx(30.0) and vals[5] == pytest.approx(110.0)
    assert cl == [0, 0, 0, 0, 1, 2]
    s = P.NdGrid([P.Axis("x", [5.0]), P.Axis("y", [0.0, 1.0])], [3.0, 7.0])
    assert s.interpolate([5.0, 0.5]) == pytest.approx(5.0)

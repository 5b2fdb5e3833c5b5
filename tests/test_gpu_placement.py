"""GPU parity of the placement path: probe down-sampling (mt19937_64 keep
masks), the fixed-frequency instance simulation, the goodput search and the
config table, against the reference's own known answers
(tests/test_placement.cpp:442-680) and the compiled reference (oracle/_ref)
bit for bit."""
from __future__ import annotations

import ctypes as C
import random

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P
from paper_2602_18755_b200 import workloads as W

pytestmark = pytest.mark.gpu

PF, DE = P.Phase.prefill, P.Phase.decode


def probe_models() -> P.ModelSet:
    """test_placement.cpp:24-40: prefill 4 / 8 tokens/ms at 500 / 1000 MHz,
    decode 2 / 1 ms per iteration, prefill 100 / 200 W, decode 50 W, idle 10 W."""
    m = P.ModelSet()
    m.latency_prefill = P.LatencyTable(PF, P.NdGrid([P.Axis("sum_len", [0.0, 131072.0]),
                                                     P.Axis("freq_mhz", [500.0, 1000.0])], [0.0, 0.0, 32768.0, 16384.0]))
    m.latency_decode = P.LatencyTable(DE, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])], [2.0, 1.0]))
    m.power_prefill = P.PowerTable(PF, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])], [100.0, 200.0]))
    m.power_decode = P.PowerTable(DE, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])], [50.0, 50.0]))
    m.idle = P.IdlePowerModel([P.TpEntry(1, [500.0, 1000.0], [10.0, 10.0])])
    return m


def fixed_interval_trace(n, interval_ms, input_len, output_len) -> P.Trace:  # test_placement.cpp:52-60
    return P.Trace([P.Request(i, float(i) * interval_ms, input_len, output_len) for i in range(n)],
                   float(n) * interval_ms)


def gpu_sim(models, traces, cfg, policy=None, slo=None, device=None):
    dev = device or P.default_device()
    keep: list = []
    tr = (A.bs_trace * len(traces))(*[P.c_trace(t, keep) for t in traces])
    ci = P.c_candidates([cfg])
    cp = P.c_policy(policy or P.SchedulerPolicy())
    cs = P.c_slo(slo or P.SLOSpec())
    out = (A.bs_sim_summary * len(traces))()
    dev.check(dev._lib.bs_simulate_instance(dev.handle, dev.models(models), tr, len(traces), ci, C.byref(cp),
                                            C.byref(cs), out))
    return [out[i] for i in range(len(traces))]


def ref_sim(ref, models, traces, cfg, policy=None, slo=None):
    keep: list = []
    cm = P.c_model_set(models, keep)
    tr = (A.bs_trace * len(traces))(*[P.c_trace(t, keep) for t in traces])
    ci = P.c_candidates([cfg])
    cp = P.c_policy(policy or P.SchedulerPolicy())
    cs = P.c_slo(slo or P.SLOSpec())
    out = (A.bs_sim_summary * len(traces))()
    assert ref.ref_simulate(C.byref(cm), tr, len(traces), ci, C.byref(cp), C.byref(cs), out) == 0
    return [out[i] for i in range(len(traces))]


def summary(s):
    return (s.status, s.meets_slo if s.status == 0 else 0, s.completed, s.busy_energy_j, s.idle_energy_j,
            s.horizon_ms) if s.status == 0 else (s.status,)


def test_slo_compliance_kats(gpu_device):  # test_placement.cpp:442-460
    m = probe_models()
    pt = fixed_interval_trace(1, 1000.0, 100, 1)
    cfg = P.InstanceConfig(PF, 1, 1000.0)
    assert gpu_sim(m, [pt], cfg, slo=P.SLOSpec(12.5, 100.0))[0].meets_slo == 1
    assert gpu_sim(m, [pt], cfg, slo=P.SLOSpec(12.49, 100.0))[0].meets_slo == 0
    dt = fixed_interval_trace(1, 1000.0, 100, 3)
    dcfg = P.InstanceConfig(DE, 1, 1000.0)
    assert gpu_sim(m, [dt], dcfg, slo=P.SLOSpec(600.0, 1.0))[0].meets_slo == 1
    assert gpu_sim(m, [dt], dcfg, slo=P.SLOSpec(600.0, 0.99))[0].meets_slo == 0


def test_energy_kats(gpu_device):  # test_placement.cpp:565-590
    m = probe_models()
    pt = fixed_interval_trace(2, 100.0, 400, 1)
    pt.duration_ms = 1000.0
    s = gpu_sim(m, [pt], P.InstanceConfig(PF, 1, 1000.0))[0]
    assert (s.busy_energy_j + s.idle_energy_j) / s.completed == 14.5
    assert s.busy_energy_j / s.completed == 10.0
    dt = fixed_interval_trace(1, 100.0, 100, 4)
    dt.duration_ms = 1000.0
    s = gpu_sim(m, [dt], P.InstanceConfig(DE, 1, 1000.0))[0]
    assert abs(s.busy_energy_j / s.completed - 0.2) < 1e-12
    assert abs((s.busy_energy_j + s.idle_energy_j) / s.completed - 10.16) < 1e-12
    empty = P.Trace([], 100.0)
    assert gpu_sim(m, [empty], P.InstanceConfig(PF, 1, 1000.0))[0].completed == 0


def test_simulation_matches_reference_bitwise(gpu_device, ref_lib):
    rng = random.Random(5)
    lad = W.ladder(8)
    m = W.llama_models(lad)
    lengths = P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7))
    traces = [P.gen_gamma_trace(rng.choice([2.0, 6.0, 12.0]), rng.choice([0.5, 1.0]), 20_000.0, lengths, seed)
              for seed in range(12)]
    for phase in (PF, DE):
        for tp in (1, 2, 4, 8):
            for f in (lad.freqs_mhz[0], lad.freqs_mhz[4], lad.freqs_mhz[-1]):
                cfg = P.InstanceConfig(phase, tp, f)
                pol = P.SchedulerPolicy(max_batch_tokens=2048, max_batch_requests=rng.choice([16, 256]),
                                        chunking=rng.random() < 0.8)
                slo = P.SLOSpec(600.0, 100.0)
                got = [summary(s) for s in gpu_sim(m, traces, cfg, pol, slo)]
                want = [summary(s) for s in ref_sim(ref_lib, m, traces, cfg, pol, slo)]
                assert got == want, (phase, tp, f)


def test_probe_traces_match_reference(gpu_device, ref_lib):  # test_placement.cpp:632-648
    base = fixed_interval_trace(600, 50.0, 600, 1)
    search = P.GoodputSearch()
    a = P.downsample_keep(base, search, 40, 0)
    assert 200 < len(a) < 400
    assert P.downsample_keep(base, search, 40, 0) == a
    assert P.downsample_keep(base, search, 40, 1) != a
    assert P.downsample_keep(base, search, 200, 0) == list(range(600))
    keep: list = []
    ct = P.c_trace(base, keep)
    for k, j in ((1, 0), (7, 0), (40, 0), (40, 1), (79, 2)):
        cg = P.c_search(search)
        idx = (C.c_int32 * 600)()
        n = C.c_int64()
        assert ref_lib.ref_downsample_keep(C.byref(ct), C.byref(cg), k, j, idx, C.byref(n)) == 0
        assert P.downsample_keep(base, search, k, j) == list(idx[:n.value])


def test_goodput_kats(gpu_device):  # test_placement.cpp:462-560
    m = probe_models()
    pol = P.SchedulerPolicy()
    base = fixed_interval_trace(600, 50.0, 600, 1)
    slo = P.SLOSpec(600.0, 100.0)
    search = P.GoodputSearch(probe_count=2)
    cfg = P.InstanceConfig(PF, 1, 1000.0)
    res = P.max_goodput(cfg, base, slo, m, pol, search)
    assert 1 <= res.k_star < 80 and not res.saturated and res.r_c == res.k_star * search.tolerance_rps

    def all_pass(k):
        for j in range(search.probe_count):
            idx = P.downsample_keep(base, search, k, j)
            if not idx:
                continue
            probe = P.Trace([base.requests[i] for i in idx], base.duration_ms)
            if not gpu_sim(m, [probe], cfg, pol, slo)[0].meets_slo:
                return False
        return True
    assert all_pass(res.k_star) and not all_pass(res.k_star + 1)

    loose = P.max_goodput(cfg, base, P.SLOSpec(1e6, 100.0), m, pol, P.GoodputSearch())
    assert loose.saturated and loose.k_star == 80 and loose.r_c == 20.0
    dres = P.max_goodput(P.InstanceConfig(DE, 1, 1000.0), fixed_interval_trace(600, 50.0, 600, 30), slo, m, pol,
                         P.GoodputSearch())
    assert dres.saturated and dres.r_c == 20.0
    z = P.max_goodput(cfg, base, P.SLOSpec(1.0, 100.0), m, pol, P.GoodputSearch())
    assert (z.r_c, z.k_star, z.saturated) == (0.0, 0, False)
    tiny = P.SchedulerPolicy(kv_capacity_tokens=100)
    assert P.max_goodput(P.InstanceConfig(DE, 1, 1000.0), base, slo, m, tiny, P.GoodputSearch()).r_c == 0.0
    assert P.max_goodput(cfg, fixed_interval_trace(2, 5000.0, 100, 1), slo, m, pol, P.GoodputSearch()).r_c == 0.0
    with pytest.raises(P.ParameterError):
        P.max_goodput(cfg, base, slo, m, pol, P.GoodputSearch(tolerance_rps=0.0))
    with pytest.raises(P.ParameterError):
        P.max_goodput(cfg, base, slo, m, pol, P.GoodputSearch(probe_count=0))


def test_candidate_evaluation_kats(gpu_device):  # test_placement.cpp:592-630
    m = probe_models()
    pol = P.SchedulerPolicy()
    base = fixed_interval_trace(600, 50.0, 600, 1)
    slo = P.SLOSpec(600.0, 100.0)
    search = P.GoodputSearch()
    e = P.evaluate_candidate(P.InstanceConfig(PF, 1, 1000.0), base, slo, m, pol, search)
    g = P.max_goodput(P.InstanceConfig(PF, 1, 1000.0), base, slo, m, pol, search)
    assert (e.r_c, e.saturated, e.g_c, e.error) == (g.r_c, g.saturated, 1, "") and e.usable()
    idx = P.downsample_keep(base, search, g.k_star, 0)
    s = gpu_sim(m, [P.Trace([base.requests[i] for i in idx], base.duration_ms)], P.InstanceConfig(PF, 1, 1000.0))[0]
    assert e.e_c == (s.busy_energy_j + s.idle_energy_j) / s.completed
    gap = P.evaluate_candidate(P.InstanceConfig(PF, 4, 1000.0), base, slo, m, pol, search)
    assert gap.error and gap.r_c == 0.0 and gap.e_c is None and not gap.usable() and gap.g_c == 4
    zero = P.evaluate_candidate(P.InstanceConfig(PF, 1, 1000.0), base, P.SLOSpec(1.0, 100.0), m, pol, search)
    assert zero.error == "" and zero.r_c == 0.0 and zero.e_c is None and not zero.usable()


def _ref_table(ref, models, base, slo, pol, search, cands):
    keep: list = []
    cm = P.c_model_set(models, keep)
    ct = P.c_trace(base, keep)
    cs, cp, cg = P.c_slo(slo), P.c_policy(pol), P.c_search(search)
    ci = P.c_candidates(cands)
    out = (A.bs_table_entry * len(cands))()
    assert ref.ref_config_table(C.byref(cm), C.byref(ct), C.byref(cs), C.byref(cp), C.byref(cg), ci, len(cands),
                                out) == 0
    return [P.entry_from_c(out[i]) for i in range(len(cands))]


def _cmp(e):
    return (e.config.phase, e.config.tp, e.config.base_freq_mhz, e.r_c, e.e_c, e.g_c, e.saturated, e.error)


def test_config_table_probe_models_matches_reference(gpu_device, ref_lib):
    m = probe_models()
    base = fixed_interval_trace(300, 50.0, 400, 1)
    cands = P.enumerate_candidates(P.FrequencyLadder([500.0, 1000.0]), [1, 4])
    for slo in (P.SLOSpec(600.0, 100.0), P.SLOSpec(60.0, 1.5)):
        for search in (P.GoodputSearch(), P.GoodputSearch(probe_count=3, tolerance_rps=0.5)):
            got = P.build_config_table(cands, base, slo, m, P.SchedulerPolicy(), search)
            want = _ref_table(ref_lib, m, base, slo, P.SchedulerPolicy(), search, cands)
            assert [_cmp(e) for e in got] == [_cmp(e) for e in want]


@pytest.mark.parametrize("seed", [7, 8])
def test_config_table_llama_matches_reference(gpu_device, ref_lib, seed):
    """C3 shape, scaled down: gamma(0.5) 12 rps window, TP {1,2,4,8} x 8 rungs
    x 2 phases = 64 candidates, max_batch_tokens 2048."""
    lad = W.ladder(8)
    m = W.llama_models(lad)
    base = P.gen_gamma_trace(12.0, 0.5, 60_000.0, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)),
                             seed)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    pol = P.SchedulerPolicy(max_batch_tokens=2048)
    slo = P.SLOSpec(600.0, 100.0)
    got = P.build_config_table(cands, base, slo, m, pol, P.GoodputSearch())
    want = _ref_table(ref_lib, m, base, slo, pol, P.GoodputSearch(), cands)
    assert [_cmp(e) for e in got] == [_cmp(e) for e in want]
    assert sum(e.usable() for e in got) > 8
    plan = P.solve_placement(P.PlacementProblem(got, 16, P.peak_rps(base, 10.0), 0.05))
    assert plan.gpus_used <= 16


def test_batched_tables_match_reference(gpu_device, ref_lib):
    """bs_goodput_tables: several windows' tables in one probe grid (with an
    empty window and a window too thin for any rate step) equal the
    reference's build_config_table of each window, entry for entry."""
    lad = W.ladder(8)
    m = W.llama_models(lad)
    day = P.gen_gamma_trace(10.0, 0.5, 3 * 60_000.0, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)),
                            19)
    wins = P.split_windows(day, 60_000.0)
    wins.append(P.Trace([], 60_000.0))
    wins.append(P.Trace([P.Request(0, 10.0, 300, 20)], 60_000.0))
    cands = P.enumerate_candidates(lad, [1, 2, 4])
    pol = P.SchedulerPolicy(max_batch_tokens=2048)
    slo = P.SLOSpec(600.0, 100.0)
    for search in (P.GoodputSearch(), P.GoodputSearch(probe_count=2, tolerance_rps=0.5)):
        tables = P.build_config_tables(wins, cands, slo, m, pol, search, gpu_device)
        assert len(tables) == len(wins)
        for w, table in zip(wins, tables):
            want = _ref_table(ref_lib, m, w, slo, pol, search, cands)
            assert [_cmp(e) for e in table] == [_cmp(e) for e in want]


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_search_pruning_random_tables_match_reference(gpu_device, ref_lib, seed):
    """Search-path pruning under stress: random grids whose latency or power
    turns non-positive above a random batch size (ModelError part-way through
    some probes, so outcomes mix pass / fail / error along the search path),
    1-3 replicates, tight and loose SLOs, traces whose feasibility is not
    monotone in the rate step -- every table entry equals the reference's."""
    rng = random.Random(seed)
    m = probe_models()
    cut = rng.choice([3000.0, 4000.0, 6000.0])
    knots = P.Axis("sum_len", [0.0, 1000.0, cut, 1.5 * cut])  # values cross zero just above `cut`
    lat = [2.0, 40.0, 300.0, -1.0 if seed % 2 else 900.0]
    pw = [100.0, 150.0, 180.0, -5.0 if seed % 4 == 0 else 200.0]
    m.latency_prefill = P.LatencyTable(PF, P.NdGrid([knots], lat))
    m.power_prefill = P.PowerTable(PF, P.NdGrid([P.Axis("sum_len", [0.0, 1000.0, cut, 1.5 * cut])], pw))
    m.latency_decode = P.LatencyTable(DE, P.NdGrid([P.Axis("n_requests", [1.0, 8.0, 64.0]),
                                                    P.Axis("freq_mhz", [500.0, 1000.0])],
                                                   [2.0, 1.0, 8.0, 5.0, -3.0 if seed % 2 == 0 else 40.0, 25.0]))
    m.idle = P.IdlePowerModel([P.TpEntry(1, [500.0, 1000.0], [10.0, 10.0]), P.TpEntry(2, [500.0, 1000.0], [12.0, 14.0])])
    reqs, t = [], 0.0
    for i in range(rng.randint(150, 400)):
        t += rng.expovariate(1.0 / rng.choice([5.0, 20.0, 80.0]))
        reqs.append(P.Request(i, t, rng.randint(50, 3000), rng.randint(1, 60)))
    base = P.Trace(reqs, t + 1000.0)
    cands = P.enumerate_candidates(P.FrequencyLadder([500.0, 750.0, 1000.0]), [1, 2])
    # batches big enough to reach the non-positive region (prefill: odd seeds; decode: even seeds)
    pol = P.SchedulerPolicy(max_batch_tokens=8192 if seed % 2 else rng.choice([2048, 8192]),
                            max_batch_requests=256 if seed % 2 == 0 else rng.choice([16, 256]))
    for slo in (P.SLOSpec(rng.uniform(30.0, 300.0), rng.uniform(3.0, 20.0)), P.SLOSpec(5000.0, 500.0)):
        search = P.GoodputSearch(tolerance_rps=rng.choice([0.25, 0.5, 1.0]), probe_count=rng.randint(1, 3),
                                 seed=rng.getrandbits(63))
        got = P.build_config_table(cands, base, slo, m, pol, search)
        want = _ref_table(ref_lib, m, base, slo, pol, search, cands)
        assert [_cmp(e) for e in got] == [_cmp(e) for e in want]


def test_empty_saturated_probe_without_idle_tp_matches_reference(gpu_device, ref_lib):
    """evaluate_candidate (placement.hpp:217-238) when the search ends on an
    EMPTY probe (an empty probe counts as a pass, placement.hpp:169) and the
    idle model lacks the candidate's tp: the E_c simulation throws ModelError,
    the catch clears r_c but keeps saturated.  Seeds are searched on the
    reference's own down-sampler until the k_max probe of replicate 0 keeps
    nothing."""
    m = probe_models()  # idle model: tp 1 only
    base = P.Trace([P.Request(0, 100.0, 200, 5), P.Request(1, 2500.0, 300, 5)], 3000.0)  # 0.667 rps: k_max 2
    keep: list = []
    ct = P.c_trace(base, keep)
    kept = (C.c_int32 * 2)()
    nk = C.c_int64()
    found = None
    for seed in range(1, 400):
        search = P.GoodputSearch(seed=seed)
        assert ref_lib.ref_downsample_keep(C.byref(ct), C.byref(P.c_search(search)), 2, 0, kept, C.byref(nk)) == 0
        if nk.value == 0:
            found = search
            break
    assert found is not None
    cands = [P.InstanceConfig(PF, 4, 1000.0), P.InstanceConfig(PF, 1, 1000.0), P.InstanceConfig(DE, 4, 500.0)]
    got = P.build_config_table(cands, base, P.SLOSpec(600.0, 100.0), m, P.SchedulerPolicy(), found)
    want = _ref_table(ref_lib, m, base, P.SLOSpec(600.0, 100.0), P.SchedulerPolicy(), found, cands)
    assert [_cmp(e) for e in got] == [_cmp(e) for e in want]
    assert want[0].saturated and want[0].r_c == 0.0 and "tp 4" in want[0].error


def test_c3_full_hour_table_matches_reference(gpu_device, ref_lib):
    """BASELINE C3 at full size: a bursty 1-hour gamma(0.5) window at 12 rps
    (~43k requests), 2 phases x TP {1,2,4,8} x 16 rungs = 128 candidates,
    max_batch_tokens 2048 -- every entry equal to the reference's
    build_config_table (placement.hpp:240-260), then the ILP for 16 GPUs."""
    lad = W.ladder(16)
    m = W.llama_models(lad)
    base = P.gen_gamma_trace(12.0, 0.5, 3600e3, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 7)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    pol, slo = P.SchedulerPolicy(max_batch_tokens=2048), P.SLOSpec(600.0, 100.0)
    got = P.build_config_table(cands, base, slo, m, pol, P.GoodputSearch(), device=gpu_device)
    want = _ref_table(ref_lib, m, base, slo, pol, P.GoodputSearch(), cands)
    assert len(base.requests) > 40000
    assert [_cmp(e) for e in got] == [_cmp(e) for e in want]
    plan = P.solve_placement(P.PlacementProblem(got, 16, P.peak_rps(base, 10.0), 0.05), gpu_device)
    assert plan.gpus_used <= 16 and sum(plan.counts) >= 2

"""The reference's simulator known-answer tests (tests/test_simulator.cpp) on
the device replay (bs_replay).  Its unit models make every interpolated
value exact: prefill runs at 8 tokens/ms at 1000 MHz (4 at 500), a decode
iteration takes 1 ms at 1000 MHz (2 at 500), prefill draws 200 W at 1000 MHz,
decode 50 W, idle 10 W (test_simulator.cpp:16-39).

The reference's instance KATs use simulate_instance; here the same requests
go through a 1P + 1D cluster (simulate_cluster), so prefill expectations are
the KATs' own, and decode expectations are the KATs' shifted by each
request's prefill completion (its decode join, simulator.hpp:840-853)."""
from __future__ import annotations

import math

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P

pytestmark = pytest.mark.gpu


def unit_models() -> P.ModelSet:
    """test_simulator.cpp:20-39."""
    m = P.ModelSet()
    m.latency_prefill = P.LatencyTable(P.Phase.prefill, P.NdGrid(
        [P.Axis("sum_len", [0.0, 131072.0]), P.Axis("freq_mhz", [500.0, 1000.0])], [0.0, 0.0, 32768.0, 16384.0]))
    m.latency_decode = P.LatencyTable(P.Phase.decode, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])], [2.0, 1.0]))
    m.power_prefill = P.PowerTable(P.Phase.prefill, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])],
                                                             [100.0, 200.0]))
    m.power_decode = P.PowerTable(P.Phase.decode, P.NdGrid([P.Axis("freq_mhz", [500.0, 1000.0])], [50.0, 50.0]))
    m.idle = P.IdlePowerModel([P.TpEntry(1, [500.0, 1000.0], [10.0, 10.0]),
                               P.TpEntry(2, [500.0, 1000.0], [16.0, 16.0])])
    return m


def run(reqs, duration_ms, *, max_tokens=8192, chunking=True, kv=1_000_000, max_req=256, prefill=((1.0,),),
        decode=((1.0,),), device=None):
    inst = [P.ClusterInstance(P.InstanceConfig(P.Phase.prefill, 1, 1000.0), w[0]) for w in prefill]
    inst += [P.ClusterInstance(P.InstanceConfig(P.Phase.decode, 1, 1000.0), w[0]) for w in decode]
    pol = P.SchedulerPolicy(max_batch_tokens=max_tokens, max_batch_requests=max_req, chunking=chunking,
                            kv_capacity_tokens=kv)
    sc = P.ReplayScenario(P.Trace([P.Request(*r) for r in reqs], duration_ms), P.ClusterSpec(inst), pol, None,
                          P.SimOptions(), P.SLOSpec(), 0.0)
    return P.replay([sc], unit_models(), device, requests=True, logs=True, raise_errors=False)[0]


def batches_of(res, instance):
    return [b for b in res.batches if b.instance == instance]


def test_single_prefill_request(gpu_device):  # test_simulator.cpp:126-152
    res = run([(0, 0.0, 100, 1)], 1000.0, device=gpu_device)
    r = res.requests[0]
    assert r.prefill_done_ms - 0.0 == 12.5 and r.prefill_instance == 0 and r.completed
    pb = batches_of(res, 0)
    assert len(pb) == 1 and (pb[0].start_ms, pb[0].end_ms, pb[0].power_w, pb[0].sum_len) == (0.0, 12.5, 200.0, 100)
    assert abs(pb[0].energy_j - 2.5) <= 1e-12
    pidle = sum(i.energy_j for i in res.idles if i.instance == 0)
    assert abs(pidle - 10.0 * 987.5 / 1000.0) <= 1e-12


def test_late_arrival_waits_idle(gpu_device):  # test_simulator.cpp:154-167
    res = run([(0, 250.0, 100, 1)], 1000.0, device=gpu_device)
    pb = batches_of(res, 0)
    assert (pb[0].start_ms, pb[0].end_ms) == (250.0, 262.5)
    assert res.requests[0].prefill_done_ms - 250.0 == 12.5
    pi = [i for i in res.idles if i.instance == 0]
    assert len(pi) == 2 and pi[0].end_ms == 250.0 and (pi[1].start_ms, pi[1].end_ms) == (262.5, 1000.0)


@pytest.mark.parametrize("chunking,want", [
    (True, [(100, 2, 12.5), (20, 1, 15.0)]),    # test_simulator.cpp:169-185
    (False, [(60, 1, 7.5), (60, 1, 15.0)]),     # test_simulator.cpp:187-201
])
def test_budget_and_chunking(gpu_device, chunking, want):
    res = run([(0, 0.0, 60, 1), (1, 0.0, 60, 1)], 1000.0, max_tokens=100, chunking=chunking, device=gpu_device)
    pb = batches_of(res, 0)
    assert [(b.sum_len, b.n_requests, b.end_ms) for b in pb] == want
    assert [r.prefill_done_ms for r in res.requests] == ([12.5, 15.0] if chunking else [7.5, 15.0])


def test_oversized_prompt(gpu_device):  # test_simulator.cpp:203-231
    res = run([(0, 0.0, 150, 1), (1, 0.0, 50, 1)], 1000.0, max_tokens=100, chunking=False, device=gpu_device)
    pb = batches_of(res, 0)
    assert [(b.sum_len, b.n_requests, b.end_ms) for b in pb] == [(150, 1, 18.75), (50, 1, 25.0)]
    assert [r.prefill_done_ms for r in res.requests] == [18.75, 25.0]
    res = run([(0, 0.0, 150, 1), (1, 0.0, 50, 1)], 1000.0, max_tokens=100, chunking=True, device=gpu_device)
    assert [b.sum_len for b in batches_of(res, 0)] == [100, 100]
    assert [r.prefill_done_ms for r in res.requests] == [25.0, 25.0]


def test_queue_head_blocks(gpu_device):  # test_simulator.cpp:233-243
    res = run([(0, 0.0, 80, 1), (1, 0.0, 30, 1), (2, 0.0, 15, 1)], 1000.0, max_tokens=100, chunking=False,
              device=gpu_device)
    pb = batches_of(res, 0)
    assert [(b.n_requests, b.sum_len) for b in pb] == [(1, 80), (2, 45)]


def test_decode_one_iteration_per_token(gpu_device):  # test_simulator.cpp:245-269
    res = run([(0, 0.0, 100, 5)], 100.0, device=gpu_device)
    r = res.requests[0]
    join = r.prefill_done_ms
    assert join == 12.5 and r.decode_first_start_ms == join
    assert (r.first_token_ms, r.last_token_ms, r.n_tokens, r.max_tbt_ms) == (join + 1.0, join + 5.0, 5, 1.0)
    db = batches_of(res, 1)
    assert [b.batch_seq for b in db] == [0, 1, 2, 3, 4]
    assert [b.sum_len for b in db] == [100, 101, 102, 103, 104] and all(b.n_requests == 1 for b in db)
    assert all(abs(b.energy_j - 0.05) <= 1e-12 for b in db)
    assert res.generated_tokens == 5 and res.completed_requests == 1


def test_kv_reservation_gates_admission(gpu_device):  # test_simulator.cpp:292-312
    # equal prompts complete together at 12.5 * 3 = 37.5 (one 300-token batch)
    res = run([(0, 0.0, 100, 5), (1, 0.0, 100, 10), (2, 0.0, 100, 5)], 100.0, kv=250, device=gpu_device)
    join = 37.5
    a, b, c = res.requests
    assert {a.prefill_done_ms, b.prefill_done_ms, c.prefill_done_ms} == {join}
    assert (a.first_token_ms, a.last_token_ms) == (join + 1.0, join + 5.0)
    assert (b.n_tokens, b.last_token_ms) == (10, join + 10.0)
    assert c.decode_first_start_ms == join + 5.0 and (c.first_token_ms, c.last_token_ms) == (join + 6.0, join + 10.0)
    assert c.max_tbt_ms == 6.0 and res.completed_requests == 3 and res.generated_tokens == 20


def test_kv_capacity_rejection(gpu_device):  # test_simulator.cpp:314-320
    res = run([(0, 0.0, 90, 20)], 100.0, kv=100, device=gpu_device)
    assert res.status == A.BS_SIMULATION_ERROR
    with pytest.raises(P.SimulationError, match="needs 110 KV tokens, capacity 100"):
        P.replay([P.ReplayScenario(P.Trace([P.Request(0, 0.0, 90, 20)], 100.0), P.ClusterSpec([
            P.ClusterInstance(P.InstanceConfig(P.Phase.prefill, 1, 1000.0), 1.0),
            P.ClusterInstance(P.InstanceConfig(P.Phase.decode, 1, 1000.0), 1.0)]),
            P.SchedulerPolicy(kv_capacity_tokens=100), None, P.SimOptions(), P.SLOSpec(), 0.0)], unit_models(),
            gpu_device)


def test_residency_cap(gpu_device):  # test_simulator.cpp:322-334
    # the cap also limits prefill batches (scheduler.hpp:44): requests 0, 1 finish prefill at 2.5 ms,
    # request 2 at 3.75 ms, mid-iteration, and waits for a resident slot
    res = run([(0, 0.0, 10, 3), (1, 0.0, 10, 3), (2, 0.0, 10, 3)], 100.0, max_req=2, device=gpu_device)
    a, b, c = res.requests
    assert [a.prefill_done_ms, b.prefill_done_ms, c.prefill_done_ms] == [2.5, 2.5, 3.75]
    assert (a.first_token_ms, a.last_token_ms) == (3.5, 5.5)
    assert (b.first_token_ms, b.last_token_ms) == (3.5, 5.5)
    assert c.decode_first_start_ms == 5.5 and (c.first_token_ms, c.last_token_ms) == (6.5, 8.5)
    assert all(b.n_requests <= 2 for b in batches_of(res, 1))


def test_cluster_conserves_requests_tokens_energy(gpu_device):  # test_simulator.cpp:452-530
    reqs = [(i, 25.0 * i, 50 + (i * 37) % 200, 3 + i % 5) for i in range(40)]
    res = run(reqs, 1000.0, prefill=((0.6,), (0.4,)), decode=((0.5,), (0.5,)), device=gpu_device)
    assert res.status == 0 and res.completed_requests == 40
    assert res.generated_tokens == sum(r[3] for r in reqs)
    prefill_in = [0, 0]
    decode_n = [0, 0]
    for r, q in zip(res.requests, reqs):
        assert r.completed and r.prefill_instance in (0, 1) and r.decode_instance in (2, 3)
        prefill_in[r.prefill_instance] += q[2]
        decode_n[r.decode_instance - 2] += 1
        assert r.n_tokens == q[3] and r.prefill_done_ms > q[1] and r.decode_first_start_ms >= r.prefill_done_ms
        assert r.first_token_ms > r.decode_first_start_ms
    total_in = sum(prefill_in)
    assert abs(prefill_in[0] - 0.6 * total_in) <= 250.0 and abs(decode_n[0] - 20) <= 1
    # each instance's busy and idle records partition [0, horizon]
    for inst in range(4):
        spans = sorted([(b.start_ms, b.end_ms) for b in res.batches if b.instance == inst] +
                       [(i.start_ms, i.end_ms) for i in res.idles if i.instance == inst])
        assert spans and abs(spans[0][0]) <= 1e-9 and abs(spans[-1][1] - res.horizon_ms) <= 1e-9
        assert all(abs(spans[k][0] - spans[k - 1][1]) <= 1e-9 for k in range(1, len(spans)))
    assert math.isfinite(res.report.prefill_energy_j)

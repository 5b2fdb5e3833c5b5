"""Row 22 of SURVEY.md §8a on the device: simulate_cluster (simulator.hpp:
758-893) with the two-tier controllers (dvfs.hpp:302-390) or at fixed
frequencies, then trim_steady_state + make_report (metrics.hpp:71-156), for
batches of scenarios in one bs_replay call.  Checked bit for bit against the
unmodified reference (oracle/_ref: ref_replay runs pdsim::simulate_cluster,
trim_steady_state and make_report): every summary field, every request
record, and the full batch / idle / decision logs in SimResult order."""
from __future__ import annotations

import ctypes as C
import math

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P
from paper_2602_18755_b200 import workloads as W

pytestmark = pytest.mark.gpu

SUMMARY_FIELDS = [f for f, _ in A.bs_replay_summary._fields_ if f != "_pad"]
REQUEST_FIELDS = [f for f, _ in A.bs_replay_request._fields_ if f != "_pad"]


def same(a, b) -> bool:
    if isinstance(a, float) and isinstance(b, float):
        return (math.isnan(a) and math.isnan(b)) or a == b
    return a == b


def fields(x, names):
    return {n: (list(getattr(x, n)) if n == "decisions_by_trigger" else getattr(x, n)) for n in names}


def record_tuple(r):
    return tuple(getattr(r, f) for f, _ in r._fields_ if f != "_pad")


def run_ref(ref_lib, scenarios, models):
    keep: list = []
    cfgs, scs, total = P.c_replay_inputs(scenarios, keep)
    n = len(scenarios)
    out = (A.bs_replay_summary * n)()
    reqs = (A.bs_replay_request * max(1, total))()
    lg = P.c_replay_logs(scenarios, keep)
    cm = P.c_model_set(models, keep)
    ctl = next((s.controllers.models for s in scenarios if s.controllers is not None), models)
    cc = P.c_model_set(ctl, keep)
    rc = ref_lib.ref_replay(C.byref(cm), C.byref(cc), cfgs, scs, n, out, reqs, lg, 16)
    assert rc == 0, ref_lib.last_error()
    res, q = [], 0
    for i, s in enumerate(scenarios):
        L = lg[i]
        res.append({
            "summary": out[i],
            "requests": [reqs[q + k] for k in range(len(s.trace.requests))],
            "batches": [L.batches[k] for k in range(L.n_batches)],
            "idles": [L.idles[k] for k in range(L.n_idles)],
            "decisions": [L.decisions[k] for k in range(L.n_decisions)],
        })
        q += len(s.trace.requests)
    return res


def check_same(gpu_dev, ref_lib, scenarios, models):
    got = P.replay(scenarios, models, gpu_dev, requests=True, logs=True, raise_errors=False)
    want = run_ref(ref_lib, scenarios, models)
    keep: list = []
    for i, (g, w) in enumerate(zip(got, want)):
        ws = w["summary"]
        assert g.status == ws.status, (i, g.status, ws.status)
        if ws.status != 0:
            continue
        gs = A.bs_replay_summary()
        # re-read the raw summary through the Python mirror's fields
        r = g.report
        gvals = {"horizon_ms": g.horizon_ms, "completed_requests": g.completed_requests,
                 "generated_tokens": g.generated_tokens, "n_batches": g.n_batches, "n_idles": g.n_idles,
                 "n_decisions": g.n_decisions, "decisions_by_trigger": list(g.decisions_by_trigger),
                 "p99_ttft_ms": r.p99_ttft_ms, "p99_mean_tpot_ms": r.p99_mean_tpot_ms,
                 "energy_per_first_token_j": r.energy_per_first_token_j,
                 "energy_per_output_token_j": r.energy_per_output_token_j,
                 "avg_power_prefill_w": r.avg_power_prefill_w, "avg_power_decode_w": r.avg_power_decode_w,
                 "prefill_energy_j": r.prefill_energy_j, "decode_energy_j": r.decode_energy_j,
                 "span_ms": r.span_ms, "report_completed": r.completed_requests,
                 "report_generated": r.generated_tokens, "ttft_violations": r.ttft_violations,
                 "tpot_violations": r.tpot_violations}
        wvals = fields(ws, SUMMARY_FIELDS)
        for k, v in gvals.items():
            wv = wvals[k]
            if k.startswith("p99") or k.startswith("energy_per"):
                has = {"p99_ttft_ms": ws.has_p99_ttft, "p99_mean_tpot_ms": ws.has_p99_tpot,
                       "energy_per_first_token_j": ws.has_e_first, "energy_per_output_token_j": ws.has_e_output}[k]
                wv = wv if has else None
            assert (v is None and wv is None) or same(v, wv), (i, k, v, wv)
        assert len(g.requests) == len(w["requests"])
        for a, b in zip(g.requests, w["requests"]):
            fa, fb = fields(a, REQUEST_FIELDS), fields(b, REQUEST_FIELDS)
            for k in REQUEST_FIELDS:
                assert same(fa[k], fb[k]), (i, a.id, k, fa[k], fb[k])
        for kind in ("batches", "idles", "decisions"):
            ga = [record_tuple(x) for x in getattr(g, kind)]
            wa = [record_tuple(x) for x in w[kind]]
            assert len(ga) == len(wa), (i, kind, len(ga), len(wa))
            for j, (x, y) in enumerate(zip(ga, wa)):
                assert all(same(p, q) for p, q in zip(x, y)), (i, kind, j, x, y)
    return got


def scenario(rps, seconds, seed, *, n_pre=1, n_dec=1, weights=None, controlled=True, ttft=600.0, tpot=100.0,
             mbt=512, chunking=True, kv=1_000_000, max_req=256, shape=1.0, mpc_k=8, mpc_n=7, horizon=-1.0,
             rampup=5.0, levels=8, switch=30.0, margin=0.05, dmargin=0.05):
    lad = W.ladder(levels)
    models = W.llama_models(lad)
    tr = P.gen_gamma_trace(rps, shape, seconds * 1000.0,
                           P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), seed)
    fmax = lad.freqs_mhz[-1]
    wp = weights[0] if weights else [1.0 / n_pre] * n_pre
    wd = weights[1] if weights else [1.0 / n_dec] * n_dec
    inst = [P.ClusterInstance(P.InstanceConfig(P.Phase.prefill, 2, fmax), w) for w in wp]
    inst += [P.ClusterInstance(P.InstanceConfig(P.Phase.decode, 4, fmax), w) for w in wd]
    pol = P.SchedulerPolicy(max_batch_tokens=mbt, max_batch_requests=max_req, chunking=chunking,
                            kv_capacity_tokens=kv)
    slo = P.SLOSpec(ttft, tpot)
    fac = None
    if controlled:
        mpc = P.MpcConfig(horizon_K=mpc_k, ladder_N=mpc_n, ladder=lad)
        mpc.slo = slo
        mpc.switch_latency_ms = switch
        mpc.margin = margin
        dec = P.DecodePolicyConfig(tbt_slo_ms=tpot, kv_threshold=0.9, ladder=lad, margin=dmargin)
        fac = P.TwoTierFactory(mpc, dec, models, pol)
    return models, P.ReplayScenario(tr, P.ClusterSpec(inst), pol, fac, P.SimOptions(switch, horizon), slo, rampup)


def test_replay_c1_two_tier(gpu_device, ref_lib):
    models, s = scenario(6.0, 60, 7)
    got = check_same(gpu_device, ref_lib, [s], models)[0]
    assert got.n_decisions > 100 and got.completed_requests > 300


def test_replay_fixed_frequency(gpu_device, ref_lib):
    models, s = scenario(8.0, 60, 11, controlled=False)
    check_same(gpu_device, ref_lib, [s], models)


def test_replay_multi_instance_bursty_tight_slo(gpu_device, ref_lib):
    models, s = scenario(12.0, 60, 3, n_pre=2, n_dec=2, weights=([0.6, 0.4], [0.3, 0.7]), ttft=400.0, shape=0.5,
                         mpc_n=5, tpot=60.0)
    got = check_same(gpu_device, ref_lib, [s], models)[0]
    assert got.decisions_by_trigger[1] > 0  # arrival-triggered decisions


def test_replay_batch_of_scenarios(gpu_device, ref_lib):
    """Several scenarios in one call; each must equal its own reference run."""
    lad = W.ladder(8)
    models = W.llama_models(lad)
    scs = []
    for k, (rps, seed, npre, ndec, ctl) in enumerate([(4.0, 1, 1, 1, True), (10.0, 2, 2, 1, True),
                                                       (6.0, 3, 1, 3, False), (14.0, 4, 3, 2, True)]):
        _, s = scenario(rps, 40, seed, n_pre=npre, n_dec=ndec, controlled=ctl, ttft=500.0 + 50 * k)
        if s.controllers is not None:
            s.controllers.models = models
        scs.append(s)
    check_same(gpu_device, ref_lib, scs, models)


def test_replay_policies_and_options(gpu_device, ref_lib):
    """No chunking, small KV capacity (admission blocks on reservations),
    few residents, a horizon beyond the trace, no switch latency."""
    lad = W.ladder(8)
    models = W.llama_models(lad)
    variants = [dict(chunking=False, mbt=2048), dict(kv=40_000, max_req=16), dict(horizon=90_000.0, switch=0.0),
                dict(rampup=0.0, margin=0.0, dmargin=0.0), dict(mpc_k=4, mpc_n=8, mbt=1024)]
    scs = []
    for k, v in enumerate(variants):
        _, s = scenario(7.0, 45, 20 + k, **v)
        if s.controllers is not None:
            s.controllers.models = models
        scs.append(s)
    check_same(gpu_device, ref_lib, scs, models)


def test_replay_error_paths(gpu_device, ref_lib):
    """The exception simulate_cluster raises: KV need above capacity
    (SimulationError), no decode instance (ConfigError), bad weights
    (ParameterError); good scenarios in the same call are unaffected."""
    lad = W.ladder(8)
    models = W.llama_models(lad)
    _, bad_kv = scenario(5.0, 20, 5, kv=600)
    _, good = scenario(5.0, 20, 6)
    _, no_dec = scenario(5.0, 20, 7)
    no_dec.cluster.instances = [ci for ci in no_dec.cluster.instances if ci.config.phase == P.Phase.prefill]
    _, bad_w = scenario(5.0, 20, 8, n_pre=2, weights=([0.5, 0.6], [1.0]))
    scs = [bad_kv, good, no_dec, bad_w]
    for s in scs:
        s.controllers.models = models
    got = check_same(gpu_device, ref_lib, scs, models)
    assert [g.status for g in got] == [A.BS_SIMULATION_ERROR, 0, A.BS_CONFIG_ERROR, A.BS_PARAMETER_ERROR]
    with pytest.raises(P.SimulationError, match="KV tokens"):
        P.replay([bad_kv], models, gpu_device)


def test_replay_miscalibrated_controller_fires_safety(gpu_device, ref_lib):
    """TwoTierFactory with its own (optimistic) controller models: the
    simulator's ground truth runs slower than predicted, so safety deadlines
    fire and switch to max (simulator.hpp:238-245)."""
    lad = W.ladder(8)
    truth = W.llama_models(lad)
    optimistic = P.synth_model_set(P.SynthFamily.compute_bound, lad, [1, 2, 4, 8],
                                   P.SynthOptions(lat_coef=250.0, power_a=1e-7, power_b=60.0),
                                   P.SynthOptions(lat_coef=4.0, power_a=1e-7, power_b=120.0))
    scs = []
    for k, (rps, npre, ndec) in enumerate([(8.0, 1, 1), (14.0, 2, 2)]):
        _, s = scenario(rps, 45, 40 + k, n_pre=npre, n_dec=ndec, ttft=450.0)
        s.controllers.models = optimistic
        scs.append(s)
    got = check_same(gpu_device, ref_lib, scs, truth)
    assert sum(g.decisions_by_trigger[2] for g in got) > 0


def test_replay_edge_traces(gpu_device, ref_lib):
    """Empty trace, single request, one-token outputs (no TPOT), a burst of
    simultaneous arrivals, and a ramp-up longer than the trace (empty view)."""
    lad = W.ladder(8)
    models = W.llama_models(lad)
    scs = []
    _, base = scenario(5.0, 20, 31)
    variants = [
        [],
        [P.Request(0, 100.0, 700, 50)],
        [P.Request(i, 10.0 * i, 300 + 10 * i, 1) for i in range(40)],
        [P.Request(i, 500.0, 200 + i, 20 + i) for i in range(64)],
    ]
    for k, reqs in enumerate(variants):
        _, s = scenario(5.0, 20, 40 + k)
        s.trace = P.Trace(reqs, 20e3)
        s.controllers.models = models
        scs.append(s)
    _, late = scenario(5.0, 20, 50, rampup=60.0)
    late.controllers.models = models
    scs.append(late)
    got = check_same(gpu_device, ref_lib, scs, models)
    assert all(g.status == 0 for g in got)

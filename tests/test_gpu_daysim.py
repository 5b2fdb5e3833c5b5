"""GPU parity of the day-sweep driver (paper_2602_18755_b200/daysim.py,
BASELINE configs[3]): every (scenario, window) planned and replayed in four
device calls must equal pdsim.run_experiment (runner.hpp:155-172, two-tier
policy) scenario by scenario -- plans, tables and window reports -- and the
buffer-based window split / peak rate must equal split_windows /
peak_rps (workload.hpp:184-201, placement.hpp:513-527)."""
from __future__ import annotations

import pytest

from paper_2602_18755_b200 import daysim as D
from paper_2602_18755_b200 import pdsim as P
from paper_2602_18755_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _cfg(lad):
    cfg = P.RunnerConfig(slo=P.SLOSpec(600.0, 100.0), total_gpus=16, tp_options=[1, 2, 4, 8], ladder=lad,
                         scheduler=P.SchedulerPolicy(max_batch_tokens=2048), rampup_s=30.0)
    cfg.plan.policy = P.SchedulerPolicy(max_batch_tokens=2048)
    return cfg


def _as_trace(day: D.DayTrace) -> P.Trace:
    r = day.requests
    return P.Trace([P.Request(int(r["id"][i]), float(r["arrival_ms"][i]), int(r["input_len"][i]),
                              int(r["output_len"][i])) for i in range(len(r))], day.duration_ms)


def test_split_and_peak_match_the_trace_functions(gpu_device):
    day = D.gen_day(3, [5.0, 9.0])
    tr = _as_trace(day)
    for wms in (300e3, 7e5):
        a = D.split(day, wms)
        b = P.split_windows(tr, wms)
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert x.duration_ms == y.duration_ms and len(x.requests) == len(y.requests)
            assert [(int(q["id"]), float(q["arrival_ms"])) for q in x.requests] == \
                [(q.id, q.arrival_ms) for q in y.requests]
            if y.requests:
                assert D.peak_rps(x, 10.0) == P.peak_rps(y, 10.0)
    hour0 = P.gen_gamma_trace(5.0, 0.5, D.HOUR_MS, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)),
                              3000)
    assert [(q.id, q.arrival_ms, q.input_len, q.output_len) for q in hour0.requests] == \
        [(q.id, q.arrival_ms, q.input_len, q.output_len) for q in tr.requests[:len(hour0.requests)]]


def test_day_sweep_equals_run_experiment(gpu_device):
    lad = W.ladder(8)
    models = W.llama_models(lad)
    cfg = _cfg(lad)
    days = [D.gen_day(s, [6.0, 14.0]) for s in (11, 12)]
    res = D.run_day_sweep(days, 300e3, cfg, models, gpu_device)
    assert res.n_windows == 2 * 24
    for s, day in enumerate(days):
        ex = P.run_experiment(_as_trace(day), 300e3, [P.Policy.two_tier], cfg, models, gpu_device)
        assert len(ex.runs) == len(res.results[s])
        for w, run in enumerate(ex.runs):
            got_plan, got = res.plans[s][w].ilp, res.results[s][w]
            assert (got_plan.counts, got_plan.objective_w, got_plan.gpus_used) == \
                (run.plan.counts, run.plan.objective_w, run.plan.gpus_used)
            assert res.plans[s][w].target_rps > 0.0
            a, b = got.report, run.result.report
            assert (got.n_decisions, got.completed_requests, got.generated_tokens) == \
                (run.result.n_decisions, run.result.completed_requests, run.result.generated_tokens)
            assert (a.prefill_energy_j, a.decode_energy_j, a.p99_ttft_ms, a.p99_mean_tpot_ms, a.ttft_violations) == \
                (b.prefill_energy_j, b.decode_energy_j, b.p99_ttft_ms, b.p99_mean_tpot_ms, b.ttft_violations)

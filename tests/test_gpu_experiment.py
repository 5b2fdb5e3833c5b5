"""run_experiment (runner.hpp:155-172) on the GPU path: per window a GPU
config table + the exact ILP / max-throughput plans (planned from the
previous window), then every (window, policy) simulate_cluster + report in
one bs_replay call.  Checked against the unmodified reference
run_experiment (oracle/_ref) run by run: plan (GPUs used, objective,
target), SimResult counters, MetricsReport fields and SLO verdicts, bit for
bit."""
from __future__ import annotations

import ctypes as C
import math

import pytest

import oracle
from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P
from paper_2602_18755_b200 import workloads as W

pytestmark = pytest.mark.gpu


def same(a, b):
    return a == b or (isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b))


def ref_config(cfg: P.RunnerConfig, keep: list) -> oracle.ref_runner_config:
    c = oracle.ref_runner_config()
    c.slo = P.c_slo(cfg.slo)
    c.total_gpus = cfg.total_gpus
    tps = (C.c_int32 * len(cfg.tp_options))(*cfg.tp_options)
    lad = (C.c_double * len(cfg.ladder.freqs_mhz))(*cfg.ladder.freqs_mhz)
    keep += [tps, lad]
    c.n_tp, c.tp_options = len(cfg.tp_options), tps
    c.ladder, c.n_ladder = lad, len(cfg.ladder.freqs_mhz)
    c.scheduler = P.c_policy(cfg.scheduler)
    c.alpha, c.peak_subwindow_s = cfg.plan.alpha, cfg.plan.peak_subwindow_s
    c.search = P.c_search(cfg.plan.search)
    c.plan_policy = P.c_policy(cfg.plan.policy)
    c.rampup_s, c.switch_latency_ms = cfg.rampup_s, cfg.switch_latency_ms
    c.mpc_k, c.mpc_n, c.mpc_margin = cfg.mpc_horizon_k, cfg.mpc_ladder_n, cfg.mpc_margin
    c.kv_threshold, c.decode_margin = cfg.kv_threshold, cfg.decode_margin
    return c


@pytest.mark.parametrize("rps,shape,minutes,window_s,gpus,seed", [
    (8.0, 1.0, 6, 120, 8, 7),
    (14.0, 0.5, 4, 60, 16, 11),
])
def test_run_experiment_matches_reference(gpu_device, ref_lib, rps, shape, minutes, window_s, gpus, seed):
    lad = W.ladder(8)
    models = W.llama_models(lad)
    trace = P.gen_gamma_trace(rps, shape, minutes * 60e3,
                              P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), seed)
    cfg = P.RunnerConfig(slo=P.SLOSpec(600.0, 100.0), total_gpus=gpus, tp_options=[1, 2, 4], ladder=lad,
                         scheduler=P.SchedulerPolicy(max_batch_tokens=1024), rampup_s=10.0)
    cfg.plan.policy = P.SchedulerPolicy(max_batch_tokens=1024)
    pols = [P.Policy.maxfreq_distserve, P.Policy.place_only, P.Policy.two_tier]
    got = P.run_experiment(trace, window_s * 1000.0, pols, cfg, models, gpu_device)

    keep: list = []
    cap = 64
    out = (oracle.ref_window_run * cap)()
    n_out, tt = C.c_int(), C.c_int32()
    cm, ct = P.c_model_set(models, keep), P.c_trace(trace, keep)
    pa = (C.c_int32 * 3)(*[int(p) for p in pols])
    rc = ref_lib.ref_run_experiment(C.byref(cm), C.byref(ct), window_s * 1000.0, pa, 3, C.byref(ref_config(cfg, keep)),
                                    out, cap, C.byref(n_out), C.byref(tt))
    assert rc == 0, ref_lib.last_error()
    assert n_out.value == len(got.runs) == 3 * math.ceil(minutes * 60 / window_s)
    assert bool(tt.value) == got.two_tier_slo_pass
    names = [f for f, _ in A.bs_replay_summary._fields_ if f not in ("_pad", "status", "decisions_by_trigger")]
    for i, run in enumerate(got.runs):
        w = out[i]
        assert (run.window_index, int(run.policy)) == (w.window, w.policy)
        assert (run.plan.gpus_used, run.plan.objective_w, run.plan.target_rps) == (w.gpus_used, w.objective_w,
                                                                                    w.target_rps), i
        assert run.slo_pass == bool(w.slo_pass)
        r, rep = run.result, run.report
        mine = {"horizon_ms": r.horizon_ms, "completed_requests": r.completed_requests,
                "generated_tokens": r.generated_tokens, "n_batches": r.n_batches, "n_idles": r.n_idles,
                "n_decisions": r.n_decisions,
                "has_p99_ttft": int(rep.p99_ttft_ms is not None), "has_p99_tpot": int(rep.p99_mean_tpot_ms is not None),
                "has_e_first": int(rep.energy_per_first_token_j is not None),
                "has_e_output": int(rep.energy_per_output_token_j is not None),
                "p99_ttft_ms": rep.p99_ttft_ms, "p99_mean_tpot_ms": rep.p99_mean_tpot_ms,
                "energy_per_first_token_j": rep.energy_per_first_token_j,
                "energy_per_output_token_j": rep.energy_per_output_token_j,
                "avg_power_prefill_w": rep.avg_power_prefill_w, "avg_power_decode_w": rep.avg_power_decode_w,
                "prefill_energy_j": rep.prefill_energy_j, "decode_energy_j": rep.decode_energy_j,
                "span_ms": rep.span_ms, "report_completed": rep.completed_requests,
                "report_generated": rep.generated_tokens, "ttft_violations": rep.ttft_violations,
                "tpot_violations": rep.tpot_violations}
        for k in names:
            want = getattr(w.report, k)
            have = mine[k]
            if have is None:
                assert not getattr(w.report, "has_" + {"p99_ttft_ms": "p99_ttft", "p99_mean_tpot_ms": "p99_tpot",
                                                       "energy_per_first_token_j": "e_first",
                                                       "energy_per_output_token_j": "e_output"}[k])
                continue
            assert same(have, want), (i, k, have, want)
        assert list(r.decisions_by_trigger) == list(w.report.decisions_by_trigger)
        assert rep.window_id == f"w{run.window_index}"

"""Golden vectors of the unmodified reference (tests/golden/mpc_golden.json,
written by tools/make_golden.py from oracle/_ref/libpdsim_ref.so): the oracle
restatement (CPU) and the sm_100a path (GPU, through the C ABI) must reproduce
every recorded decision bit for bit, without /root/reference or the reference
driver being present."""
from __future__ import annotations

import json
from pathlib import Path

import pytest

from helpers import cpu_decode, cpu_mpc, gpu_result_tuple, result_tuple
from paper_2602_18755_b200 import pdsim as P

GOLDEN = json.loads((Path(__file__).parent / "golden" / "mpc_golden.json").read_text())
SET_IDS = [f"{s['kind']}-{s['generator']}-{s['seed']:#x}" for s in GOLDEN["mpc_sets"]]


def _instances(s):
    from make_golden import instances
    return instances(s["generator"], s["seed"], len(s["records"]), s["kwargs"])


def _expect(rec, kind):
    exp = tuple(tuple(x) if isinstance(x, list) else x for x in rec["result"])
    exp = exp[:4] + (tuple(exp[4]),) + exp[5:6] + (tuple(tuple(lv) for lv in rec["result"][6]),)
    extra = (rec["feasible_count"], rec["best_code"], rec["trajectories"]) if kind == "exhaustive" else None
    return exp, extra


@pytest.fixture(scope="module", autouse=True)
def _tools_path():
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))


@pytest.mark.parametrize("s", GOLDEN["mpc_sets"], ids=SET_IDS)
def test_oracle_reproduces_reference_golden(oracle_lib, s):
    for inst, rec in zip(_instances(s), s["records"]):
        rc, r = cpu_mpc(oracle_lib, s["kind"], *inst)
        assert rc == rec["status"]
        exp, extra = _expect(rec, s["kind"])
        assert result_tuple(r) == exp
        if extra:
            assert (r.feasible_count, r.best_code, r.trajectories) == extra


def test_oracle_decode_golden(oracle_lib):
    from make_golden import decode_instances
    d = GOLDEN["decode"]
    for (m, cfg, batch, kv), rec in zip(decode_instances(d["seed"], d["count"]), d["records"]):
        o = cpu_decode(oracle_lib, m, cfg, batch, kv, 1)
        assert [o.status, o.freq_mhz, o.eval_count, o.kv_override] == rec


@pytest.mark.gpu
@pytest.mark.parametrize("s", GOLDEN["mpc_sets"], ids=SET_IDS)
def test_gpu_reproduces_reference_golden(gpu_device, s):
    insts = list(_instances(s))
    for (m, cfg, pol, q), rec in zip(insts, s["records"]):
        fn = P.greedy_freq_select if s["kind"] == "greedy" else P.exhaustive_freq_select
        g = fn(q, cfg, m, pol)
        exp, extra = _expect(rec, s["kind"])
        assert gpu_result_tuple(g, exp[0]) == exp
        if extra:
            assert (g.feasible_count, g.best_code, g.trajectories) == extra


@pytest.mark.gpu
def test_gpu_c2_golden(gpu_device):
    """BASELINE C2 (horizon 6 x 16 rungs, 16,777,216 trajectories per decision)."""
    from paper_2602_18755_b200.workloads import c2_corpus
    c2 = GOLDEN["c2"]
    m, cfg, pol, snaps = c2_corpus(c2["seed"], c2["count"])
    got = P.exhaustive_freq_select_batch(snaps, cfg, m, pol)
    for g, rec in zip(got, c2["records"]):
        exp, extra = _expect(rec, "exhaustive")
        assert gpu_result_tuple(g, exp[0]) == exp
        assert (g.feasible_count, g.best_code, g.trajectories) == extra


@pytest.mark.gpu
def test_gpu_decode_golden(gpu_device):
    from make_golden import decode_instances
    d = GOLDEN["decode"]
    for (m, cfg, batch, kv), rec in zip(decode_instances(d["seed"], d["count"]), d["records"]):
        g = P.select_decode_freq_ex(batch, kv, cfg, m, 1)
        assert [0, g.freq_mhz, g.eval_count, int(g.kv_override)] == rec


def test_placement_golden_inputs_regenerate():
    """The C3-shaped windows regenerate with the recorded request counts (the
    host trace generator is bit-identical to gen_gamma_trace, workload.hpp)."""
    from make_golden import placement_inputs
    for t in GOLDEN["placement"]:
        _, base, cands, _, _ = placement_inputs(t["seed"])
        assert len(base.requests) == t["n_requests"] and len(cands) == len(t["rows"])


@pytest.mark.gpu
@pytest.mark.parametrize("t", GOLDEN["placement"], ids=lambda t: f"seed{t['seed']}-probes{t['probe_count']}")
def test_gpu_config_table_golden(gpu_device, t):
    """build_config_table (placement.hpp:240-260) on the GPU probe grid equals
    the reference's table entry for entry (r_c, E_c, G_c, saturated, error)."""
    from make_golden import placement_inputs, table_row
    m, base, cands, pol, slo = placement_inputs(t["seed"])
    search = P.GoodputSearch(probe_count=t["probe_count"], tolerance_rps=t["tolerance_rps"])
    got = P.build_config_table(cands, base, slo, m, pol, search)
    assert [table_row(e) for e in got] == t["rows"]

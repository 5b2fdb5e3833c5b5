"""GPU parity of the placement ILPs (bs_ilp.cu): solve_placement
(placement.hpp:357-416) and solve_max_throughput (placement.hpp:421-499) on
the device against the compiled reference -- the reference's known answers
(tests/test_placement.cpp:120-188), random tables with exact duplicates
(ties follow the lexicographic rule), C3-sized tables (128 entries, 16 GPUs)
and the batched entry point."""
from __future__ import annotations

import ctypes as C
import random

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import _lib
from paper_2602_18755_b200 import pdsim as P
from paper_2602_18755_b200 import workloads as W

pytestmark = pytest.mark.gpu

PF, DE = P.Phase.prefill, P.Phase.decode


def entry(phase, tp, f, r, e):  # test_placement.cpp:42-50
    return P.ConfigTableEntry(P.InstanceConfig(phase, tp, f), r, e, tp)


def lib_solve(table, G, target, alpha, max_freq=None, ctx=None):
    """Through the C ABI; ctx None = the library's default context (as the
    reference-shaped C++ drop-ins call it)."""
    L = _lib.lib()
    tab = P.c_table(table)
    n = len(table)
    counts = (C.c_int64 * max(1, n))()
    obj, used = C.c_double(), C.c_int32()
    if max_freq is None:
        rc = L.bs_placement_solve(ctx, tab, n, G, target, alpha, counts, C.byref(obj), C.byref(used))
    else:
        rc = L.bs_placement_max_throughput(ctx, tab, n, G, target, alpha, max_freq, counts, C.byref(obj),
                                           C.byref(used))
    msg = (L.bs_last_error(ctx) or b"").decode()
    return rc, list(counts[:n]), obj.value, used.value, msg if rc else ""


def ref_solve(ref, table, G, target, alpha, max_freq=None):
    tab = P.c_table(table)
    n = len(table)
    counts = (C.c_int64 * max(1, n))()
    obj, used = C.c_double(), C.c_int32()
    if max_freq is None:
        rc = ref.ref_solve_placement(tab, n, G, target, alpha, counts, C.byref(obj), C.byref(used))
    else:
        rc = ref.ref_solve_max_throughput(tab, n, G, target, alpha, max_freq, counts, C.byref(obj), C.byref(used))
    return rc, list(counts[:n]), obj.value, used.value, ref.last_error().decode() if rc else ""


def test_ilp_kats(gpu_device):  # test_placement.cpp:120-188
    t = [entry(PF, 1, 1000.0, 10.0, 5.0), entry(PF, 1, 500.0, 10.0, 3.0),
         entry(DE, 1, 1000.0, 10.0, 4.0), entry(DE, 1, 500.0, 10.0, 2.0)]
    rc, counts, obj, used, _ = lib_solve(t, 4, 10.0, 0.0)
    assert rc == 0 and counts == [0, 1, 0, 1] and used == 2
    assert obj == 10.0 * 3.0 + 10.0 * 2.0
    rc, *_, msg = lib_solve([t[0]], 4, 10.0, 0.0)
    assert rc == A.BS_INFEASIBLE_ERROR and msg.startswith("goodput-decode|")
    rc, *_, msg = lib_solve(t, 1, 10.0, 0.0)
    assert rc == A.BS_INFEASIBLE_ERROR and msg.startswith("capacity|prefill needs 1 GPUs, decode needs 1")
    plan = P.solve_placement(P.PlacementProblem(t, 4, 10.0, 0.0), gpu_device)
    assert plan.counts == [0, 1, 0, 1] and [i.weight for i in plan.instances] == [1.0, 1.0]
    with pytest.raises(P.InfeasibleError) as ei:
        P.solve_placement(P.PlacementProblem(t, 1, 10.0, 0.0), gpu_device)
    assert ei.value.binding_constraint() == "capacity"


def _random_table(rng, n_lo=3, n_hi=8, dup=2):
    n = rng.randint(n_lo, n_hi)
    tab = []
    for _ in range(n):
        ph = rng.choice([PF, DE])
        tp = rng.choice([1, 2, 4, 8])
        f = rng.choice([500.0, 1000.0, 1500.0])
        r = rng.choice([0.0, rng.uniform(0.5, 30.0)])
        e = rng.uniform(0.5, 20.0) if r > 0 else None
        tab.append(P.ConfigTableEntry(P.InstanceConfig(ph, tp, f), r, e, tp))
    for _ in range(rng.randint(0, dup)):  # exact duplicates force ties (lexicographic rule)
        tab.append(tab[rng.randrange(len(tab))])
    return tab


def test_ilp_matches_reference_random(gpu_device, ref_lib):
    """400 small random tables (the survey's B&B-vs-enumeration set shape)."""
    rng = random.Random(0xFEEDFACE)
    solved = 0
    for _ in range(400):
        tab = _random_table(rng)
        G = rng.randint(2, 16)
        target = rng.uniform(1.0, 40.0)
        alpha = rng.choice([0.0, 0.05])
        a = lib_solve(tab, G, target, alpha, ctx=gpu_device.handle)
        b = ref_solve(ref_lib, tab, G, target, alpha)
        assert a == b
        solved += a[0] == 0
        a = lib_solve(tab, G, target, alpha, 1500.0, ctx=gpu_device.handle)
        b = ref_solve(ref_lib, tab, G, target, alpha, 1500.0)
        assert a == b
    assert solved > 50


@pytest.mark.parametrize("seed", range(4))
def test_ilp_wider_tables(gpu_device, ref_lib, seed):
    """Wider trees than the frontier (12-40 entries, up to 32 GPUs): the
    frontier / subtree split and the key's subtree order matter here."""
    rng = random.Random(0x1A0 + seed)
    for _ in range(25):
        tab = _random_table(rng, 12, 40, 6)
        G = rng.randint(8, 32)
        target = rng.uniform(5.0, 120.0)
        alpha = rng.choice([0.0, 0.05])
        assert lib_solve(tab, G, target, alpha, ctx=gpu_device.handle) == ref_solve(ref_lib, tab, G, target, alpha)
        mf = rng.choice([1000.0, 1500.0])
        if G <= 20:
            assert lib_solve(tab, G, target, alpha, mf, ctx=gpu_device.handle) == \
                ref_solve(ref_lib, tab, G, target, alpha, mf)


def _c3_table(rng, lad):
    """A C3-shaped table: 2 phases x TP {1,2,4,8} x 16 rungs = 128 entries,
    goodput rising with TP and frequency, energy per request falling with
    frequency towards a knee; some candidates unusable."""
    tab = []
    for ph in (PF, DE):
        for tp in (1, 2, 4, 8):
            for f in lad.freqs_mhz:
                if rng.random() < 0.1:
                    tab.append(P.ConfigTableEntry(P.InstanceConfig(ph, tp, f), 0.0, None, tp))
                    continue
                r = 0.25 * int(tp * (0.6 + f / 1830.0) * rng.uniform(2.0, 4.0) / 0.25)
                e = (40.0 + 1e-5 * f * f) * tp * rng.uniform(0.8, 1.2) / max(r, 0.25)
                tab.append(P.ConfigTableEntry(P.InstanceConfig(ph, tp, f), r, e if r > 0 else None, tp))
    return tab


@pytest.mark.parametrize("seed", range(3))
def test_ilp_c3_sized_tables(gpu_device, ref_lib, seed):
    rng = random.Random(0xC3 + seed)
    lad = W.ladder(16)
    for target in (4.0, 12.0, 20.0):
        tab = _c3_table(rng, lad)
        for G in (8, 16):
            assert lib_solve(tab, G, target, 0.05, ctx=gpu_device.handle) == \
                ref_solve(ref_lib, tab, G, target, 0.05)
            assert lib_solve(tab, G, target, 0.05, lad.max_mhz(), ctx=gpu_device.handle) == \
                ref_solve(ref_lib, tab, G, target, 0.05, lad.max_mhz())


def test_ilp_real_config_table(gpu_device, ref_lib):
    """A config table built by the device goodput search on a C3-shaped
    window, solved for 16 GPUs at the window's peak rate."""
    lad = W.ladder(8)
    m = W.llama_models(lad)
    base = P.gen_gamma_trace(12.0, 0.5, 60_000.0, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)),
                             7)
    cands = P.enumerate_candidates(lad, [1, 2, 4, 8])
    table = P.build_config_table(cands, base, P.SLOSpec(600.0, 100.0), m, P.SchedulerPolicy(max_batch_tokens=2048),
                                 P.GoodputSearch(), device=gpu_device)
    peak = P.peak_rps(base, 10.0)
    for alpha in (0.0, 0.05):
        assert lib_solve(table, 16, peak, alpha, ctx=gpu_device.handle) == ref_solve(ref_lib, table, 16, peak, alpha)
        assert lib_solve(table, 16, peak, alpha, lad.max_mhz(), ctx=gpu_device.handle) == \
            ref_solve(ref_lib, table, 16, peak, alpha, lad.max_mhz())


def test_ilp_batch_equals_single_calls(gpu_device, ref_lib):
    """bs_placement_solve_batch: 120 problems of both kinds (feasible,
    infeasible, parameter errors) in one call, each equal to the reference."""
    rng = random.Random(0xBA7C)
    probs = []
    for k in range(120):
        tab = _random_table(rng, 3, 24, 3)
        G = rng.randint(1, 20)
        mf = rng.choice([None, 1500.0])
        probs.append((P.PlacementProblem(tab, G, rng.uniform(1.0, 60.0), rng.choice([0.0, 0.05])), mf))
    probs.append((P.PlacementProblem(_random_table(rng), 0, 5.0, 0.0), None))  # total_gpus < 1
    got = P.solve_placement_batch(probs, gpu_device)
    for (p, mf), g in zip(probs, got):
        rc, counts, obj, used, msg = ref_solve(ref_lib, p.table, p.total_gpus, p.target_rps, p.alpha, mf)
        if rc:
            assert isinstance(g, P.PdsimError)
            if rc == A.BS_INFEASIBLE_ERROR:
                assert isinstance(g, P.InfeasibleError) and f"{g.binding_constraint()}|{g}" == msg
        else:
            assert (g.counts, g.objective_w, g.gpus_used) == (counts, obj, used)

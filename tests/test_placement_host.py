"""CPU-side parity of the placement path's host logic (no GPU): trace
synthesis (gen_gamma_trace, workload.hpp:95-116) and the exact ILPs
(solve_placement placement.hpp:357-416, solve_max_throughput 421-499) of
libbiscale_gpu.so against the compiled reference, on the reference's own
known answers (tests/test_placement.cpp) and random tables."""
from __future__ import annotations

import ctypes as C
import random

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import _lib
from paper_2602_18755_b200 import pdsim as P


def entry(phase, tp, f, r, e):  # test_placement.cpp:42-50
    return P.ConfigTableEntry(P.InstanceConfig(phase, tp, f), r, e, tp)


def lib_solve(table, G, target, alpha, max_freq=None):
    L = _lib.lib()
    tab = P.c_table(table)
    n = len(table)
    counts = (C.c_int64 * max(1, n))()
    obj, used = C.c_double(), C.c_int32()
    if max_freq is None:
        rc = L.bs_placement_solve(None, tab, n, G, target, alpha, counts, C.byref(obj), C.byref(used))
    else:
        rc = L.bs_placement_max_throughput(None, tab, n, G, target, alpha, max_freq, counts, C.byref(obj),
                                           C.byref(used))
    msg = (L.bs_last_error(None) or b"").decode()
    return rc, list(counts[:n]), obj.value, used.value, msg


def ref_solve(ref, table, G, target, alpha, max_freq=None):
    tab = P.c_table(table)
    n = len(table)
    counts = (C.c_int64 * max(1, n))()
    obj, used = C.c_double(), C.c_int32()
    if max_freq is None:
        rc = ref.ref_solve_placement(tab, n, G, target, alpha, counts, C.byref(obj), C.byref(used))
    else:
        rc = ref.ref_solve_max_throughput(tab, n, G, target, alpha, max_freq, counts, C.byref(obj), C.byref(used))
    return rc, list(counts[:n]), obj.value, used.value, ref.last_error().decode()


PF, DE = P.Phase.prefill, P.Phase.decode


def test_ilp_kats():  # test_placement.cpp:120-188
    t = [entry(PF, 1, 1000.0, 10.0, 5.0), entry(PF, 1, 500.0, 10.0, 3.0),
         entry(DE, 1, 1000.0, 10.0, 4.0), entry(DE, 1, 500.0, 10.0, 2.0)]
    rc, counts, obj, used, _ = lib_solve(t, 4, 10.0, 0.0)
    assert rc == 0 and counts == [0, 1, 0, 1] and used == 2
    assert obj == 10.0 * 3.0 + 10.0 * 2.0
    rc, *_ , msg = lib_solve([t[0]], 4, 10.0, 0.0)
    assert rc == A.BS_INFEASIBLE_ERROR and msg.startswith("goodput-decode|")
    rc, *_ , msg = lib_solve(t, 1, 10.0, 0.0)
    assert rc == A.BS_INFEASIBLE_ERROR and msg.startswith("capacity|prefill needs 1 GPUs, decode needs 1")


def _random_table(rng):
    n = rng.randint(3, 8)
    tab = []
    for _ in range(n):
        ph = rng.choice([PF, DE])
        tp = rng.choice([1, 2, 4, 8])
        f = rng.choice([500.0, 1000.0, 1500.0])
        r = rng.choice([0.0, rng.uniform(0.5, 30.0)])
        e = rng.uniform(0.5, 20.0) if r > 0 else None
        tab.append(P.ConfigTableEntry(P.InstanceConfig(ph, tp, f), r, e, tp))
    # exact duplicates force ties (lexicographic rule)
    for _ in range(rng.randint(0, 2)):
        tab.append(tab[rng.randrange(len(tab))])
    return tab


def test_ilp_matches_reference_random(ref_lib):
    rng = random.Random(0xFEEDFACE)
    solved = 0
    for _ in range(400):
        tab = _random_table(rng)
        G = rng.randint(2, 16)
        target = rng.uniform(1.0, 40.0)
        alpha = rng.choice([0.0, 0.05])
        a = lib_solve(tab, G, target, alpha)
        b = ref_solve(ref_lib, tab, G, target, alpha)
        assert a == b
        solved += a[0] == 0
        a = lib_solve(tab, G, target, alpha, 1500.0)
        b = ref_solve(ref_lib, tab, G, target, alpha, 1500.0)
        assert a == b
    assert solved > 50


def _ref_trace(ref, rps, shape, dur, lengths, seed):
    keep: list = []
    cl = P.c_lengths(lengths, keep)
    n = C.c_int64()
    assert ref.ref_gen_gamma_trace(rps, shape, dur, C.byref(cl), seed, None, 0, C.byref(n)) == 0
    out = (A.bs_request * max(1, n.value))()
    assert ref.ref_gen_gamma_trace(rps, shape, dur, C.byref(cl), seed, out, n.value, C.byref(n)) == 0
    return [(out[i].id, out[i].arrival_ms, out[i].input_len, out[i].output_len) for i in range(n.value)]


@pytest.mark.parametrize("shape", [0.5, 1.0, 2.5])
def test_gen_gamma_trace_bit_identical(ref_lib, shape):
    lengths = P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7))
    t = P.gen_gamma_trace(12.0, shape, 60_000.0, lengths, 7)
    got = [(r.id, r.arrival_ms, r.input_len, r.output_len) for r in t.requests]
    assert got == _ref_trace(ref_lib, 12.0, shape, 60_000.0, lengths, 7)
    pool = P.LengthDistribution(samples=[(100, 10), (2000, 300), (512, 64)])
    t = P.gen_gamma_trace(5.0, shape, 30_000.0, pool, 11)
    assert [(r.id, r.arrival_ms, r.input_len, r.output_len) for r in t.requests] == \
        _ref_trace(ref_lib, 5.0, shape, 30_000.0, pool, 11)


def test_split_windows_and_peak():  # workload.hpp:184-201, placement.hpp:513-527
    t = P.Trace([P.Request(i, 1000.0 * i + 0.5, 10, 5) for i in range(25)], 25_000.0)
    w = P.split_windows(t, 10_000.0)
    assert [len(x.requests) for x in w] == [10, 10, 5]
    assert w[1].requests[0].arrival_ms == 0.5 and w[2].duration_ms == 5_000.0
    assert P.peak_rps(t, 10.0) == 1.0

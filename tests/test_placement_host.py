"""CPU-side parity of the placement path's host logic (no GPU): trace
synthesis (gen_gamma_trace, workload.hpp:95-116), window splitting and the
peak rate against the compiled reference.  The ILPs run on the device:
tests/test_gpu_ilp.py."""
from __future__ import annotations

import ctypes as C

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import pdsim as P


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

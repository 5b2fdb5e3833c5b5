"""The N>1 host path on CPU: world_size-2 gloo process groups exercising the
sharding used by bench.py --gpus N.  The per-unit work is done
by the CPU oracle here (test infrastructure); what is under test is the
partitioning, the gather order and the two-step (objective, code) MIN
all-reduce of a decision sliced across ranks."""
from __future__ import annotations

import ctypes as C
import os
import random
import socket
import struct

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_18755_b200 import sharding as S


def test_shard_bounds_partition():
    for n in (0, 1, 7, 256, 1001):
        for world in (1, 2, 3, 8):
            spans = [S.shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_code_slices_cover_whole_subtrees():
    for nc, K, world in ((16, 6, 2), (16, 6, 8), (24, 8, 8), (3, 4, 5), (7, 2, 4)):
        spans = [S.code_slice(nc, K, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == nc ** K
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_prefix_slices_partition_leading_digits():
    for nc, world in ((16, 2), (16, 8), (24, 8), (5, 8), (2, 8), (3, 3)):
        spans = [S.prefix_slice(nc, r, world) for r in range(world)]
        digits = spans[0][0]
        assert all(d == digits for d, _, _ in spans) and digits == (1 if nc >= world else 2)
        assert spans[0][1] == 0 and spans[-1][2] == nc ** digits
        assert all(spans[i][2] == spans[i + 1][1] for i in range(world - 1))


def test_combine_slices_takes_lexicographic_minimum():
    assert S.combine_slices([(False, 9.0, 5, 0), (False, 1.0, 2, 0)]) == (None, None, 0)
    # equal objectives: the smaller code wins whatever the slice order
    assert S.combine_slices([(True, 2.5, 40, 3), (True, 2.5, 7, 4), (True, 3.0, 1, 1)]) == (2.5, 7, 8)
    assert S.combine_slices([(True, 0.0, 99, 1), (False, 0.0, 0, 0)]) == (0.0, 99, 1)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import oracle
        from paper_2602_18755_b200 import _abi as A
        from paper_2602_18755_b200 import pdsim as P
        from paper_2602_18755_b200 import workloads as W

        orc = oracle.load_oracle()
        lad = W.ladder(5)
        m = W.llama_models(lad)
        cfg = P.MpcConfig(horizon_K=4, ladder_N=5, ladder=lad)
        pol = P.SchedulerPolicy(max_batch_tokens=512)
        rng = random.Random(0x5A)
        snaps = [W.synthetic_snapshot(rng, lad, n_lo=4, n_hi=9) for _ in range(11)]
        keep: list = []
        cm, cc, cp = P.c_model_set(m, keep), P.c_mpc_config(cfg, keep), P.c_policy(pol)

        # 1. decisions sharded across ranks, rows gathered in global order
        lo, hi = S.shard_bounds(len(snaps), rank, world)
        rows = []
        for q in snaps[lo:hi]:
            r = A.bs_mpc_result()
            assert orc.orc_exhaustive(C.byref(cm), C.byref(cc), C.byref(cp), C.byref(P.c_snapshot(q, keep)),
                                      C.byref(r)) == 0
            bits = struct.unpack("<q", struct.pack("<d", r.objective_w))[0]
            rows.append([bits, r.best_code, r.feasible_count])
        got = S.gather_rows(torch.tensor(rows, dtype=torch.int64).reshape(-1, 3), len(snaps))

        # 2. one decision sliced by leading digits, two-step MIN all-reduce
        q = snaps[3]
        nc, K = 5, 4
        a, b = S.code_slice(nc, K, rank, world)
        codes = (C.c_uint64 * (b - a))(*range(a, b))
        feas = (C.c_int32 * (b - a))()
        obj = (C.c_double * (b - a))()
        assert orc.orc_eval_codes(C.byref(cm), C.byref(cc), C.byref(cp), C.byref(P.c_snapshot(q, keep)), codes,
                                  b - a, feas, obj) == 0
        best = None
        for i in range(b - a):
            if feas[i] and (best is None or obj[i] < best[0]):  # first strict min = smallest code
                best = (obj[i], a + i)
        gobj, gcode = S.argmin_over_ranks(best[0] if best else None, best[1] if best else None)
        t = S.max_over_ranks(float(rank + 1))
        outq.put((rank, got.tolist(), (gobj, gcode), t))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_gather_and_sliced_argmin(oracle_lib):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort()
    assert outs[0][1] == outs[1][1]  # every rank holds the same gathered table
    assert outs[0][2] == outs[1][2] and outs[0][3] == outs[1][3] == 2.0

    # single-process reference of the same work
    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as W

    lad = W.ladder(5)
    m = W.llama_models(lad)
    cfg = P.MpcConfig(horizon_K=4, ladder_N=5, ladder=lad)
    pol = P.SchedulerPolicy(max_batch_tokens=512)
    rng = random.Random(0x5A)
    snaps = [W.synthetic_snapshot(rng, lad, n_lo=4, n_hi=9) for _ in range(11)]
    keep: list = []
    cm, cc, cp = P.c_model_set(m, keep), P.c_mpc_config(cfg, keep), P.c_policy(pol)
    want = []
    for s in snaps:
        r = A.bs_mpc_result()
        assert oracle_lib.orc_exhaustive(C.byref(cm), C.byref(cc), C.byref(cp), C.byref(P.c_snapshot(s, keep)),
                                         C.byref(r)) == 0
        want.append([struct.unpack("<q", struct.pack("<d", r.objective_w))[0], r.best_code, r.feasible_count])
        if s is snaps[3]:
            whole = r
    assert outs[0][1] == want
    if whole.feasible:
        assert outs[0][2] == (whole.objective_w, whole.best_code)
    else:
        assert outs[0][2] == (None, None)


def _table_worker(rank: int, world: int, port: int, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2602_18755_b200 import _abi as A
        from paper_2602_18755_b200 import pdsim as P
        from paper_2602_18755_b200 import workloads as W

        ref = oracle.load_ref()
        lad = W.ladder(5)
        m = W.llama_models(lad)
        day = P.gen_gamma_trace(6.0, 0.5, 5 * 20_000.0,
                                P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 4)
        wins = P.split_windows(day, 20_000.0)
        cands = P.enumerate_candidates(lad, [2, 4])
        lo, hi = S.shard_bounds(len(wins), rank, world)
        keep: list = []
        cm = P.c_model_set(m, keep)
        local = []
        for w in wins[lo:hi]:  # the CPU reference stands in for each rank's device here
            out = (A.bs_table_entry * len(cands))()
            assert ref.ref_config_table(C.byref(cm), C.byref(P.c_trace(w, keep)), C.byref(P.c_slo(P.SLOSpec())),
                                        C.byref(P.c_policy(P.SchedulerPolicy(max_batch_tokens=1024))),
                                        C.byref(P.c_search(P.GoodputSearch())), P.c_candidates(cands), len(cands),
                                        out) == 0
            local.append([P.entry_from_c(out[i]) for i in range(len(cands))])
        tables = S.gather_tables(local, len(wins))
        outq.put((rank, [[(e.config.tp, e.r_c, e.e_c, e.saturated, e.error) for e in t] for t in tables]))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_gather_tables(ref_lib):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_table_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[0][1] == outs[1][1] and len(outs[0][1]) == 5
    # single process: the same five tables
    from paper_2602_18755_b200 import _abi as A
    from paper_2602_18755_b200 import pdsim as P
    from paper_2602_18755_b200 import workloads as W

    lad = W.ladder(5)
    m = W.llama_models(lad)
    day = P.gen_gamma_trace(6.0, 0.5, 5 * 20_000.0, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 4)
    cands = P.enumerate_candidates(lad, [2, 4])
    keep: list = []
    cm = P.c_model_set(m, keep)
    want = []
    for w in P.split_windows(day, 20_000.0):
        out = (A.bs_table_entry * len(cands))()
        assert ref_lib.ref_config_table(C.byref(cm), C.byref(P.c_trace(w, keep)), C.byref(P.c_slo(P.SLOSpec())),
                                        C.byref(P.c_policy(P.SchedulerPolicy(max_batch_tokens=1024))),
                                        C.byref(P.c_search(P.GoodputSearch())), P.c_candidates(cands), len(cands),
                                        out) == 0
        want.append([(e.config.tp, e.r_c, e.e_c, e.saturated, e.error)
                     for e in (P.entry_from_c(out[i]) for i in range(len(cands)))])
    assert outs[0][1] == want

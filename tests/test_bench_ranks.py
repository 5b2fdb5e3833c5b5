"""CPU test of bench.py's multi-rank plumbing (world size 2 over gloo): the
rank environment check, the barrier-aligned max-over-ranks timing, the
whole-job value (units of every rank / the slowest rank's time), the final
all-gather of per-decision rows in rank order, and rank 0 alone printing the
JSON line.  The per-rank device measurement (measure_c2, which needs a B200)
is replaced by fixed numbers; everything after it is bench.py's own code."""
from __future__ import annotations

import contextlib
import io
import json
import multiprocessing as mp
import os
import socket
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_measure(args, dev, rank, world, local):
    D = 4
    return {"D": D, "total_ms": 10.0 + 2.0 * rank, "step_ms": [5.0 + rank, 5.0 + rank], "launches": 10,
            "leaf_ms": [1.0], "phase_ms": [[0.1, 0.0, 0.2, 1.0, 0.05]], "e2e_s": 0.01 * (rank + 1), "h2d": 1000,
            "d2h": 100, "same": True, "clocks": {"sm_mhz": None}, "trajectories": D * 16 ** 6, "feasible": 7,
            "rows": [[rank * 100 + i, i, rank] for i in range(D)], "peak": 1.8e13, "corpus": None, "out": None}


def _rank(rank: int, port: int, q):
    os.environ.update(WORLD_SIZE="2", RANK=str(rank), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import bench

    bench.make_device = lambda local: object()
    bench.measure_c2 = _fake_measure
    sys.argv = ["bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-extras", "--no-cpu-baseline",
                "--dist-backend", "gloo"]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = bench.main()
    q.put((rank, rc, buf.getvalue()))


def test_world2_bench_line():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, rc0, text0), (r1, rc1, text1) = outs
    assert rc0 == rc1 == 0 and text1 == ""  # rank 0 alone prints
    line = json.loads(text0.strip().splitlines()[-1])
    traj = 16 ** 6
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["scaling"] == "weak"
    assert line["ms_per_step"] == 12.0 / 2  # the slowest rank
    assert line["value"] == pytest.approx(2 * 4 * traj * 2 / 12e-3)
    assert line["e2e"]["value"] == pytest.approx(2 * 4 * traj / 0.02)
    assert line["gather"]["rows"] == 8 and line["gather"]["rank0_rows_match"] is True
    assert line["gpu_launches"] == 10 and line["config"]["parallelism"].endswith("2 GPU(s)")


def test_world_size_must_match_gpus(monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench

    monkeypatch.setenv("WORLD_SIZE", "3")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    with pytest.raises(SystemExit, match="WORLD_SIZE=3"):
        bench.main()

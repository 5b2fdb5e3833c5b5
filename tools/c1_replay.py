"""Run the C1 scenario once through bs_replay (for ncu captures of the
replay kernels on a single, latency-bound scenario)."""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2602_18755_b200 import _abi as A  # noqa: E402
from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import workloads as W  # noqa: E402

models, sc = W.c1_scenario()
dev = P.default_device()
keep: list = []
cfgs, scs, _ = P.c_replay_inputs([sc], keep)
out = (A.bs_replay_summary * 1)()
mh = dev.models(models)
dev.check(dev._lib.bs_replay(dev.handle, mh, mh, cfgs, 1, scs, 1, out, None, None))
print("status", out[0].status, "decisions", out[0].n_decisions)

"""C5 exhaustive at N = 1, 2, 4, 8: contiguous shards (sharding.shard_bounds)
against strided ones (decision i to rank i mod N), every rank's shard timed
on this GPU (the job takes the slowest rank's time)."""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_18755_b200 import _abi as A  # noqa: E402
from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import sharding as S  # noqa: E402
from paper_2602_18755_b200 import workloads as Wk  # noqa: E402

dev = P.Device(0)
lib = dev._lib
models, cfg, pol, snaps = Wk.c5_corpus(0xC5, 4096)
keep: list = []
cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
probs = P.c_problems(snaps, None, keep)
mh = dev.models(models)
res = (A.bs_mpc_result * 4096)()


def run(idx):
    arr = (A.bs_mpc_problem * len(idx))(*[probs[i] for i in idx])
    dev.check(lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, arr, len(idx), res))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        dev.check(lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, arr, len(idx), res))
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


for mode in ("contiguous", "strided"):
    t1 = None
    for N in (1, 2, 4, 8):
        ts = []
        for r in range(N):
            if mode == "contiguous":
                lo, hi = S.shard_bounds(4096, r, N)
                idx = list(range(lo, hi))
            else:
                idx = list(range(r, 4096, N))
            ts.append(run(idx))
        t = max(ts)
        t1 = t if N == 1 else t1
        print(mode, N, f"slowest {t * 1e3:.2f} ms", "eff", round(t1 / (N * t), 3), [round(x * 1e3, 2) for x in ts],
              flush=True)

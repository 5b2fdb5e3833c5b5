"""Host phases of the C2 end-to-end call (bs_mpc_exhaustive, 1024 decisions,
host buffers): run with BS_DEBUG_TIMING=1 for the library's breakdown."""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_18755_b200 import _abi as A  # noqa: E402
from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import workloads as Wk  # noqa: E402

dev = P.Device(0)
lib = dev._lib
m, cfg, pol, snaps = Wk.c2_corpus(0xC2, 1024)
keep: list = []
cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
probs = P.c_problems(snaps, None, keep)
mh = dev.models(m)
res = (A.bs_mpc_result * 1024)()
for _ in range(3):
    dev.check(lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, probs, 1024, res))
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    dev.check(lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, probs, 1024, res))
    ts.append(time.perf_counter() - t0)
print(f"e2e median {statistics.median(ts) * 1e3:.3f} ms")

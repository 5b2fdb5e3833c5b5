"""Per-call latency of the drop-in greedy controller path (one decision per
bs_mpc_greedy call, host buffers), as GpuPrefillMpcController::decide makes
it; with BS_DEBUG_TIMING=1 the library prints its host phases per call."""
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
mc, cfg, pol, snaps = Wk.c1_corpus(n=256)
keep: list = []
carr = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
parr = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
probs = [P.c_problems([q], None, keep) for q in snaps]
one = (A.bs_mpc_result * 1)()
mh = dev.models(mc)
for pr in probs[:16]:
    dev.check(lib.bs_mpc_greedy(dev.handle, mh, carr, parr, 1, pr, 1, one))
raw = []
for pr in probs:
    t0 = time.perf_counter()
    dev.check(lib.bs_mpc_greedy(dev.handle, mh, carr, parr, 1, pr, 1, one))
    raw.append((time.perf_counter() - t0) * 1e6)
raw.sort()
print(f"c_abi p50 {raw[len(raw) // 2]:.1f} us  p99 {raw[int(0.99 * (len(raw) - 1))]:.1f} us  mean {statistics.mean(raw):.1f}")

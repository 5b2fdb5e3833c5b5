"""Time the device ILPs (bs_placement_solve / _batch) on C3-shaped tables:
one problem, a run_experiment's 24, and a C4 day sweep's 4608."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import random  # noqa: E402

from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import workloads as W  # noqa: E402
from test_gpu_ilp import _c3_table  # noqa: E402

dev = P.Device(0)
rng = random.Random(5)
lad = W.ladder(8)
tabs = [_c3_table(rng, lad) for _ in range(64)]
for n in (1, 24, 256, 4608):
    probs = [(P.PlacementProblem(tabs[i % 64], 16, 12.0, 0.05), None if i % 2 == 0 else lad.max_mhz()) for i in range(n)]
    P.solve_placement_batch(probs, dev)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        P.solve_placement_batch(probs, dev)
        ts.append(time.perf_counter() - t0)
    print(f"{n} problems: {min(ts) * 1e3:.2f} ms ({min(ts) / n * 1e6:.1f} us/problem)")

"""List sizes of a C5 exhaustive batch (resident plan; BS_DEBUG_COUNTS=1)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_18755_b200 import _abi as A  # noqa: E402
from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import workloads as Wk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = P.Device(0)
lib = dev._lib
m, cfg, pol, snaps = Wk.c5_corpus(0xC5, n)
keep: list = []
cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep))
cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
probs = P.c_problems(snaps, None, keep)
plan = C.c_void_p()
dev.check(lib.bs_mpc_plan_create(dev.handle, dev.models(m), cc, cp, 1, probs, n, 0, C.byref(plan)))
out = (A.bs_mpc_result * n)()
for _ in range(2):
    dev.check(lib.bs_mpc_plan_run(dev.handle, plan, 1))
    dev.check(lib.bs_mpc_plan_results(dev.handle, plan, out))
ms = (C.c_float * 5)()
lib.bs_mpc_plan_kernel_ms(dev.handle, plan, ms, 5)
print("phases ms", [round(x, 3) for x in ms])

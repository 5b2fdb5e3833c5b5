"""The C3 table's longest probe alone: a full-rate hour (12 rps gamma(0.5),
seed 7) on a decode TP8 instance at 1830 MHz, through bs_simulate_instance
(the probe kernel's warp decode simulator) -- for ncu source profiles."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_18755_b200 import _abi as A  # noqa: E402
from paper_2602_18755_b200 import pdsim as P  # noqa: E402
from paper_2602_18755_b200 import workloads as Wk  # noqa: E402

dev = P.Device(0)
lad = Wk.ladder(16)
m = Wk.llama_models(lad)
base = P.gen_gamma_trace(12.0, 0.5, 3600e3, P.LengthDistribution(lognormal=P.Lognormal(6.2, 0.6, 5.3, 0.7)), 7)
keep: list = []
tr = (A.bs_trace * 1)(P.c_trace(base, keep))
ci = A.bs_instance_config(int(P.Phase.decode), 8, lad.max_mhz())
cp = P.c_policy(P.SchedulerPolicy(max_batch_tokens=2048))
cs = P.c_slo(P.SLOSpec(600.0, 100.0))
out = (A.bs_sim_summary * 1)()
for i in range(3):
    t0 = time.perf_counter()
    dev.check(dev._lib.bs_simulate_instance(dev.handle, dev.models(m), tr, 1, C.byref(ci), C.byref(cp), C.byref(cs),
                                            out))
    print(f"{(time.perf_counter() - t0) * 1e3:.1f} ms, completed {out[0].completed}, meets {out[0].meets_slo}")

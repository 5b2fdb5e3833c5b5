import ctypes as C, statistics, sys, time
from pathlib import Path
sys.path.insert(0, '/root/repo')
from paper_2602_18755_b200 import _abi as A, pdsim as P, workloads as Wk
dev = P.Device(0); lib = dev._lib
models, cfg, pol, snaps = Wk.c5_corpus(0xC5, 4096)
keep = []
cc = (A.bs_mpc_config * 1)(P.c_mpc_config(cfg, keep)); cp = (A.bs_scheduler_policy * 1)(P.c_policy(pol))
probs = P.c_problems(snaps, None, keep); mh = dev.models(models)
res = (A.bs_mpc_result * 1)()
out = []
for i in range(512, 1024):
    arr = (A.bs_mpc_problem * 1)(probs[i])
    lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, arr, 1, res)
    t0 = time.perf_counter(); lib.bs_mpc_exhaustive(dev.handle, mh, cc, cp, 1, arr, 1, res); t = time.perf_counter() - t0
    q = snaps[i]
    out.append((t, i, len(q.waiting), res[0].feasible_count, q.now_ms - (q.waiting[0].arrival_ms if q.waiting else q.now_ms)))
out.sort(reverse=True)
for r in out[:12]: print(f"{r[0]*1e3:.2f} ms  i={r[1]} n_wait={r[2]} feasible={r[3]} age={r[4]:.1f}")
print('median', statistics.median(o[0] for o in out) * 1e3)

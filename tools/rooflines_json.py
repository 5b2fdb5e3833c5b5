"""profiles/r02_rooflines.json from tools/ncu_rooflines.sh's CSVs: per
sub-benchmark, the dominant kernel's executed FP64-pipe and issue fractions,
occupancy, DRAM bytes and duration (one ncu launch, --clock-control none)."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = {"gpu__time_duration.sum": "duration_us",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_active_frac",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_frac",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy",
        "dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
        "smsp__thread_inst_executed_per_inst_executed.ratio": "avg_active_threads_per_warp",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid", "launch__block_size": "block"}
SCALE = {"B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1,
         "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3, "s": 1e6, "second": 1e6}


def parse(path: Path) -> dict | None:
    if not path.exists():
        return None
    rows = list(csv.reader(l for l in path.read_text().splitlines() if not l.startswith("==")))
    if not rows:
        return None
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    out = {}
    for r in rows[1:]:
        if len(r) != len(h) or r[mi] not in KEYS:
            continue
        out["kernel"] = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        v = float(r[vi].replace(",", ""))
        k = KEYS[r[mi]]
        if k.endswith("_frac") or k == "achieved_occupancy":
            v /= 100.0
        elif k.endswith("_bytes") or k == "duration_us":
            v *= SCALE.get(r[ui], 1)
        out[k] = v
    return out or None


def main():
    src = ROOT / "gpurun_out"
    res = {}
    for cfg in ("c1", "c2l", "c3", "c4", "c4d", "c4x", "c5g", "c5x"):
        p = parse(src / f"roof_{cfg}.csv")
        if p:
            res[cfg] = p
    doc = {"source": "ncu --metrics (fp64 pipe, issue, occupancy, DRAM) --clock-control none, one launch of each "
                     "sub-benchmark's dominant kernel after warm-up: tools/ncu_rooflines.sh", "configs": res}
    out = ROOT / "profiles" / (sys.argv[1] if len(sys.argv) > 1 else "r02_rooflines.json")
    out.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()

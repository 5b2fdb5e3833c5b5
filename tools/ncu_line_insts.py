"""Per-source-line executed warp instructions (and min/max per SASS
instruction: the execution count of a line) of one kernel in an ncu report.

usage: python tools/ncu_line_insts.py REPORT.ncu-rep KERNEL_REGEX LIB.so [FILE]
"""
import collections
import csv
import io
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
import ncu_lines as N  # noqa: E402

rep, kernel, lib = sys.argv[1:4]
only = sys.argv[4] if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
ai, ei = hdr.index("Address"), hdr.index("Instructions Executed")
seen, data = set(), []
for r in rows:
    if len(r) != len(hdr) or r[0] == "Address":
        continue
    a = int(r[ai], 16)
    if a in seen:
        continue
    seen.add(a)
    data.append((a, float(r[ei] or 0)))
base = min(a for a, _ in data)
lines = N.line_map(lib, kernel)
tot = collections.Counter()
mx = collections.defaultdict(float)
for a, e in data:
    k = lines.get(a - base, ("?", 0))
    tot[k] += e
    mx[k] = max(mx[k], e)
s = sum(tot.values())
print(f"total warp instructions {s:.0f}")
for (f, ln), e in sorted(tot.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if only and f != only:
        continue
    if e > 0.002 * s:
        print(f"{f}:{ln:5d}  {e:12.0f} ({100 * e / s:5.2f}%)  max/instr {mx[(f, ln)]:10.0f}")

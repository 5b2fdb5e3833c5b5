"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX[@SASS_REGEX] [LIB.so] [TOP]

SASS_REGEX selects the kernel's section in the library when several
instantiations share the name (e.g. sweep_kernel@sweep_kernelILi3E for
sweep_kernel<3>): offsets from another instantiation would mislabel lines.

ncu's source page gives per-SASS-instruction samples with runtime
addresses; nvdisasm -g on the library's cubin gives per-instruction source
lines (the library is built with -lineinfo).  Offsets from the kernel's first
instruction join the two.
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def sass_samples(rep: str, kernel: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    si, ai, srci = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address"), hdr.index("Source")
    seen, data = set(), []
    for r in rows:
        if len(r) != len(hdr) or r[0] == "Address":
            continue
        a = int(r[ai], 16)
        if a in seen:  # one launch only
            continue
        seen.add(a)
        try:
            data.append((a, float(r[si] or 0), r[srci].strip()))
        except ValueError:
            pass
    base = min(a for a, _, _ in data)
    return [(a - base, s, src) for a, s, src in data]


def line_map(lib: str, kernel: str):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=d, capture_output=True)
        for cub in Path(d).glob("*.cubin"):
            txt = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout
            m = re.search(r"\.text\.(\S*" + kernel + r"\S*):", txt)
            if not m:
                continue
            body = txt[m.end():]
            nxt = re.search(r"\n\s*\.text\.", body)
            body = body[:nxt.start()] if nxt else body
            cur, res = None, {}
            for ln in body.splitlines():
                fm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                if fm:
                    cur = (Path(fm.group(1)).name, int(fm.group(2)))
                    continue
                om = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
                if om and cur:
                    res[int(om.group(1), 16)] = cur
            return res
    return {}


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    kernel, _, sass_kernel = kernel.partition("@")
    lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2602_18755_b200/libbiscale_gpu.so"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    samples = sass_samples(rep, kernel)
    lines = line_map(lib, sass_kernel or kernel)
    tot = sum(s for _, s, _ in samples) or 1.0
    agg = collections.Counter()
    for off, s, _ in samples:
        agg[lines.get(off, ("?", 0))] += s
    print(f"{kernel}: {tot:.0f} samples, {len(samples)} instructions, {len(lines)} mapped")
    for (f, ln), s in agg.most_common(top):
        print(f"{100 * s / tot:6.2f}%  {f}:{ln}")


if __name__ == "__main__":
    main()

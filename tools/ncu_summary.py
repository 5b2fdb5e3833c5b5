"""Summarise an ncu report: key metrics per kernel (used to write profiles/)."""
import csv
import subprocess
import sys

WANT = ['Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'Registers Per Thread',
        'Achieved Occupancy', 'Theoretical Occupancy', 'Executed Ipc Active', 'Issue Slots Busy', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp',
        'Dynamic Shared Memory Per Block', 'Block Limit Shared Mem', 'Block Limit Registers', 'Grid Size',
        'Block Size']


def main(path, raw_metrics=()):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    idi = h.index('ID')
    seen = set()
    for r in rows[1:]:
        key = (r[idi], r[mi])
        if r[mi] in WANT and key not in seen:
            seen.add(key)
            print(f"{r[idi]:>3s} {r[ki][:28]:28s} {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
    if raw_metrics:
        out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h = rows[0]
        cols = [i for i, name in enumerate(h) if any(m in name for m in raw_metrics)]
        ki = h.index('Kernel Name')
        for r in rows[2:]:
            print(r[ki][:28], {h[i]: r[i] for i in cols})


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2:])

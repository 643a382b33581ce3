"""Summaries of ncu outputs for profiles/ (run here, no GPU needed).

    python scripts/summarize_ncu.py launches <launches.csv> [--title T]   # per-kernel share table
    python scripts/summarize_ncu.py report <prof.ncu-rep> [--title T]     # key metrics of a --set full capture

The launch list comes from the recipe's ``ncu --metrics gpu__time_duration.sum
--clock-control none`` pass (cold-cache, serialised: compare shares, not
absolutes); the report from ``ncu --set full``.
"""

import argparse
import collections
import csv
import io
import re
import subprocess
import sys


def _rows(text):
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if '"Kernel Name"' in l or "Kernel Name" in l.split(",")[:8])
    return list(csv.reader(io.StringIO("\n".join(lines[start:]))))


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("pl::", "")
    return name[:60]


def launches(path, title):
    r = _rows(open(path).read())
    h, data = r[0], r[1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    tot = collections.Counter()
    cnt = collections.Counter()
    grids = {}
    for x in data:
        if len(x) <= vi or not x[vi]:
            continue
        k = short(x[ki])
        ns = float(x[vi].replace(",", ""))
        tot[k] += ns
        cnt[k] += 1
        if gi is not None:
            grids.setdefault(k, x[gi])
    all_ns = sum(tot.values())
    print(f"### {title}\n")
    print(f"{sum(cnt.values())} launches, {all_ns / 1e3:.1f} us total (serialised, cold-cache)\n")
    print("| kernel | launches | total us | share | avg us | grid |")
    print("|---|---:|---:|---:|---:|---|")
    for k, ns in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {ns / 1e3:.1f} | {100 * ns / all_ns:.1f}% | {ns / cnt[k] / 1e3:.2f} | "
              f"{grids.get(k, '')} |")


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]


def report(path, title):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, rows = r[0], r[1], r[2:]
    ki = h.index("Kernel Name")
    print(f"### {title}\n")
    for row in rows:
        print(f"**{short(row[ki])}**\n")
        print("| metric | value |")
        print("|---|---:|")
        seen = set()
        for key, label in KEYS:
            if key in h and label not in seen:
                i = h.index(key)
                seen.add(label)
                print(f"| {label} (`{key}`) | {row[i]} {units[i]} |")
        print()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "report"])
    ap.add_argument("path")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    (launches if a.mode == "launches" else report)(a.path, a.title or a.path)


if __name__ == "__main__":
    sys.exit(main())

"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into
markdown (per kernel and grid size: launches, total time, share). Whole-scene
launches and the host path's 1024-row strip launches have different grids.

    python tools/launch_summary.py gpurun_out/launches.csv "<command>" > profiles/rNN_launches_summary.md
"""
import csv
import sys
from collections import defaultdict


def main(path: str, command: str) -> None:
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = (r["Kernel Name"].split("(")[0][:64], r["Grid Size"].replace(" ", ""))
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0,
                 "ms": 1e3}[unit]
        tot[name] += v * scale
        cnt[name] += 1
    grand = sum(tot.values())
    print(f"# ncu launch list summary: `{command}`\n")
    print("Cold-cache, serialised per-launch times (compare shares, not absolutes).\n")
    print("| kernel | grid | launches | total time (us) | mean per launch (us) | share |")
    print("|---|---|---|---|---|---|")
    for (name, grid), t in sorted(tot.items(), key=lambda kv: -kv[1]):
        n = cnt[(name, grid)]
        print(f"| `{name}` | {grid} | {n} | {t:.0f} | {t / n:.1f} | {100 * t / grand:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")

"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [--skip REGEX]
"""
import collections
import csv
import re
import sys


def load(path):
    with open(path) as f:
        lines = f.read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        out.append((r["Kernel Name"], v * scale))
    return out


def main():
    rows = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        key = re.sub(r"\(.*", "", name)[:90]
        agg[key][0] += 1
        agg[key][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'total_us':>10} {'n':>5}  share  kernel   (total {tot:.1f} us over {len(rows)} launches)")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{us:10.1f} {n:5d} {us / tot:6.3f}  {k}")


if __name__ == "__main__":
    main()

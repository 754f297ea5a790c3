"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

usage: python tools/launch_summary.py launches.csv [header comment lines ...]
Prints one line per kernel (launches, total/avg microseconds, share of the listed time),
the format of profiles/r1*_launches.txt. ncu times are cold-cache and serialised: use the
shares, not the absolute times.
"""
import collections
import csv
import sys


def main(path, header=()):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
        name = name.split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        rows.append((name, us))
    agg = collections.OrderedDict()
    for name, us in rows:
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values()) or 1.0
    for h in header:
        print("#", h)
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:32s} launches={n:5d} total_us={t:10.1f} avg_us={t / n:9.2f} share={t / total:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])

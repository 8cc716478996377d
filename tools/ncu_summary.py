"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X ...`): total device time per kernel name, launch counts and share.

usage: python tools/ncu_summary.py launches.csv [top_n]"""
import collections
import csv
import sys


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        rows.append((short, v * scale))
    return rows


def main():
    rows = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    tot = collections.Counter()
    cnt = collections.Counter()
    for n, us in rows:
        tot[n] += us
        cnt[n] += 1
    all_us = sum(tot.values())
    print(f"{len(rows)} launches, {all_us:.1f} us total")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for n, us in tot.most_common(top):
        print(f"{n[:60]:60s} {cnt[n]:8d} {us:10.1f} {us / cnt[n]:9.2f} {100 * us / all_us:5.1f}%")


if __name__ == "__main__":
    main()

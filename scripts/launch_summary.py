"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file F ...`):
one line per kernel with launches, mean duration and share of the total.

    python scripts/launch_summary.py F.csv [--markdown]
"""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    head = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            head = r
            continue
        if head is None or len(r) != len(head):
            continue
        d = dict(zip(head, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        agg.setdefault(d["Kernel Name"], []).append(us)
    total = sum(sum(v) for v in agg.values()) or 1.0
    return [(k, len(v), sum(v) / len(v), sum(v) / total) for k, v in agg.items()]


def main():
    md = "--markdown" in sys.argv
    for path in [a for a in sys.argv[1:] if not a.startswith("--")]:
        rows = summarise(path)
        if md:
            print("| kernel | launches | mean (us) | share |\n|---|---|---|---|")
        for k, n, mean, share in rows:
            name = k if len(k) < 90 else k[:87] + "..."
            if md:
                print(f"| `{name}` | {n} | {mean:.1f} | {share:.2f} |")
            else:
                print(f"{n:5d} {mean:10.1f} us {share:6.2f}  {name}")


if __name__ == "__main__":
    main()

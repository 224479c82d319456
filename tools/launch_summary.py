"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
    python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= mi:
            continue
        ms = float(r[mi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(a[1] for a in agg.values())
    print(f"{sum(a[0] for a in agg.values())} launches, {tot:.3f} ms device time (cold-cache, serialised)")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k[:60]:60s} {c:8d} {t:10.3f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()

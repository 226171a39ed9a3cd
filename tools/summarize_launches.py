"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into
a markdown table (share of device time per kernel)."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        unit = r[ui]
        name = r[ki].split("(")[0].replace("void ", "")[:90]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
    print(f"| kernel | launches | total us | mean us | share |")
    print(f"|---|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| `{k}` | {c} | {v * scale:.1f} | {v * scale / c:.2f} | {100 * v / tot:.1f}% |")
    print(f"\n{sum(c for c, _ in agg.values())} launches, {tot * scale:.1f} us total (cold-cache, serialised under ncu)")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

    python tools/summarize_launches.py profiles/r01_launches.csv > profiles/r01_launches.md
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ig, ib = hdr.index("Grid Size"), hdr.index("Block Size")
    agg = collections.OrderedDict()
    tot = 0.0
    for r in data:
        name = r[ik].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r[iv].replace(",", ""))
        us = {"ns": v / 1e3, "us": v, "ms": v * 1e3, "s": v * 1e6}.get(r[iu], v)
        a = agg.setdefault(name, [0, 0.0, r[ig], r[ib]])
        a[0] += 1
        a[1] += us
        tot += us
    print(f"# ncu launch list: {path}\n")
    print(f"{len(data)} launches, {tot:.1f} us total (cold-cache, serialised: compare shares, not absolutes)\n")
    print("| kernel | launches | total us | share | grid | block |")
    print("|---|---|---|---|---|---|")
    for k, (n, us, g, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {us:.1f} | {100 * us / tot:.1f}% | {g} | {b} |")


if __name__ == "__main__":
    main(sys.argv[1])

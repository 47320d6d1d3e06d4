"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys


def summarize(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    seq = []
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1000 if u in ("nsecond", "ns") else (v * 1000 if u == "msecond" else v)
        seq.append((r[ki].split("(")[0].replace("void ", "")[:70], v))
    agg = collections.OrderedDict()
    for n, v in seq:
        agg.setdefault(n, []).append(v)
    tot = sum(v for _, v in seq)
    print(f"{len(seq)} launches, {tot:.1f} us total")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:70s} n={len(v):5d} mean={sum(v)/len(v):9.2f}us sum={sum(v):10.1f}us "
              f"share={sum(v)/tot*100:5.1f}%")


if __name__ == "__main__":
    summarize(sys.argv[1])

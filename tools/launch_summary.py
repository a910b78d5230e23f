"""Summarise ncu --csv launch lists (tools/launches.sh): per kernel, launches,
mean / total duration and share of the motif's kernel time."""
import csv
import sys
from collections import defaultdict


def summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        u = r[iu].lower()
        v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        agg[r[ik].split("(")[0][:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:72s} {len(v):6d} {sum(v) / len(v):10.2f} {sum(v):12.1f} {100 * sum(v) / tot:6.2f}%")


for p in sys.argv[1:]:
    print(f"# {p}: kernel | launches | mean us | total us | share (cold, serialised: compare shares)")
    summary(p)

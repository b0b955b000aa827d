"""Per-kernel launch count, median and max duration (us) of an ncu
--metrics gpu__time_duration.sum --csv launch list, and the durations of
the first launches of the kernels named on the command line."""
import csv
import statistics
import sys
from collections import defaultdict

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
seq = defaultdict(list)
for r in rows:
    k = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    seq[k].append(v)
for k in sorted(seq, key=lambda k: -statistics.median(seq[k]) * len(seq[k])):
    print(f"{k:24s} n={len(seq[k]):4d} median={statistics.median(seq[k]):8.1f} us  max={max(seq[k]):8.1f} us")
for k in sys.argv[2:]:
    print(k, [round(x, 1) for x in seq.get(k, [])[:40]])

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total and per-launch time, share of the total."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    k = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Unit"] in ("usecond", "us"):
        v *= 1e3
    elif r["Metric Unit"] in ("msecond", "ms"):
        v *= 1e6
    tot[k] += v
    cnt[k] += 1
all_ns = sum(tot.values())
print(f"launches {sum(cnt.values())}, total {all_ns / 1e6:.3f} ms")
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{k:28s} n={cnt[k]:4d} total={tot[k] / 1e6:8.3f} ms  per-launch={tot[k] / cnt[k] / 1e3:9.1f} us"
          f"  share={100 * tot[k] / all_ns:5.1f}%")

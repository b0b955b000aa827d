"""Per-source-line totals from `ncu --page source --csv --print-source cuda,sass`:
warp-stall samples and executed warp instructions, attributed to the CUDA
line each SASS instruction maps to.  Usage: source_hotspots.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

samples = defaultdict(int)
insts = defaultdict(int)
text = {}
path = None
cur = None
for row in csv.reader(open(sys.argv[1])):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0].isdigit():
        cur = (path, int(row[0]))
        text[cur] = row[1].strip()[:70]
        continue
    if cur is not None and len(row) > 6 and row[0] == "" and row[2].startswith("0x"):
        try:
            samples[cur] += int(row[4] or 0)
            insts[cur] += int(row[7] or 0)
        except ValueError:
            pass
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ts, ti = sum(samples.values()) or 1, sum(insts.values()) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
for k in sorted(samples, key=samples.get, reverse=True)[:top]:
    print(f"{k[0]}:{k[1]:5d} samp {100 * samples[k] / ts:5.1f}% inst {100 * insts[k] / ti:5.1f}%  {text.get(k, '')}")

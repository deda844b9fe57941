"""Aggregate warp-stall samples per CUDA source line from an ncu
--page source --print-source cuda,sass CSV.  usage: ncu_line_hot.py f.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cur = None
samples = defaultdict(float)
execd = defaultdict(float)
text = {}
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] not in ("", "-"):
        cur = f"{fname}:{r[0]}"
        text[cur] = r[1]
        continue
    try:
        samples[cur] += float(r[4])
        execd[cur] += float(r[7])
    except ValueError:
        pass
tot = sum(samples.values())
print(f"total samples {tot:.0f}")
for line, v in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:7.0f} {100*v/tot:5.1f}% exec {execd[line]:8.0f}  {line}: {text.get(line,'')[:90]}")

"""Print an ncu --metrics gpu__time_duration.sum CSV as (kernel, grid, us),
second half only (the first half is the warm-up tree) unless --all."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
if "--all" not in sys.argv:
    rows = rows[len(rows) // 2:]
tot = 0.0
for r in rows:
    us = float(r[vi].replace(",", "")) / 1e3
    tot += us
    print(f"{r[ki][:58]:58s} {r[gi]:>14s} {us:10.1f}")
print(f"{'total':58s} {'':>14s} {tot:10.1f}")

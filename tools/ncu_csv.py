"""Print 'metric value' pairs of an `ncu --csv` capture read from stdin (one kernel launch)."""
import csv
import sys

rows = [r for r in csv.reader(line for line in sys.stdin if line.startswith('"'))]
if not rows:
    sys.exit(print("no csv rows"))
h = rows[0]
mi, vi, ki = h.index("Metric Name"), h.index("Metric Value"), h.index("Kernel Name")
for r in rows[1:]:
    print("  ", r[ki][:28], r[mi], r[vi])

"""Print kernel name and duration (ns) of each launch in an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[hdr + 1:]:
    print(f"{r[ki][:60]:60s} {r[vi]:>10s}")

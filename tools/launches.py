"""Print kernel name and duration (ns) from an ncu --csv launch list: python tools/launches.py FILE"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == "ID"][0]
i, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
for r in rows:
    if len(r) > v and r[0] != "ID":
        print(r[i][:60], r[v])
